"""configs[3] (IGB-large-shaped, 100M nodes, batch 8192 per GPU, shared cache over 8 B200) at
its full node count, counts-only on ONE B200.

By invariant I8 (pinned on the oracle for every policy, and GPU-vs-GPU in
tests/test_gpu_multiproc.py) a G-GPU shared cache of L lines per GPU gives exactly the same
counters as one home of G*L lines on the merged batches (pvp = 0). So the 8-GPU box's cache
behaviour — hit ratio, storage reads per iteration — is computed here with one home of
8 x L lines, 16-byte rows (counters do not depend on the payload; bytes are reported for
4 KiB rows). The batches come from the GPU UVA sampler (lsmgnn_sample) over the 100M-node
CSR pinned in host memory. NVLink throughput of the real 8-GPU run is not measured here.

usage: python tools/cfg4_counts.py OUT.json [--iters 60] [--lines-per-gpu 4194304,262144]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--nodes", type=int, default=100_000_000)
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--warm", type=int, default=10)
    ap.add_argument("--lines-per-gpu", default="4194304,262144")
    ap.add_argument("--policies", default="hybrid,static,lru")
    args = ap.parse_args()
    import torch
    import synth
    from paper_2407_15264_b200 import LsmGnn, Sampler, STATS_FIELDS
    F = {n: i for i, n in enumerate(STATS_FIELDS)}
    N, G, B, fan, W = args.nodes, 8, 8192, (10, 5, 5), 256
    t0 = time.time()
    g = synth.plcite_c(N, 12)
    t_graph = time.time() - t0
    t0 = time.time()
    scores = synth.static_scores(g)
    t_scores = time.time() - t0
    dev = torch.device("cuda", 0)
    perm = torch.from_numpy(synth.epoch_seeds(N, 0)).to(dev)
    K = args.warm + args.iters
    total = K + W + 1
    res = {"config": "configs[3] IGB-large-shaped", "N": N, "G_virtual": G, "batch_per_gpu": B, "fanout": list(fan),
           "W": W, "T": W // 8, "ways": 32, "iterations": {"warm": args.warm, "measured": args.iters},
           "graph_s": round(t_graph, 1), "scores_s": round(t_scores, 1),
           "method": "one home x (8 x L) lines on the merged 8-rank batches (I8, pvp = 0), 16-B rows, GPU sampler",
           "runs": []}
    samp = Sampler(g.indptr, g.indices)  # pins the 100M-node CSR once
    table = torch.zeros((N, 16), dtype=torch.uint8, pin_memory=True)
    for lpg in [int(x) for x in args.lines_per_gpu.split(",")]:
        for pol in args.policies.split(","):
            bound = Sampler.bound(B, fan) * G
            c = LsmGnn(N, 4, G * lpg, 32, 0, scores, policy=pol, pvp=0, window=W, max_batch_ids=bound)
            c.attach_storage(table)
            samp.reattach()  # lsmgnn_finalize of the previous run forgot the CSR
            batches = {}
            t_samp = [0.0]

            def merged(k):
                if k not in batches:
                    if k >= K + W:  # the window of every measured iteration is full
                        batches[k] = torch.zeros(0, dtype=torch.int64, device=dev)
                    else:
                        ts = time.time()
                        parts = []
                        for r in range(G):
                            seeds = perm[(k * G + r) * B:(k * G + r + 1) * B]
                            o, cn = samp.sample(seeds, fan, 4, k, r)
                            parts.append(o[: int(cn.item())])
                        batches[k] = torch.cat(parts)
                        t_samp[0] += time.time() - ts
                    batches.pop(k - W - 2, None)
                return batches[k]

            t0 = time.time()
            for k in range(1, W + 1):
                c.prefetch([merged(k)], first_iter=k)
            out = torch.empty((bound, 16), dtype=torch.uint8, device=dev)
            for t in range(K):
                c.gather(merged(t), out)
                c.prefetch([merged(t + 1 + W)], first_iter=t + 1 + W)
            torch.cuda.synchronize()
            h = c.history(args.warm, args.iters)
            c.close()
            e = h.sum(axis=0)
            u = max(int(e[F["unique"]]), 1)
            run = {"policy": pol, "lines_per_gpu": lpg, "cache_pct_boxwide": round(100 * G * lpg / N, 2),
                   "requests_per_iter": int(e[F["requests"]]) // args.iters, "unique_per_iter": u // args.iters,
                   "hit_ratio": round(int(e[F["hits"]]) / u, 4),
                   "storage_GB_per_iter_4KiB": round(int(e[F["storage_reads"]]) * 4096 / args.iters / 1e9, 3),
                   "bypassed_per_iter": int(e[F["bypassed"]]) // args.iters, "wall_s": round(time.time() - t0, 1),
                   "sampler_s": round(t_samp[0], 1)}
            res["runs"].append(run)
            print(json.dumps(run), flush=True)
            json.dump(res, open(args.out, "w"), indent=1)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Config 5 (BASELINE.json configs[4]): eviction-policy sweep on an IGBH-shaped graph —
storage-tier bytes per epoch for hybrid vs static-only vs LRU (and RR, dynamic-only,
hybrid+PVP) at cache sizes 1/2/5/10/20% of the nodes, G = 2/4/8 GPUs.

Runs the CUDA path (liblsmgnn.so) counts-only with 16-byte rows (counts do not depend
on the payload; bytes are reported x 4096 for 4 KiB rows). A G-GPU shared cache of L
lines per GPU is run as ONE home with G*L lines on the merged batches: with pvp = 0 the
counters are identical (invariant I8, pinned by tests/test_oracle_invariants.py
::test_shared_cache_equivalence for every policy). The hybrid+PVP row uses G*V victim
lines in W queues (equal to the G homes' total only when no queue overflows; flagged).

Graph: plcite with N = 10M nodes in typed ID ranges scaled from IGBH-large
(paper 46%, author 53.7%, fos 0.3%, institute 0.014%; SPEC S:99 models heterogeneity as
one ID space); training seeds = 10% of the paper range; fanout (5,2,2,2), batch 2048
per GPU; W = 256, T = 32. Epoch 0 warms up, epoch 1 is measured (R23).

usage: python tools/policy_sweep.py OUT.json [--nodes N] [--gpus 2,4,8] [--sizes 1,2,5,10,20]
                                     [--window W] [--period P] [--policies ...] [--private] [--scores rpr]
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


def typed_trace(g, N, G, batch, fanout, iters_per_epoch, epochs, train, W, seed_s=4):
    import synth
    trace = []
    total = iters_per_epoch * epochs + W + 1
    for t in range(total):
        ep, te = divmod(t, iters_per_epoch)
        perm = np.random.default_rng(3 + ep).permutation(train)
        row = []
        for r in range(G):
            lo = (te * G + r) * batch
            seeds = perm[lo:lo + batch] if ep < epochs else perm[:0]
            row.append(synth.sample_batch(g, seeds, fanout, seed_s, t, r) if seeds.size else np.zeros(0, np.int64))
        trace.append(row)
    return trace


def run_point(trace_merged, N, lines, ways, scores, policy, pvp, W, V, iters_per_epoch, period=1):
    import torch
    from paper_2407_15264_b200 import LsmGnn
    D = 4  # 16-byte rows
    K = len(trace_merged)
    dev = torch.device("cuda", 0)
    ids = [torch.from_numpy(np.asarray(x, np.int64)).to(dev) for x in trace_merged]
    mb = max(1, max(x.numel() for x in ids))
    c = LsmGnn(N, D, lines, ways, V, scores, policy=policy, pvp=pvp, window=W, max_batch_ids=mb, period=period)
    table = torch.zeros((N, 16), dtype=torch.uint8, pin_memory=True)
    c.attach_storage(table)
    empty = torch.zeros(0, dtype=torch.int64, device=dev)
    c.prefetch([ids[k] if k < K else empty for k in range(1, W + 1)], first_iter=1)
    out = torch.empty((mb, 16), dtype=torch.uint8, device=dev)
    n_iter = 2 * iters_per_epoch
    for t in range(n_iter):
        c.gather(ids[t], out)
        k = t + 1 + W
        c.prefetch([ids[k] if k < K else empty], first_iter=k)
    h = c.history(0, n_iter)
    c.close()
    from paper_2407_15264_b200 import STATS_FIELDS
    F = {n: i for i, n in enumerate(STATS_FIELDS)}
    e1 = h[iters_per_epoch:n_iter]
    res = {f: int(e1[:, F[f]].sum()) for f in ("requests", "unique", "hits", "victim_hits", "storage_reads",
                                                  "bypassed", "evictions", "victim_admitted", "victim_dropped")}
    res["storage_bytes_epoch_4KiB"] = res["storage_reads"] * 4096
    res["hit_ratio"] = round((res["hits"] + res["victim_hits"]) / max(res["unique"], 1), 4)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--nodes", type=int, default=10_000_000)
    ap.add_argument("--gpus", default="2,4,8")
    ap.add_argument("--sizes", default="1,2,5,10,20")
    ap.add_argument("--policies", default="hybrid,static,lru,rr,dynamic")
    ap.add_argument("--private", action="store_true", help="add M-GIDS rows: independent per-GPU caches")
    ap.add_argument("--scores", default="degree", choices=["degree", "rpr"],
                    help="static information: degree, or reverse PageRank (the paper's choice, P:645)")
    ap.add_argument("--window", type=int, default=256, help="W (the paper: 256, P:607; 64 in its W sweep)")
    ap.add_argument("--period", type=int, default=1, help="dynamic-information update period P (the paper: 4)")
    ap.add_argument("--no-pvp-row", action="store_true", help="skip the hybrid+PVP row")
    args = ap.parse_args()
    import synth
    N = args.nodes
    W, ways, batch, fanout = args.window, 32, 2048, (5, 2, 2, 2)
    n_paper = int(0.46 * N)
    train = np.arange(0, n_paper, 10, dtype=np.int64)  # 10% of the paper range (a typed ID range)
    t0 = time.time()
    g = synth.plcite(N, 12)
    if args.scores == "rpr":
        t1 = time.time()
        scores = synth.quantize_scores(synth.reverse_pagerank(g))
        print(f"reverse PageRank in {time.time() - t1:.0f}s", flush=True)
    else:
        scores = synth.static_scores(g)
    print(f"graph {N} nodes in {time.time() - t0:.0f}s", flush=True)
    results = {"workload": {"N": N, "typed_ranges": {"paper": [0, n_paper], "author": [n_paper, int(0.997 * N)],
                                                     "fos+institute": [int(0.997 * N), N]},
                            "train": int(train.size), "fanout": list(fanout), "batch_per_gpu": batch, "W": W,
                            "T": max(1, W // 8), "period": args.period, "ways": ways, "scores": "u8 rank-quantised " + ("reverse PageRank (d=0.85, tol 1e-6, <=100 it)"
                                                                           if args.scores == "rpr" else "degree"), "row_bytes_run": 16,
                            "bytes_reported_for_row": 4096,
                            "note": "G-GPU runs executed as 1 home x G*L lines on merged batches (I8, exact "
                                    "for pvp=0); hybrid+pvp uses G*V victim lines"},
               "points": []}
    for G in [int(x) for x in args.gpus.split(",")]:
        ipe = -(-train.size // (batch * G))
        t0 = time.time()
        tr = typed_trace(g, N, G, batch, fanout, ipe, 2, train, W)
        merged = [np.concatenate(row) for row in tr]
        print(f"G={G}: {ipe} iterations/epoch, trace in {time.time() - t0:.0f}s", flush=True)
        for pct in [float(x) for x in args.sizes.split(",")]:
            lines_total = int(N * pct / 100) // (ways * G) * ways * G
            runs = [(p, 0) for p in args.policies.split(",")] + ([] if args.no_pvp_row else [("hybrid", 1)])
            for pol, pvp in runs:
                V = 16384 * W * G if pvp else 0
                r = run_point(merged, N, lines_total, ways, scores, pol, pvp, W, V, ipe, args.period)
                r.update({"G": G, "cache_pct": pct, "lines_per_gpu": lines_total // G, "policy": pol, "pvp": pvp,
                          "W": W, "P": args.period})
                results["points"].append(r)
                print(json.dumps(r), flush=True)
            # M-GIDS baseline: G independent PRIVATE caches of L lines each, every
            # GPU caching its own requests (no communication layer) — RR as in the paper, and hybrid
            if args.private:
                for pol in ("rr", "hybrid"):
                    tot = None
                    for rk in range(G):
                        mine = [row[rk] for row in tr]
                        pr = run_point(mine, N, lines_total // G, ways, scores, pol, 0, W, 0, ipe)
                        tot = pr if tot is None else {k: tot[k] + pr[k] for k in tot if k != "hit_ratio"}
                    tot["hit_ratio"] = round((tot["hits"] + tot["victim_hits"]) / max(tot["unique"], 1), 4)
                    tot.update({"G": G, "cache_pct": pct, "lines_per_gpu": lines_total // G, "policy": "private_" + pol,
                                "pvp": 0})
                    results["points"].append(tot)
                    print(json.dumps(tot), flush=True)
        json.dump(results, open(args.out, "w"), indent=1)
    json.dump(results, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

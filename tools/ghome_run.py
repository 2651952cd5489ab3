"""configs[3] / configs[4] at full node count through the G-HOME data path (one process per home,
CUDA IPC + stream-memory-op flags, one-sided pulls): launched with torch.distributed.run, G ranks
(on a 1-GPU pool all ranks share the device; run it under MPS so they execute concurrently).

Every rank samples its own batches on the GPU (lsmgnn_sample over the CSR, which rank 0 builds
and shares through /dev/shm; each rank page-locks the same pages and reads them zero-copy, the
paper's UVA placement P:251), keeps each list on the device until its gather and feeds the
shared window with lsmgnn_prefetch; rank r at
iteration t takes seeds perm[(t*G + r)*B : +B]. Counts-only: 16-byte rows (the counters do not
depend on the payload; bytes are reported for 4 KiB rows).

  --workload igb   configs[3] IGB-large-shaped: plcite N = 100M, m = 12, batch 8192 per GPU,
                   fanout (10,5,5), W = 256, warm-up + measured iterations of one epoch slice.
                   By I8 the summed per-home counters must EQUAL the one-home x G*L run of
                   tools/cfg4_counts.py on the same merged batches (profiles/r01_cfg4_counts.json):
                   a full-scale check of the directory and the exchange.
  --workload igbh  configs[4] IGBH-shaped point: typed ID ranges (paper 46%, author 53.7%, fos +
                   institute 0.3%) at N nodes, training seeds = 10% of the paper range, fanout
                   (5,2,2,2), batch 2048 per GPU; epoch 0 warms up, epoch 1 is measured
                   (R23); storage bytes per epoch per policy at one cache size.

usage: python -m torch.distributed.run --nproc-per-node G tools/ghome_run.py OUT.json
           [--workload igb|igbh] [--nodes N] [--lines-per-gpu L] [--cache-pct P]
           [--policies hybrid,static,lru,dynamic] [--period 1] [--iters 60 --warm 10]
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
SHM = "/dev/shm/lsmgnn_ghome"


def log(*a):
    print(f"[rank {os.environ.get('RANK', '0')}]", *a, file=sys.stderr, flush=True)


def shared_graph(rank, N, dist):
    """Rank 0 builds the graph + u8 scores once and writes them to /dev/shm; every rank maps them."""
    import synth
    t0 = time.time()
    if rank == 0:
        os.makedirs(SHM, exist_ok=True)
        g = synth.plcite_c(N, 12)
        g.indptr.tofile(f"{SHM}/indptr.bin")  # raw, so the mapping starts page-aligned
        g.indices.tofile(f"{SHM}/indices.bin")
        np.save(f"{SHM}/scores.npy", synth.static_scores(g))
        del g
    dist.barrier()
    # shared, writable mappings (cudaHostRegister refuses the read-only mapping np.load gives)
    indptr = np.memmap(f"{SHM}/indptr.bin", dtype=np.int64, mode="r+")
    indices = np.memmap(f"{SHM}/indices.bin", dtype=np.int32, mode="r+")
    scores = np.load(f"{SHM}/scores.npy")
    log(f"graph N={N} nnz={indices.size} ready in {time.time() - t0:.0f}s")
    return indptr, indices, scores


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--workload", default="igb", choices=["igb", "igbh"])
    ap.add_argument("--nodes", type=int, default=100_000_000)
    ap.add_argument("--lines-per-gpu", type=int, default=4_194_304)
    ap.add_argument("--cache-pct", type=float, default=None, help="igbh: box-wide cache size in % of the nodes")
    ap.add_argument("--policies", default="hybrid")
    ap.add_argument("--period", type=int, default=1)
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--warm", type=int, default=10)
    ap.add_argument("--max-ids", type=int, default=0, help="max_batch_ids per rank (0: from the workload)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, G = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dev = torch.device("cuda", torch.cuda.current_device())
    import synth
    from paper_2407_15264_b200 import LsmGnn, Sampler, STATS_FIELDS
    F = {n: i for i, n in enumerate(STATS_FIELDS)}
    N, W = args.nodes, 256
    indptr, indices, scores = shared_graph(rank, N, dist)
    if args.workload == "igb":
        B, fan = 8192, (10, 5, 5)
        perm = torch.from_numpy(synth.epoch_seeds(N, 0)).to(dev)
        K = args.warm + args.iters
        ipe = None
        lpg = args.lines_per_gpu
    else:
        B, fan = 2048, (5, 2, 2, 2)
        n_paper = int(0.46 * N)
        train = np.arange(0, n_paper, 10, dtype=np.int64)
        ipe = -(-train.size // (B * G))
        K = 2 * ipe
        perms = [torch.from_numpy(train[np.random.default_rng(3 + ep).permutation(train.size)]).to(dev)
                 for ep in range(2)]
        lpg = int(N * args.cache_pct / 100) // (32 * G) * 32
    bound = Sampler.bound(B, fan)
    cap = args.max_ids or bound
    samp = Sampler(indptr, indices, pin=False)  # page-locks the shared /dev/shm pages, zero-copy reads (UVA)
    Q = (N - rank + G - 1) // G
    table = torch.zeros((Q, 16), dtype=torch.uint8, pin_memory=True)
    res = {"workload": args.workload, "N": N, "G": G, "batch_per_gpu": B, "fanout": list(fan), "W": W,
           "lines_per_gpu": lpg, "cache_pct_boxwide": round(100 * G * lpg / N, 3), "period": args.period,
           "max_batch_ids": cap, "path": "G homes (one process each), CUDA IPC + stream-memory-op flags, GPU "
           "sampler (batches kept on the device until their gather) feeding lsmgnn_prefetch; 16-B rows, bytes reported x 4096", "runs": []}
    if ipe:
        res["iterations_per_epoch"] = ipe
    for pol in args.policies.split(","):
        c = LsmGnn(N, 4, lpg, 32, 0, scores, policy=pol, pvp=0, window=W, max_batch_ids=cap, period=args.period,
                   rank=rank, world=G, group=dist.group.WORLD)
        c.attach_storage(table)
        samp.reattach()
        bufs = {}
        scratch = torch.empty(bound, dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        empty = torch.zeros(0, dtype=torch.int64, device=dev)

        def batch(k):
            """this rank's list of iteration k (sampled once, kept compact until its gather)"""
            if k not in bufs:
                ids = empty
                # igb: every measured iteration sees a full window (batches sampled through K + W,
                # as tools/cfg4_counts.py did); igbh: the trace ends after two epochs
                if k < (K + W if not ipe else K):
                    if ipe:
                        ep, te = divmod(k, ipe)
                        lo = (te * G + rank) * B
                        seeds = perms[ep][lo:lo + B]
                    else:
                        seeds = perm[(k * G + rank) * B:(k * G + rank + 1) * B]
                    if seeds.numel():
                        samp.sample(seeds, fan, 4, k, rank, out=scratch, count=cnt)
                        ids = scratch[:int(cnt.item())].clone()
                bufs[k] = ids
                bufs.pop(k - W - 3, None)
            return bufs[k]

        t0 = time.time()
        c.prefetch([batch(k) for k in range(1, W + 1)], first_iter=1)
        out = torch.empty((cap, 16), dtype=torch.uint8, device=dev)
        for t in range(K):
            c.gather(batch(t), out)
            c.prefetch([batch(t + 1 + W)], first_iter=t + 1 + W)
        torch.cuda.synchronize()
        wall = time.time() - t0
        first, nrec = (args.warm, args.iters) if not ipe else (ipe, ipe)
        h = c.history(first, nrec).astype(np.int64)
        c.close()
        allh = [None] * G
        dist.all_gather_object(allh, h)
        if rank == 0:
            tot = sum(allh)  # summed over homes
            e = tot.sum(axis=0)
            u = max(int(e[F["unique"]]), 1)
            run = {"policy": pol, "hit_ratio": round(int(e[F["hits"]]) / u, 4),
                   "requests": int(e[F["requests"]]), "unique": u, "peer_requests": int(e[F["peer_requests"]]),
                   "storage_reads": int(e[F["storage_reads"]]), "bypassed": int(e[F["bypassed"]]),
                   "evictions": int(e[F["evictions"]]), "wall_s": round(wall, 1),
                   "per_home_unique": [int(x[:, F["unique"]].sum()) for x in allh]}
            if ipe:
                run["storage_GB_per_epoch_4KiB"] = round(run["storage_reads"] * 4096 / 1e9, 3)
            else:
                run["requests_per_iter"] = run["requests"] // args.iters
                run["unique_per_iter"] = u // args.iters
                run["storage_GB_per_iter_4KiB"] = round(run["storage_reads"] * 4096 / args.iters / 1e9, 3)
            res["runs"].append(run)
            print(json.dumps(run), flush=True)
            json.dump(res, open(args.out, "w"), indent=1)
        dist.barrier()
    if rank == 0:
        json.dump(res, open(args.out, "w"), indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Worker for multi-process tests: one rank of a G-rank run of the CUDA path.

Launched by tests/test_gpu_multiproc.py (GPU) and tests/test_mp_cpu.py (CPU, gloo) with
torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1. Every rank may share one
physical GPU (CUDA IPC within a device stands in for NVLink P2P on a 1-GPU pool).

usage: python -m torch.distributed.run ... tests/mp_worker.py MODE OUTDIR [policy pvp]
  MODE = gather  : run a config-1-shaped trace, save this home's per-iteration counters and
                   the number of rows that differ from F(v)
  MODE = cpu     : CPU-only host logic (handle exchange through gloo, layout checks)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    mode, outdir = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    if mode == "cpu":
        # host-side bootstrap logic of lsmgnn_connect, across two real processes over gloo: each
        # rank plans the handle it would export (lsmgnn_plan_handle, no GPU), the blobs are
        # all-gathered in rank order, and lsmgnn_connect's validation (lsmgnn_check_handles) runs
        # on every rank — matching layouts pass; rank order, world and layout mismatches fail
        from paper_2407_15264_b200 import LsmGnnError, check_handles, last_error, plan_handle
        ECOMM = -6
        res = {"rank": rank}

        def exchange(blob):
            blobs = [None] * world
            dist.all_gather_object(blobs, blob)
            return blobs

        base = dict(num_nodes=16384, feat_dim=128, lines_per_gpu=1024, ways=8, victim_lines=512, pvp=1, window=8,
                    max_batch_ids=4096)
        mine = plan_handle(**base, rank=rank, world=world)
        blobs = exchange(mine)
        res["ok"] = check_handles(blobs, mine)
        res["reversed"] = check_handles(blobs[::-1], mine)
        res["reversed_msg"] = last_error()
        res["short"] = check_handles(blobs[:1], mine)  # fewer handles than the world
        # rank 1 initialised with different arguments / options / world: every rank must refuse
        for name, change in (("lines", dict(lines_per_gpu=2048)), ("max_batch_ids", dict(max_batch_ids=4097)),
                             ("pvp", dict(pvp=0)), ("window", dict(window=16)), ("row_bytes", dict(feat_dim=132))):
            b = plan_handle(**dict(base, **change), rank=rank, world=world) if rank == 1 else mine
            res[name] = check_handles(exchange(b), mine)
            res[name + "_msg"] = last_error()
        w3 = plan_handle(**base, rank=rank, world=3) if rank == 1 else mine
        res["world"] = check_handles(exchange(w3), mine)
        res["world_msg"] = last_error()
        try:
            plan_handle(**dict(base, feat_dim=3), rank=rank, world=world)  # R = 12 bytes
            res["bad_args"] = "accepted"
        except LsmGnnError as e:
            res["bad_args"] = str(e)
        try:
            plan_handle(**base, rank=world, world=world)
            res["bad_rank"] = "accepted"
        except LsmGnnError as e:
            res["bad_rank"] = str(e)
        # the home partition each rank's batches are routed by (v mod G)
        import synth
        g = synth.plcite(4096, 4)
        tr = synth.make_trace(g, world, 32, (4, 2), 3)
        res["homes"] = [np.unique(tr[t][rank] % world).tolist() for t in range(3)]
        res["ECOMM"] = ECOMM
        json.dump(res, open(os.path.join(outdir, f"r{rank}.json"), "w"))
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "fuzz":  # many random small cases in one launch (the library re-initialises per case)
        torch.cuda.set_device(rank % torch.cuda.device_count())
        from tests.harness import run_gpu
        from tests.test_gpu_multiproc import random_mp_case
        ncases = int(sys.argv[3])
        for case in range(ncases):
            cfg, tr, sc = random_mp_case(case, world)
            hist, _, bad = run_gpu(tr, scores=sc, rank=rank, world=world, group=dist.group.WORLD,
                                   max_batch_ids=max(1, max(len(x) for row in tr for x in row)), **cfg)
            np.save(os.path.join(outdir, f"fz{case}_h{rank}.npy"), hist)
            assert bad == 0, (case, rank)
            dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "edge":  # ragged / empty / duplicate-heavy batches across ranks, tiny victim queues
        torch.cuda.set_device(rank % torch.cuda.device_count())
        from tests.harness import run_gpu
        z = np.load(os.path.join(outdir, "trace.npz"))
        K = len([k for k in z.files if k.endswith("_r0")])
        tr = [[z[f"t{t}_r{r}"] for r in range(world)] for t in range(K)]
        cfg = json.load(open(os.path.join(outdir, "cfg.json")))
        if cfg.pop("file", 0):  # file tier: this home's rows in its own file
            from tests.harness import write_table_file
            cfg["storage_file"] = write_table_file(os.path.join(outdir, f"home{rank}.bin"), cfg["N"], cfg["D"],
                                                   home=rank, G=world)
        hist, _, bad = run_gpu(tr, scores=z["scores"], rank=rank, world=world, group=dist.group.WORLD,
                               max_batch_ids=max(1, max(len(x) for row in tr for x in row)), **cfg)
        np.save(os.path.join(outdir, f"hist{rank}.npy"), hist)
        json.dump({"rank": rank, "bad": int(bad)}, open(os.path.join(outdir, f"r{rank}.json"), "w"))
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "mismatch":  # lsmgnn_connect must refuse a peer whose layout differs (ECOMM)
        torch.cuda.set_device(rank % torch.cuda.device_count())
        from paper_2407_15264_b200 import LsmGnn, LsmGnnError
        from tests.harness import table_for
        res = {"rank": rank, "mismatch_error": None}
        try:
            LsmGnn(4096, 32, 256 if rank == 0 else 512, 8, 0, None, window=4, max_batch_ids=64, rank=rank,
                   world=world, group=dist.group.WORLD)
        except LsmGnnError as e:
            res["mismatch_error"] = str(e)
        from paper_2407_15264_b200 import binding
        binding._LIB.lsmgnn_finalize()
        dist.barrier()
        c = LsmGnn(4096, 32, 256, 8, 0, None, window=4, max_batch_ids=64, rank=rank, world=world,
                   group=dist.group.WORLD)
        c.attach_storage(table_for(4096, 32, pinned=True, home=rank, G=world))
        ids = torch.arange(rank, 64 + rank, dtype=torch.int64, device="cuda")
        out = torch.empty((64, 128), dtype=torch.uint8, device="cuda")
        c.prefetch([ids] * 4, first_iter=1)
        c.gather(ids, out)
        torch.cuda.synchronize()
        import synth
        res["bad"] = int(synth.check_rows(out.cpu().numpy().view(np.uint32).reshape(64, 32), ids.cpu().numpy(), 32)[0])
        res["retry_ok"] = True
        c.close()
        json.dump(res, open(os.path.join(outdir, f"r{rank}.json"), "w"))
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "cfg3":  # full-size configs[2]: trace from the driver's npz
        torch.cuda.set_device(rank % torch.cuda.device_count())
        import synth
        from tests.harness import run_gpu
        wl = synth.CONFIGS["cfg3"]
        z = np.load(os.path.join(outdir, "trace.npz"))
        K = len([k for k in z.files if k.endswith("_r0")])
        tr = [[z[f"t{t}_r{r}"] for r in range(world)] for t in range(K)]
        hist, _, bad = run_gpu(tr, N=wl.N, D=wl.D, L=wl.lines_per_gpu, A=wl.ways, scores=z["scores"],
                               policy="hybrid", pvp=1, W=wl.window, V=wl.victim_lines, rank=rank, world=world,
                               group=dist.group.WORLD, max_batch_ids=max(len(x) for row in tr for x in row))
        np.save(os.path.join(outdir, f"hist{rank}.npy"), hist)
        json.dump({"rank": rank, "bad": int(bad)}, open(os.path.join(outdir, f"r{rank}.json"), "w"))
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "sampler":  # NEXT N3 at G > 1: each rank's GPU sampler feeds the shared window
        torch.cuda.set_device(rank % torch.cuda.device_count())
        import synth
        from paper_2407_15264_b200 import LsmGnn, Sampler, prefetch_dev
        from tests.harness import table_for
        pvp = int(sys.argv[3])
        N, D, W, K, B, fan = 16384, 128, 8, 20, 256, (10, 5)
        g = synth.plcite(N, 8)
        perm = synth.epoch_seeds(N, 0)
        bound = Sampler.bound(B, fan)
        c = LsmGnn(N, D, 1024, 8, 512, synth.static_scores(g), policy="hybrid", pvp=pvp, window=W,
                   max_batch_ids=bound, rank=rank, world=world, group=dist.group.WORLD)
        c.attach_storage(table_for(N, D, pinned=True, home=rank, G=world))
        s = Sampler(g.indptr, g.indices)
        lists = {}

        def sampled(k):  # batch k of this rank: seeds slot (k, rank) of the epoch permutation
            if k not in lists:
                if k < K:
                    sd = torch.from_numpy(perm[(k * world + rank) * B:(k * world + rank + 1) * B]).cuda()
                    lists[k] = s.sample(sd, fan, 4, k, rank)
                else:
                    lists[k] = (torch.zeros(1, dtype=torch.int64, device="cuda"),
                                torch.zeros(1, dtype=torch.int64, device="cuda"))
            return lists[k]

        for k in range(1, W + 1):
            prefetch_dev(*sampled(k), first_iter=k)
        out = torch.empty((bound, 4 * D), dtype=torch.uint8, device="cuda")
        bad = 0
        for t in range(K):
            ids, cnt = sampled(t)
            n = int(cnt.item())
            c.gather(ids[:n], out)
            prefetch_dev(*sampled(t + 1 + W), first_iter=t + 1 + W)
            c.prefetch([], first_iter=0)
            rows = out[:n].cpu().numpy().view(np.uint32).reshape(n, D)
            bad += synth.check_rows(rows, ids[:n].cpu().numpy(), D)[0]
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"hist{rank}.npy"), c.history(0, K))
        json.dump({"rank": rank, "bad": int(bad)}, open(os.path.join(outdir, f"r{rank}.json"), "w"))
        c.close()
        dist.destroy_process_group()
        return
    policy = sys.argv[3] if len(sys.argv) > 3 else "hybrid"
    pvp = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(rank % ndev)
    import synth
    from tests.harness import run_gpu
    N, D = 16384, 128
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, world, 256, (10, 5), 20)
    sc = synth.static_scores(g)
    hist, _, bad = run_gpu(tr, N=N, D=D, L=1024, A=8, scores=sc, policy=policy, pvp=pvp, W=8, V=512,
                           rank=rank, world=world, group=dist.group.WORLD,
                           max_batch_ids=max(len(x) for row in tr for x in row))
    np.save(os.path.join(outdir, f"hist{rank}.npy"), hist)
    json.dump({"rank": rank, "bad": int(bad)}, open(os.path.join(outdir, f"r{rank}.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

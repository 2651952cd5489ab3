"""Shared driver for parity tests and the bench: runs a trace through the CUDA path
(via the C-ABI binding) and through the CPU oracle on identical seeded inputs.

Both sides consume the same inputs from `synth` (graph, trace, scores, feature table);
neither computes anything for the other.
"""
from __future__ import annotations

import numpy as np

import synth


def table_for(N: int, D: int, seed_f: int = 5, pinned: bool = False, home: int = 0, G: int = 1):
    """Host feature table rows of home `home` (node home + k*G at row k), uint8 [rows, 4D]."""
    import torch
    rows = (N - home + G - 1) // G
    if pinned:
        t = torch.empty((rows, 4 * D), dtype=torch.uint8, pin_memory=True)
    else:
        t = torch.empty((rows, 4 * D), dtype=torch.uint8)
    if G == 1:
        synth.fill_features(t.data_ptr(), 0, rows, D, seed_f)
    else:
        ids = np.arange(home, N, G, dtype=np.int64)
        synth._lib().synth_fill_f32_ids(t.data_ptr(), ids.ctypes.data, ids.size, D, seed_f)
    return t


def run_gpu(trace, *, N, D, L, A, scores, policy="hybrid", pvp=0, W=8, T=0, V=0, reinsert=1, table=None,
            check_rows="full", max_batch_ids=None, rank=0, world=1, group=None, seed_f=5, keep_outs=False, P=1,
            state_cb=None, storage_file=None, two_streams=False, overlap=False):
    """Run trace[t][rank] through the library. Returns (history [K, 24] uint64, outs or None, bad_rows).

    check_rows: "full" compares every row with the closed form F(v); "none" skips it.
    overlap: no host synchronisation between the gathers (each into its own `out`, all rows
    checked at the end), so consecutive gathers can run concurrently (kernels.cuh k_dedup
    `early`); otherwise each `out` is read back right after its gather."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    K = len(trace)
    R = 4 * D
    mine = [np.asarray(trace[t][rank], np.int64) for t in range(K)]
    mb = max_batch_ids or max(1, max(x.size for x in mine))
    c = LsmGnn(N, D, L, A, V, scores, policy=policy, pvp=pvp, window=W, threshold=T, reinsert=reinsert,
               max_batch_ids=mb, rank=rank, world=world, group=group, period=P)
    if storage_file is not None:  # file tier: the same rows, read from a file per batch
        c.attach_storage_file(storage_file)
    else:
        if table is None:
            table = table_for(N, D, seed_f, pinned=True, home=rank, G=world)
        c.attach_storage(table)
    dev = torch.device("cuda", torch.cuda.current_device())
    ids_d = [torch.from_numpy(x).to(dev) for x in mine]
    empty = torch.zeros(0, dtype=torch.int64, device=dev)
    sb = None
    if two_streams:  # window feeds on their own stream (the library orders them by events)
        sb = torch.cuda.Stream()
        torch.cuda.synchronize()
    c.prefetch([ids_d[k] if k < K else empty for k in range(1, W + 1)], first_iter=1, stream=sb)
    outs = []
    pending = []
    bad = 0

    def check(t, out):
        nonlocal bad
        host = out[: ids_d[t].numel()].cpu().numpy()
        nb, _ = synth.check_rows(host.view(np.uint32).reshape(-1, D), mine[t], D, seed_f)
        bad += nb
        if keep_outs:
            outs.append(host)

    for t in range(K):
        out = torch.empty((max(1, ids_d[t].numel()), R), dtype=torch.uint8, device=dev)
        c.gather(ids_d[t], out)
        k = t + 1 + W
        c.prefetch([ids_d[k] if k < K else empty], first_iter=k, stream=sb)
        if check_rows == "full" and ids_d[t].numel():
            if overlap:
                pending.append((t, out))
            else:
                check(t, out)
    torch.cuda.synchronize()
    for t, out in pending:
        check(t, out)
    hist = c.history(0, K)
    if state_cb is not None:  # inspect the final cache state before the home is freed
        state_cb(c)
    c.close()
    return hist, (outs if keep_outs else None), bad


def run_oracle(trace, *, G, N, D, L, A, scores, policy="hybrid", pvp=0, W=8, T=0, V=0, reinsert=1, P=1):
    from oracle import Oracle, run_trace
    o = Oracle(G, N, 4 * D, L, A, scores, policy=policy, pvp=pvp, W=W, T=T, V=V, reinsert=reinsert, P=P)
    return run_trace(o, trace)


def small_workload(N=16384, m=8, G=1, batch=256, fanout=(10, 5), iters=20, dedup=True, seed_s=4):
    g = synth.plcite(N, m)
    tr = synth.make_trace(g, G, batch, fanout, iters, dedup=dedup, seed_s=seed_s)
    return g, tr, synth.static_scores(g)


def write_table_file(path, N: int, D: int, seed_f: int = 5, home: int = 0, G: int = 1, chunk: int = 1 << 16):
    """The file-tier layout of home `home`: its rows (node home + k*G at row k) back to back."""
    import torch
    rows = (N - home + G - 1) // G
    with open(path, "wb") as f:
        for r0 in range(0, rows, chunk):
            n = min(chunk, rows - r0)
            t = torch.empty((n, 4 * D), dtype=torch.uint8)
            ids = np.arange(home + r0 * G, home + (r0 + n) * G, G, dtype=np.int64)
            synth._lib().synth_fill_f32_ids(t.data_ptr(), ids.ctypes.data, ids.size, D, seed_f)
            f.write(t.numpy().tobytes())
    return str(path)

"""CUDA-graph step (-m gpu): one captured launch per iteration (gather + window feed, all
per-iteration values on the device) gives exactly the oracle's counters and F(v) rows, also
when mixed with direct gather/prefetch calls and with the PVP / periodic update on."""
import numpy as np
import pytest

import synth

from .harness import run_oracle, small_workload, table_for
from .test_gpu_parity import compare

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy,pvp,P", [("hybrid", 0, 1), ("hybrid", 1, 1), ("lru", 1, 2), ("dynamic", 0, 3)])
def test_graph_replay_parity(policy, pvp, P):
    import torch
    from paper_2407_15264_b200 import LsmGnn
    N, D, W = 16384, 128, 8
    g, tr, sc = small_workload(N, 8, G=1, batch=256, fanout=(10, 5), iters=20)
    K = len(tr)
    kw = dict(N=N, D=D, L=1024, A=8, scores=sc, policy=policy, pvp=pvp, W=W, V=512, P=P)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    mb = max(len(x[0]) for x in tr)
    c = LsmGnn(N, D, 1024, 8, 512, sc, policy=policy, pvp=pvp, window=W, max_batch_ids=mb, period=P)
    c.attach_storage(table_for(N, D, pinned=True))
    ring = [torch.from_numpy(np.asarray(tr[k][0], np.int64)).cuda() if k < K else
            torch.zeros(0, dtype=torch.int64, device="cuda") for k in range(K + W + 1)]
    out = torch.empty((mb, 4 * D), dtype=torch.uint8, device="cuda")
    c.prefetch(ring[1:W + 1], first_iter=1)
    # two direct steps, then capture and replay the rest (the styles mix)
    for t in range(2):
        c.gather(ring[t], out)
        c.prefetch([ring[t + 1 + W]], first_iter=t + 1 + W)
    c.graph_capture(ring, out)
    for t in range(2, K):
        c.graph_replay()
        n = ring[t].numel()
        rows = out[:n].cpu().numpy().view(np.uint32).reshape(n, D)
        assert synth.check_rows(rows, tr[t][0], D)[0] == 0, t
    torch.cuda.synchronize()
    compare(c.history(0, K), ho, f"graph {policy}/pvp{pvp}/P{P}")
    c.close()


@pytest.mark.parametrize("pvp", [0, 1])
def test_gather_and_prefetch_on_different_streams(pvp):
    """gather(t) on one stream, the window feed + PVP copy on another: the library orders
    them by events (a feed waits only for gather(t-1), the next gather waits for the feed),
    so the two may overlap — and the result is still the oracle's, bit for bit."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    N, D, W = 16384, 128, 8
    g, tr, sc = small_workload(N, 8, G=1, batch=256, fanout=(10, 5), iters=20)
    K = len(tr)
    kw = dict(N=N, D=D, L=1024, A=8, scores=sc, policy="hybrid", pvp=pvp, W=W, V=512)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    mb = max(len(x[0]) for x in tr)
    c = LsmGnn(N, D, 1024, 8, 512, sc, policy="hybrid", pvp=pvp, window=W, max_batch_ids=mb)
    c.attach_storage(table_for(N, D, pinned=True))
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ids = [torch.from_numpy(np.asarray(tr[k][0], np.int64)).cuda() if k < K else
           torch.zeros(0, dtype=torch.int64, device="cuda") for k in range(K + W + 1)]
    torch.cuda.synchronize()
    outs = [torch.empty((mb, 4 * D), dtype=torch.uint8, device="cuda") for _ in range(K)]
    c.prefetch(ids[1:W + 1], first_iter=1, stream=sb)
    for t in range(K):
        c.gather(ids[t], outs[t], stream=sa)
        c.prefetch([ids[t + 1 + W]], first_iter=t + 1 + W, stream=sb)
    torch.cuda.synchronize()
    for t in range(K):
        n = ids[t].numel()
        rows = outs[t][:n].cpu().numpy().view(np.uint32).reshape(n, D)
        assert synth.check_rows(rows, tr[t][0], D)[0] == 0, t
    compare(c.history(0, K), ho, f"two streams pvp{pvp}")
    c.close()


@pytest.mark.parametrize("pvp", [0, 1])
def test_gathers_alternate_streams(pvp):
    """gather(t) on alternating streams (and the feeds on a third): a gather on a new stream
    first waits for the previous gather (its k_dedup would otherwise reset the per-iteration
    state and scratch the previous k_serve still uses) — bit-exact rows and counters."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    N, D, W = 16384, 128, 8
    g, tr, sc = small_workload(N, 8, G=1, batch=256, fanout=(10, 5), iters=20)
    K = len(tr)
    kw = dict(N=N, D=D, L=1024, A=8, scores=sc, policy="hybrid", pvp=pvp, W=W, V=512)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    mb = max(len(x[0]) for x in tr)
    c = LsmGnn(N, D, 1024, 8, 512, sc, policy="hybrid", pvp=pvp, window=W, max_batch_ids=mb)
    c.attach_storage(table_for(N, D, pinned=True))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    sf = torch.cuda.Stream()
    ids = [torch.from_numpy(np.asarray(tr[k][0], np.int64)).cuda() if k < K else
           torch.zeros(0, dtype=torch.int64, device="cuda") for k in range(K + W + 1)]
    torch.cuda.synchronize()
    outs = [torch.empty((mb, 4 * D), dtype=torch.uint8, device="cuda") for _ in range(K)]
    c.prefetch(ids[1:W + 1], first_iter=1, stream=sf)
    for t in range(K):
        c.gather(ids[t], outs[t], stream=streams[t % 2])
        c.prefetch([ids[t + 1 + W]], first_iter=t + 1 + W, stream=sf if t % 3 else streams[t % 2])
    torch.cuda.synchronize()
    for t in range(K):
        n = ids[t].numel()
        rows = outs[t][:n].cpu().numpy().view(np.uint32).reshape(n, D)
        assert synth.check_rows(rows, tr[t][0], D)[0] == 0, t
    compare(c.history(0, K), ho, f"alternating streams pvp{pvp}")
    c.close()

"""GPU parity: CUDA path (through the C-ABI) vs the CPU oracle, bit-exact (-m gpu).

Bytes: every gathered row equals the closed form F(v) (= the oracle's plain gather
of the same synth table). Counts: every field of every per-iteration record equals
the oracle's, integer for integer.
"""
import numpy as np
import pytest

import synth
from oracle import COUNT_FIELDS

from .harness import run_gpu, run_oracle, small_workload

pytestmark = pytest.mark.gpu

F = {n: i for i, n in enumerate(COUNT_FIELDS)}


def compare(hg, ho, label=""):
    assert hg.shape == ho.shape, (hg.shape, ho.shape)
    if not np.array_equal(hg, ho):
        bad = np.argwhere(hg != ho)
        t, f = bad[0]
        raise AssertionError(f"{label}: first mismatch iter {t} field {COUNT_FIELDS[f]}: gpu {hg[t, f]} oracle "
                             f"{ho[t, f]} ({len(bad)} mismatching cells)\n gpu {hg[t]}\n orc {ho[t]}")


@pytest.fixture(scope="module")
def cfg1_g1():
    # configs[0] shape (16,384 nodes / 131,072 edges, fanout (10,5), batch 256, 8-way, 512 victim
    # lines, 20 batches) on ONE home: 1,024 lines
    return small_workload(16384, 8, G=1, batch=256, fanout=(10, 5), iters=20)


@pytest.mark.parametrize("policy", ["hybrid", "static", "lru", "rr", "dynamic"])
@pytest.mark.parametrize("pvp", [0, 1])
def test_cfg1_single_home(cfg1_g1, policy, pvp):
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=128, L=1024, A=8, scores=sc, policy=policy, pvp=pvp, W=8, V=512)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"{policy}/pvp{pvp}")
    assert ho[:, F["bypassed"]].sum() > 0  # the oversubscribed regime of config 1 is exercised
    if pvp:
        assert ho[:, F["victim_admitted"]].sum() > 0 and ho[:, F["victim_hits"]].sum() > 0


def test_duplicates_and_ragged():
    """Raw sampler lists with duplicates and ragged batch sizes."""
    g, tr, sc = small_workload(4096, 6, G=1, batch=64, fanout=(6, 3), iters=15, dedup=False)
    tr = [[x[: (7 * t) % len(x) + 1]] for t, (x,) in enumerate(tr)]
    kw = dict(N=4096, D=32, L=256, A=4, scores=sc, policy="hybrid", pvp=1, W=5, V=40)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho)
    assert ho[:, F["requests"]].sum() > ho[:, F["unique"]].sum()


@pytest.mark.parametrize("case", ["empty", "one_way", "full_assoc", "w1", "reinsert0", "tiny_queue", "thresh",
                                  "same_node", "no_window"])
def test_edge_cases(case):
    rng = np.random.default_rng(7)
    N, D = 2000, 4
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = [[rng.integers(0, N, int(rng.integers(0, 300)))] for _ in range(25)]
    kw = dict(N=N, D=D, L=64, A=8, scores=sc, policy="hybrid", pvp=1, W=6, V=60)
    if case == "empty":
        tr = [[np.zeros(0, np.int64)] if t % 3 == 0 else x for t, x in enumerate(tr)]
    elif case == "one_way":
        kw.update(L=32, A=1)
    elif case == "full_assoc":
        kw.update(L=32, A=32)
    elif case == "w1":
        kw.update(W=1, V=4)
    elif case == "reinsert0":
        kw.update(reinsert=0)
    elif case == "tiny_queue":
        kw.update(V=6)  # C = 1: queue overflow -> admission by node order
    elif case == "thresh":
        kw.update(T=4)
    elif case == "same_node":
        tr = [[np.full(50, 17, np.int64)] for _ in range(10)]
    elif case == "no_window":
        kw.update(pvp=0, policy="dynamic", W=1)
    hg, _, bad = run_gpu(tr, max_batch_ids=400, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, case)


def test_bad_ids_sticky_erange():
    import torch
    from paper_2407_15264_b200 import LsmGnn, LsmGnnError
    from .harness import table_for
    N, D = 100, 4
    c = LsmGnn(N, D, 16, 4, 0, np.zeros(N, np.uint8), window=2, max_batch_ids=16)
    c.attach_storage(table_for(N, D, pinned=True))
    ids = torch.tensor([1, 2, 150, 3], dtype=torch.int64, device="cuda")
    out = torch.full((4, 16), 7, dtype=torch.uint8, device="cuda")
    c.gather(ids, out)
    torch.cuda.synchronize()
    assert out[2].sum().item() == 0
    good = out[[0, 1, 3]].cpu().numpy().view(np.uint32).reshape(3, D)
    assert synth.check_rows(good, [1, 2, 3], D)[0] == 0
    with pytest.raises(LsmGnnError):
        c.stats()
    with pytest.raises(LsmGnnError):
        c.gather(ids, out)
    c.close()


def test_device_count_overflow_sticky():
    """A device-resident batch length beyond max_batch_ids (lsmgnn_prefetch_dev / graph ring)
    is clamped on the device — no out-of-bounds write — and reported as a sticky EINVAL."""
    import torch
    from paper_2407_15264_b200 import LsmGnn, LsmGnnError, prefetch_dev
    from .harness import table_for
    c = LsmGnn(100, 4, 16, 4, 0, None, window=2, max_batch_ids=8)
    c.attach_storage(table_for(100, 4, pinned=True))
    ids = torch.arange(20, dtype=torch.int64, device="cuda")
    prefetch_dev(ids, torch.tensor([20], dtype=torch.int64, device="cuda"), first_iter=1)
    torch.cuda.synchronize()
    with pytest.raises(LsmGnnError):
        c.stats()
    c.close()


def test_abi_errors():
    from paper_2407_15264_b200 import LsmGnn, LsmGnnError
    with pytest.raises(LsmGnnError):
        LsmGnn(100, 3, 16, 4)  # R = 12 bytes: not a multiple of 16
    with pytest.raises(LsmGnnError):
        LsmGnn(100, 4, 18, 4)  # lines not a multiple of ways
    with pytest.raises(LsmGnnError, match="2\\^31"):
        LsmGnn(2**31 + 8, 4, 64, 8, max_batch_ids=8)  # one home cannot index 2^31 rows in a fill record
    c = LsmGnn(100, 4, 16, 4, max_batch_ids=8)
    import torch
    ids = torch.zeros(9, dtype=torch.int64, device="cuda")
    out = torch.empty((9, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(LsmGnnError):
        c.gather(ids, out)  # no storage attached / n > max_batch_ids
    c.close()


@pytest.mark.parametrize("policy,pvp", [("hybrid", 0), ("hybrid", 1), ("static", 0), ("lru", 0)])
def test_cfg2_shape_reduced(policy, pvp):
    """configs[1] shape (IGB-small: 1M nodes, fanout (10,5,5), batch 1024, 10% cache, 32-way,
    W=256) with 64-dim rows and 12 iterations; counts must match exactly."""
    g = synth.plcite(1_000_000, 12)
    tr = synth.make_trace(g, 1, 1024, (10, 5, 5), 12)
    sc = synth.static_scores(g)
    kw = dict(N=1_000_000, D=16, L=100_000, A=32, scores=sc, policy=policy, pvp=pvp, W=256, V=256 * 64)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"cfg2/{policy}/pvp{pvp}")


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("policy,pvp", [("hybrid", 0), ("hybrid", 1), ("dynamic", 0)])
def test_update_period(cfg1_g1, P, policy, pvp):
    """NEXT N1: the paper's periodic dynamic-information update (P = 4 in P:607)
    with the Fresh class: the GPU's every-P-th window scan (k_snapshot) matches the
    oracle bit-exactly."""
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=128, L=1024, A=8, scores=sc, policy=policy, pvp=pvp, W=8, V=512, P=P)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"P={P}/{policy}/pvp{pvp}")
    kw1 = dict(kw, P=1)
    assert not np.array_equal(ho, run_oracle(tr, G=1, **kw1)[:, 0, :])  # the period changes decisions


@pytest.mark.parametrize("policy,pvp", [("hybrid", 1), ("lru", 0), ("rr", 0), ("dynamic", 1)])
def test_oversized_set_buckets(policy, pvp):
    """A few sets receiving thousands of distinct nodes per batch (more than k_set's shared
    memory holds): those sets are processed in global scratch — still bit-exact."""
    rng = np.random.default_rng(11)
    N, D = 200_000, 4
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = [[rng.integers(0, N, int(rng.integers(3000, 9000)))] for _ in range(12)]
    kw = dict(N=N, D=D, L=64, A=32, scores=sc, policy=policy, pvp=pvp, W=4, V=400)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"big sets {policy}/pvp{pvp}")


@pytest.mark.parametrize("policy,pvp", [("hybrid", 1), ("lru", 0)])
def test_multi_tile_set_scan(policy, pvp):
    """S = 12,000 sets: the set-offset scan spans three 4096-count tiles (k_scan's look-back
    carries), and two sets in later tiles receive > 1024 distinct nodes per batch, so their
    global-scratch regions are placed by the carried oversized-set offsets — bit-exact."""
    rng = np.random.default_rng(23)
    S, A = 12_000, 4
    N = 1_120 * S
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = []
    for _ in range(10):
        big = [s + S * rng.choice(1_120, 1_100, replace=False) for s in (5_000, 9_000)]
        tr.append([rng.permutation(np.concatenate(big + [rng.integers(0, N, 20_000)])).astype(np.int64)])
    kw = dict(N=N, D=4, L=S * A, A=A, scores=sc, policy=policy, pvp=pvp, W=4, V=4_000)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"multi-tile scan {policy}/pvp{pvp}")


@pytest.mark.parametrize("policy,pvp,P", [("hybrid", 1, 1), ("lru", 0, 1), ("rr", 1, 1), ("dynamic", 1, 2)])
def test_cache_state_parity(cfg1_g1, policy, pvp, P):
    """Stronger than equal counters: after every iteration the GPU's cache state equals the
    oracle's — the tag and last-use of every way of every set (way placement included) and
    the content of every victim queue (as a set: slot order within a batch's admissions is
    the atomic arrival order on the GPU)."""
    import torch
    from oracle import Oracle
    from paper_2407_15264_b200 import LsmGnn
    from .harness import table_for
    g, tr, sc = cfg1_g1
    N, D, L, A, W, V = 16384, 128, 1024, 8, 8, 512
    K = len(tr)
    o = Oracle(1, N, 4 * D, L, A, sc, policy=policy, pvp=pvp, W=W, V=V, P=P)
    mb = max(len(x[0]) for x in tr)
    c = LsmGnn(N, D, L, A, V, sc, policy=policy, pvp=pvp, window=W, max_batch_ids=mb, period=P)
    c.attach_storage(table_for(N, D, pinned=True))
    ids = [torch.from_numpy(np.asarray(x[0], np.int64)).cuda() for x in tr]
    ids += [torch.zeros(0, dtype=torch.int64, device="cuda")] * (W + 1)
    empty = [np.zeros(0, np.int64)]
    for k in range(1, W + 1):
        o.feed(k, tr[k] if k < K else empty)
    c.prefetch(ids[1:W + 1], first_iter=1)
    out = torch.empty((mb, 4 * D), dtype=torch.uint8, device="cuda")
    C = V // W
    for t in range(K):
        o.gather(t, tr[t])
        o.pvp_prefetch(t)
        o.feed(t + 1 + W, tr[t + 1 + W] if t + 1 + W < K else empty)
        c.gather(ids[t], out)
        c.prefetch([ids[t + 1 + W]], first_iter=t + 1 + W)
        ot, olu = o.tags(0)
        gt = c.debug_state(0, L).astype(np.int64)
        gt[gt == 0xFFFFFFFF] = -1
        assert np.array_equal(gt.reshape(ot.shape), ot), t
        assert np.array_equal(c.debug_state(1, L).astype(np.int64).reshape(olu.shape), olu), t
        if pvp:
            qlen = c.debug_state(2, W)
            qn = c.debug_state(3, W * C)
            for k in range(W):
                onodes, _ = o.queue(0, k)
                assert sorted(qn[k * C:k * C + qlen[k]].tolist()) == sorted(onodes.tolist()), (t, k)
    c.close()


def test_bf16_rows():
    """dtype only sets the row size (R = feat_dim x 2 for bf16/fp16): the gathered bytes and
    the counters are those of the same rows moved as bytes."""
    import torch
    from paper_2407_15264_b200 import BF16, LsmGnn
    from .harness import table_for
    rng = np.random.default_rng(3)
    N, D = 5000, 8  # 8 u32 words = 32 bytes = 16 bf16 values per row
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = [[rng.integers(0, N, 200)] for _ in range(10)]
    ho = run_oracle(tr, G=1, N=N, D=D, L=64, A=8, scores=sc, policy="hybrid", pvp=0, W=4)[:, 0, :]
    c = LsmGnn(N, 2 * D, 64, 8, 0, sc, dtype=BF16, window=4, max_batch_ids=200)
    c.attach_storage(table_for(N, D, pinned=True))
    ids = [torch.from_numpy(x[0]).cuda() for x in tr] + [torch.zeros(0, dtype=torch.int64, device="cuda")] * 5
    c.prefetch(ids[1:5], first_iter=1)
    out = torch.empty((200, 4 * D), dtype=torch.uint8, device="cuda")
    for t in range(10):
        c.gather(ids[t], out)
        c.prefetch([ids[t + 5]], first_iter=t + 5)
        assert synth.check_rows(out.cpu().numpy().view(np.uint32).reshape(200, D), tr[t][0], D)[0] == 0
    compare(c.history(0, 10), ho, "bf16")
    c.close()


def test_long_run_history_wrap():
    """6,000 iterations (the on-device history keeps the last 4,094): the cumulative counters
    and the last 4,094 per-iteration records still equal the oracle's (stamps, rings, wraps)."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    from .harness import table_for
    from oracle import Oracle, run_trace
    rng = np.random.default_rng(5)
    N, D, K, W = 3000, 4, 6000, 3
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = [[rng.integers(0, N, int(rng.integers(0, 60)))] for _ in range(K)]
    ho = run_trace(Oracle(1, N, 16, 64, 4, sc, policy="hybrid", pvp=1, W=W, V=8 * W), tr)[:, 0, :]
    c = LsmGnn(N, D, 64, 4, 8 * W, sc, policy="hybrid", pvp=1, window=W, max_batch_ids=60)
    c.attach_storage(table_for(N, D, pinned=True))
    ids = [torch.from_numpy(np.asarray(x[0], np.int64)).cuda() for x in tr]
    ids += [torch.zeros(0, dtype=torch.int64, device="cuda")] * (W + 1)
    c.prefetch(ids[1:W + 1], first_iter=1)
    out = torch.empty((64, 4 * D), dtype=torch.uint8, device="cuda")
    for t in range(K):
        c.gather(ids[t], out)
        c.prefetch([ids[t + 1 + W]], first_iter=t + 1 + W)
    torch.cuda.synchronize()
    compare(c.history(K - 4094, 4094), ho[K - 4094:], "history tail")
    with pytest.raises(Exception):
        c.history(K - 4095, 4095)  # the two slots ahead are already zeroed (end_record)
    cum = c.stats(1)
    from paper_2407_15264_b200 import STATS_FIELDS
    for i, f in enumerate(STATS_FIELDS[1:], 1):
        assert cum[f] == int(ho[:, i].sum()), f
    c.close()


def test_determinism_launch_geometry(cfg1_g1, monkeypatch):
    """I9: identical counters and bytes under a different launch geometry (one warp per CTA
    in k_set, one CTA per SM for every grid-stride kernel) — the batch-synchronous rules make
    the result independent of thread scheduling."""
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=128, L=1024, A=8, scores=sc, policy="hybrid", pvp=1, W=8, V=512)
    h1, _, bad1 = run_gpu(tr, **kw)
    monkeypatch.setenv("LSMGNN_GEOMETRY", "small")
    h2, _, bad2 = run_gpu(tr, **kw)
    assert bad1 == 0 and bad2 == 0
    compare(h1, h2, "geometry")


@pytest.mark.parametrize("D", [128, 1024])
@pytest.mark.parametrize("out_kind", ["pinned", "pageable"])
def test_gather_host_end_to_end(cfg1_g1, out_kind, D):
    """lsmgnn_gather_host (the e2e entry point: host IDs in, host rows out, copies inside the
    call): rows equal F(v) and every per-iteration counter equals the oracle's. Pinned `out`
    is written by the serve kernel over PCIe; pageable `out` goes through device staging."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    from .harness import table_for
    _, tr, sc = cfg1_g1
    N, W, K = 16384, 8, len(tr)
    mine = [np.asarray(tr[t][0], np.int64) for t in range(K)]
    # D = 1024: the bench's 4 KiB rows (k_serve<8, kHost> for pinned out — the e2e path)
    c = LsmGnn(N, D, 1024, 8, 512, sc, policy="hybrid", pvp=1, window=W, max_batch_ids=max(x.size for x in mine))
    c.attach_storage(table_for(N, D, 5, pinned=True))
    dev = torch.device("cuda", torch.cuda.current_device())
    ids_d = [torch.from_numpy(x).to(dev) for x in mine]
    empty = torch.zeros(0, dtype=torch.int64, device=dev)
    c.prefetch([ids_d[k] if k < K else empty for k in range(1, W + 1)], first_iter=1)
    bad = 0
    for t in range(K):
        hid = torch.from_numpy(mine[t]).pin_memory()
        n = mine[t].size
        if out_kind == "pinned":
            hout = torch.empty((max(n, 1), 4 * D), dtype=torch.uint8, pin_memory=True)
            c.gather_host(hid, hout)
            rows = hout[:n].numpy()
        else:
            hout = np.empty((max(n, 1), 4 * D), np.uint8)
            c.gather_host(hid, hout)
            rows = hout[:n]
        k = t + 1 + W
        c.prefetch([ids_d[k] if k < K else empty], first_iter=k)
        if n:
            nb, _ = synth.check_rows(rows.view(np.uint32).reshape(-1, D), mine[t], D, 5)
            bad += nb
    torch.cuda.synchronize()
    hg = c.history(0, K)
    c.close()
    assert bad == 0
    ho = run_oracle(tr, G=1, N=N, D=D, L=1024, A=8, scores=sc, policy="hybrid", pvp=1, W=W, V=512)[:, 0, :]
    compare(hg, ho, f"gather_host {out_kind} D{D}")


def test_launch_count_and_profile(cfg1_g1):
    """lsmgnn_kernel_launches and lsmgnn_profile/_read (what bench.py's gpu_launches and phases
    come from): a G = 1 step without PVP or periodic update is 4 kernels (dedup (+ the iteration's
    values, the clear of the leaving window slot and the hit probe), set (the sets with a miss),
    serve (its last CTA closes the record) + the window feed's route_local), and the profiled
    phase spans cover the step's phases with non-negative times."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    from .harness import table_for
    _, tr, sc = cfg1_g1
    N, D, W, K = 16384, 128, 8, len(tr)
    mine = [np.asarray(tr[t][0], np.int64) for t in range(K)]
    c = LsmGnn(N, D, 1024, 8, 0, sc, policy="hybrid", pvp=0, window=W, max_batch_ids=max(x.size for x in mine))
    c.attach_storage(table_for(N, D, 5, pinned=True))
    dev = torch.device("cuda", torch.cuda.current_device())
    ids_d = [torch.from_numpy(x).to(dev) for x in mine]
    out = torch.empty((max(x.size for x in mine), 4 * D), dtype=torch.uint8, device=dev)
    c.prefetch(ids_d[1:W + 1], first_iter=1)
    steps = K - W - 1
    c.profile(True)
    c.profile_read()
    n0 = c.kernel_launches()
    for t in range(steps):
        c.gather(ids_d[t], out)
        c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
    torch.cuda.synchronize()
    n1 = c.kernel_launches()
    prof = c.profile_read()
    c.profile(False)
    c.close()
    assert n1 - n0 == 4 * steps, (n1 - n0, steps)
    for ph in ("route", "dedup", "probe_replace", "fill", "window"):
        ms, cnt = prof[ph]
        assert cnt == steps and ms >= 0.0, (ph, prof[ph])
    assert prof["fill"][0] > 0.0

# ----------------------------------------------------------------------------- full row width
# The bench's rows are 4 KiB (1024 fp32 words): nvec = 256 selects the UNROLL = 8 kernel
# instantiations (k_serve<8>, k_pvp<8>, k_fill<8>, k_pull<8,..>). These cases run them against
# the oracle at that width.

@pytest.mark.parametrize("policy,V", [("hybrid", 64), ("hybrid", 512), ("dynamic", 64)])
def test_full_row_width_pvp(cfg1_g1, policy, V):
    """configs[0] trace on one home at R = 4 KiB with the PVP on: k_serve<8> fills with victim
    D2H into the pinned queues, serves staged rows and bypass rows; k_pvp<8> copies 4 KiB
    victim rows back. V = 64 (C = 8 per queue) overflows the queues (admission by node order)."""
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=1024, L=1024, A=8, scores=sc, policy=policy, pvp=1, W=8, V=V)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"4KiB {policy}/V{V}")
    assert ho[:, F["victim_hits"]].sum() > 0 and ho[:, F["victim_admitted"]].sum() > 0
    assert ho[:, F["bypassed"]].sum() > 0
    if V == 64:
        assert ho[:, F["victim_dropped"]].sum() > 0


def test_full_row_width_pvp_unused():
    """Windows that differ from the gathered batches (§8(b): "pvp_unused counts the
    mismatches"): staged 4 KiB rows the batch does not request are counted, not served."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    from oracle import Oracle
    from .harness import table_for
    rng = np.random.default_rng(41)
    N, D, L, A, W, V, K = 3000, 1024, 64, 8, 4, 4 * 32, 30
    sc = rng.integers(0, 256, N).astype(np.uint8)
    win = [[rng.integers(0, N, int(rng.integers(20, 120)))] for _ in range(K)]
    # gathered batch = the window batch with a random third of its IDs replaced
    gat = []
    for (x,) in win:
        y = x.copy()
        sel = rng.random(y.size) < 0.33
        y[sel] = rng.integers(0, N, int(sel.sum()))
        gat.append([y])
    o = Oracle(1, N, 4 * D, L, A, sc, policy="hybrid", pvp=1, W=W, V=V)
    empty = [np.zeros(0, np.int64)]
    for k in range(1, W + 1):
        o.feed(k, win[k])
    c = LsmGnn(N, D, L, A, V, sc, policy="hybrid", pvp=1, window=W, max_batch_ids=200)
    c.attach_storage(table_for(N, D, pinned=True))
    dw = [torch.from_numpy(np.asarray(x[0], np.int64)).cuda() for x in win] + \
        [torch.zeros(0, dtype=torch.int64, device="cuda")] * (W + 1)
    dg = [torch.from_numpy(np.asarray(x[0], np.int64)).cuda() for x in gat]
    c.prefetch(dw[1:W + 1], first_iter=1)
    out = torch.empty((200, 4 * D), dtype=torch.uint8, device="cuda")
    rows, bad = [], 0
    for t in range(K):
        oc, _ = o.gather(t, gat[t])
        rows.append(oc[0])
        o.pvp_prefetch(t)
        o.feed(t + 1 + W, win[t + 1 + W] if t + 1 + W < K else empty)
        c.gather(dg[t], out)
        c.prefetch([dw[t + 1 + W]], first_iter=t + 1 + W)
        n = dg[t].numel()
        bad += synth.check_rows(out[:n].cpu().numpy().view(np.uint32).reshape(n, D), gat[t][0], D)[0]
    hg = c.history(0, K)
    c.close()
    ho = np.stack(rows)
    assert bad == 0
    compare(hg, ho, "pvp_unused 4KiB")
    assert ho[:, F["pvp_unused"]].sum() > 0 and ho[:, F["victim_hits"]].sum() > 0


@pytest.mark.parametrize("D", [128, 1024])
@pytest.mark.parametrize("st", ["0", "3"])
def test_g1_pull_path(cfg1_g1, monkeypatch, D, st):
    """LSMGNN_G1_PULL=1 (the profiling aid) runs the G > 1 serve path on one home — k_fill, then
    k_pull phase 0 (rows in place) and phase 1 (rows filled this batch), k_end — with TMA rings
    (st = 3) or 16-B vector copies (st = 0): same rows and counters as the oracle."""
    monkeypatch.setenv("LSMGNN_G1_PULL", "1")
    monkeypatch.setenv("LSMGNN_SERVE_ST", st)
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=D, L=1024, A=8, scores=sc, policy="hybrid", pvp=1, W=8, V=512)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"g1 pull D{D} st{st}")


@pytest.mark.parametrize("st,tail,rounds,ahead", [("0", "8", "2", "1"), ("2", "1", "64", "1"), ("8", "32", "2", "0"),
                                                 ("6", "3", "0", "1"), ("6", "4", "1", "0")])
def test_serve_geometry(cfg1_g1, monkeypatch, st, tail, rounds, ahead):
    """k_serve's delivery with TMA rings of 2..8 stages per warp (8 is clamped to the shared
    memory) and with 16-B vector copies (LSMGNN_SERVE_ST), and guided chunk sizes down to one
    request (LSMGNN_SERVE_TAIL / _ROUNDS) at 4 KiB rows: identical rows and counters (I9 for the
    serve geometry)."""
    monkeypatch.setenv("LSMGNN_SERVE_ST", st)
    monkeypatch.setenv("LSMGNN_SERVE_CPS", "1")
    monkeypatch.setenv("LSMGNN_SERVE_TAIL", tail)
    monkeypatch.setenv("LSMGNN_SERVE_TAIL_ROUNDS", rounds)
    monkeypatch.setenv("LSMGNN_SERVE_AHEAD", ahead)
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=1024, L=1024, A=8, scores=sc, policy="lru", pvp=0, W=8)
    hg, _, bad = run_gpu(tr, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"serve st{st} tail{tail}/{rounds} ahead{ahead}")


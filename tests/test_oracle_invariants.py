"""Invariants I1-I10 (DESIGN.md §"Invariants") on random traces (-m "not gpu").

The oracle simulates any number of homes G in one process, so the multi-GPU
semantics (directory, exchange, shared-cache equivalence) are pinned here on CPU.
"""
import numpy as np
import pytest

import synth
from oracle import COUNT_FIELDS, Oracle, run_trace

F = {n: i for i, n in enumerate(COUNT_FIELDS)}
POLS = ["hybrid", "static", "lru", "rr", "dynamic"]


def rand_trace(rng, G, N, K, maxlen, dup=True):
    tr = []
    for _ in range(K):
        row = []
        for _ in range(G):
            n = int(rng.integers(0, maxlen + 1))
            x = rng.zipf(1.3, n) % N if n else np.zeros(0, np.int64)
            if not dup:
                x = synth.first_occurrence_unique(x)
            row.append(np.asarray(x, np.int64))
        tr.append(row)
    return tr


def run_checked(o, trace, C):
    """Drive the oracle like run_trace and check I2-I6 after every gather."""
    K, W, G = len(trace), o.W, o.G
    empty = [np.zeros(0, np.int64)] * G
    for k in range(1, W + 1):
        o.feed(k, trace[k] if k < K else empty)
    allc = []
    for t in range(K):
        before = [o.tags(g)[0].copy() for g in range(G)]
        c, _ = o.gather(t, trace[t])
        allc.append(c)
        # R10: a line hit by batch t is protected for the whole batch — still resident after it
        req = set(np.concatenate(trace[t]).tolist()) if trace[t] else set()
        for g in range(G):
            hit = req & set(before[g][before[g] >= 0].tolist())
            after = o.tags(g)[0]
            assert hit <= set(after[after >= 0].tolist()), f"t={t} home {g}: a hit line was evicted"
        # I3: requests = sum of list lengths routed by v mod G; unique = |union| (brute force)
        ids = np.concatenate(trace[t]) if trace[t] else np.zeros(0, np.int64)
        for g in range(G):
            mine = ids[ids % G == g]
            assert c[g, F["requests"]] == mine.size
            assert c[g, F["unique"]] == len(set(mine.tolist()))
            # I2
            assert c[g, F["hits"]] + c[g, F["victim_hits"]] + c[g, F["storage_reads"]] == c[g, F["unique"]]
            assert c[g, F["evictions"]] == c[g, F["evict_noreuse"]] + c[g, F["evict_far"]] + \
                c[g, F["evict_fresh"]] + c[g, F["evict_near"]]
            assert c[g, F["evictions"]] == c[g, F["victim_admitted"]] + c[g, F["victim_dropped"]] + \
                c[g, F["evicted_no_reuse"]]
        # I4 + I5 (exclusivity; homes own only their nodes)
        for g in range(G):
            tags, _ = o.tags(g)
            valid = tags[tags >= 0]
            assert valid.size == len(set(valid.tolist())), "node cached twice"
            assert np.all(valid % G == g)
            for s in range(o.S):
                row = tags[s][tags[s] >= 0]
                assert np.all((row // G) % o.S == s)
            in_q = []
            for k in range(W):
                nodes, reuse = o.queue(g, k)
                assert nodes.size <= C
                assert np.all(reuse % W == k)
                in_q += nodes.tolist()
            assert len(in_q) == len(set(in_q))
        # I6 class-minimality inside each set (not for RR, which has no key order)
        if o.policy != 3:
            ev = o.events()
            for (g, s) in set(map(tuple, ev[:, :2].tolist())):
                e = ev[(ev[:, 0] == g) & (ev[:, 1] == s)]
                keys = lambda kind: [tuple(r[4:7]) for r in e if r[2] == kind]
                evk, surv, byp, ins = keys(0), keys(1), keys(2), keys(3)
                if evk and surv:
                    assert max(evk) <= min(surv)
                if byp and ins:
                    assert max(byp) <= min(ins)
        o.pvp_prefetch(t)
        # I5 including the PVP staging buffer: a staged node is this home's, is staged once,
        # and is neither cached nor still queued (the copy empties its queue)
        for g in range(G):
            stg = o.staging(g).tolist()
            assert len(stg) == len(set(stg)) and all(x % G == g for x in stg)
            tags, _ = o.tags(g)
            assert not set(stg) & set(tags[tags >= 0].tolist()), f"t={t} home {g}: staged node also cached"
            queued = set()
            for k in range(W):
                queued |= set(o.queue(g, k)[0].tolist())
            assert not set(stg) & queued, f"t={t} home {g}: staged node still queued"
        o.feed(t + 1 + W, trace[t + 1 + W] if t + 1 + W < K else empty)
    return np.stack(allc)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("policy", POLS)
@pytest.mark.parametrize("pvp", [0, 1])
def test_invariants_random(G, policy, pvp):
    rng = np.random.default_rng(G * 100 + POLS.index(policy) * 10 + pvp)
    A, S, W = 4, 4, 6
    N = 40 * G
    C = 3
    o = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy=policy, pvp=pvp, W=W,
               V=C * W)
    trace = rand_trace(rng, G, N, 30, 25)
    c = run_checked(o, trace, C)
    # I10 cold start
    assert np.all(c[0, :, F["storage_reads"]] == c[0, :, F["unique"]])
    if pvp == 0:
        assert c[..., F["victim_hits"]].sum() == 0 and c[..., F["victim_admitted"]].sum() == 0


@pytest.mark.parametrize("seed", range(4))
def test_pvp_exactness(seed):
    """I7: windows = batches, prefetch every iteration => victim_hits(t) = pvp_prefetched(t),
    pvp_unused = 0."""
    rng = np.random.default_rng(seed)
    G, A, S, W = 2, 4, 2, 8
    N = 60
    o = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy="hybrid", pvp=1, W=W,
               V=1000 * W)
    trace = rand_trace(rng, G, N, 40, 20)
    c = run_trace(o, trace)
    assert np.array_equal(c[..., F["victim_hits"]], c[..., F["pvp_prefetched"]])
    assert c[..., F["pvp_unused"]].sum() == 0
    assert c[..., F["victim_admitted"]].sum() > 0  # the scenario exercises the PVP
    # with reinsert=0 the staged rows still match exactly
    o2 = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy="hybrid", pvp=1, W=W,
                V=1000 * W, reinsert=0)
    c2 = run_trace(o2, trace)
    assert np.array_equal(c2[..., F["victim_hits"]], c2[..., F["pvp_prefetched"]])


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("policy", POLS)
@pytest.mark.parametrize("pvp", [0, 1])
def test_shared_cache_equivalence(G, policy, pvp):
    """I8 (P:629 'comparable to ... twice as large'): G homes x L lines == 1 home x G*L lines
    on the merged batches, for every counter except peer_requests (pvp=1: no queue overflow)."""
    rng = np.random.default_rng(G + 7 * POLS.index(policy) + 50 * pvp)
    A, S, W = 4, 3, 5
    N = 30 * G
    sc = rng.integers(0, 256, N).astype(np.uint8)
    V = 10_000 * W
    trace = rand_trace(rng, G, N, 25, 20)
    merged = [[np.concatenate(row)] for row in trace]
    cg = run_trace(Oracle(G, N, 16, S * A, A, sc, policy=policy, pvp=pvp, W=W, V=V), trace)
    c1 = run_trace(Oracle(1, N, 16, G * S * A, A, sc, policy=policy, pvp=pvp, W=W, V=V), merged)
    sg = cg.sum(axis=1)
    s1 = c1.sum(axis=1)
    for name in COUNT_FIELDS:
        if name in ("iter", "peer_requests", "bytes_nvlink"):
            continue
        assert np.array_equal(sg[:, F[name]], s1[:, F[name]]), name


def test_determinism_and_bytes():
    """I9 (replay) and I1 (every out row is F(id), P1: index_select on the host table)."""
    g = synth.plcite(2048, 4)
    tr = synth.make_trace(g, 2, 32, (5, 3), 8, dedup=False)
    D = 8
    table = synth.features(np.arange(2048), D).view(np.uint8).reshape(2048, 4 * D)
    sc = synth.static_scores(g)
    runs = []
    for _ in range(2):
        o = Oracle(2, 2048, 4 * D, 64, 8, sc, policy="hybrid", pvp=1, W=4, V=64)
        c, outs = run_trace(o, tr, table=table)
        runs.append(c)
        for t, out in enumerate(outs):
            ids = np.concatenate(tr[t])
            assert synth.check_rows(out.view(np.uint32).reshape(-1, D), ids, D)[0] == 0
            assert np.array_equal(out, table[ids])
    assert np.array_equal(runs[0], runs[1])


def test_bad_ids_rejected():
    o = Oracle(1, 10, 16, 4, 2, np.zeros(10, np.uint8))
    with pytest.raises(RuntimeError):
        o.gather(0, [np.array([3, 10])])
    with pytest.raises(RuntimeError):
        o.feed(1, [np.array([-1])])


@pytest.mark.parametrize("P", [2, 3, 5])
@pytest.mark.parametrize("policy", ["hybrid", "dynamic"])
@pytest.mark.parametrize("pvp", [0, 1])
def test_invariants_update_period(P, policy, pvp):
    """I2-I6 hold with the periodic update (N1)."""
    rng = np.random.default_rng(P * 10 + pvp)
    G, A, S, W, C = 2, 4, 4, 6, 3
    N = 80
    o = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy=policy, pvp=pvp, W=W,
               V=C * W, P=P)
    c = run_checked(o, rand_trace(rng, G, N, 30, 25), C)
    assert c[..., F["evict_fresh"]].sum() > 0


@pytest.mark.parametrize("seed", range(6))
def test_north_star_reuse_protected(seed):
    """The north star's invariant, exact for hybrid with pvp = 0 and P = 1 (R21):
    a line whose dynamic reuse count is > 0 (Far/Near, key level > 0) is evicted only when no
    other candidate — no unprotected NoReuse line (level 0) — survives in its set."""
    rng = np.random.default_rng(seed)
    G, A, S, W = 2, 4, 3, 8
    N = 90
    o = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy="hybrid", pvp=0, W=W)
    trace = rand_trace(rng, G, N, 40, 30)
    K = len(trace)
    empty = [np.zeros(0, np.int64)] * G
    for k in range(1, W + 1):
        o.feed(k, trace[k] if k < K else empty)
    evicted_with_reuse = 0
    for t in range(K):
        o.gather(t, trace[t])
        ev = o.events()
        for (g, s) in set(map(tuple, ev[:, :2].tolist())):
            e = ev[(ev[:, 0] == g) & (ev[:, 1] == s)]
            if any(r[2] == 0 and r[4] > 0 for r in e):  # a line with reuse was evicted ...
                evicted_with_reuse += 1
                assert not any(r[2] == 1 and r[4] == 0 for r in e)  # ... so no NoReuse line survived
        o.pvp_prefetch(t)
        o.feed(t + 1 + W, trace[t + 1 + W] if t + 1 + W < K else empty)
    assert evicted_with_reuse > 0  # the situation occurs


@pytest.mark.parametrize("seed", range(6))
def test_pvp_staging_single_use(seed):
    """P:397-400 (R15-R17): the prefetching buffer holds the rows staged for the next
    iteration only. When the PVP copy is skipped after some gathers (the caller did not call
    prefetch), no victim-buffer hit can occur in the following gather: victim_hits(t) <=
    pvp_prefetched(t) at every t, and every row is served once from staging at most."""
    rng = np.random.default_rng(900 + seed)
    G, A, S, W, C = 1 + seed % 2, 2, 3, 4, 4
    N = 30 * G
    o = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy="hybrid", pvp=1, W=W,
               V=C * W, reinsert=int(seed % 3 == 0))
    trace = rand_trace(rng, G, N, 40, 20)
    K = len(trace)
    empty = [np.zeros(0, np.int64)] * G
    for k in range(1, W + 1):
        o.feed(k, trace[k] if k < K else empty)
    vh = 0
    for t in range(K):
        c, _ = o.gather(t, trace[t])
        assert np.all(c[:, F["victim_hits"]] <= c[:, F["pvp_prefetched"]]), t
        vh += int(c[:, F["victim_hits"]].sum())
        if rng.random() < 0.6:
            o.pvp_prefetch(t)
        o.feed(t + 1 + W, trace[t + 1 + W] if t + 1 + W < K else empty)
    assert vh > 0  # the case exercises the victim buffer


"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the pin (DESIGN.md §"Oracle pins") and the
passage it follows. None of them re-types the oracle's formulas: expected values
come from hand derivations, textbook algorithms written independently here
(dictionary LRU, cursor round-robin, brute-force Belady), or exhaustive
enumeration checked against the paper's prose ordering.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import COUNT_FIELDS, Oracle, run_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")
F = {n: i for i, n in enumerate(COUNT_FIELDS)}


def tot(counts, name):
    return int(counts[..., F[name]].sum())


# ----------------------------------------------------------------------------- P9
@pytest.mark.parametrize("run", json.load(open(os.path.join(GOLD, "appendix_a.json")))["runs"],
                         ids=lambda r: f"{r['policy']}-pvp{r['pvp']}")
def test_appendix_a_hand_derived(run):
    """P9: SURVEY.md Appendix A, hand-derived from P:360-371."""
    gold = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    su = gold["setup"]
    o = Oracle(su["G"], su["N"], su["R"], su["L"], su["A"], np.zeros(su["N"], np.uint8), policy=run["policy"],
               pvp=run["pvp"], W=su["W"], T=su["T"], V=su["V"])
    trace = [[np.array(b)] for b in gold["batches"]]
    c = run_trace(o, trace)
    for k in ("hits", "victim_hits", "storage_reads", "evictions", "victim_admitted", "pvp_prefetched"):
        assert tot(c, k) == run[k], k
    assert tot(c, "unique") == gold["unique_total"]
    assert tot(c, "hits") + tot(c, "victim_hits") + tot(c, "storage_reads") == gold["unique_total"]


def test_appendix_a_pvp_trajectory():
    """Appendix A notes: 2 evicted at t=1 with reuse 3 into queue 3, staged after gather(2),
    a VHIT at t=3 and re-inserted, evicting 1 (NoReuse, discarded)."""
    o = Oracle(1, 4, 16, 2, 2, np.zeros(4, np.uint8), policy="hybrid", pvp=1, W=4, V=16)
    trace = [[np.array(b)] for b in [[1, 2], [3], [1], [2], [3]]]
    for k in range(1, 5):
        o.feed(k, trace[k])
    o.gather(0, trace[0]); o.pvp_prefetch(0); o.feed(5, [np.zeros(0)])
    c1, _ = o.gather(1, trace[1])
    nodes, reuse = o.queue(0, 3)
    assert list(nodes) == [2] and list(reuse) == [3]
    assert c1[0, F["evict_far"]] == 1
    o.pvp_prefetch(1); o.feed(6, [np.zeros(0)])
    o.gather(2, trace[2]); o.pvp_prefetch(2); o.feed(7, [np.zeros(0)])
    assert list(o.staging(0)) == [2]
    c3, _ = o.gather(3, trace[3])
    assert c3[0, F["victim_hits"]] == 1 and c3[0, F["evict_noreuse"]] == 1
    assert c3[0, F["victim_admitted"]] == 0 and c3[0, F["evicted_no_reuse"]] == 1
    tags, _ = o.tags(0)
    assert sorted(tags[0]) == [2, 3]


# ----------------------------------------------------------------------------- P6
def test_p410_worked_example_queue_slot():
    """P6: P:410 — reuse 4 and counter 5 -> slot 5 of victim buffer 4."""
    gold = json.load(open(os.path.join(GOLD, "p410_worked_example.json")))
    A, W = 6, 8
    o = Oracle(1, 64, 16, A, A, np.zeros(64, np.uint8), policy="hybrid", pvp=1, W=W, T=1, V=16 * W)
    b0 = np.arange(10, 16)
    trace = [[b0], [np.arange(20, 26)], [np.zeros(0)], [np.zeros(0)], [b0]]
    for k in range(1, W + 1):
        o.feed(k, trace[k] if k < len(trace) else [np.zeros(0)])
    o.gather(0, trace[0]); o.pvp_prefetch(0); o.feed(W + 1, [np.zeros(0)])
    o.gather(1, trace[1])
    nodes, reuse = o.queue(0, gold["queue_index"])
    assert len(nodes) == gold["counter_before"] + 1
    # the entry that saw counter value 5 sits in slot 5 and carries reuse 4
    assert reuse[gold["slot"]] == gold["reuse"]
    assert nodes[gold["slot"]] == 15 and list(nodes) == list(range(10, 16))


# ----------------------------------------------------------------------------- P3 textbook
def _single_request_trace(rng, n_req, n_nodes):
    return [[np.array([int(rng.integers(0, n_nodes))])] for _ in range(n_req)]


def _textbook_lru(trace, S, A):
    sets = [[] for _ in range(S)]  # most-recent last
    hits = misses = ev = 0
    for b in trace:
        v = int(b[0][0])
        s = sets[v % S]
        if v in s:
            hits += 1
            s.remove(v)
            s.append(v)
        else:
            misses += 1
            if len(s) == A:
                s.pop(0)
                ev += 1
            s.append(v)
    return hits, misses, ev


def _textbook_rr(trace, S, A):
    ways = [[None] * A for _ in range(S)]
    cur = [0] * S
    hits = misses = ev = 0
    for b in trace:
        v = int(b[0][0])
        w = ways[v % S]
        if v in w:
            hits += 1
            continue
        misses += 1
        if None in w:
            w[w.index(None)] = v
        else:
            w[cur[v % S]] = v
            cur[v % S] = (cur[v % S] + 1) % A
            ev += 1
    return hits, misses, ev


def _textbook_static(trace, S, A, score):
    sets = [set() for _ in range(S)]
    hits = misses = ev = 0
    for b in trace:
        v = int(b[0][0])
        s = sets[v % S]
        if v in s:
            hits += 1
            continue
        misses += 1
        if len(s) == A:
            s.remove(min(s, key=lambda x: (score[x], x)))
            ev += 1
        s.add(v)
    return hits, misses, ev


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("policy", ["lru", "rr", "static"])
def test_textbook_reductions(seed, policy):
    """P3: G=1, one request per batch, pvp=0 — LRU / RR / STATIC reduce to the textbook
    per-set algorithms (dictionary+list LRU, cursor round-robin, evict-min-score)."""
    rng = np.random.default_rng(seed)
    S, A, N = int(rng.integers(1, 4)), int(rng.integers(1, 5)), int(rng.integers(4, 24))
    score = rng.integers(0, 256, N).astype(np.uint8)
    trace = _single_request_trace(rng, 60, N)
    o = Oracle(1, N, 16, S * A, A, score, policy=policy, pvp=0, W=4)
    c = run_trace(o, trace)
    want = {"lru": lambda: _textbook_lru(trace, S, A), "rr": lambda: _textbook_rr(trace, S, A),
            "static": lambda: _textbook_static(trace, S, A, score)}[policy]()
    assert (tot(c, "hits"), tot(c, "storage_reads"), tot(c, "evictions")) == want
    assert tot(c, "bypassed") == 0


def _belady_bruteforce(seq, A):
    """Minimum misses over all eviction choices, allocate-on-miss, one fully associative set."""
    best = [len(seq)]

    def rec(i, cache, misses):
        if misses >= best[0]:
            return
        if i == len(seq):
            best[0] = misses
            return
        v = seq[i]
        if v in cache:
            rec(i + 1, cache, misses)
        elif len(cache) < A:
            rec(i + 1, cache | {v}, misses + 1)
        else:
            for x in cache:
                rec(i + 1, (cache - {x}) | {v}, misses + 1)

    rec(0, frozenset(), 0)
    return best[0]


@pytest.mark.parametrize("seed", range(25))
def test_dynamic_is_belady(seed):
    """P3: DYNAMIC with W >= trace length is Belady's MIN — its miss count equals the
    brute-force minimum over all replacement choices (<=12 requests, <=3 ways)."""
    rng = np.random.default_rng(100 + seed)
    A = int(rng.integers(1, 4))
    n = int(rng.integers(4, 13))
    N = int(rng.integers(2, 7))
    seq = [int(x) for x in rng.integers(0, N, n)]
    trace = [[np.array([v])] for v in seq]
    o = Oracle(1, N, 16, A, A, np.zeros(N, np.uint8), policy="dynamic", pvp=0, W=n + 1)
    c = run_trace(o, trace)
    assert tot(c, "storage_reads") == _belady_bruteforce(seq, A)


# ----------------------------------------------------------------------------- P4 exhaustive
def _paper_victim(classes, scores, pvp):
    """P:361-369 (and P:434 with PVP): the lowest priority level first — no reuse, then
    reuse beyond the threshold, then recently inserted, then near reuse; with PVP the two
    lowest are swapped. Within a level, the lowest static value; then the lowest node ID."""
    order = ["far", "noreuse", "fresh", "near"] if pvp else ["noreuse", "far", "fresh", "near"]
    cands = [(order.index(classes[i]), scores[i], i + 1) for i in range(4)]
    return min(cands)[2]


@pytest.mark.parametrize("pvp", [0, 1])
def test_hybrid_victim_exhaustive(pvp):
    """P4: exhaustive {NoReuse, Far, Near} x {0,128,255} for 4 ways."""
    W, T = 8, 1
    cls_vals = ["noreuse", "far", "near"]
    score_vals = [0, 128, 255]
    n_checked = 0
    for classes in itertools.product(cls_vals, repeat=4):
        for scores in itertools.product(score_vals, repeat=4):
            N = 8
            sc = np.zeros(N, np.uint8)
            sc[1:5] = scores
            # nodes 1..4 resident after t=0; node 5 misses at t=1 and evicts one line.
            batches = {0: [1, 2, 3, 4], 1: [5]}
            for i, cl in enumerate(classes):
                k = {"near": 2, "far": 5}.get(cl)  # d = 1 <= T (near), d = 4 > T (far)
                if k is not None:
                    batches.setdefault(k, []).append(i + 1)
            trace = [[np.array(batches.get(k, []), np.int64)] for k in range(6)]
            o = Oracle(1, N, 16, 4, 4, sc, policy="hybrid", pvp=pvp, W=W, T=T, V=W * 4)
            for k in range(1, W + 1):
                o.feed(k, trace[k] if k < len(trace) else [np.zeros(0)])
            o.gather(0, trace[0])
            o.pvp_prefetch(0)
            o.feed(W + 1, [np.zeros(0)])
            c, _ = o.gather(1, trace[1])
            tags, _ = o.tags(0)
            gone = set(range(1, 5)) - set(tags[0].tolist())
            assert gone == {_paper_victim(classes, scores, pvp)}, (classes, scores)
            n_checked += 1
    assert n_checked == 81 * 81


# ----------------------------------------------------------------------------- P5
def _brute_next(trace_sets, v, t, W):
    for k in range(t + 1, t + W + 1):
        if k < len(trace_sets) and v in trace_sets[k]:
            return k
    return -1


@pytest.mark.parametrize("seed", range(6))
def test_next_reuse_linear_scan(seed):
    """P5: next_t(v) equals an independent linear window scan."""
    rng = np.random.default_rng(seed)
    G, N, W, K = int(rng.integers(1, 4)), 40, int(rng.integers(1, 9)), 25
    trace = [[rng.integers(0, N, int(rng.integers(0, 8))) for _ in range(G)] for _ in range(K)]
    sets = [set(np.concatenate(b).tolist()) if b else set() for b in trace]
    o = Oracle(G, N, 16, 4 * G, 2, np.zeros(N, np.uint8), W=W)
    empty = [np.zeros(0, np.int64)] * G
    for k in range(1, W + 1):
        o.feed(k, trace[k] if k < K else empty)
    for t in range(K):
        o.gather(t, trace[t])
        for v in range(N):
            assert o.next_use(v, t) == _brute_next(sets, v, t, W), (t, v)
        o.pvp_prefetch(t)
        o.feed(t + 1 + W, trace[t + 1 + W] if t + 1 + W < K else empty)


def test_next_reuse_spec_example():
    """a line reused at t+3 and t+90 has next reuse t+3."""
    gold = json.load(open(os.path.join(GOLD, "spec_examples.json")))["next_reuse"]
    W = gold["W"]
    o = Oracle(1, 8, 16, 2, 2, np.zeros(8, np.uint8), W=W)
    for k in range(1, W + 1):
        o.feed(k, [np.array([5]) if k in gold["appears_at_offsets"] else np.zeros(0)])
    o.gather(0, [np.array([5])])
    assert o.next_use(5, 0) == gold["expected_offset"]


# ----------------------------------------------------------------------------- P7
@pytest.mark.parametrize("seed", range(8))
def test_compulsory_misses_only(seed):
    """P7: if every set's distinct demand over the whole trace is <= A, storage_reads =
    distinct nodes ever requested, bypassed = 0 and evictions = 0."""
    rng = np.random.default_rng(seed)
    G, A, S = int(rng.integers(1, 4)), 4, 8
    N = G * S * A  # exactly A distinct nodes per (home, set)
    trace = [[rng.integers(0, N, 10) for _ in range(G)] for _ in range(15)]
    for pol in ["hybrid", "static", "lru", "rr", "dynamic"]:
        o = Oracle(G, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy=pol, W=4)
        c = run_trace(o, trace)
        distinct = len(set(np.concatenate([np.concatenate(b) for b in trace]).tolist()))
        assert tot(c, "storage_reads") == distinct
        assert tot(c, "bypassed") == 0 and tot(c, "evictions") == 0


# ----------------------------------------------------------------------------- split
def test_spec_split_example():
    """P2: SPEC S:295 — [9,4,2,7] on 2 devices -> home0 {4,2}, home1 {9,7}."""
    gold = json.load(open(os.path.join(GOLD, "spec_examples.json")))["split"]
    o = Oracle(gold["G"], 16, 16, 4, 2, np.zeros(16, np.uint8), W=2)
    c, _ = o.gather(0, [np.array(gold["ids"]), np.zeros(0, np.int64)])
    assert c[0, F["requests"]] == len(gold["home0"]) and c[1, F["requests"]] == len(gold["home1"])
    assert c[0, F["peer_requests"]] == 0 and c[1, F["peer_requests"]] == len(gold["home1"])


def test_quantize_example():
    gold = json.load(open(os.path.join(GOLD, "spec_examples.json")))["quantize"]
    assert synth.quantize_scores(np.array(gold["raw"])).tolist() == gold["scores"]


# ----------------------------------------------------------------------------- N1: update period P > 1
def test_update_period_hand_derived():
    """P:357-358 periodic update, P = 2, on the Appendix-A trace (hybrid, pvp = 0). Hand
    derivation: t0 (scan) 1,2 miss -> Fresh; t1 (no scan) 3 misses, both lines Fresh,
    lowest node 1 evicted; t2 (scan: 2 -> reuse 3 Near, 3 -> reuse 4 Far) 1 misses, 3
    evicted; t3 2 hits; t4 (scan: 1, 2 no reuse) 3 misses, 1 evicted. Totals: hits 1,
    storage 5, evictions 3 = Fresh 1 + Far 1 + NoReuse 1 (vs hits 2 / storage 4 at P = 1)."""
    o = Oracle(1, 4, 16, 2, 2, np.zeros(4, np.uint8), policy="hybrid", pvp=0, W=4, P=2)
    c = run_trace(o, [[np.array(b)] for b in [[1, 2], [3], [1], [2], [3]]])
    assert (tot(c, "hits"), tot(c, "storage_reads"), tot(c, "evictions")) == (1, 5, 3)
    assert (tot(c, "evict_noreuse"), tot(c, "evict_far"), tot(c, "evict_fresh"), tot(c, "evict_near")) == (1, 1, 1, 0)


def test_update_period_stale_snapshot_is_fresh():
    """R6: with P = 4 the window scan runs at t = 0 and t = 4 only. Hand
    derivation (1 line, W = 8): t0 node 0 missed and installed; t4 scan records its next
    reuse 5; t5 hit; t6 (no scan) node 1 misses and evicts node 0, whose recorded reuse 5
    has passed (<= 6) — no valid dynamic information, so the line is Fresh, not Near."""
    o = Oracle(1, 4, 16, 1, 1, np.zeros(4, np.uint8), policy="hybrid", pvp=0, W=8, P=4)
    c = run_trace(o, [[np.array(b, np.int64)] for b in [[0], [], [], [], [], [0], [1]]])
    assert (tot(c[5], "hits"), tot(c[6], "evictions")) == (1, 1)
    assert (tot(c[6], "evict_noreuse"), tot(c[6], "evict_far"), tot(c[6], "evict_fresh"),
            tot(c[6], "evict_near")) == (0, 0, 1, 0)


@pytest.mark.parametrize("T,cls", [(0, "evict_far"), (2, "evict_far"), (3, "evict_near")])
def test_threshold_default_w_over_8(T, cls):
    """P:365 (R4): the threshold defaults to W/8. Hand derivation (1 line, W = 16): node 0
    installed at t0, node 1 evicts it at t1 while its next reuse is iteration 4, d = 3:
    Far under the default T = 16/8 = 2 (and T = 2), Near once T >= 3."""
    o = Oracle(1, 4, 16, 1, 1, np.zeros(4, np.uint8), policy="hybrid", pvp=0, W=16, T=T)
    c = run_trace(o, [[np.array(b, np.int64)] for b in [[0], [1], [], [], [0]]])
    assert tot(c[1], "evictions") == 1 and tot(c[1], cls) == 1


@pytest.mark.parametrize("seed", range(8))
def test_update_period_never_reduces_to_static(seed):
    """With P longer than the trace, only the t = 0 scan happens (on an empty cache): every
    resident line is 'recently inserted' (Fresh) for the whole run, so HYBRID orders
    victims by (score, node) = STATIC, and DYNAMIC by node = STATIC with all-zero scores
    (no bypass at t = 0, where incoming misses still carry exact information)."""
    rng = np.random.default_rng(seed)
    N, S, A = 30, 2, 3
    sc = rng.integers(0, 256, N).astype(np.uint8)
    trace = [[np.array([int(rng.integers(0, N))])] for _ in range(40)]
    want = run_trace(Oracle(1, N, 16, S * A, A, sc, policy="static", W=6), trace)
    got = run_trace(Oracle(1, N, 16, S * A, A, sc, policy="hybrid", W=6, P=1000), trace)
    assert np.array_equal(want[..., 1:10], got[..., 1:10])
    z = np.zeros(N, np.uint8)
    want = run_trace(Oracle(1, N, 16, S * A, A, z, policy="static", W=6), trace)
    got = run_trace(Oracle(1, N, 16, S * A, A, sc, policy="dynamic", W=6, P=1000), trace)
    assert np.array_equal(want[..., 1:10], got[..., 1:10])
    # all lines Fresh: nothing carries reuse information, so PVP admits nothing
    c = run_trace(Oracle(1, N, 16, S * A, A, sc, policy="hybrid", pvp=1, W=6, V=60, P=1000), trace)
    assert tot(c, "victim_admitted") == 0 and tot(c, "evict_fresh") == tot(c, "evictions")


@pytest.mark.parametrize("seed", range(6))
def test_admission_order_on_overflow(seed):
    """R14 (P:408-409 leaves the order to the atomic race): when more victims with the same
    reuse iteration arrive than their queue has room for, the ones with the smallest node IDs
    are admitted — checked by brute force from the eviction log of each batch."""
    rng = np.random.default_rng(seed)
    A, S, W = 4, 4, 6
    N, C = 400, 2
    o = Oracle(1, N, 16, S * A, A, rng.integers(0, 256, N).astype(np.uint8), policy="hybrid", pvp=1, W=W,
               V=C * W)
    trace = [[rng.integers(0, N, 40)] for _ in range(30)]
    K = len(trace)
    empty = [np.zeros(0, np.int64)]
    for k in range(1, W + 1):
        o.feed(k, trace[k] if k < K else empty)
    overflowed = 0
    for t in range(K):
        before = {k: set(o.queue(0, k)[0].tolist()) for k in range(W)}
        c, _ = o.gather(t, trace[t])
        ev = o.events()
        evicted = [int(r[3]) for r in ev if r[2] == 0]
        # candidates: evicted lines that carried a reuse iteration (next use at decision time)
        cands = {}
        for x in evicted:
            nx = o.next_use(x, t)
            if nx >= 0:
                cands.setdefault(nx % W, []).append(x)
        for k, xs in cands.items():
            room = C - len(before[k])
            admitted = set(o.queue(0, k)[0].tolist()) - before[k]
            want = set(sorted(xs)[:max(0, room)])
            assert admitted == want, (t, k, sorted(xs), room, admitted)
            overflowed += len(xs) > room
        o.pvp_prefetch(t)
        o.feed(t + 1 + W, trace[t + 1 + W] if t + 1 + W < K else empty)
    assert overflowed > 0

def test_pvp_unused_window_mismatch():
    """§8(b) "pvp_unused counts the mismatches" when the window batches differ from the gathered
    ones: hand-derived trace (tests/golden/pvp_unused_window_mismatch.json) where the victim
    staged for iteration 3 (the window said {2}) is not requested by the batch gathered ({4})."""
    gold = json.load(open(os.path.join(GOLD, "pvp_unused_window_mismatch.json")))
    su = gold["setup"]
    o = Oracle(su["G"], su["N"], su["R"], su["L"], su["A"], np.zeros(su["N"], np.uint8), policy=su["policy"],
               pvp=su["pvp"], W=su["W"], T=su["T"], V=su["V"])
    win = [[np.array(b)] for b in gold["window_batches"]]
    gat = [[np.array(b)] for b in gold["gathered_batches"]]
    W, K = su["W"], len(gat)
    empty = [np.zeros(0, np.int64)]
    for k in range(1, W + 1):
        o.feed(k, win[k] if k < K else empty)
    rows = []
    for t in range(K):
        c, _ = o.gather(t, gat[t])
        rows.append(c[0])
        o.pvp_prefetch(t)
        o.feed(t + 1 + W, win[t + 1 + W] if t + 1 + W < K else empty)
    rows = np.stack(rows)
    for k, want in gold["per_iteration"].items():
        assert rows[:, F[k]].tolist() == want, k
    assert o.staging(0).size == 0  # single use: nothing staged after the last prefetch

"""Soft checks of the paper's reported trends on a synthetic power-law workload (-m "not gpu").
These are not exact pins (the paper's datasets are out of scope); they check that the oracle's
semantics reproduce the directions the paper reports:
  - P:629  the communication layer makes G shared caches behave like one G-times larger cache:
           shared hit ratio above private (M-GIDS) caches of the same size;
  - P:657, P:670  hybrid > static-only > Round-Robin in hit ratio;
  - P:692  the PVP raises the (hit + victim-hit) ratio of the hybrid policy;
  - P:657, "hybrid ... outperforms ... dynamic-only" — holds with the paper's periodic
           update of the dynamic information (P = 4; lines go stale or Fresh between
           scans), NOT with exact per-iteration information (P = 1, this build's
           default, R6): then dynamic-only is a windowed Belady MIN (pinned in
           test_oracle_pins::test_dynamic_is_belady) and the static score only adds noise.
           test_policy_ordering_by_update_period records which ordering holds at which P.
"""
import numpy as np
import pytest

import synth
from oracle import COUNT_FIELDS, Oracle, run_trace

F = {n: i for i, n in enumerate(COUNT_FIELDS)}


@pytest.fixture(scope="module")
def workload():
    N, G = 40000, 2
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, G, 128, (5, 2, 2), 60)
    return N, G, tr, synth.static_scores(g)


def hit_ratio(c, skip=20):
    c = c[skip:]
    return (c[..., F["hits"]].sum() + c[..., F["victim_hits"]].sum()) / c[..., F["unique"]].sum()


def test_shared_cache_beats_private(workload):
    N, G, tr, sc = workload
    L, A, W = 2048, 32, 32
    shared = hit_ratio(run_trace(Oracle(G, N, 16, L, A, sc, policy="rr", W=W), tr))
    private = np.mean([hit_ratio(run_trace(Oracle(1, N, 16, L, A, sc, policy="rr", W=W), [[row[r]] for row in tr]))
                       for r in range(G)])
    private2x = np.mean([hit_ratio(run_trace(Oracle(1, N, 16, 2 * L, A, sc, policy="rr", W=W),
                                             [[row[r]] for row in tr])) for r in range(G)])
    assert shared > private
    assert abs(shared - private2x) < abs(private - private2x) + 0.02  # "comparable to ... twice as large"


def test_policy_ordering(workload):
    N, G, tr, sc = workload
    L, A, W = 4096, 32, 32
    h = {p: hit_ratio(run_trace(Oracle(G, N, 16, L, A, sc, policy=p, W=W), tr)) for p in ("hybrid", "static", "rr")}
    assert h["hybrid"] > h["static"] > h["rr"], h


def test_pvp_raises_hit_ratio(workload):
    N, G, tr, sc = workload
    L, A, W = 4096, 32, 32
    off = hit_ratio(run_trace(Oracle(G, N, 16, L, A, sc, policy="hybrid", pvp=0, W=W), tr))
    on = hit_ratio(run_trace(Oracle(G, N, 16, L, A, sc, policy="hybrid", pvp=1, W=W, V=W * 2048), tr))
    assert on > off


@pytest.mark.parametrize("L", [2048, 4096])
def test_policy_ordering_by_update_period(workload, L):
    """Which of hybrid / dynamic-only wins depends on the update period P:
    P = 4 and 8 (the paper's periodic scan): hybrid > dynamic-only;
    P = 1 (exact information every iteration): dynamic-only >= hybrid. Hybrid beats static-only
    at every P."""
    N, G, tr, sc = workload
    A, W = 32, 32
    res = {}
    for P in (1, 4, 8):
        res[P] = {p: hit_ratio(run_trace(Oracle(G, N, 16, L, A, sc, policy=p, W=W, P=P), tr))
                  for p in ("hybrid", "dynamic", "static")}
    assert res[1]["dynamic"] >= res[1]["hybrid"], res
    for P in (4, 8):
        assert res[P]["hybrid"] > res[P]["dynamic"], (P, res)
    for P in res:
        assert res[P]["hybrid"] > res[P]["static"], (P, res)
    # exact information never hurts dynamic-only (stale/Fresh information is what hybrid's score covers)
    assert res[1]["dynamic"] > res[4]["dynamic"] > res[8]["dynamic"], res

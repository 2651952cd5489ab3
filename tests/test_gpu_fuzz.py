"""Randomised parity (-m gpu): many small random configurations — ways, sets, window,
threshold, policy, PVP, victim capacity, re-insertion, update period, row size, batch
shapes with duplicates and empty batches — each compared with the oracle counter by counter
and row by row. A net for corner cases the structured tests do not enumerate."""
import os

import numpy as np
import pytest

from .harness import run_gpu, run_oracle
from .test_gpu_parity import compare

pytestmark = pytest.mark.gpu

POLICIES = ["hybrid", "static", "lru", "rr", "dynamic"]


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    A = int(rng.choice([1, 2, 3, 4, 7, 8, 16, 32]))
    S = int(rng.integers(1, 40))
    N = int(rng.integers(max(2, A * S // 2), A * S * 6 + 50))
    W = int(rng.integers(1, 12))
    cfg = dict(N=N, D=int(rng.choice([4, 8, 32])), L=A * S, A=A, policy=str(rng.choice(POLICIES)),
               pvp=int(rng.integers(0, 2)), W=W, T=int(rng.integers(0, W + 1)), V=int(rng.integers(W, 8 * W)),
               reinsert=int(rng.integers(0, 2)), P=int(rng.choice([1, 1, 2, 3])))
    K = int(rng.integers(5, 30))
    tr = []
    for _ in range(K):
        n = int(rng.integers(0, 3 * A * S + 5)) if rng.random() > 0.1 else 0
        x = rng.zipf(1.3, n) % N if rng.random() < 0.5 else rng.integers(0, N, n)
        tr.append([np.asarray(x, np.int64)])
    sc = rng.integers(0, 256, N).astype(np.uint8)
    return cfg, tr, sc


@pytest.mark.parametrize("seed", range(int(os.environ.get("LSMGNN_FUZZ", "40"))))
def test_fuzz_parity(seed):
    from oracle import Oracle, run_trace
    cfg, tr, sc = random_case(seed)
    state = {}
    hg, _, bad = run_gpu(tr, scores=sc, max_batch_ids=max(1, max(len(x[0]) for x in tr)),
                         state_cb=lambda c: state.update(tags=c.debug_state(0, cfg["L"]),
                                                         lu=c.debug_state(1, cfg["L"])), **cfg)
    o = Oracle(1, cfg["N"], 4 * cfg["D"], cfg["L"], cfg["A"], sc, policy=cfg["policy"], pvp=cfg["pvp"], W=cfg["W"],
               T=cfg["T"], V=cfg["V"], reinsert=cfg["reinsert"], P=cfg["P"])
    ho = run_trace(o, tr)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"fuzz {seed}: {cfg}")
    # the final cache state, way by way
    ot, olu = o.tags(0)
    gt = state["tags"].astype(np.int64)
    gt[gt == 0xFFFFFFFF] = -1
    assert np.array_equal(gt, ot.reshape(-1)) and np.array_equal(state["lu"].astype(np.int64), olu.reshape(-1))


@pytest.mark.parametrize("seed", range(int(os.environ.get("LSMGNN_FUZZ_OVERLAP", "20"))))
def test_fuzz_parity_overlapped(seed):
    """The same random configurations without a victim buffer (the condition for consecutive
    gathers to overlap) and without any host synchronisation between the gathers."""
    from oracle import Oracle, run_trace
    cfg, tr, sc = random_case(500 + seed)
    cfg["pvp"] = 0
    cfg["V"] = 0  # no victim buffer: the overlap is off whenever one exists
    hg, _, bad = run_gpu(tr, scores=sc, max_batch_ids=max(1, max(len(x[0]) for x in tr)), overlap=True, **cfg)
    o = Oracle(1, cfg["N"], 4 * cfg["D"], cfg["L"], cfg["A"], sc, policy=cfg["policy"], pvp=0, W=cfg["W"],
               T=cfg["T"], V=cfg["V"], reinsert=cfg["reinsert"], P=cfg["P"])
    ho = run_trace(o, tr)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"overlapped fuzz {seed}: {cfg}")

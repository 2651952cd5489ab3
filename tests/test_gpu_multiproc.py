"""G > 1 parity (-m gpu): G processes, one home each, exchanging node IDs, flags and rows
through CUDA IPC mappings and stream memory operations — the communication layer of
P:294-313. On a 1-GPU pool all ranks share cuda:0. Every home's per-iteration counters
must equal the oracle's G-home simulation, and every row must equal F(v)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth

from .harness import run_oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(G, tmp, *args, timeout=600, split=1):
    """split: LSMGNN_SPLIT_PULL for the ranks — 1 forces pull phase 0 onto its own stream
    concurrent with k_fill (the default on distinct GPUs), 0 runs both phases after "served"
    (the default when ranks share a GPU, as here); both must be bit-exact."""
    env = dict(os.environ)
    env.pop("LSMGNN_SPLIT_PULL", None)
    if split is not None:  # None: the library's own choice (ranks here share a GPU => unsplit)
        env["LSMGNN_SPLIT_PULL"] = str(split)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mp_worker.py"), *args]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]


def random_mp_case(seed, G):
    """A random small G-home case (same for every rank: derived from the seed only)."""
    rng = np.random.default_rng(5000 + 37 * seed + G)
    A = int(rng.choice([1, 2, 4, 8, 32]))
    S = int(rng.integers(1, 20))
    N = int(rng.integers(G * A * S // 2 + G, G * A * S * 5 + 50))
    W = int(rng.integers(1, 10))
    cfg = dict(N=N, D=int(rng.choice([4, 16])), L=A * S, A=A,
               policy=str(rng.choice(["hybrid", "static", "lru", "rr", "dynamic"])), pvp=int(rng.integers(0, 2)),
               W=W, T=int(rng.integers(0, W + 1)), V=int(rng.integers(W, 6 * W)), reinsert=int(rng.integers(0, 2)),
               P=int(rng.choice([1, 1, 2])))
    K = int(rng.integers(4, 16))
    tr = [[np.asarray(rng.integers(0, N, int(rng.integers(0, 2 * A * S * G + 3))) if rng.random() > 0.15
                      else np.zeros(0, np.int64), np.int64) for _ in range(G)] for _ in range(K)]
    return cfg, tr, rng.integers(0, 256, N).astype(np.uint8)


@pytest.mark.parametrize("split", [0, 1])
@pytest.mark.parametrize("G", [2, 3])
def test_multiprocess_fuzz(tmp_path, G, split):
    """Random small G-home cases (one process launch runs them all): every home's counters
    equal the oracle's."""
    n = int(os.environ.get("LSMGNN_MP_FUZZ", "12"))
    launch(G, tmp_path, "fuzz", str(tmp_path), str(n), timeout=1200, split=split)
    for case in range(n):
        cfg, tr, sc = random_mp_case(case, G)
        ho = run_oracle(tr, G=G, scores=sc, **cfg)
        for r in range(G):
            hg = np.load(tmp_path / f"fz{case}_h{r}.npy")
            assert np.array_equal(hg, ho[:, r, :]), (case, r, cfg, np.argwhere(hg != ho[:, r, :])[:3])


@pytest.mark.parametrize("G,case,split", [(2, "ragged", 1), (3, "dups", 0), (3, "dups", 1), (2, "period", 1),
                                          (4, "rr", None), (2, "file", 1), (3, "two_streams", 1), (3, "skew", 1)])
def test_multiprocess_edge_cases(tmp_path, G, case, split):
    """Ranks with empty batches, cross-rank duplicates, raw lists, victim-queue overflow,
    reinsert = 0, the periodic update, RR, and a home whose window slots overflow the ring (every
    rank's batch homed there: the slot's bits are cleared by a sweep) — per-home counters equal
    the oracle's."""
    rng = np.random.default_rng(G * 7 + len(case))
    N, D, K = 3000, 4, 18
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = []
    for t in range(K):
        row = []
        for r in range(G):
            n = 0 if (case == "ragged" and (t + r) % 3 == 0) else int(rng.integers(1, 400))
            x = rng.zipf(1.2, n) % N if case == "dups" else rng.integers(0, N, n)
            if case == "skew":  # every ID at home 0 on odd iterations: its window slot overflows the
                n = 399        # ring (3 ranks x max_batch_ids > 2 x max_batch_ids) and is swept instead
                x = 3 * rng.integers(0, N // 3, n) if t % 2 else rng.integers(0, N, n)
            row.append(np.asarray(x, np.int64))
        tr.append(row)
    cfg = dict(N=N, D=D, L=64 * 8, A=8, policy="hybrid", pvp=1, W=5, V=5 * 2, reinsert=1, P=1)
    if case == "period":
        cfg.update(P=3, reinsert=0)
    if case == "rr":
        cfg.update(policy="rr", pvp=0)
    if case == "file":  # NEXT N2: every home reads its rows from its own file (k_fill path)
        cfg.update(D=128, file=1)
    if case == "two_streams":  # window feeds (and their exchange) on a second stream
        cfg.update(two_streams=True)
    np.savez(tmp_path / "trace.npz", scores=sc, **{f"t{t}_r{r}": tr[t][r] for t in range(K) for r in range(G)})
    json.dump(cfg, open(tmp_path / "cfg.json", "w"))
    launch(G, tmp_path, "edge", str(tmp_path), split=split)
    cfg.pop("file", None)
    cfg.pop("two_streams", None)
    ho = run_oracle(tr, G=G, scores=sc, **cfg)
    for r in range(G):
        assert json.load(open(tmp_path / f"r{r}.json"))["bad"] == 0
        hg = np.load(tmp_path / f"hist{r}.npy")
        assert np.array_equal(hg, ho[:, r, :]), (case, r, np.argwhere(hg != ho[:, r, :])[:3])


@pytest.mark.parametrize("G,policy,pvp,split", [(2, "hybrid", 1, 1), (2, "lru", 0, 0), (3, "hybrid", 0, 1),
                                               (4, "static", 1, 0), (8, "hybrid", 1, 1), (8, "hybrid", 0, 0)])
def test_multiprocess_parity(tmp_path, G, policy, pvp, split):
    launch(G, tmp_path, "gather", str(tmp_path), policy, str(pvp), split=split)
    N, D = 16384, 128
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, G, 256, (10, 5), 20)
    sc = synth.static_scores(g)
    ho = run_oracle(tr, G=G, N=N, D=D, L=1024, A=8, scores=sc, policy=policy, pvp=pvp, W=8, V=512)
    for r in range(G):
        meta = json.load(open(tmp_path / f"r{r}.json"))
        assert meta["bad"] == 0
        hg = np.load(tmp_path / f"hist{r}.npy")
        if not np.array_equal(hg, ho[:, r, :]):
            bad = np.argwhere(hg != ho[:, r, :])
            raise AssertionError(f"home {r}: {len(bad)} mismatches, first {bad[0]}: gpu {hg[bad[0][0]]} "
                                 f"oracle {ho[bad[0][0], r]}")
    assert ho[:, :, 2].sum() > 0  # peer requests crossed homes
    if pvp == 0:
        # SURVEY.md §4 "Equivalence" on the GPU: G homes x L lines == 1 home x G*L lines on the
        # merged batches (I8) — pins the directory and the exchange GPU against GPU
        from .harness import run_gpu
        merged = [[np.concatenate(row)] for row in tr]
        h1, _, bad = run_gpu(merged, N=N, D=D, L=G * 1024, A=8, scores=sc, policy=policy, pvp=0, W=8)
        assert bad == 0
        hg = sum(np.load(tmp_path / f"hist{r}.npy").astype(np.int64) for r in range(G))
        skip = {0, 2, 20}  # iter, peer_requests, bytes_nvlink
        for f in range(hg.shape[1]):
            if f not in skip:
                assert np.array_equal(hg[:, f], h1[:, f].astype(np.int64)), f


@pytest.mark.parametrize("G,pvp,split", [(2, 1, 1), (3, 0, 0)])
def test_multiprocess_gpu_sampler_window(tmp_path, G, pvp, split):
    """NEXT N3 at G > 1: every rank samples its own batches on the GPU and feeds the shared
    window with lsmgnn_prefetch_dev (the length never leaves the device); per-home counters
    equal the oracle's G-home run over the sampler oracle's lists, rows equal F(v)."""
    import oracle
    launch(G, tmp_path, "sampler", str(tmp_path), str(pvp), split=split)
    N, D, W, K, B, fan = 16384, 128, 8, 20, 256, (10, 5)
    g = synth.plcite(N, 8)
    perm = synth.epoch_seeds(N, 0)
    tr = [[oracle.sample_batch(g.indptr, g.indices, perm[(t * G + r) * B:(t * G + r + 1) * B], fan, 4, t, r)
           for r in range(G)] for t in range(K)]
    ho = run_oracle(tr, G=G, N=N, D=D, L=1024, A=8, scores=synth.static_scores(g), policy="hybrid", pvp=pvp, W=W,
                    V=512)
    for r in range(G):
        assert json.load(open(tmp_path / f"r{r}.json"))["bad"] == 0
        hg = np.load(tmp_path / f"hist{r}.npy")
        assert np.array_equal(hg, ho[:, r, :]), (r, np.argwhere(hg != ho[:, r, :])[:3])
    assert ho[:, :, 2].sum() > 0

def _run_edge(tmp_path, G, tr, sc, cfg, split):
    np.savez(tmp_path / "trace.npz", scores=sc, **{f"t{t}_r{r}": tr[t][r] for t in range(len(tr)) for r in range(G)})
    json.dump(cfg, open(tmp_path / "cfg.json", "w"))
    launch(G, tmp_path, "edge", str(tmp_path), split=split)
    cfg = dict(cfg)
    cfg.pop("file", None)
    cfg.pop("two_streams", None)
    ho = run_oracle(tr, G=G, scores=sc, **cfg)
    for r in range(G):
        assert json.load(open(tmp_path / f"r{r}.json"))["bad"] == 0
        hg = np.load(tmp_path / f"hist{r}.npy")
        assert np.array_equal(hg, ho[:, r, :]), (r, np.argwhere(hg != ho[:, r, :])[:3])
    return ho


@pytest.mark.parametrize("G,split,V", [(2, 0, 512), (2, 1, 512), (3, 1, 64), (3, 0, 64)])
def test_multiprocess_full_row_width(tmp_path, G, split, V):
    """configs[0]'s trace across G homes at the bench's 4 KiB rows with the PVP on: k_fill<8>
    (victim D2H + fills), k_pull<8, kDev, 0/1> (both pull orders), k_pvp<8> per home; V = 64
    overflows the victim queues."""
    N = 16384
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, G, 256, (10, 5), 20)
    sc = synth.static_scores(g)
    cfg = dict(N=N, D=1024, L=1024, A=8, policy="hybrid", pvp=1, W=8, V=V, reinsert=1, P=1)
    ho = _run_edge(tmp_path, G, tr, sc, cfg, split)
    assert ho[..., 5].sum() > 0 and ho[..., 14].sum() > 0  # victim hits, admissions
    assert ho[..., 2].sum() > 0  # peer requests crossed homes


def test_multiprocess_file_tier_full_row_width(tmp_path):
    """File tier (N2) at 4 KiB rows across 2 homes (O_DIRECT reads into the bounce buffer,
    k_fill<8> reads it), PVP on."""
    N = 16384
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, 2, 256, (10, 5), 14)
    sc = synth.static_scores(g)
    cfg = dict(N=N, D=1024, L=1024, A=8, policy="hybrid", pvp=1, W=8, V=512, reinsert=1, P=1, file=1)
    _run_edge(tmp_path, 2, tr, sc, cfg, 1)


def test_connect_rejects_mismatched_layout(tmp_path):
    """lsmgnn_connect on the GPU: rank 1 initialised with other arguments -> both ranks get
    LSMGNN_ECOMM before anything is mapped; a matching retry in the same processes connects."""
    launch(2, tmp_path, "mismatch", str(tmp_path))
    for r in range(2):
        d = json.load(open(tmp_path / f"r{r}.json"))
        assert d["mismatch_error"] and "layout" in d["mismatch_error"], d
        assert d["retry_ok"] and d["bad"] == 0, d


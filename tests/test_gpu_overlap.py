"""GPU parity with consecutive gathers in flight together (-m gpu).

A direct G = 1 gather whose predecessor on the stream is the previous gather (or the window feed
behind it) starts its k_dedup and k_set while the previous k_serve still delivers (kernels.cuh
k_dedup `early`: parity-indexed node_loc / request lists / fill lists / counters, finished-CTA
counters instead of programmatic waits). The harness in test_gpu_parity reads every `out` back
right after its gather, which synchronises the stream, so those tests never overlap two gathers.
Here the host issues the whole trace without synchronising and checks rows and counters at the
end: (a) every gather into its own `out`; (b) one shared `out` that a consumer kernel of the
caller copies away between the gathers (stream order must still hold for it).
"""
import numpy as np
import pytest

import synth

from .harness import run_oracle, table_for
from .test_gpu_parity import compare

pytestmark = pytest.mark.gpu


def _trace(N, batch, fanout, K, W):
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, 1, batch, fanout, K + W + 1, seed_s=11)
    return tr, synth.static_scores(g)


def _run(tr, K, *, N, D, L, A, sc, W, shared_out, steps_mode="direct"):
    import torch
    from paper_2407_15264_b200 import LsmGnn
    dev = torch.device("cuda", torch.cuda.current_device())
    ids = [torch.from_numpy(np.asarray(tr[t][0], np.int64)).to(dev) for t in range(len(tr))]
    n_max = max(x.numel() for x in ids)
    c = LsmGnn(N, D, L, A, 0, sc, policy="hybrid", pvp=0, window=W, max_batch_ids=n_max)
    c.attach_storage(table_for(N, D, pinned=True))
    R = 4 * D
    c.prefetch(ids[1:W + 1], first_iter=1)
    torch.cuda.synchronize()
    outs = []
    shared = torch.empty((n_max, R), dtype=torch.uint8, device=dev) if shared_out else None
    for t in range(K):
        n = ids[t].numel()
        if shared_out:
            c.gather(ids[t], shared)
            outs.append(shared[:n].clone())  # the caller's consumer kernel, between the gathers
        else:
            o = torch.empty((max(1, n), R), dtype=torch.uint8, device=dev)
            c.gather(ids[t], o)
            outs.append(o[:n])
        c.prefetch([ids[t + 1 + W]], first_iter=t + 1 + W)
    torch.cuda.synchronize()
    hist = c.history(0, K)
    c.close()
    bad = 0
    for t in range(K):
        host = outs[t].cpu().numpy()
        nb, _ = synth.check_rows(host.view(np.uint32).reshape(-1, D), np.asarray(tr[t][0], np.int64), D)
        bad += nb
    return hist, bad


@pytest.mark.parametrize("regime", ["hits", "misses"])
@pytest.mark.parametrize("shared_out", [False, True])
def test_overlapped_gathers_parity(regime, shared_out):
    N, D, A, W, K = 60000, 256, 32, 6, 40
    L = N - N % A if regime == "hits" else 6016  # whole table vs ~10% (oversubscribed sets)
    tr, sc = _trace(N, 256, (10, 5, 5), K, W)
    hg, bad = _run(tr, K, N=N, D=D, L=L, A=A, sc=sc, W=W, shared_out=shared_out)
    ho = run_oracle(tr, G=1, N=N, D=D, L=L, A=A, scores=sc, policy="hybrid", pvp=0, W=W)[:, 0, :]
    assert bad == 0
    compare(hg, ho[:K], f"overlap {regime} shared_out={shared_out}")


@pytest.mark.parametrize("switches", [{"LSMGNN_DEDUP_EARLY": "0"},
                                      {"LSMGNN_META_EVICT_LAST": "0", "LSMGNN_MASK_EVICT_LAST": "0",
                                       "LSMGNN_SERVE_STATIC_FIRST": "0"},
                                      {"LSMGNN_L2_EVICT_FIRST": "1", "LSMGNN_EARLY_DEDUP_PER_SM": "1"}])
def test_overlap_toggle_identical(monkeypatch, switches):
    """The timing switches (no overlap: every kernel waits for its predecessor; no L2 policies;
    other geometries) give the same records and rows as the defaults."""
    N, D, A, W, K = 60000, 64, 32, 6, 30
    L = 12000
    tr, sc = _trace(N, 256, (10, 5, 5), K, W)
    h1, bad1 = _run(tr, K, N=N, D=D, L=L, A=A, sc=sc, W=W, shared_out=False)
    for k, v in switches.items():
        monkeypatch.setenv(k, v)
    h0, bad0 = _run(tr, K, N=N, D=D, L=L, A=A, sc=sc, W=W, shared_out=False)
    assert bad1 == 0 and bad0 == 0
    compare(h1, h0, f"defaults vs {switches}")


def test_overlap_slow_feed():
    """Tiny gathers behind huge window feeds: the early k_set of gather t+1 would start while the
    feed of t+1+W still sets reuse bits unless it waits for the feeds issued before it (their
    finished-CTA count). Eviction classes and victims depend on those bits (hybrid, W = 4)."""
    N, D, A, W, K = 1_000_000, 4, 8, 4, 40
    L = 16384
    rng = np.random.default_rng(21)
    tr = []
    for t in range(K + W + 1):
        n = 1_500_000 if t % 3 == 0 else 96
        tr.append([rng.integers(0, N, n).astype(np.int64)])
    sc = rng.integers(0, 256, N).astype(np.uint8)
    hg, bad = _run(tr, K, N=N, D=D, L=L, A=A, sc=sc, W=W, shared_out=False)
    ho = run_oracle(tr, G=1, N=N, D=D, L=L, A=A, scores=sc, policy="hybrid", pvp=0, W=W)[:, 0, :]
    assert bad == 0
    compare(hg, ho[:K], "overlap slow feed")


@pytest.mark.parametrize("static_first", ["1", "0"])
def test_hit_dominated_large_batches(monkeypatch, static_first):
    """Batches of ~10^5 requests that nearly all hit (the bench's hit-path shape at 256-B rows):
    k_serve hands each warp its first delivery chunk statically when every fill warp has at most
    one fill (LSMGNN_SERVE_STATIC_FIRST), the rest from the counter; overlapped gathers."""
    monkeypatch.setenv("LSMGNN_SERVE_STATIC_FIRST", static_first)
    N, D, A, W, K = 200_000, 64, 32, 8, 30
    g = synth.plcite(N, 8)
    tr = synth.make_trace(g, 1, 1024, (10, 5, 5), K + W + 1, seed_s=12)
    sc = synth.static_scores(g)
    L = N - N % A
    hg, bad = _run(tr, K, N=N, D=D, L=L, A=A, sc=sc, W=W, shared_out=False)
    ho = run_oracle(tr, G=1, N=N, D=D, L=L, A=A, scores=sc, policy="hybrid", pvp=0, W=W)[:, 0, :]
    assert bad == 0
    compare(hg, ho[:K], f"hit-dominated static_first={static_first}")
    assert ho[K // 2:, 4].sum() > 0.9 * ho[K // 2:, 3].sum()  # hits / unique: the hit path

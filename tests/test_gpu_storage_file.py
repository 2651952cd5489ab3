"""NEXT N2 on the GPU (-m gpu): the file tier. The backing rows live in a file (O_DIRECT
when R % 512 == 0, buffered otherwise); each gather reads the rows its fills need into a
pinned bounce buffer. Counters must equal the oracle's and every row must equal F(v) —
the storage medium changes where bytes come from, never what the cache decides."""
import numpy as np
import pytest

import synth

from .harness import run_gpu, run_oracle, write_table_file
from .test_gpu_parity import cfg1_g1, compare  # noqa: F401 (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("buffered", [False, True])
@pytest.mark.parametrize("policy,pvp", [("hybrid", 1), ("lru", 0)])
def test_file_tier_parity(tmp_path, monkeypatch, cfg1_g1, policy, pvp, buffered):
    if buffered:
        monkeypatch.setenv("LSMGNN_STORAGE_BUFFERED", "1")
    g, tr, sc = cfg1_g1
    kw = dict(N=16384, D=128, L=1024, A=8, scores=sc, policy=policy, pvp=pvp, W=8, V=512)
    path = write_table_file(tmp_path / "home0.bin", 16384, 128)
    hg, _, bad = run_gpu(tr, storage_file=path, **kw)
    ho = run_oracle(tr, G=1, **kw)[:, 0, :]
    assert bad == 0
    compare(hg, ho, f"file tier {policy}/pvp{pvp}/buffered{int(buffered)}")


def test_file_tier_small_rows_and_edge_batches(tmp_path):
    """R = 16 B (buffered reads), empty and duplicate-heavy batches, oversubscribed sets."""
    rng = np.random.default_rng(3)
    N = 5000
    sc = rng.integers(0, 256, N).astype(np.uint8)
    tr = [[np.asarray(rng.zipf(1.3, int(n)) % N if n else np.zeros(0), np.int64)] for n in
          rng.integers(0, 900, 15)]
    tr[4] = [np.zeros(0, np.int64)]
    kw = dict(N=N, D=4, L=64, A=8, scores=sc, policy="hybrid", pvp=1, W=3, V=30)
    path = write_table_file(tmp_path / "h.bin", N, 4)
    hg, _, bad = run_gpu(tr, storage_file=path, **kw)
    assert bad == 0
    compare(hg, run_oracle(tr, G=1, **kw)[:, 0, :], "file tier small rows")


def test_file_tier_errors(tmp_path):
    import torch
    from paper_2407_15264_b200 import LsmGnn, LsmGnnError
    c = LsmGnn(1000, 128, 64, 8, 0, None, window=2, max_batch_ids=64)
    with pytest.raises(LsmGnnError, match="open"):
        c.attach_storage_file(str(tmp_path / "missing.bin"))
    short = tmp_path / "short.bin"
    short.write_bytes(b"\0" * 512 * 10)
    with pytest.raises(LsmGnnError, match="bytes"):
        c.attach_storage_file(str(short))
    c.attach_storage_file(write_table_file(tmp_path / "ok.bin", 1000, 128))
    ids = [torch.arange(10, dtype=torch.int64, device="cuda") for _ in range(6)]
    out = torch.empty((64, 512), dtype=torch.uint8, device="cuda")
    c.prefetch(ids[1:3], first_iter=1)
    with pytest.raises(LsmGnnError, match="graph"):
        c.graph_capture(ids, out)
    c.gather(ids[0], out)
    rows = out[:10].cpu().numpy().view(np.uint32).reshape(10, 128)
    assert synth.check_rows(rows, np.arange(10), 128)[0] == 0
    c.close()

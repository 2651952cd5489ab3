"""World-size-2 gloo test of the N>1 host logic on CPU (-m "not gpu"): the connect-time
handle validation of liblsmgnn.so (lsmgnn_plan_handle / lsmgnn_check_handles, the checks
lsmgnn_connect runs before mapping any peer) across two processes exchanging their blobs over
gloo, and the home partition of each rank's batches (v mod G)."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gloo_world2(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_worker.py"), "cpu", str(tmp_path)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-4000:]
    for rank in range(2):
        d = json.load(open(tmp_path / f"r{rank}.json"))
        assert d["rank"] == rank
        E = d["ECOMM"]
        assert d["ok"] == 0
        assert d["reversed"] == E and "rank order" in d["reversed_msg"]
        assert d["short"] == E
        for name in ("lines", "max_batch_ids", "pvp", "window", "row_bytes"):
            assert d[name] == E and "layout" in d[name + "_msg"], (name, d[name], d[name + "_msg"])
        assert d["world"] == E and "world" in d["world_msg"]
        assert "multiple of 16" in d["bad_args"]
        assert "rank/world" in d["bad_rank"]
        assert all(set(h) <= {0, 1} for h in d["homes"])

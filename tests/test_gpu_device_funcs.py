"""Device helper functions against their plain definitions (-m gpu): next_reuse_d (the
window mask's next reuse distance, R5) in its register form and its word-by-word
form vs a host scan of positions t+1..t+W, every W in 1..600 and every p0."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_next_reuse_distance(tmp_path):
    exe = tmp_path / "nrc"
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o",
                           str(exe), os.path.join(ROOT, "tests", "cuda", "next_reuse_check.cu")])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 mismatches" in r.stdout

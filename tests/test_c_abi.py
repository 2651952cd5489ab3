"""The boundary from plain C: tests/c_abi_demo.c includes only include/lsmgnn.h (+ the CUDA
runtime for its own buffers) and links liblsmgnn.so — no Python or torch on the call path.
CPU: it compiles and links against the header and the library; GPU: it runs, every row equals
the table row and hits + victim hits + storage reads = unique per iteration."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build(tmp_path):
    exe = str(tmp_path / "c_abi_demo")
    lib = os.path.join(ROOT, "paper_2407_15264_b200")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "c_abi_demo.c"), "-L", lib, "-llsmgnn",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{lib}:{os.path.join(CUDA, 'lib64')}",
           "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_consumer_builds(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_c_consumer_runs(tmp_path):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c abi ok" in r.stdout

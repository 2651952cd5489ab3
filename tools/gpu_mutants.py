"""Sensitivity of the GPU parity tests: build liblsmgnn.so variants, each with ONE plausible
kernel mistake (paper_2407_15264_b200/csrc/kernels.cuh), into ab/mut_<name>.so. Run on the GPU
box with tools/gpu_mutants.sh, which swaps each variant in and runs the parity tests; every
mutant must fail them (results: profiles/r01_gpu_mutants.txt).

usage: python tools/gpu_mutants.py build
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2407_15264_b200", "csrc")

# (name, original, mutated, what it breaks)
MUTANTS = [
    ("threshold_strict", "((uint32_t)d <= T ? kNear : kFar)", "((uint32_t)d < T ? kNear : kFar)", "R4 Near iff d <= T"),
    ("no_level_swap", "if (cls == kNoReuse) return pvp ? 1 : 0;\n  if (cls == kFar) return pvp ? 0 : 1;",
     "if (cls == kNoReuse) return 0;\n  if (cls == kFar) return 1;", "P:434 level swap"),
    ("bypass_largest", "const uint32_t v = (uint32_t)skey[k];", "const uint32_t v = (uint32_t)skey[nM - 1 - k];",
     "R10 bypass the smallest incoming keys"),
    ("admit_strict", "if (!none && c.x <= thresh) {", "if (!none && c.x < thresh) {", "R14 admission of the room smallest"),
    ("pvp_wrong_queue", "const uint32_t k = (uint32_t)(t1 % W), stamp1", "const uint32_t k = (uint32_t)(it->t % W), stamp1",
     "R17 queue t+1 after gather(t)"),
    ("mask_never_cleared", "const uint32_t m = ~(1u << (bit & 31));", "const uint32_t m = ~0u;",
     "S10 bits of iteration t cleared"),
    ("deliver_first_only", "for (uint32_t pos = first; pos != kInvalid; pos = nxt[pos]) {",
     "for (uint32_t pos = first; pos != kInvalid; pos = kInvalid) {", "S8 every requester of a node"),
    ("no_victim_d2h", "      if (f.victim != kInvalid) warp_copy_row<UNROLL, kDev, kHost>(hostq + (size_t)f.victim * nvec, slot, nvec);\n      const bool from_host",
     "      const bool from_host", "S6 victim row D2H before the slot is overwritten"),
    ("rr_cursor", "p.rr[s] = (svict[e - 1] + 1) % A;", "p.rr[s] = svict[e - 1];", "P:612 round robin"),
    ("stale_not_fresh", "if (info == kInfoFresh || info <= t) return kFresh;", "if (info == kInfoFresh) return kFresh;",
     "R6 stale snapshot is Fresh"),
    ("pull_phase1_skips", "if (((loc & kDelivered) != 0) != (PHASE == 1)) continue;",
     "if ((loc & kDelivered) != 0) continue;", "G > 1 filled rows pulled after served"),
]


def build():
    out = os.path.join(ROOT, "ab")
    os.makedirs(out, exist_ok=True)
    src = open(os.path.join(CSRC, "kernels.cuh")).read()
    for name, old, new, _ in MUTANTS:
        assert src.count(old) == 1, name
        d = tempfile.mkdtemp()
        shutil.copytree(CSRC, os.path.join(d, "csrc"))
        os.makedirs(os.path.join(d, "include"))
        shutil.copy(os.path.join(ROOT, "include", "lsmgnn.h"), os.path.join(d, "include"))
        open(os.path.join(d, "csrc", "kernels.cuh"), "w").write(src.replace(old, new))
        # same relative layout as the package (csrc/ includes ../../include/lsmgnn.h)
        pkg = os.path.join(d, "pkg")
        os.makedirs(pkg)
        shutil.move(os.path.join(d, "csrc"), os.path.join(pkg, "csrc"))
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
                               "--expt-relaxed-constexpr", "-o", os.path.join(out, f"mut_{name}.so"),
                               os.path.join(pkg, "csrc", "lsmgnn.cu"), "-ldl", "-lrt", "-lpthread"])
        shutil.rmtree(d)
        print("built", name, flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()

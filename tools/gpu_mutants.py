"""Sensitivity of the GPU parity tests: build liblsmgnn.so variants, each with ONE plausible
kernel mistake (paper_2407_15264_b200/csrc/kernels.cuh or device_common.cuh), into ab/mut_<name>.so. Run on the GPU
box with tools/gpu_mutants.sh, which swaps each variant in and runs the parity tests; every
mutant must fail them (results: profiles/r01_gpu_mutants.txt, profiles/r02_gpu_mutants.txt).

usage: python tools/gpu_mutants.py build
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2407_15264_b200", "csrc")

# (name, original, mutated, what it breaks) — kernels.cuh unless the name starts with "dc_"
# (device_common.cuh). Round 2 replaced the patterns of the rewritten kernels and added mutants
# for the new mechanisms (the hit probe in k_dedup, the slow-set list, the TMA rings, guided
# delivery chunks, the pipelined file tier).
MUTANTS = [
    ("threshold_strict", "((uint32_t)d <= T ? kNear : kFar)", "((uint32_t)d < T ? kNear : kFar)", "R4 Near iff d <= T"),
    ("no_level_swap", "if (cls == kNoReuse) return pvp ? 1 : 0;\n  if (cls == kFar) return pvp ? 0 : 1;",
     "if (cls == kNoReuse) return 0;\n  if (cls == kFar) return 1;", "P:434 level swap"),
    ("bypass_largest", "const uint32_t v = (uint32_t)skey[k];", "const uint32_t v = (uint32_t)skey[nM - 1 - k];",
     "R10 bypass the smallest incoming keys"),
    ("admit_strict", "if (!none && c.x <= thresh) {", "if (!none && c.x < thresh) {", "R14 admission of the room smallest"),
    ("pvp_wrong_queue", "const uint32_t k = (uint32_t)(t1 % W), stamp1", "const uint32_t k = (uint32_t)(it->t % W), stamp1",
     "R17 queue t+1 after gather(t)"),
    ("mask_never_cleared", "const uint32_t m = ~(1u << (slot & 31));", "const uint32_t m = ~0u;",
     "S10 bits of iteration t cleared (in k_dedup)"),
    ("deliver_first_only", "for (uint32_t pos = first; pos != kInvalid; pos = a.nxt[pos]) {",
     "for (uint32_t pos = first; pos != kInvalid; pos = kInvalid) {", "S8 every requester of a node"),
    ("no_victim_d2h", "      if (f.victim != kInvalid) warp_copy_row<UNROLL, kDev, kHost>(a.hostq + (size_t)f.victim * nvec, slot, nvec);\n",
     "", "S6 victim row D2H before the slot is overwritten"),
    ("rr_cursor", "p.rr[s] = (svict[e - 1] + 1) % A;", "p.rr[s] = svict[e - 1];", "P:612 round robin"),
    ("stale_not_fresh", "if (info == kInfoFresh || info <= t) return kFresh;", "if (info == kInfoFresh) return kFresh;",
     "R6 stale snapshot is Fresh"),
    ("pull_phase1_skips", "const uint32_t need = __ballot_sync(0xffffffffu, valid && (((loc & kDelivered) != 0) == (PHASE == 1)));",
     "const uint32_t need = __ballot_sync(0xffffffffu, valid && !(loc & kDelivered));", "G > 1 filled rows pulled after served"),
    ("probe_no_last_use", "    a.last_use[s * a.A + (uint32_t)way] = t;\n    ++*nhit;", "    ++*nhit;",
     "R10/R20 a hit's last use is t (k_dedup probe)"),
    ("slow_set_dropped", "      a.slow_list[atomicAdd(&a.scr->nslow, 1u)] = s;  // first miss of the set: k_set processes it",
     "      (void)s;", "S4/S5 every set with a miss is replaced"),
    ("miss_not_listed", "    if (a.head) list_join(a, q, pos, stamp);  // a fill will deliver this row",
     "", "S8 a filled node's first requester receives the row"),
    ("fast_set_cnt_kept", "    if (p.set_cnt[sl] && p.slow_stamp[sl] != stamp_) p.set_cnt[sl] = 0;  // ready for the next batch",
     "    ;", "S3 the all-hit sets' buckets start empty next batch"),
    ("hit_counted_twice", "        if (way >= 0) {  // (node_loc and the hit count were written by k_dedup's probe)\n          kind = kHit;",
     "        if (way >= 0) {\n          kind = kHit;\n          ++ctr[C_HIT];", "S9 hits counted once"),
    ("pvp_unused_inverted", "      unused += p.mark[stg[j] / G] != stamp_;", "      unused += p.mark[stg[j] / G] == stamp_;",
     "R28 pvp_unused = staged rows not requested"),
    ("file_no_wait", "      if (from_host && a.bounce) io_wait(a.io_ready, e, stamp);  // file tier: row e read yet?\n",
     "", "N2 a fill reads its bounce row only after the host released its chunk"),
    ("dc_ring_no_read_wait", "      if (r.nl >= r.ST) bulk_wait_read(r.ns + r.ST - 1 - r.nl);\n", "",
     "a stage is reloaded only after its store has read it (TMA rings)"),
    ("dc_ring_store_wrong_row", "    bulk_s2g(dst[r.pend[s]], r.buf + (size_t)s * r.R, r.R);",
     "    bulk_s2g(dst[r.pend[(s + 1) % r.ST]], r.buf + (size_t)s * r.R, r.R);", "each stage stored to its own row"),
]


def build():
    out = os.path.join(ROOT, "ab")
    os.makedirs(out, exist_ok=True)
    for name, old, new, _ in MUTANTS:
        if os.path.exists(os.path.join(out, f"mut_{name}.so")):
            continue  # (delete ab/ to rebuild everything)
        fname = "device_common.cuh" if name.startswith("dc_") else "kernels.cuh"
        src = open(os.path.join(CSRC, fname)).read()
        assert src.count(old) == 1, name
        d = tempfile.mkdtemp()
        shutil.copytree(CSRC, os.path.join(d, "csrc"))
        os.makedirs(os.path.join(d, "include"))
        shutil.copy(os.path.join(ROOT, "include", "lsmgnn.h"), os.path.join(d, "include"))
        open(os.path.join(d, "csrc", fname), "w").write(src.replace(old, new))
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

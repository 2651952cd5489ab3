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
# delivery chunks, the pipelined file tier, the overlap of consecutive gathers).
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
    ("deliver_first_only", "for (uint32_t pos = first; pos != kInvalid; pos = nxt[pos]) {",
     "for (uint32_t pos = first; pos != kInvalid; pos = kInvalid) {", "S8 every requester of a node"),
    ("no_victim_d2h", "      if (f.victim != kInvalid) warp_copy_row<UNROLL, kDev, kHost>(a.hostq + (size_t)f.victim * nvec, slot, nvec);\n",
     "", "S6 victim row D2H before the slot is overwritten"),
    ("rr_cursor", "p.rr[s] = (svict[e - 1] + 1) % A;", "p.rr[s] = svict[e - 1];", "P:612 round robin"),
    ("stale_not_fresh", "if (info == kInfoFresh || info <= t) return kFresh;", "if (info == kInfoFresh) return kFresh;",
     "R6 stale snapshot is Fresh"),
    ("pull_phase1_skips", "const uint32_t need = __ballot_sync(0xffffffffu, valid && (((loc & kDelivered) != 0) == (PHASE == 1)));",
     "const uint32_t need = __ballot_sync(0xffffffffu, valid && !(loc & kDelivered));", "G > 1 filled rows pulled after served"),
    ("probe_no_last_use", "      st_u32_hint(&a.last_use[s * a.A + (uint32_t)way], t, pp.pol);\n", "",
     "R10/R20 a hit's last use is t (k_dedup probe, L2-hinted path; k_set protects the ways used at t)"),
    ("slow_set_dropped", "      a.slow_list[atomicAdd(pp.nslow, 1u)] = s;  // first miss of the set: k_set processes it",
     "      (void)s;", "S4/S5 every set with a miss is replaced"),
    ("miss_not_listed", "    if (pp.head) list_join(pp, q, pos, stamp);  // a fill will deliver this row",
     "", "S8 a filled node's first requester receives the row"),
    ("hit_into_bucket", "  if (way >= 0) {\n    if (pp.hint) {",
     "  if (way >= 0) {\n    a.bucket[(size_t)s * a.BC + atomicAdd(&a.set_cnt[s], 1u)] = v;\n    if (pp.hint) {",
     "S3/S4 the buckets hold the misses only (a hit re-installed would be counted twice)"),
    ("protect_none", "const uint32_t protm = __ballot_sync(0xffffffffu, lane < A && tg != kInvalid && lu == t_);",
     "const uint32_t protm = 0u;", "R10 hits of the batch are protected from eviction"),
    # the overlap of consecutive gathers (k_dedup / k_set `early`)
    ("set_no_dedup_wait", "      while (ld_acquire_u64(&p.it->dedup_ctas_done) < p.dedup_wait) __nanosleep(64);\n", "",
     "an early k_set starts after its gather's k_dedup finished"),
    ("set_no_feed_wait", "      while (ld_acquire_u64(&p.it->feed_ctas_done) < p.feed_wait) __nanosleep(64);\n", "",
     "an early k_set reads the window bits after the feeds issued before its gather"),
    ("serve_no_prev_wait", "      while (ld_acquire_u64(&a.it->t_next) < (uint64_t)a.t_host) __nanosleep(64);\n", "",
     "an early k_serve fills slots only after the previous gather completed"),
    ("loc_no_parity", "  pp.node_loc = a.node_loc + par * a.loc_stride;", "  pp.node_loc = a.node_loc;",
     "node_loc of gather t+1 does not overwrite the table k_serve(t) reads"),
    ("lists_no_parity", "  pp.head = a.head ? a.head + (size_t)par * a.Q : nullptr;", "  pp.head = a.head;",
     "request lists of gather t+1 do not overwrite those k_serve(t) walks"),
    ("fills_no_parity", "  FillEnt* const fills_ = p.fills + (size_t)par_ * p.fstride;", "  FillEnt* const fills_ = p.fills;",
     "the fill list of gather t+1 does not overwrite the one k_serve(t) reads"),
    ("pending_not_resolved", "if (__ballot_sync(0xffffffffu, loc == kPending) && loc == kPending) loc = loc_of(ids[c0 + lane]);",
     "if (__ballot_sync(0xffffffffu, loc == kPending) && loc == kPending) loc = kDelivered;",
     "S8 requests k_dedup left pending (repeats, staged rows) are delivered through node_loc"),
    ("record_zeroed_early", "  unsigned long long* nrec = hist + (size_t)((t + 2) % kHist) * F_NFIELDS;",
     "  unsigned long long* nrec = hist + (size_t)((t + 1) % kHist) * F_NFIELDS;",
     "the record of t+1 (already being counted by an early k_dedup) is not zeroed by gather t"),
    ("pvp_unused_inverted", "      unused += p.mark[stg[j] / G] != stamp_;", "      unused += p.mark[stg[j] / G] == stamp_;",
     "R28 pvp_unused = staged rows not requested"),
    ("file_no_wait", "      if (from_host && a.bounce) io_wait(a.io_ready, e, stamp);  // file tier: row e read yet?\n",
     "", "N2 a fill reads its bounce row only after the host released its chunk"),
    ("dc_ring_no_read_wait", "      if (r.nl >= r.ST) bulk_wait_read(r.ns + r.ST - 1 - r.nl);\n", "",
     "a stage is reloaded only after its store has read it (TMA rings)"),
    ("dc_ring_store_wrong_row", "    else bulk_s2g(dst[r.pend[s]], r.buf + (size_t)s * r.R, r.R);",
     "    else bulk_s2g(dst[r.pend[(s + 1) % r.ST]], r.buf + (size_t)s * r.R, r.R);", "each stage stored to its own row"),
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

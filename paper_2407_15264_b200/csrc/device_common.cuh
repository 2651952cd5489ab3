// device_common.cuh — small device helpers for the LSM-GNN gather path (sm_100a).
//
// Nothing here is shared with oracle/: the two implement the paper independently.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lsm {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;  // empty cache way / "no victim slot"
constexpr uint32_t kHostBit = 0x80000000u;  // FillEnt::src: bit 31 set => backing-table row q
constexpr uint32_t kInfoNone = 0xFFFFFFFFu;  // line snapshot: no reuse found in the window
constexpr uint32_t kInfoFresh = 0xFFFFFFFEu; // line snapshot: inserted after the last scan

// Dynamic-information classes; index of evict_by_class[].
enum Cls : int { kNoReuse = 0, kFar = 1, kFresh = 2, kNear = 3 };
// Probe outcome per unique request.
enum Kind : uint32_t { kStorage = 0, kHit = 1, kVHit = 2 };

// Counter fields, in lsmgnn_stats_t order.
enum Field : int {
  F_ITER = 0, F_REQ, F_PEER, F_UNIQUE, F_HIT, F_VHIT, F_STOR, F_INS, F_BYP, F_EVICT,
  F_EV0, F_EV1, F_EV2, F_EV3, F_VADM, F_VDROP, F_ENR, F_PREF, F_UNUSED,
  F_BOUT, F_BNVL, F_BH2D, F_BPVP, F_BD2H, F_NFIELDS
};

// One row copy the fill kernel performs.
struct FillEnt {
  uint32_t src;     // kHostBit|q: backing-table row q; else a pool row (PVP staging)
  uint32_t dst;     // pool row (cache slot or bypass staging)
  uint32_t victim;  // host victim-queue row the OLD content of dst goes to first, or kInvalid
  uint32_t node;    // node v whose row this is (fused delivery walks its request list)
};
constexpr uint32_t kDelivered = 0x80000000u;  // node_loc bit: row delivered to `out` by the fill
// One victim-buffer candidate.
struct Cand {
  uint32_t x;      // evicted node
  uint32_t reuse;  // its next reuse iteration
  uint32_t fill;   // index of the FillEnt overwriting its slot
  uint32_t pad;
};

// Per-batch scratch counters (u32, device).
// (unique nodes and requests are counted straight into the iteration's record by k_dedup)
struct Scratch {
  uint32_t nfill[2];   // FillEnt entries, by iteration parity (k_set of t + 1 may run while k_serve
                       // of t still reads its list: k_dedup/k_set `early`)
  uint32_t ncand;      // victim candidates (PVP: never early)
  uint32_t nbypass[2]; // bypass-staging rows used, by iteration parity
  uint32_t bad_ids;    // sticky count of node IDs >= N (ERANGE)
  uint32_t staged[2];  // rows the PVP staged, by iteration parity
  uint32_t pvp_done;   // grid-completion counter of the PVP kernel
  uint32_t pull_next;  // k_serve: next request index handed to a delivering warp
  uint32_t serve_done; // k_serve: CTAs finished (the last one closes the record)
  uint32_t io_done;    // k_io_export: CTAs finished (the last one publishes the list)
  uint32_t nslow[2];   // sets with a miss (k_dedup's slow list), by iteration parity: k_dedup(t+1)
                       // may count while gather t closes (k_dedup `early`)
  uint32_t pull_phase_next[2];  // k_pull: next request index per phase
};

// Per-iteration values, resident on the device. k_begin / k_win_begin write them (from host
// arguments, or — when a captured CUDA graph replays — from the device's own counters and the
// caller's ring of batch pointers); every other kernel reads them, so a whole step can be
// replayed without any per-iteration host parameter.
constexpr uint32_t kHist = 4096;  // per-iteration records kept on the device
struct IterState {
  uint64_t t;                 // iteration of the current gather
  uint64_t t_next;            // graph replay: the next gather iteration
  const int64_t* ids;         // this rank's request IDs of gather t (device)
  int64_t n;                  // their count
  uint32_t stamp, p0, par, upd;  // t+1; (t+1) mod (W+1); t & 1; periodic scan at t
  uint32_t rec_idx;           // t mod kHist (history record)
  uint32_t stage_base;        // pool row of the PVP staging buffer for parity t & 1
  // window feed (lsmgnn_prefetch): the batch of iteration wk
  uint64_t wk, wk_next;
  const int64_t* wids;
  int64_t wn;
  uint32_t wslot;             // wk mod (W+1): ring slot and mask bit
  // G = 1 window feeds: CTAs of k_route_local that finished their work (monotonic; the host
  // counts the CTAs it launched, and an early k_set waits for that many, kernels.cuh k_set)
  unsigned long long feed_ctas_done;
  // G = 1 direct gathers: CTAs of k_dedup that finished (monotonic, counted the same way)
  unsigned long long dedup_ctas_done;
  unsigned long long set_ctas_done;  // ... and of early k_set launches
};

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream
// serialization may start while its predecessor on the stream is still running; it waits
// here until the predecessor has completed and its memory is visible, then lets its own
// successor be scheduled early. Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// CTA-wide reservation of one slot per thread with want == true: one atomicAdd per CTA on the
// shared counter instead of one per warp (a hot single address). Every thread of the CTA must
// call it (CTA-uniform control flow), and blockDim.x must be a multiple of 32 (full-warp
// ballots; every launch of a kernel using it has 256 threads). Slot order within the CTA
// follows thread order.
__device__ __forceinline__ uint32_t block_reserve(uint32_t* ctr, bool want) {
  __shared__ uint32_t s_cnt[32];
  __shared__ uint32_t s_base;
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const uint32_t b = __ballot_sync(0xffffffffu, want);
  if (lane == 0) s_cnt[w] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (uint32_t i = 0; i < nw; ++i) {
      const uint32_t c = s_cnt[i];
      s_cnt[i] = tot;
      tot += c;
    }
    s_base = tot ? atomicAdd(ctr, tot) : 0u;
  }
  __syncthreads();
  const uint32_t r = s_base + s_cnt[w] + __popc(b & ((1u << lane) - 1u));
  __syncthreads();  // s_cnt / s_base are reused by the next call
  return r;
}
// Warp-aggregated atomicAdd of `inc` per lane: one atomic per warp. Must be called
// by all 32 lanes (inactive lanes pass inc = 0). Returns this lane's base offset.
__device__ __forceinline__ uint32_t warp_reserve(uint32_t* ctr, uint32_t inc) {
  const uint32_t lane = lane_id();
  uint32_t incl = inc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t base = 0;
  if (lane == 31 && total) base = atomicAdd(ctr, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - inc;
}

// First set bit in [lo, hi) of a bitmask row; -1 if none.
__device__ __forceinline__ int first_bit_in(const uint32_t* row, int lo, int hi) {
  if (lo >= hi) return -1;
  int w = lo >> 5, wl = (hi - 1) >> 5;
  uint32_t bits = row[w] & (~0u << (lo & 31));
  while (true) {
    if (w == wl) {
      int top = hi - (w << 5);  // 1..32 valid bits in this word
      if (top < 32) bits &= (1u << top) - 1u;
    }
    if (bits) return (w << 5) + __ffs(bits) - 1;
    if (++w > wl) return -1;
    bits = row[w];
  }
}

// Next reuse distance d in 1..W of a node from its window mask row, 0 = none.
// Bit position of iteration k is k mod (W+1); at gather(t) the window is t+1..t+W
// (PAPER.md P:352-354 window buffer; R5). p0 = (t+1) mod (W+1).
// Rows of up to 16 words (W <= 511) are loaded in one round trip (independent loads into
// registers) and scanned there; longer rows take the word-by-word scan below.
__device__ __forceinline__ int next_reuse_d_seq(const uint32_t* row, int p0, int W);
__device__ __forceinline__ int next_reuse_d(const uint32_t* row, int p0, int W) {
  const int Wp1 = W + 1, MW = (Wp1 + 31) >> 5;
  if (MW > 16) return next_reuse_d_seq(row, p0, W);
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = i < MW ? row[i] : 0u;
  // positions [p0, Wp1) come first (d = pos - p0 + 1), then the wrapped part [0, p0 - 1)
  // (d = Wp1 - p0 + pos + 1); position p0 - 1 (iteration t) is not in the window
  // (p0 = 0: the window is [0, W) and position W is iteration t)
  const int hi_end = p0 == 0 ? W : Wp1;
  int first_hi = -1, first_lo = -1;
#pragma unroll
  for (int i = 15; i >= 0; --i) {
    if (i >= MW) continue;
    const int b0 = i << 5;
    const uint32_t x = w[i];
    // bits at positions in [p0, hi_end)
    uint32_t hi = x, lo = x;
    if (p0 > b0) hi &= (p0 - b0 >= 32) ? 0u : (~0u << (p0 - b0));
    if (hi_end - b0 < 32) hi &= hi_end - b0 <= 0 ? 0u : ((1u << (hi_end - b0)) - 1u);
    // bits at positions < p0 - 1
    const int lim = p0 - 1 - b0;
    lo &= lim <= 0 ? 0u : (lim >= 32 ? ~0u : ((1u << lim) - 1u));
    if (hi) first_hi = b0 + __ffs(hi) - 1;
    if (lo) first_lo = b0 + __ffs(lo) - 1;
  }
  if (first_hi >= 0) return first_hi - p0 + 1;
  if (first_lo >= 0) return (Wp1 - p0) + first_lo + 1;
  return 0;
}
__device__ __forceinline__ int next_reuse_d_seq(const uint32_t* row, int p0, int W) {
  const int Wp1 = W + 1;
  int end1 = p0 + W < Wp1 ? p0 + W : Wp1;
  int pos = first_bit_in(row, p0, end1);
  if (pos >= 0) return pos - p0 + 1;
  int end2 = p0 + W - Wp1;  // wrapped part [0, p0-1)
  pos = first_bit_in(row, 0, end2);
  if (pos >= 0) return (Wp1 - p0) + pos + 1;
  return 0;
}

// Acquire load of a 64-bit device counter (spin-waits on flags another kernel publishes).
__device__ __forceinline__ uint64_t ld_acquire_u64(const void* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// 16-byte vector copies.
// Device-memory rows are streamed (.nc, no L1 allocation, .cs stores); rows in host
// memory mapped over PCIe use plain ld/st (cache-policy qualifiers are not valid on
// the system address space).
enum Mem : int { kDev = 0, kHost = 1 };
template <int M>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 r;
  if (M == kDev)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  return r;
}
template <int M>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
  if (M == kDev)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Warp copies one row of `nvec` 16-byte vectors, UNROLL vectors in flight per lane.
template <int UNROLL, int SRC, int DST>
__device__ __forceinline__ void warp_copy_row(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                              int nvec) {
  const int lane = (int)lane_id();
  int i = lane;
  for (; i + 32 * (UNROLL - 1) < nvec; i += 32 * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = ld16<SRC>(src + i + 32 * u);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) st16<DST>(dst + i + 32 * u, v[u]);
  }
  for (; i < nvec; i += 32) st16<DST>(dst + i, ld16<SRC>(src + i));
}

// ---- TMA bulk row copies (cp.async.bulk, sm_90+; the B200 path for whole-row HBM copies)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(g), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}
// The same copies with an L2 eviction-priority policy (createpolicy): the row streams of a step
// are touched once, so they are loaded and stored evict_first and the metadata the next
// step's latency-bound kernels walk (tags, stamps, node_loc, reuse masks) stays in L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem, const void* g, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem)),
      "l"(g), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* g, const void* smem, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(g),
               "r"(smem_u32(smem)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most k committed bulk groups still have to READ their shared-memory source
__device__ __forceinline__ void bulk_wait_read(uint32_t k) {
  switch (k) {
    case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory"); break;
  }
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// A warp's ring of ST row stages in shared memory, driven by its lane 0: rows are loaded with
// cp.async.bulk (global -> shared, completion on the stage's mbarrier) and stored with
// cp.async.bulk (shared -> global, bulk groups). At most ST - 1 loads are in flight, so the stage
// a new load reuses is the one stored one step EARLIER: its store has (almost always) finished
// reading shared memory, and the store just issued may still be reading (wait_group.read 1).
// (Reloading the stage just stored would wait for every store to drain: measured as the top
// stall of the first version, profiles/r02_ncu_hit.md.) Counters run across calls so that the
// stage phases stay consistent.
constexpr uint32_t kMaxStages = 8;
struct RowRing {
  uint8_t* buf;    // ST * R bytes of this warp's shared memory
  uint64_t* bar;   // ST mbarriers
  uint32_t* pend;  // ST entries: the row index (into dst[]) whose load occupies the stage
  uint32_t ST, R;
  uint32_t nl, ns, phase;  // loads issued, stores issued (lane 0), phase bit per stage
  uint32_t hint;           // 1: rows loaded and stored with the L2 evict_first policy `pol`; 2: stored only
  uint64_t pol;
};
__device__ __forceinline__ void ring_init(RowRing& r) {  // lane 0; then __syncwarp
  for (uint32_t s = 0; s < r.ST; ++s) mbar_init(&r.bar[s], 1);
  mbar_fence_init();
  r.nl = r.ns = r.phase = 0;
  r.pol = r.hint ? l2_policy_evict_first() : 0;
}
// Lane 0: copy rows j in `mask` (bit j) from src[j] to dst[j] (R bytes each, 16-B aligned),
// returning when every store has been issued (its completion is awaited by ring_drain or the
// next stage reuse).
__device__ __forceinline__ void ring_copy(RowRing& r, const void* const* src, void* const* dst, uint32_t mask) {
  const uint32_t total = __popc(mask);
  uint32_t issued = 0, stored = 0;
  while (stored < total) {
    while (issued < total && r.nl - r.ns < r.ST - 1) {
      const uint32_t j = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t s = r.nl % r.ST;
      // the stage's last store (number nl - ST) must have read it; later stores may still read
      if (r.nl >= r.ST) bulk_wait_read(r.ns + r.ST - 1 - r.nl);
      mbar_expect_tx(&r.bar[s], r.R);
      if (r.hint == 1) bulk_g2s_hint(r.buf + (size_t)s * r.R, src[j], r.R, &r.bar[s], r.pol);
      else bulk_g2s(r.buf + (size_t)s * r.R, src[j], r.R, &r.bar[s]);
      r.pend[s] = j;
      ++r.nl;
      ++issued;
    }
    const uint32_t s = r.ns % r.ST;
    mbar_wait_parity(&r.bar[s], (r.phase >> s) & 1u);
    r.phase ^= 1u << s;
    if (r.hint) bulk_s2g_hint(dst[r.pend[s]], r.buf + (size_t)s * r.R, r.R, r.pol);
    else bulk_s2g(dst[r.pend[s]], r.buf + (size_t)s * r.R, r.R);
    bulk_commit();
    ++r.ns;
    ++stored;
  }
}
__device__ __forceinline__ void ring_drain() { bulk_wait_all(); }  // lane 0, before the kernel ends

template <typename T>
__device__ __forceinline__ void warp_bitonic_sort(T* a, int P) {
  const int lane = (int)lane_id();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = (i & k) == 0;
          T x = a[i], y = a[ixj];
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace lsm

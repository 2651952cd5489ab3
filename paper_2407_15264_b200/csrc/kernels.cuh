// kernels.cuh — sm_100a kernels of the LSM-GNN gather hot path.
//
// Step names follow SURVEY.md §8(a) (S1..S11) and DESIGN.md §"Kernels":
//   k_begin/k_end  S9  per-iteration state (IterState: t, stamps, batch pointer) and counters
//   k_route_peer   S1  G > 1: bucket by home (v mod G), store into the homes' inboxes (P2P)
//   k_dedup        S1+S3 home: unique nodes (node-indexed stamp table) + per-set counts; at G = 1 it
//                       reads the caller's IDs directly and threads the request lists
//   k_scan         S3  home: exclusive scan of per-set counts; oversized-set scratch; PVP "unused"
//   k_bucket       S3  home: scatter unique nodes into set buckets
//   k_snapshot     S4  period > 1: the paper's periodic window scan of every resident line
//   k_set          S4+S5 home: warp per touched set — tag probe, staging probe, bypass selection,
//                       way assignment by the policy key, eviction classes, victim candidates
//   k_qscatter/k_admit  S5  victim admission per queue (PVP); k_set builds the histogram
//   k_serve        S6+S8 G = 1: fill (victim D2H, storage/staging row -> slot) fused with delivery
//                       to every requester; 1 warp in 8 copies the hits
//   k_fill         S6  G > 1: victim row D2H then new row -> slot / bypass staging
//   k_pull         S7+S8 G > 1: location lookup at the home + row copy (local or peer HBM)
//   k_win_begin, k_mask_clear, k_win_gather (+ k_route_local)  S10  window feed (reuse bitmask)
//   k_pvp          S11 PVP copy of victim queue (t+1) mod W into home staging (side stream)
#pragma once
#include "device_common.cuh"

namespace lsm {

// Build-time timeline probe (nvcc -DLSMGNN_TRACE, experiments only, never in the product build):
// per kernel and iteration parity, the earliest CTA start and the latest CTA end (%globaltimer).
#ifdef LSMGNN_TRACE
__device__ unsigned long long g_trace[8][2][2];
__device__ __forceinline__ unsigned long long trace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE_AT(k, par, e) \
  do { if (threadIdx.x == 0) { if (e) atomicMax(&g_trace[k][par][1], trace_now()); else atomicMin(&g_trace[k][par][0], trace_now()); } } while (0)
#else
#define TRACE_AT(k, par, e) do { } while (0)
#endif

// Reuse-bitmask updates with an L2 eviction-priority policy (evict_last: the mask rows the window
// feed sets, k_dedup clears and k_set reads stay in L2 while the row stream passes through)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void red_or_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_and_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("red.global.and.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// ------------------------------------------------------------------------------ S9
// Start gather t: publish the iteration's values (IterState), zero its record and the per-batch
// scratch counters. t_host >= 0: t and the batch come from the
// host; t_host < 0 (graph replay): t = it->t_next, batch = ids_ring[t mod ring_len].
struct BeginArgs {
  int64_t t_host;
  const int64_t* ids_host;
  int64_t n_host;
  const int64_t* const* ids_ring;  // graph replay: device array of batch pointers
  const int64_t* n_ring;           // and their lengths
  uint32_t ring_len;
  uint32_t Wp1, period, L, C;
  int64_t cap;                     // max_batch_ids: a longer device-resident batch is clamped ...
  volatile uint32_t* overflow;     // ... and flagged here (pinned host word, sticky EINVAL)
};
// The per-iteration values of gather t, from the host arguments (direct calls) or from the
// device's own iteration counter and the caller's ring of batches (graph replay). `clamped` is
// set when a device-resident length exceeded max_batch_ids.
struct IterVals {
  uint64_t t;
  const int64_t* ids;
  int64_t n;
  bool clamped;
};
__device__ __forceinline__ IterVals begin_values(const BeginArgs& a, const IterState* it) {
  IterVals v;
  v.t = a.t_host >= 0 ? (uint64_t)a.t_host : it->t_next;
  v.clamped = false;
  if (a.t_host >= 0) {
    v.ids = a.ids_host;
    v.n = a.n_host;
  } else {
    const uint32_t k = (uint32_t)(v.t % a.ring_len);
    v.ids = a.ids_ring[k];
    v.n = a.n_ring[k];
    if (v.n > a.cap || v.n < 0) {
      v.n = v.n < 0 ? 0 : a.cap;
      v.clamped = true;
    }
  }
  return v;
}
// Publish them in IterState for the kernels that follow (one thread).
__device__ __forceinline__ void begin_publish(const BeginArgs& a, const IterVals& v, IterState* it,
                                              unsigned long long* hist) {
  const uint64_t t = v.t;
  it->t = t;
  it->ids = v.ids;
  it->n = v.n;
  if (v.clamped) *a.overflow = 1u;
  it->stamp = (uint32_t)(t + 1);
  it->p0 = (uint32_t)((t + 1) % a.Wp1);
  it->par = (uint32_t)(t & 1);
  it->upd = a.period <= 1 || t % a.period == 0;
  it->rec_idx = (uint32_t)(t % kHist);
  it->stage_base = a.L + (uint32_t)(t & 1) * a.C;
  hist[(size_t)(t % kHist) * F_NFIELDS + F_ITER] = t;
}
// G > 1 (the route kernels read the batch before k_dedup runs): publish the iteration's values.
// The record of t and the per-batch scratch counters were zeroed by end_record of t - 1 (and
// by allocation before the first gather); at G = 1 k_dedup publishes them itself.
__global__ void k_begin(IterState* it, unsigned long long* hist, Scratch* scr, BeginArgs a) {
  pdl_prologue();
  if (threadIdx.x == 0) begin_publish(a, begin_values(a, it), it, hist);
}

// Close the record (G > 1, after the pulls; at G = 1 the last CTA of k_serve does it):
// end_record below, one warp.
struct EndArgs {
  IterState* it;
  unsigned long long* hist;
  unsigned long long* cum;
  Scratch* scr;
  uint32_t R;
  volatile uint32_t* bad_mirror;
};
__device__ __forceinline__ void end_record(uint64_t t, IterState* it, unsigned long long* hist, unsigned long long* cum,
                                           Scratch* scr, uint32_t R, volatile uint32_t* bad_mirror);
__global__ void k_end(EndArgs a) {
  pdl_prologue();
  end_record(a.it->t, a.it, a.hist, a.cum, a.scr, a.R, a.bad_mirror);
}

// Start the window feed of one batch (iteration wk): k_host >= 0 from the host, else (graph
// replay) wk = it->wk_next with the batch from the ring.
__global__ void k_win_begin(IterState* it, int64_t k_host, const int64_t* ids_host, int64_t n_host,
                            const int64_t* n_dev, const int64_t* const* ids_ring, const int64_t* n_ring,
                            uint32_t ring_len, uint32_t Wp1, int64_t cap, volatile uint32_t* overflow) {
  pdl_prologue();
  if (threadIdx.x != 0) return;
  const uint64_t k = k_host >= 0 ? (uint64_t)k_host : it->wk_next;
  it->wk = k;
  it->wslot = (uint32_t)(k % Wp1);
  if (k_host >= 0) {
    it->wids = ids_host;
    it->wn = n_dev ? *n_dev : n_host;  // n_dev: a length produced on the device (lsmgnn_sample)
  } else {
    const uint32_t j = (uint32_t)(k % ring_len);
    it->wids = ids_ring[j];
    it->wn = n_ring[j];
  }
  if (it->wn > cap || it->wn < 0) {  // a device-resident length beyond max_batch_ids
    it->wn = it->wn < 0 ? 0 : cap;
    *overflow = 1u;
  }
  it->wk_next = k + 1;
}

// ------------------------------------------------------------------------------ S10 (G = 1)
// Window feed at one home, one launch: store the batch of iteration k (u32, position i of the
// caller's list at slot entry i; an invalid ID counts toward ERANGE and is stored as kInvalid)
// into ring slot k mod (W+1) and set each node's reuse bit of the slot. The slot's previous
// bits (iteration k - W - 1) were cleared by k_dedup of gather(k - W - 1), which this launch
// follows. k_host >= 0: iteration, IDs and count are kernel arguments (direct calls; block 0
// also advances it->wk_next so that graph replays can follow); k_host < 0 (graph replay):
// k_win_begin published them in IterState. (The gather side of S1 at G = 1 is fused into
// k_dedup.)
// wait_prev = 0 (the host sets it only when the library's previous launch on this stream was
// the k_serve of gather t): no griddepcontrol.wait — the feed of iteration k = t+1+W depends on
// nothing gather t writes (k_dedup(t) cleared its slot, and k_dedup/k_set completed before
// k_serve(t) could trigger this launch), and the caller's IDs were produced before gather(t) (a
// kernel or copy of the caller's in between is not a programmatic predecessor: no early start).
// So it runs alongside k_serve(t) on the SMs k_serve leaves free, and waits for k_serve(t) only
// at its END (in one CTA): the launch completes after k_serve(t) did, so the programmatic wait of
// k_dedup(t+1) still covers gather t, and so does any later work the caller puts on the stream.
__global__ void k_route_local(IterState* it, int64_t k_host, const int64_t* ids_host, int64_t n_host, uint32_t Wp1,
                              uint64_t N, uint32_t* __restrict__ ring, uint64_t stride, uint32_t* __restrict__ ring_len,
                              Scratch* scr, uint32_t* __restrict__ mask, uint32_t MW, uint32_t wait_prev,
                              uint32_t mask_hint) {
  if (wait_prev || k_host < 0) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t mpol = mask_hint ? l2_evict_last_policy() : 0;
  const int64_t* __restrict__ ids;
  int64_t n;
  uint32_t slot;
  if (k_host >= 0) {
    ids = ids_host;
    n = n_host;
    slot = (uint32_t)((uint64_t)k_host % Wp1);
  } else {
    ids = it->wids;
    n = it->wn;
    slot = it->wslot;
  }
  uint32_t* __restrict__ list = ring + (size_t)slot * stride;
  TRACE_AT(4, (uint32_t)(k_host & 1), 0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = ids[i];
    if (x >= 0 && (uint64_t)x < N) {
      list[i] = (uint32_t)x;
      if (mask_hint) red_or_hint(&mask[(size_t)x * MW + (slot >> 5)], 1u << (slot & 31), mpol);  // G = 1: q = v
      else atomicOr(&mask[(size_t)x * MW + (slot >> 5)], 1u << (slot & 31));
    } else {
      list[i] = kInvalid;
      atomicAdd(&scr->bad_ids, 1u);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ring_len[slot] = (uint32_t)n;
    // (feeds of consecutive iterations may overlap: the latest one wins)
    if (k_host >= 0) atomicMax(reinterpret_cast<unsigned long long*>(&it->wk_next), (unsigned long long)k_host + 1);
  }
  TRACE_AT(4, (uint32_t)(k_host & 1), 1);
  // early feed (behind a G = 1 gather): this CTA's list entries and bits are written — count it
  // (an early k_set waits for the count of the early feeds the host launched; a feed that is not
  // early is followed by a gather that is not early either)
  if (!wait_prev && k_host >= 0) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&it->feed_ctas_done, 1ull);
    }
  }
  // complete after k_serve(t): one CTA waits, the others exit and free their SM slots (for the
  // early k_dedup of gather t + 1)
  if (!wait_prev && k_host >= 0 && blockIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------------------------ S1 (G > 1)
// Requester side of the communication layer: bucket each valid ID by its
// home g = v mod G and store it straight into home g's inbox slot [me] through the
// peer mapping. Counts go to route_cnt[g] (local) and are published by k_route_publish.
struct RouteArgs {
  uint32_t* inbox[8];  // inbox base of each home (peer-mapped), slot [me] already applied
  uint32_t* route_cnt; // [G] local counters
  uint32_t G;
};
__global__ void k_route_peer(const IterState* it, uint32_t window, uint64_t N, RouteArgs a, Scratch* scr) {
  pdl_prologue();
  __shared__ uint32_t s_cnt[8], s_base[8];
  const int64_t* __restrict__ ids = window ? it->wids : it->ids;
  const int64_t n = window ? it->wn : it->n;
  const int64_t tile = blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * tile; base < n; base += (int64_t)gridDim.x * tile) {
    if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    bool ok = false;
    uint32_t v = 0, g = 0, local = 0;
    if (i < n) {
      const int64_t x = ids[i];
      ok = x >= 0 && (uint64_t)x < N;
      if (!ok) atomicAdd(&scr->bad_ids, 1u);
      v = (uint32_t)x;
      g = v % a.G;
      if (ok) local = atomicAdd(&s_cnt[g], 1u);
    }
    __syncthreads();
    if (threadIdx.x < a.G) s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(&a.route_cnt[threadIdx.x], s_cnt[threadIdx.x]) : 0;
    __syncthreads();
    if (ok) a.inbox[g][s_base[g] + local] = v;
    __syncthreads();
  }
}
// Publish this requester's per-home counts into every home's inbox header [me].
struct PublishArgs {
  uint32_t* peer_cnt[8];  // inbox_cnt array of each home (peer-mapped)
  uint32_t G, me;
};
__global__ void k_route_publish(const uint32_t* route_cnt, PublishArgs a) {
  pdl_prologue();
  const uint32_t g = threadIdx.x;
  if (g < a.G) {
    a.peer_cnt[g][a.me] = route_cnt[g];
    __threadfence_system();
  }
}

// ------------------------------------------------------------------------------ S3
// Home: one representative per distinct node (stamp table indexed by q = v / G), written
// straight into its cache set's bucket: bucket[s * BC + set_cnt[s]++] (BC = the most distinct
// nodes one set can receive in a batch, ceil(Q / S) capped by the batch capacity), so no scan
// or scatter pass is needed; k_set sorts each bucket before any order-dependent step and
// resets set_cnt. Requests and peer requests are counted here (every count but `requests` is
// over unique nodes, R11).
// G = 1 (direct): the caller's int64 IDs are read straight from it->ids and validated here
// (S1 fused away; an ID >= N counts toward ERANGE and is skipped), and every request
// position i is threaded onto its node's list for the fused delivery of k_serve:
// head[q] = stamp<<32 | last position, nxt[i] = previous (kInvalid = end).
// G > 1: the IDs come from the inbox segments of the nsrc requesters.
// S10 (window): the same launch drops the reuse bits of iteration t (ring slot t mod (W+1)):
// gather(t) reads iterations t+1..t+W only, and gather(t-1), the last reader of those bits,
// has completed; the feed of t+1+W (which rewrites the slot) is ordered after this kernel.
struct DedupArgs;
struct DedupPar;
__device__ __forceinline__ uint32_t dedup_one(uint32_t v, uint32_t pos, const DedupArgs& a, const DedupPar& pp,
                                              uint32_t stamp, uint32_t t, uint32_t* nhit);
struct DedupArgs {
  const uint32_t* inbox;
  const uint32_t* inbox_cnt;
  uint32_t nsrc, cap, me, G, S, BC;
  uint32_t* mark;
  uint32_t* bucket;
  uint32_t* set_cnt;
  unsigned long long* head;  // G = 1: request lists of the fused delivery (two parities of Q entries)
  uint32_t* nxt;             // (two parities of cap entries)
  uint32_t direct;
  uint64_t N;
  // window slot of iteration t: its list and the reuse mask (bit t mod (W+1) is cleared)
  const uint32_t* ring;
  uint64_t ring_stride;
  const uint32_t* ring_len;
  uint32_t* mask;
  uint32_t MW, Wp1;
  uint64_t Q;  // home rows (the overflow sweep)
  // S4 hit probe of every distinct node (the cache state is final: the previous k_serve is done):
  // a hit writes node_loc and the way's last use (hits are protected, R10) and is counted here;
  // a node that is not resident marks its set for k_set (slow_stamp[s] = stamp)
  const uint32_t* tags;
  uint32_t* last_use;
  uint32_t* node_loc;
  uint64_t loc_stride;  // G = 1: node_loc has one table per iteration parity (Q apart); G > 1: 0
  uint32_t* req_loc;    // G = 1: per-request locations, one table per iteration parity (cap apart)
  uint32_t meta_evict_last;  // L2 evict_last policy on the probe's metadata accesses (A/B)
  uint32_t mask_hint;        // ... and on the window clear's mask updates
  uint32_t* slow_stamp;
  uint32_t* slow_list;  // the sets with a miss this batch (count scr->nslow[t & 1])
  uint32_t A;
};
// The tables of iteration t's parity: with `early` (below) k_dedup(t+1) runs while k_serve(t)
// still reads node_loc, the request lists and its counters of parity t & 1.
struct DedupPar {
  uint32_t* node_loc;
  unsigned long long* head;
  uint32_t* nxt;
  uint32_t* nslow;
  uint32_t* req_loc;  // G = 1: per request position, the slot of a first-occurrence hit, else kPending
  uint32_t hint;      // 1: the probe's metadata accesses carry the L2 policy pol
  uint64_t pol;
};
constexpr uint32_t kPending = 0xFFFFFFFEu;  // req_loc: look the location up in node_loc (k_serve)
// One request: first occurrence of its node (returns 1) is probed against its set's A tags; a
// hit writes node_loc and the way's last use (= t: hits are protected, R10, and k_set reads the
// protection from last_use), a miss goes into the set's bucket (the bucket holds the batch's
// MISSES only: k_set works on those and on the resident lines).
// The tag loads are issued with the stamp exchange (speculatively for a repeated occurrence, one
// extra 128-B read), so a hit costs two dependent round trips: IDs, then stamp + tags.
// G = 1: request position pos joins node q's list (head[q] = stamp<<32 | pos, nxt[pos] = previous)
// — the positions a fill of q delivers its row to (k_serve). A hit is delivered through node_loc,
// so the FIRST occurrence of a hit node never needs to be on the list (the common case skips the
// atomic); later occurrences join it before they know whether the node hit (harmless).
__device__ __forceinline__ void list_join(const DedupPar& pp, uint32_t q, uint32_t pos, uint32_t stamp) {
  const unsigned long long old = atomicExch(&pp.head[q], ((unsigned long long)stamp << 32) | pos);
  pp.nxt[pos] = (uint32_t)(old >> 32) == stamp ? (uint32_t)old : kInvalid;
}
// 16-byte load that the compiler may neither drop nor sink into the branch that uses it
__device__ __forceinline__ uint4 ld16_issue(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// ... and the same accesses with an L2 eviction-priority policy (DedupPar::pol, evict_last): the
// probe's scattered metadata stays in L2 while the previous gather's row stream passes through
__device__ __forceinline__ uint4 ld16_issue_hint(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t atom_exch_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  uint32_t r;
  asm volatile("atom.global.exch.L2::cache_hint.b32 %0, [%1], %2, %3;" : "=r"(r) : "l"(p), "r"(v), "l"(pol) : "memory");
  return r;
}
__device__ __forceinline__ void st_u32_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t dedup_one(uint32_t v, uint32_t pos, const DedupArgs& a, const DedupPar& pp,
                                              uint32_t stamp, uint32_t t, uint32_t* nhit) {
  const uint32_t q = v / a.G;
  const uint32_t s = q % a.S;
  const uint32_t* tg = a.tags + (size_t)s * a.A;
  const bool vec = (a.A & 3u) == 0;  // a set's tags are whole 16-B words (A = 4, 8, ..., 32)
  uint4 w[8];
  if (vec) {
    const uint4* t4 = reinterpret_cast<const uint4*>(tg);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      w[i] = 4u * i < a.A ? (pp.hint ? ld16_issue_hint(t4 + i, pp.pol) : ld16_issue(t4 + i))
                          : make_uint4(kInvalid, kInvalid, kInvalid, kInvalid);
  }
  const bool first = (pp.hint ? atom_exch_hint(&a.mark[q], stamp, pp.pol) : atomicExch(&a.mark[q], stamp)) != stamp;
  if (!first) {
    if (pp.head) list_join(pp, q, pos, stamp);
    if (pp.req_loc) pp.req_loc[pos] = kPending;
    return 0;
  }
  int way = -1;
  if (vec) {
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      if (w[i].w == v) way = 4 * i + 3;
      if (w[i].z == v) way = 4 * i + 2;
      if (w[i].y == v) way = 4 * i + 1;
      if (w[i].x == v) way = 4 * i;
    }
  } else {
    for (uint32_t k = 0; k < a.A; ++k)
      if (tg[k] == v) way = (int)k;
  }
  if (way >= 0) {
    if (pp.hint) {
      st_u32_hint(&pp.node_loc[q], s * a.A + (uint32_t)way, pp.pol);
      st_u32_hint(&a.last_use[s * a.A + (uint32_t)way], t, pp.pol);
    } else {
      pp.node_loc[q] = s * a.A + (uint32_t)way;
      a.last_use[s * a.A + (uint32_t)way] = t;
    }
    if (pp.req_loc) pp.req_loc[pos] = s * a.A + (uint32_t)way;
    ++*nhit;
  } else {
    const uint32_t slot = atomicAdd(&a.set_cnt[s], 1u);
    a.bucket[(size_t)s * a.BC + slot] = v;
    if (pp.head) list_join(pp, q, pos, stamp);  // a fill will deliver this row
    if (pp.req_loc) pp.req_loc[pos] = kPending;
    if (a.slow_stamp[s] != stamp && atomicExch(&a.slow_stamp[s], stamp) != stamp)
      a.slow_list[atomicAdd(pp.nslow, 1u)] = s;  // first miss of the set: k_set processes it
  }
  return 1;
}
// early = 1 (the host sets it for a direct G = 1 gather whose programmatic predecessor on the
// stream is the k_serve of gather t - 1, or the early window feed that followed it): no wait at
// the start. Everything this launch reads is final once k_serve(t-1) has started — the cache
// state (k_set(t-1) completed before k_serve(t-1) could trigger), the caller's IDs (produced
// before gather(t-1) or by a non-programmatic predecessor), the window slot of t — and what it
// writes is not read by k_serve(t-1): node_loc, the request lists, the per-request locations and
// the slow-set counter are parity-indexed, the record of t is its own, and k_serve(t-1) of a
// direct call takes its iteration's values from its arguments, not from IterState. So the dedup
// and hit probe of t run alongside the delivery of t-1 and so does k_set(t) behind it (it waits
// for this launch's finished-CTA count and the window feeds issued before gather t, and writes
// nothing k_serve(t-1) reads: fill list, counters and node_loc are parity-indexed); k_serve(t)
// then waits for k_set(t)'s count and k_serve(t-1)'s published t_next before it fills any slot.
__global__ void __launch_bounds__(256, 4) k_dedup(DedupArgs a, IterState* it, Scratch* scr, unsigned long long* hist, BeginArgs ba,
                        uint32_t fused_begin, uint32_t early) {
  // (every thread reaches the __syncthreads below: no early exit before it)
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint64_t t64;
  const int64_t* ids_b;
  int64_t n_b;
  if (fused_begin) {
    const IterVals v = begin_values(ba, it);
    t64 = v.t;
    ids_b = v.ids;
    n_b = v.n;
    if (blockIdx.x == 0 && threadIdx.x == 0) begin_publish(ba, v, it, hist);
  } else {
    t64 = it->t;
    ids_b = it->ids;
    n_b = it->n;
  }
  const uint32_t stamp = (uint32_t)(t64 + 1);
  unsigned long long* rec = hist + (size_t)(t64 % kHist) * F_NFIELDS;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t par = (uint32_t)(t64 & 1);
  DedupPar pp;
  pp.node_loc = a.node_loc + par * a.loc_stride;
  pp.head = a.head ? a.head + (size_t)par * a.Q : nullptr;
  pp.nxt = a.nxt ? a.nxt + (size_t)par * a.cap : nullptr;
  pp.nslow = &scr->nslow[par];
  pp.req_loc = a.req_loc ? a.req_loc + (size_t)par * a.cap : nullptr;
  pp.hint = a.meta_evict_last;
  pp.pol = 0;
  if (pp.hint) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pp.pol));
  TRACE_AT(0, par, 0);
  {  // S10: clear the bits of iteration t (its window list is in ring slot t mod (W+1))
    const uint32_t slot = (uint32_t)(t64 % a.Wp1);
    const uint32_t* __restrict__ list = a.ring + (size_t)slot * a.ring_stride;
    const uint32_t nl = a.ring_len[slot];
    const uint32_t m = ~(1u << (slot & 31));
    const uint64_t mpol = a.mask_hint ? l2_evict_last_policy() : 0;
    if (nl == 0xFFFFFFFFu) {  // the slot's list did not fit its ring slot (k_win_gather): sweep
      for (uint64_t q = blockIdx.x * blockDim.x + threadIdx.x; q < a.Q; q += stride)
        atomicAnd(&a.mask[q * a.MW + (slot >> 5)], m);
    } else {
      for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
        const uint32_t v = list[i];
        if (v == kInvalid) continue;
        if (a.mask_hint) red_and_hint(&a.mask[(size_t)(v / a.G) * a.MW + (slot >> 5)], m, mpol);
        else atomicAnd(&a.mask[(size_t)(v / a.G) * a.MW + (slot >> 5)], m);
      }
    }
  }
  uint32_t nreq = 0, npeer = 0, nfirst = 0, nhit = 0;
  const uint32_t t = (uint32_t)t64;
  if (a.direct) {
    const int64_t* __restrict__ ids = ids_b;
    const int64_t n = n_b;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const int64_t x = ids[i];
      if (x >= 0 && (uint64_t)x < a.N) {
        nfirst += dedup_one((uint32_t)x, (uint32_t)i, a, pp, stamp, t, &nhit);
        ++nreq;
      } else {
        atomicAdd(&scr->bad_ids, 1u);
        if (pp.req_loc) pp.req_loc[i] = kInvalid;  // ERANGE: k_serve zero-fills the row
      }
    }
  } else {
    for (uint32_t r = 0; r < a.nsrc; ++r) {
      const uint32_t n = a.inbox_cnt[r];
      const uint32_t* in = a.inbox + (size_t)r * a.cap;
      for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        nfirst += dedup_one(in[i], i, a, pp, stamp, t, &nhit);
        ++nreq;
        if (r != a.me) ++npeer;
      }
    }
  }
  // counters: warp -> CTA (shared memory) -> one atomic per CTA and counter (a warp-level atomic
  // on these four hot addresses serialised thousands of atomics per batch at L2)
  __shared__ uint32_t s_cnt[4];
  if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  nreq = __reduce_add_sync(0xffffffffu, nreq);
  npeer = __reduce_add_sync(0xffffffffu, npeer);
  nfirst = __reduce_add_sync(0xffffffffu, nfirst);
  nhit = __reduce_add_sync(0xffffffffu, nhit);
  if (lane_id() == 0) {
    if (nreq) atomicAdd(&s_cnt[0], nreq);
    if (nfirst) atomicAdd(&s_cnt[1], nfirst);
    if (nhit) atomicAdd(&s_cnt[2], nhit);
    if (npeer) atomicAdd(&s_cnt[3], npeer);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_cnt[0]) atomicAdd(&rec[F_REQ], (unsigned long long)s_cnt[0]);
    if (s_cnt[1]) atomicAdd(&rec[F_UNIQUE], (unsigned long long)s_cnt[1]);
    if (s_cnt[2]) atomicAdd(&rec[F_HIT], (unsigned long long)s_cnt[2]);
    if (s_cnt[3]) atomicAdd(&rec[F_PEER], (unsigned long long)s_cnt[3]);
  }
  TRACE_AT(0, par, 1);
  // early: this CTA's stores are done — count it (the early k_set of this gather waits for the
  // count of the early k_dedup CTAs the host launched)
  if (early) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&it->dedup_ctas_done, 1ull);
    }
  }
}

// Exclusive prefix of one value per thread over a 1024-thread CTA.
__device__ __forceinline__ uint32_t block_exclusive_1024(uint32_t v, uint32_t* s_warp) {
  const uint32_t tid = threadIdx.x;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((tid & 31) >= (uint32_t)o) x += y;
  }
  __syncthreads();
  if ((tid & 31) == 31) s_warp[tid >> 5] = x;
  __syncthreads();
  if (tid < 32) {
    uint32_t w = s_warp[tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (tid >= (uint32_t)o) w += y;
    }
    s_warp[tid] = w;
  }
  __syncthreads();
  return x - v + ((tid >> 5) ? s_warp[(tid >> 5) - 1] : 0u);
}
__device__ __forceinline__ uint32_t pow2_at_least_32(uint32_t m) {
  uint32_t p = 32;
  while (p < m) p <<= 1;
  return p;
}

// Exclusive scan of cnt[0..n) into off[0..n], one CTA (1024 threads) per tile of 4096 counts
// (the per-queue victim-candidate counts of the admission step). Each CTA scans its tile in
// shared memory (coalesced loads and stores; each thread owns 4 contiguous counts, skewed
// against bank conflicts), publishes the tile total, and takes its carry from the totals of the
// tiles before it (look-back on per-tile flags stamped with `seq`, unique per iteration).
constexpr uint32_t kScanTile = 4096;
struct ScanSync {
  uint32_t* flag;  // [tiles] seq once agg of the tile is published
  uint32_t* agg;   // [tiles] tile totals
};
__device__ __forceinline__ uint32_t scan_skew(uint32_t j) { return j + (j >> 5); }
__global__ void __launch_bounds__(1024) k_scan(const uint32_t* __restrict__ cnt, uint32_t* __restrict__ off,
                                               uint32_t n, const IterState* it, ScanSync sy) {
  pdl_prologue();
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  __shared__ uint32_t s_c[kScanTile + kScanTile / 32];
  const uint32_t tid = threadIdx.x, b = blockIdx.x;
  const uint32_t base = b * kScanTile;
  const uint32_t seq = it->stamp;
  for (uint32_t j = tid; j < kScanTile; j += 1024) s_c[scan_skew(j)] = base + j < n ? cnt[base + j] : 0u;
  __syncthreads();
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = s_c[scan_skew(tid * 4 + k)];
    sum += v[k];
  }
  uint32_t run = block_exclusive_1024(sum, s_warp);
  const uint32_t total = s_warp[31];
  if (gridDim.x > 1) {
    if (tid == 0) {  // publish this tile's total
      sy.agg[b] = total;
      __threadfence();
      *(volatile uint32_t*)&sy.flag[b] = seq;
    }
    if (tid < 32) {  // carry = totals of the tiles before this one
      uint32_t c = 0;
      for (uint32_t j = tid; j < b; j += 32) {
        while (*(volatile const uint32_t*)&sy.flag[j] != seq) {
        }
        __threadfence();
        c += *(volatile const uint32_t*)&sy.agg[j];
      }
      c = __reduce_add_sync(0xffffffffu, c);
      if (tid == 0) s_carry = c;
    }
    __syncthreads();
    run += s_carry;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    s_c[scan_skew(tid * 4 + k)] = run;
    run += v[k];
  }
  __syncthreads();
  for (uint32_t j = tid; j < kScanTile && base + j < n; j += 1024) off[base + j] = s_c[scan_skew(j)];
  if (b == gridDim.x - 1 && tid == 1023) off[n] = run;  // the grand total
}

// ------------------------------------------------------------------------------ S4 (period > 1)
// Window scan of every resident line ("scans the sampled nodes in the window buffer to
// determine the next reuse iteration for the cache-lines that currently reside in the cache
// before the feature aggregation stage"), run every P-th iteration.
__global__ void k_snapshot(const uint32_t* __restrict__ tags, uint32_t L, uint32_t G, const uint32_t* __restrict__ mask,
                           uint32_t MW, uint32_t W, const IterState* it, uint32_t* __restrict__ line_info) {
  pdl_prologue();
  if (!it->upd) return;  // not a scan iteration (t mod P != 0)
  const uint32_t p0 = it->p0, t = (uint32_t)it->t;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const uint32_t x = tags[i];
    uint32_t info = kInfoNone;
    if (x != kInvalid) {
      const int d = next_reuse_d(mask + (size_t)(x / G) * MW, (int)p0, (int)W);
      if (d) info = t + (uint32_t)d;
    }
    line_info[i] = info;
  }
}

// ------------------------------------------------------------------------------ S4 + S5
struct SetParams {
  uint32_t* set_cnt;     // distinct nodes per set this batch (k_dedup); k_set resets it to 0
  const uint32_t* slow_stamp;  // == stamp: a node of the set missed in k_dedup's probe
  const uint32_t* slow_list;   // those sets (count scr->nslow)
  const uint32_t* bucket;  // set s's nodes at bucket[s * BC, + set_cnt[s])
  uint32_t BC, BCp;      // bucket capacity per set; global-scratch region per oversized set (pow2 >= BC)
  uint32_t* tags;
  uint32_t* last_use;
  uint32_t* rr;
  const uint8_t* score;
  const uint32_t* mask;
  uint32_t* node_loc;
  uint64_t loc_stride;  // G = 1: one node_loc table per iteration parity (Q apart); G > 1: 0
  const uint32_t* vst_stamp;
  const uint32_t* vst_idx;
  FillEnt* fills;        // two parities of fstride entries
  uint64_t fstride;
  uint64_t dedup_wait;   // early: k_dedup CTAs (cumulative) that must have finished; 0 = not early
  uint64_t feed_wait;    // early: window-feed CTAs (cumulative) that must have finished
  Cand* cands;
  uint32_t* qcnt;        // per-queue candidate counts (pvp = 1), zero on entry
  Scratch* scr;
  IterState* it;             // t, stamp, p0, staging parity, record of this iteration (early: done counter)
  unsigned long long* hist;
  uint32_t S, A, G, W, T, MW;
  uint32_t policy, pvp, reinsert;
  uint32_t P;            // per-warp shared capacity (power of two); larger buckets use g_* scratch
  uint32_t *g_sv, *g_sk, *g_sidx;
  unsigned long long* g_skey;
  uint32_t period;       // dynamic-information update period; 1 = exact every batch
  uint32_t* line_info;   // period > 1: per-line snapshot (reuse iteration / kInfoNone / kInfoFresh)
  uint32_t warp_bytes;   // per-warp shared memory
  uint32_t bypass_base;  // pool row of the bypass staging area
  uint32_t deliver;      // kDelivered: node_loc marks rows filled this batch (k_serve / k_pull phases)
  // pvp_unused: PVP-staged rows (stg_nodes, by parity) whose node this batch did not request
  const uint32_t* stg_nodes;
  const uint32_t* mark;
  uint32_t C;
};

enum { C_HIT, C_VHIT, C_STOR, C_INS, C_BYP, C_EVICT, C_EV0, C_EV1, C_EV2, C_EV3, C_ENR, C_N };
__device__ __constant__ int kCtrField[C_N] = {F_HIT, F_VHIT, F_STOR, F_INS, F_BYP, F_EVICT,
                                              F_EV0, F_EV1, F_EV2, F_EV3, F_ENR};

// Priority level of a class: NoReuse 0, Far 1, Fresh 2, Near 3; with PVP the
// two lowest are swapped: Far 0, NoReuse 1.
__device__ __forceinline__ uint64_t level_of(int cls, uint32_t pvp) {
  if (cls == kNoReuse) return pvp ? 1 : 0;
  if (cls == kFar) return pvp ? 0 : 1;
  return (uint64_t)cls;  // Fresh 2, Near 3
}
__device__ __forceinline__ int class_of(int d, uint32_t T) {
  return d == 0 ? kNoReuse : ((uint32_t)d <= T ? kNear : kFar);
}
// Class and reuse distance of a line from its snapshot (period > 1): none -> NoReuse;
// inserted after the scan, or a recorded reuse already passed -> Fresh (R7).
__device__ __forceinline__ int class_of_info(uint32_t info, uint32_t t, uint32_t T, int* d) {
  *d = 0;
  if (info == kInfoNone) return kNoReuse;
  if (info == kInfoFresh || info <= t) return kFresh;
  *d = (int)(info - t);
  return (uint32_t)*d <= T ? kNear : kFar;
}
// 64-bit eviction key, smallest evicted first; the node ID in the low 32 bits makes
// every key unique (tie-break by node, R8).
__device__ __forceinline__ uint64_t policy_key(const SetParams& p, uint32_t v, uint32_t lu, int cls, int d) {
  switch (p.policy) {
    case 0:  // HYBRID: (level, static score, node)
      return (level_of(cls, p.pvp) << 40) | ((uint64_t)p.score[v / p.G] << 32) | v;
    case 1:  // STATIC: (score, node)
      return ((uint64_t)p.score[v / p.G] << 32) | v;
    case 2:  // LRU: (last use, node)
      return ((uint64_t)lu << 32) | v;
    case 4:  // DYNAMIC: no reuse first, then recently inserted, then farthest reuse
      return cls == kNoReuse ? (uint64_t)v
             : cls == kFresh ? ((1ull << 48) | v)
                             : ((2ull << 48) | ((uint64_t)(p.W - d) << 32) | v);
    default:  // RR: bypass order only
      return v;
  }
}

__global__ void __launch_bounds__(256, 4) k_set(SetParams p) {
  // early (dedup_wait > 0; kernels.cuh k_dedup): this launch may run while k_serve of the
  // previous gather still delivers. A programmatic wait would also wait for that k_serve (stream
  // work completes in order), so it is replaced by two counters: the CTAs of this gather's
  // k_dedup that finished (their IterState, buckets and node_loc are then visible), and the CTAs
  // of every window feed issued before this gather (the reuse bits it reads). Everything written
  // here is parity-indexed or not read by k_serve.
  if (p.dedup_wait) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
      while (ld_acquire_u64(&p.it->dedup_ctas_done) < p.dedup_wait) __nanosleep(64);
      while (ld_acquire_u64(&p.it->feed_ctas_done) < p.feed_wait) __nanosleep(64);
    }
  } else {
    pdl_prologue();
  }
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long s_ctr[C_N];
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  if (threadIdx.x < C_N) s_ctr[threadIdx.x] = 0;
  __syncthreads();

  unsigned char* wbase = smem + (size_t)wib * p.warp_bytes;
  uint32_t* sv_s = reinterpret_cast<uint32_t*>(wbase);  // sorted nodes of the set
  uint32_t* sk_s = sv_s + p.P;                         // per node: kind | way<<2 | inM<<10 | byp<<11
  uint32_t* sidx_s = sk_s + p.P;                       // M list, then insert list (indices into sv)
  unsigned long long* skey_s = reinterpret_cast<unsigned long long*>(sidx_s + p.P);
  uint32_t* stag = reinterpret_cast<uint32_t*>(skey_s + p.P);
  uint32_t* svict = stag + 32;
  int* sd = reinterpret_cast<int*>(svict + 32);
  int* scls = sd + 32;
  // per-iteration values (device-resident, written by k_begin)
  const uint32_t t_ = (uint32_t)p.it->t, stamp_ = p.it->stamp, p0_ = p.it->p0, stage_base_ = p.it->stage_base;
  unsigned long long* rec_ = p.hist + (size_t)p.it->rec_idx * F_NFIELDS;
  const uint32_t par_ = p.it->par;
  uint32_t* const node_loc_ = p.node_loc + par_ * p.loc_stride;  // this iteration's parity (k_dedup)
  FillEnt* const fills_ = p.fills + (size_t)par_ * p.fstride;
  uint32_t* const nfill_ = &p.scr->nfill[par_];
  uint32_t* const nbypass_ = &p.scr->nbypass[par_];
  TRACE_AT(2, par_, 0);
  const bool upd = p.it->upd != 0;  // exact information for incoming misses

  uint32_t ctr[C_N];
#pragma unroll
  for (int c = 0; c < C_N; ++c) ctr[c] = 0;
  const uint32_t A = p.A, G = p.G;

  if (p.stg_nodes) {  // pvp_unused (§8(b)): staged rows whose node this batch did not request
    const uint32_t par = par_;
    const uint32_t* stg = p.stg_nodes + (size_t)par * p.C;
    const uint32_t ns = p.scr->staged[par];
    uint32_t unused = 0;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < ns; j += gridDim.x * blockDim.x)
      unused += p.mark[stg[j] / G] != stamp_;
    unused = __reduce_add_sync(0xffffffffu, unused);
    if (lane == 0 && unused) atomicAdd(&rec_[F_UNUSED], (unsigned long long)unused);
  }

  // A set whose nodes all hit was fully handled by k_dedup's probe (node_loc, last use, hit
  // count) and has an empty bucket. The sets with a miss (k_dedup's slow list) are processed by
  // one warp each: the bucket holds the set's misses, and its hits are the resident lines whose
  // last use is t (written by the probe).
  const uint32_t gwarp = blockIdx.x * nwb + wib, nwarps = gridDim.x * nwb;
  const uint32_t nslow = p.scr->nslow[par_];
  for (uint32_t i = gwarp; i < nslow; i += nwarps) {
    const uint32_t s = p.slow_list[i];
    uint32_t m = lane == 0 ? p.set_cnt[s] : 0u;
    // one round trip for the set: its first 32 bucket entries (the bucket array is padded by 32
    // entries) and its resident lines (lane w holds way w)
    const uint32_t* bk = p.bucket + (size_t)s * p.BC;
    const uint32_t b0 = bk[lane];
    uint32_t tg = kInvalid, lu = 0;
    if (lane < A) {
      tg = p.tags[s * A + lane];
      lu = p.last_use[s * A + lane];
    }
    m = __shfl_sync(0xffffffffu, m, 0);
    if (lane == 0) p.set_cnt[s] = 0;  // ready for the next batch
    stag[lane] = tg;
    __syncwarp();
    uint32_t Pm = 32;
    while (Pm < m) Pm <<= 1;
    // a bucket larger than the warp's shared-memory capacity works in its own power-of-two
    // region of global scratch (rare: only when one set receives > P distinct nodes)
    uint32_t* sv = sv_s;
    uint32_t* sk = sk_s;
    uint32_t* sidx = sidx_s;
    unsigned long long* skey = skey_s;
    if (m > p.P) {
      const size_t po = (size_t)s * p.BCp;
      sv = p.g_sv + po;
      sk = p.g_sk + po;
      sidx = p.g_sidx + po;
      skey = p.g_skey + po;
    }
    sv[lane] = lane < m ? b0 : kInvalid;
    for (uint32_t j = 32 + lane; j < Pm; j += 32) sv[j] = j < m ? bk[j] : kInvalid;
    __syncwarp();
    warp_bitonic_sort(sv, (int)Pm);  // nodes ascending (R10: misses installed in node order)

    // ---- probe (S4): the hits were found by k_dedup's tag probe, which set their ways' last
    // use to t (protected, R10); the bucket's misses are looked up in the PVP staging directory
    const uint32_t protm = __ballot_sync(0xffffffffu, lane < A && tg != kInvalid && lu == t_);
    const uint32_t mr = (m + 31) & ~31u;
    for (uint32_t j = lane; j < mr; j += 32) {
      if (j < m) {
        const uint32_t v = sv[j], q = v / G;
        uint32_t kind;
        if (p.vst_stamp[q] == stamp_) {
          kind = kVHit;
          ++ctr[C_VHIT];
        } else {
          kind = kStorage;
          ++ctr[C_STOR];
        }
        const uint32_t inM = kind == kStorage || p.reinsert;
        sk[j] = kind | (inM << 10);
      }
    }
    __syncwarp();
    const uint32_t nH = __popc(protm);

    // ---- M = misses to insert, ascending node order
    uint32_t nM = 0;
    for (uint32_t j0 = 0; j0 < mr; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool f = j < m && ((sk[j] >> 10) & 1u);
      const uint32_t b = __ballot_sync(0xffffffffu, f);
      if (f) sidx[nM + __popc(b & ((1u << lane) - 1u))] = j;
      nM += __popc(b);
    }
    __syncwarp();
    const uint32_t avail = A - nH;
    const uint32_t nbyp = nM > avail ? nM - avail : 0;
    if (nbyp) {
      // more misses than unprotected ways: bypass the nbyp smallest incoming keys (R10)
      uint32_t PM = 32;
      while (PM < nM) PM <<= 1;
      for (uint32_t k = lane; k < PM; k += 32) {
        unsigned long long key = ~0ull;
        if (k < nM) {
          const uint32_t v = sv[sidx[k]];
          int dv = 0, cv = kFresh;  // a miss has no information until the next scan ...
          if (upd && (p.policy == 0 || p.policy == 4)) {  // ... except at a scan iteration
            dv = next_reuse_d(p.mask + (size_t)(v / G) * p.MW, p0_, p.W);
            cv = class_of(dv, p.T);
          }
          key = policy_key(p, v, t_, cv, dv);
        }
        skey[k] = key;
      }
      __syncwarp();
      warp_bitonic_sort(skey, (int)PM);
      for (uint32_t k = lane; k < nbyp; k += 32) {
        const uint32_t v = (uint32_t)skey[k];
        uint32_t lo = 0, hi = m;  // lower_bound in sv
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (sv[mid] < v) lo = mid + 1; else hi = mid;
        }
        sk[lo] |= 1u << 11;
      }
      __syncwarp();
      // drop bypassed entries from the insert list (stable, in place)
      uint32_t nI = 0;
      const uint32_t nMr = (nM + 31) & ~31u;
      for (uint32_t k0 = 0; k0 < nMr; k0 += 32) {
        const uint32_t k = k0 + lane;
        uint32_t j = 0;
        bool keep = false;
        if (k < nM) {
          j = sidx[k];
          keep = !((sk[j] >> 11) & 1u);
        }
        const uint32_t b = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) sidx[nI + __popc(b & ((1u << lane) - 1u))] = j;
        nI += __popc(b);
        __syncwarp();
      }
      ctr[C_BYP] += lane == 0 ? nbyp : 0;
    }
    const uint32_t nI = nM - nbyp;

    // ---- way assignment (S5): free ways first (ascending), then victims by policy key
    const bool cand = lane < A && tg != kInvalid && !((protm >> lane) & 1u);
    const uint32_t freem = __ballot_sync(0xffffffffu, lane < A && tg == kInvalid);
    const uint32_t candm = __ballot_sync(0xffffffffu, cand);
    const uint32_t nF = __popc(freem);
    const uint32_t e = nI > nF ? nI - nF : 0;
    if (e) {
      // next reuse distance (0 = none) and class of each resident line: needed only when
      // lines are evicted (victim keys, eviction classes, victim candidates)
      int d = 0, cls = kNoReuse;
      if (tg != kInvalid) {
        if (p.period <= 1) {  // exact, from the window bitmask (P = 1)
          d = next_reuse_d(p.mask + (size_t)(tg / G) * p.MW, p0_, p.W);
          cls = class_of(d, p.T);
        } else {              // the last window scan's snapshot
          cls = class_of_info(p.line_info[s * A + lane], t_, p.T, &d);
        }
      }
      sd[lane] = d;
      scls[lane] = cls;
      uint32_t rank;
      if (p.policy == 3) {  // RR: candidates in cyclic order from the cursor
        const uint32_t c0 = p.rr[s];
        const uint32_t pos = (lane + A - c0) % A;
        uint32_t before = 0;
        for (uint32_t w = 0; w < A; ++w)
          if (((candm >> w) & 1u) && ((w + A - c0) % A) < pos) ++before;
        rank = before;
      } else {
        const unsigned long long key = cand ? policy_key(p, tg, lu, cls, d) : ~0ull;
        rank = 0;
        for (int w = 0; w < 32; ++w) {
          const unsigned long long kw = __shfl_sync(0xffffffffu, key, w);
          if (((candm >> w) & 1u) && kw < key) ++rank;
        }
      }
      if (cand && rank < e) svict[rank] = lane;
      __syncwarp();
      if (p.policy == 3 && lane == 0) p.rr[s] = (svict[e - 1] + 1) % A;
    }
    __syncwarp();

    // ---- install the kept misses; evicted lines become victim candidates
    const uint32_t nIr = (nI + 31) & ~31u;
    for (uint32_t k0 = 0; k0 < nIr; k0 += 32) {
      const uint32_t k = k0 + lane;
      const bool act = k < nI;
      uint32_t v = 0, q = 0, way = 0, kind = 0, x = kInvalid;
      if (act) {
        const uint32_t j = sidx[k];
        v = sv[j];
        q = v / G;
        kind = sk[j] & 3u;
        if (k < nF) {
          uint32_t fm = freem;
          for (uint32_t z = 0; z < k; ++z) fm &= fm - 1u;  // k-th free way
          way = __ffs(fm) - 1;
        } else {
          way = svict[k - nF];
        }
        x = stag[way];
      }
      bool is_cand = false;
      uint32_t reuse = 0;
      if (act && x != kInvalid) {
        const int dx = sd[way], cx = scls[way];
        ++ctr[C_EVICT];
        ++ctr[C_EV0 + cx];
        if (p.pvp && (cx == kNear || cx == kFar)) {
          is_cand = true;
          reuse = t_ + (uint32_t)dx;
        } else {
          ++ctr[C_ENR];
        }
      }
      const uint32_t fidx = warp_reserve(nfill_, act ? 1u : 0u);
      const uint32_t cidx = warp_reserve(&p.scr->ncand, is_cand ? 1u : 0u);
      if (act) {
        const uint32_t slot = s * A + way;
        FillEnt f;
        f.src = kind == kVHit ? stage_base_ + p.vst_idx[q] : (kHostBit | q);
        f.dst = slot;
        f.victim = kInvalid;
        f.node = v;
        fills_[fidx] = f;
        node_loc_[q] = slot | p.deliver;
        p.tags[slot] = v;
        p.last_use[slot] = t_;
        if (p.period > 1) p.line_info[slot] = kInfoFresh;
        ++ctr[C_INS];
        if (is_cand) {
          Cand c;
          c.x = x;
          c.reuse = reuse;
          c.fill = fidx;
          c.pad = 0;
          p.cands[cidx] = c;
          atomicAdd(&p.qcnt[reuse % p.W], 1u);  // per-queue histogram for the admission scan
        }
      }
    }

    // ---- rows not installed: bypassed storage misses go to bypass staging; victim-buffer
    // hits not installed are served from the PVP staging buffer
    for (uint32_t j0 = 0; j0 < mr; j0 += 32) {
      const uint32_t j = j0 + lane;
      bool bs = false;
      uint32_t v = 0;
      if (j < m) {
        const uint32_t info = sk[j];
        const uint32_t kind = info & 3u;
        const bool inM = (info >> 10) & 1u, byp = (info >> 11) & 1u;
        v = sv[j];
        if (kind == kVHit && (!inM || byp)) node_loc_[v / G] = stage_base_ + p.vst_idx[v / G];
        bs = kind == kStorage && byp;
      }
      const uint32_t b = warp_reserve(nbypass_, bs ? 1u : 0u);
      const uint32_t fidx = warp_reserve(nfill_, bs ? 1u : 0u);
      if (bs) {
        FillEnt f;
        f.src = kHostBit | (v / G);
        f.dst = p.bypass_base + b;
        f.victim = kInvalid;
        f.node = v;
        fills_[fidx] = f;
        node_loc_[v / G] = (p.bypass_base + b) | p.deliver;
      }
    }
    __syncwarp();
  }

  // ---- counters: warp -> CTA -> global
#pragma unroll
  for (int c = 0; c < C_N; ++c) {
    const uint32_t x = __reduce_add_sync(0xffffffffu, ctr[c]);
    if (lane == 0 && x) atomicAdd(&s_ctr[c], (unsigned long long)x);
  }
  __syncthreads();
  if (threadIdx.x < C_N && s_ctr[threadIdx.x]) atomicAdd(&rec_[kCtrField[threadIdx.x]], s_ctr[threadIdx.x]);
  TRACE_AT(2, par_, 1);
  if (p.dedup_wait) {  // early: count this CTA done (the early k_serve of this gather waits for it)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&p.it->set_ctas_done, 1ull);
    }
  }
}

// ------------------------------------------------------------------------------ S5: admission
// Candidates grouped by queue k = reuse mod W ("fourth victim buffer"): qcnt (built by
// k_set) is scanned into qoff, then counted back down to zero here.
__global__ void k_qscatter(const Cand* __restrict__ cands, const Scratch* scr, uint32_t W,
                           const uint32_t* __restrict__ qoff, uint32_t* __restrict__ qcnt,
                           uint32_t* __restrict__ qb) {
  pdl_prologue();
  const uint32_t n = scr->ncand;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t k = cands[i].reuse % W;
    qb[qoff[k] + atomicSub(&qcnt[k], 1u) - 1u] = i;
  }
}
// One CTA per queue: admit the candidates with the smallest node IDs into the free slots
// (R14), slot = queue counter before the increment. Admitted rows are copied to
// the pinned host queue by k_fill before their slot is overwritten.
__global__ void __launch_bounds__(256) k_admit(const Cand* __restrict__ cands, const uint32_t* __restrict__ qoff,
                                               const uint32_t* __restrict__ qb, uint32_t* __restrict__ qlen,
                                               uint32_t* __restrict__ qnode, uint32_t* __restrict__ qreuse,
                                               FillEnt* __restrict__ fills, uint64_t fstride, uint32_t C, const IterState* it,
                                               unsigned long long* rec_hist) {
  pdl_prologue();
  __shared__ uint32_t hist[256];
  unsigned long long* rec = rec_hist + (size_t)it->rec_idx * F_NFIELDS;
  __shared__ uint32_t s_prefix, s_want, s_taken;
  const uint32_t k = blockIdx.x;
  const uint32_t lo = qoff[k], nk = qoff[k + 1] - lo;
  if (nk == 0) return;
  const uint32_t len0 = qlen[k];
  const uint32_t room = len0 < C ? C - len0 : 0;
  uint32_t thresh = 0xFFFFFFFFu;  // admit x <= thresh
  bool none = room == 0;
  if (!none && nk > room) {
    // radix select: the room-th smallest node ID (IDs of one batch's victims are distinct)
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_want = room;
    }
    uint32_t pmask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const uint32_t prefix = s_prefix;
      for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) {
        const uint32_t x = cands[qb[lo + i]].x;
        if ((x & pmask) == prefix) atomicAdd(&hist[(x >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t want = s_want, dd = 0;
        for (; dd < 256; ++dd) {
          if (hist[dd] >= want) break;
          want -= hist[dd];
        }
        s_want = want;
        s_prefix = prefix | (dd << shift);
      }
      pmask |= 255u << shift;
      __syncthreads();
    }
    thresh = s_prefix;
  }
  if (threadIdx.x == 0) s_taken = 0;
  __syncthreads();
  uint32_t adm = 0;
  for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) {
    const Cand c = cands[qb[lo + i]];
    if (!none && c.x <= thresh) {
      const uint32_t slot = len0 + atomicAdd(&s_taken, 1u);
      qnode[(size_t)k * C + slot] = c.x;
      qreuse[(size_t)k * C + slot] = c.reuse;
      fills[(size_t)it->par * fstride + c.fill].victim = k * C + slot;
      ++adm;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    qlen[k] = len0 + s_taken;
    atomicAdd(&rec[F_VADM], (unsigned long long)s_taken);
    atomicAdd(&rec[F_VDROP], (unsigned long long)(nk - s_taken));
  }
  (void)adm;
}

// ------------------------------------------------------------------------------ S6 file tier (N2)
// The fills of this batch are decided on the device (k_set); the host reads their storage rows
// from the file. k_io_export publishes the list to pinned host memory — io->src[e] = backing
// row of fill entry e (kInvalid: a PVP staging row, nothing to read), io->n, then io->list =
// stamp (system-scope release) — and the host, which polls io->list, reads the rows into the
// bounce buffer (row e = entry e) chunk by chunk, setting io->ready[c] = stamp after chunk c's
// kIoChunk entries. The fill kernel, launched right behind, waits per entry for its chunk's flag
// (io_wait), so the storage reads and the fills overlap and the stream is never synchronised.
constexpr uint32_t kIoChunk = 64;
struct IoShared {     // pinned, mapped host memory (device pointer)
  uint32_t list;      // stamp of the batch whose list is published
  uint32_t n;         // fill entries of that batch
  uint32_t pad[30];
  // followed by: ready[ceil(ucap / kIoChunk)], then src[ucap]
};
__device__ __forceinline__ uint32_t ld_acquire_sys(const volatile uint32_t* p) {
  uint32_t r;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_sys(volatile uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__global__ void k_io_export(const FillEnt* __restrict__ fills_base, uint64_t fstride, Scratch* scr, const IterState* it,
                            IoShared* io, uint32_t* io_src) {
  pdl_prologue();
  const uint32_t n = scr->nfill[it->par];
  const FillEnt* __restrict__ fills = fills_base + (size_t)it->par * fstride;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const uint32_t src = fills[e].src;
    io_src[e] = (src & kHostBit) ? (src & ~kHostBit) : kInvalid;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&scr->io_done, 1u) == gridDim.x - 1) {  // last CTA: the whole list is out
      scr->io_done = 0;
      __threadfence_system();
      *(volatile uint32_t*)&io->n = n;
      st_release_sys(&io->list, it->stamp);
    }
  }
}
// Lane 0 spins until chunk e / kIoChunk of this batch is in the bounce buffer (acquire: the
// row's bytes are visible after it), then the warp proceeds.
__device__ __forceinline__ void io_wait(const uint32_t* ready, uint32_t e, uint32_t stamp) {
  if (lane_id() == 0) {
    const volatile uint32_t* f = ready + e / kIoChunk;
    uint32_t ns = 64;
    while (ld_acquire_sys(f) != stamp) {
      __nanosleep(ns);
      if (ns < 2048) ns <<= 1;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------ S6
// Warp per fill entry: first the victim row (old slot content) to the pinned host queue
// (eviction D2H), then the new row from the backing table (zero-copy over PCIe,
// P:249 "directly fetched by GPU threads") or from PVP staging into the slot.
template <int UNROLL>
__global__ void k_fill(const FillEnt* __restrict__ fills_base, uint64_t fstride, const Scratch* scr, uint4* __restrict__ pool,
                       const uint4* __restrict__ table, uint4* __restrict__ hostq, uint32_t nvec,
                       uint32_t bounce, const uint32_t* io_ready, const IterState* it) {
  pdl_prologue();
  const uint32_t n = scr->nfill[it->par];
  const FillEnt* __restrict__ fills = fills_base + (size_t)it->par * fstride;
  const uint32_t stamp = it->stamp;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = warp; e < n; e += nwarps) {
    const FillEnt f = fills[e];
    uint4* dst = pool + (size_t)f.dst * nvec;
    if (f.victim != kInvalid) warp_copy_row<UNROLL, kDev, kHost>(hostq + (size_t)f.victim * nvec, dst, nvec);
    if ((f.src & kHostBit) && bounce) io_wait(io_ready, e, stamp);  // file tier: row e read yet?
    if (f.src & kHostBit)
      warp_copy_row<UNROLL, kHost, kDev>(dst, table + (size_t)(bounce ? e : (f.src & ~kHostBit)) * nvec, nvec);
    else
      warp_copy_row<UNROLL, kDev, kDev>(dst, pool + (size_t)f.src * nvec, nvec);
  }
}

// ------------------------------------------------------------------------------ S7 + S8
// Requester: out[i] = row of ids[i] at its home. The location (cache slot, staging row)
// is looked up in the home's node_loc table (peer-mapped when home != me) — the
// "respond" step as a one-sided read — and the row is copied with 16-byte vectors.
// Two phases per batch (G > 1): PHASE 0 copies the rows already in place when the homes
// have finished k_set (hits, PVP-staged rows served in place) and zero-fills bad IDs; it runs
// on a second stream concurrently with the homes' PCIe-bound k_fill. PHASE 1 copies the
// rows k_fill wrote (node_loc bit kDelivered = "filled this batch") once every home has
// signalled "served".
struct PullArgs {
  const uint4* pool[8];
  const uint32_t* node_loc[8];
  Scratch* scr;  // per-phase chunk counters
  uint32_t G;
  uint32_t ST;  // TMA ring stages per warp (TMA = 1)
  uint32_t l2ef;  // rows moved with the L2 evict_first policy (RowRing::hint)
  uint32_t tail_chunk, tail_rounds;
  uint64_t loc_stride;  // G = 1 (LSMGNN_G1_PULL): node_loc table of the iteration's parity
};
// TMA = 1: rows move (local or peer) HBM -> shared -> `out` with TMA bulk copies through each
// warp's ring of ST stages (the source of a peer row is its IPC mapping: over NVLink on
// distinct GPUs); TMA = 0: 16-byte vector loads/stores (pinned host `out`).
template <int UNROLL, int OUT, int PHASE, int TMA>
__global__ void k_pull(const IterState* it, uint64_t N, PullArgs a, uint4* __restrict__ out, uint32_t nvec) {
  pdl_prologue();
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[8][kMaxStages];
  __shared__ uint32_t s_pend[8][kMaxStages];
  __shared__ const void* s_src[8][32];
  __shared__ void* s_dst[8][32];
  const int64_t* __restrict__ ids = it->ids;
  const int64_t n = it->n;
  const uint64_t loc_off = (uint64_t)it->par * a.loc_stride;
  const int lane = (int)lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  RowRing ring{};
  if (TMA) {
    ring.buf = smem + (size_t)wib * a.ST * nvec * 16;
    ring.bar = s_bar[wib];
    ring.pend = s_pend[wib];
    ring.ST = a.ST;
    ring.hint = a.l2ef;
    ring.R = nvec * 16;
    if (lane == 0) ring_init(ring);
    __syncwarp();
  }
  // A warp takes chunks of consecutive requests from a per-phase counter (guided sizes: 32,
  // then a.tail_chunk near the end; see k_serve): its lanes read the IDs and the (local or peer)
  // node_loc words at once — one dependent round trip per chunk instead of two per row, which
  // matters most when node_loc is a peer's (NVLink latency) — then its rows are copied.
  constexpr uint32_t kChunk = 32;
  uint32_t* counter = &a.scr->pull_phase_next[PHASE];
  uint32_t size = kChunk;
  for (;;) {
    uint32_t c0u = 0;
    if (lane == 0) c0u = atomicAdd(counter, size);
    const int64_t c0 = __shfl_sync(0xffffffffu, c0u, 0);
    if (c0 >= n) break;
    const int64_t end = min(c0 + (int64_t)size, n);
    const uint32_t m = (uint32_t)(end - c0);
    uint32_t loc = kInvalid, g = 0;
    bool valid = false;
    if ((uint32_t)lane < m) {
      const int64_t x = ids[c0 + lane];
      if (x >= 0 && (uint64_t)x < N) {
        const uint32_t v = (uint32_t)x;
        g = v % a.G;
        loc = a.node_loc[g][loc_off + v / a.G];
        valid = true;
      }
    }
    if (PHASE == 0) {  // ERANGE: zero-filled rows
      uint32_t zero = __ballot_sync(0xffffffffu, (uint32_t)lane < m && !valid);
      while (zero) {
        const uint32_t j = __ffs(zero) - 1;
        zero &= zero - 1;
        uint4* dst = out + (size_t)(c0 + j) * nvec;
        for (uint32_t k = lane; k < nvec; k += 32) st16<OUT>(dst + k, make_uint4(0, 0, 0, 0));
      }
    }
    const uint32_t need = __ballot_sync(0xffffffffu, valid && (((loc & kDelivered) != 0) == (PHASE == 1)));
    if (TMA) {
      s_src[wib][lane] = a.pool[g] + (size_t)(loc & ~kDelivered) * nvec;
      s_dst[wib][lane] = out + (size_t)(c0 + lane) * nvec;
      __syncwarp();
      if (lane == 0 && need) ring_copy(ring, s_src[wib], s_dst[wib], need);
      __syncwarp();
    } else {
      uint32_t mk = need;
      while (mk) {
        const uint32_t j = __ffs(mk) - 1;
        mk &= mk - 1;
        const uint32_t lj = __shfl_sync(0xffffffffu, loc, (int)j);
        const uint32_t gj = __shfl_sync(0xffffffffu, g, (int)j);
        warp_copy_row<UNROLL, kDev, OUT>(out + (size_t)(c0 + j) * nvec, a.pool[gj] + (size_t)(lj & ~kDelivered) * nvec,
                                         nvec);
      }
    }
    if (c0 + (int64_t)a.tail_rounds * nwarps * kChunk >= n) size = a.tail_chunk;
  }
  if (TMA && lane == 0) ring_drain();
}

// ------------------------------------------------------------------------------ S6+S8 fused (G = 1)
// One launch serves the whole batch. Fill warps stream each missing row from the backing
// table (PCIe) or PVP staging into registers once and store it to its cache slot / bypass
// row AND to every requester position of that node (the request list built by k_dedup) —
// the storage read and the delivery overlap, and the row is never re-read from HBM. The
// remaining warps (1 in 8) start copying the rows not delivered by a fill (hits, staged rows
// served in place) from HBM into `out`, concurrently with the PCIe-bound fills; fill warps
// join them once the fills are handed out. Delivery work is taken in chunks of 32 requests
// from a shared counter, so a hit-dominated batch gets the whole grid and a miss-dominated one
// keeps 7/8 of it on the fills.
// TMA = 1 (device `out`): delivery rows move HBM -> shared -> HBM with TMA bulk copies through
// each warp's ring of `ST` row stages (lane 0 drives it; RowRing), so the bytes in flight are set
// by shared memory, not registers. TMA = 0: 16-byte vector loads/stores (pinned host `out`).
// The last CTA to finish closes the iteration's record (S9, end_record).
struct ServeArgs {
  const FillEnt* fills;  // two parities of fstride entries
  uint64_t fstride;
  uint64_t set_wait;     // early: k_set CTAs (cumulative) that must have finished; 0 = not early
  int64_t t_host;        // direct call: the iteration and its batch (graph replay: -1, from IterState)
  const int64_t* ids_host;
  int64_t n_host;
  Scratch* scr;
  uint4* pool;
  const uint4* table;
  uint4* hostq;
  uint32_t nvec;
  const unsigned long long* head;  // request lists, one table per iteration parity:
  const uint32_t* nxt;             // head Q entries apart, nxt cap entries apart
  uint64_t Q, cap;
  IterState* it;
  uint64_t N;
  const uint32_t* node_loc;
  uint64_t loc_stride;  // node_loc tables Q apart (parity)
  const uint32_t* req_loc;  // k_dedup's per-request locations, tables cap apart (parity)
  uint4* out;
  uint32_t bounce;
  uint32_t tail_chunk;  // delivery chunk size near the end of the batch (guided; 32 = fixed)
  uint32_t tail_rounds; // ... once fewer than tail_rounds rounds of 32-request chunks remain
  uint32_t ahead;       // keep one 32-request chunk in reserve before the tail phase
  uint32_t static_first;  // hit-dominated batch: warp w's first delivery chunk is chunk w
  const uint32_t* io_ready;  // file tier: per-chunk "rows read" flags (pinned host, stamped)
  uint32_t ST;  // TMA ring stages per warp
  uint32_t l2ef;  // rows moved with the L2 evict_first policy (RowRing::hint)
  // S9, closed by the last CTA
  unsigned long long* hist;
  unsigned long long* cum;
  volatile uint32_t* bad_mirror;
};

// S9: close iteration t's record — algorithmic bytes per tier, cumulative sums; the staging
// count of the next parity is reset so that a missing PVP call stages nothing; the ERANGE
// counter is mirrored to pinned host memory; it->t_next = t + 1. One warp (lane = field).
// What the next gathers need comes first — the counters and the record of t + 2 start at zero,
// then t_next is published (an early k_serve of t + 1 waits for it) — and the bookkeeping of
// t's own record and the cumulative sums after it (read only once the stream is synchronised).
__device__ __forceinline__ void end_record(uint64_t t, IterState* it, unsigned long long* hist, unsigned long long* cum,
                                           Scratch* scr, uint32_t R, volatile uint32_t* bad_mirror) {
  const uint32_t f = lane_id();
  // prepare gather t + 2 (k_dedup / k_set of t + 1 may already be counting into the record of
  // t + 1 and the parity counters of t + 1; those were zeroed here by gather t - 1): the record
  // of t + 2 and the parity counters of t (= those of t + 2) start at zero; the counters only
  // k_serve / k_pull of t + 1 use (they start after gather t completed) are reset for t + 1
  unsigned long long* nrec = hist + (size_t)((t + 2) % kHist) * F_NFIELDS;
  if (f < F_NFIELDS) nrec[f] = 0;
  if (f == 0) {
    scr->nfill[t & 1] = 0;
    scr->ncand = 0;
    scr->nbypass[t & 1] = 0;
    scr->pull_next = 0;
    scr->pull_phase_next[0] = 0;
    scr->pull_phase_next[1] = 0;
    scr->nslow[t & 1] = 0;
  }
  __syncwarp();
  if (f == 0) {  // gather t is complete (an early k_serve of t + 1 waits for this)
    __threadfence();
    *(volatile uint64_t*)&it->t_next = t + 1;  // direct calls and graph replays may be mixed
  }
  unsigned long long* rec = hist + (size_t)(t % kHist) * F_NFIELDS;
  if (f == 0) {
    rec[F_PREF] = scr->staged[t & 1];  // rows the PVP staged for t (its copy completed before gather t)
    rec[F_BOUT] = rec[F_REQ] * R;
    rec[F_BNVL] = rec[F_PEER] * R;
    rec[F_BH2D] = rec[F_STOR] * R;
    rec[F_BPVP] = rec[F_PREF] * R;
    rec[F_BD2H] = rec[F_VADM] * R;
  }
  __syncwarp();
  __threadfence_block();
  unsigned long long v = 0;
  if (f < F_NFIELDS) v = rec[f];
  __syncwarp();
  if (f > 0 && f < F_NFIELDS) cum[f] += v;
  if (f == 0) {
    cum[F_ITER] = t;
    scr->staged[(t + 1) & 1] = 0;
    *bad_mirror = scr->bad_ids;
  }
}

template <int UNROLL, int OUT, int TMA>
__global__ void k_serve(ServeArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[8][kMaxStages];
  __shared__ uint32_t s_pend[8][kMaxStages];
  __shared__ const void* s_src[8][32];
  __shared__ void* s_dst[8][32];
  __shared__ uint32_t s_last;
  __shared__ uint64_t s_t;
  __shared__ const int64_t* s_ids;
  __shared__ int64_t s_n;
  // Early (set_wait > 0, kernels.cuh k_dedup): no programmatic wait (it would also wait for the
  // in-flight chain behind the previous k_serve); this gather's k_set is awaited through its
  // finished-CTA count, and the previous gather — it must be complete before this one fills
  // slots — through the t_next its last CTA publishes (end_record).
  // A direct call takes the iteration's values from its arguments (an early k_dedup of the next
  // gather may republish IterState while this launch runs); a graph replay reads IterState (the
  // next gather of a replay is never early).
  if (a.set_wait) {  // early
    if (threadIdx.x == 0) {
      while (ld_acquire_u64(&a.it->set_ctas_done) < a.set_wait) __nanosleep(64);
      while (ld_acquire_u64(&a.it->t_next) < (uint64_t)a.t_host) __nanosleep(64);
    }
    __syncthreads();
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.t_host >= 0) {
    if (threadIdx.x == 0) {
      s_t = (uint64_t)a.t_host;
      s_ids = a.ids_host;
      s_n = a.n_host;
    }
  } else if (threadIdx.x == 0) {
    s_t = a.it->t;
    s_ids = a.it->ids;
    s_n = a.it->n;
  }
  __syncthreads();
  constexpr uint32_t kChunk = 32;
  const uint64_t t_it = s_t;
  const uint32_t stamp = (uint32_t)(t_it + 1);
  const int64_t* __restrict__ ids = s_ids;
  const int64_t n = s_n;
  const uint32_t par = (uint32_t)(t_it & 1);
  TRACE_AT(3, par, 0);
  const unsigned long long* __restrict__ head = a.head + (size_t)par * a.Q;
  const uint32_t* __restrict__ nxt = a.nxt + (size_t)par * a.cap;
  const uint32_t* __restrict__ node_loc = a.node_loc + par * a.loc_stride;
  const uint32_t* __restrict__ req_loc = a.req_loc + (size_t)par * a.cap;
  const uint32_t nvec = a.nvec;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t npull = nw >= 8 ? nw / 8 : 1;
  const int lane = (int)lane_id();
  RowRing ring{};
  if (TMA) {
    ring.buf = smem + (size_t)wib * a.ST * nvec * 16;
    ring.bar = s_bar[wib];
    ring.pend = s_pend[wib];
    ring.ST = a.ST;
    ring.hint = a.l2ef;
    ring.R = nvec * 16;
    if (lane == 0) ring_init(ring);
    __syncwarp();
  }
  if (gw >= npull) {  // ---- fill warps
    const uint32_t nf = a.scr->nfill[par];
    const FillEnt* __restrict__ fills = a.fills + (size_t)par * a.fstride;
    for (uint32_t e = gw - npull; e < nf; e += nw - npull) {
      const FillEnt f = fills[e];
      uint4* slot = a.pool + (size_t)f.dst * nvec;
      if (f.victim != kInvalid) warp_copy_row<UNROLL, kDev, kHost>(a.hostq + (size_t)f.victim * nvec, slot, nvec);
      const bool from_host = (f.src & kHostBit) != 0;
      if (from_host && a.bounce) io_wait(a.io_ready, e, stamp);  // file tier: row e read yet?
      // host row: the backing table's row q, or (file tier) bounce-buffer row e
      const uint4* src = from_host ? a.table + (size_t)(a.bounce ? e : (f.src & ~kHostBit)) * nvec
                                   : a.pool + (size_t)f.src * nvec;
      const unsigned long long h = head[f.node];
      const uint32_t first = (uint32_t)(h >> 32) == stamp ? (uint32_t)h : kInvalid;
      for (uint32_t base = 0; base < nvec; base += 32 * UNROLL) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const uint32_t k = base + lane + 32 * u;
          if (k < nvec) v[u] = from_host ? ld16<kHost>(src + k) : ld16<kDev>(src + k);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const uint32_t k = base + lane + 32 * u;
          if (k < nvec) st16<kDev>(slot + k, v[u]);
        }
        for (uint32_t pos = first; pos != kInvalid; pos = nxt[pos]) {
          uint4* dst = a.out + (size_t)pos * nvec;  // list positions are request indices
#pragma unroll
          for (int u = 0; u < UNROLL; ++u) {
            const uint32_t k = base + lane + 32 * u;
            if (k < nvec) st16<OUT>(dst + k, v[u]);
          }
        }
      }
    }
  }
  // ---- delivery of the rows no fill delivers, in chunks of 32 requests. The chunk's IDs and
  // locations are looked up by its lanes at once (one dependent round trip per chunk instead of
  // two per row), then its rows are copied.
  auto copy_chunk = [&](int64_t c0, uint32_t loc) {
    uint32_t zero = __ballot_sync(0xffffffffu, loc == kInvalid);
    while (zero) {  // ERANGE: zero-filled rows (rare)
      const uint32_t j = __ffs(zero) - 1;
      zero &= zero - 1;
      uint4* dst = a.out + (size_t)(c0 + j) * nvec;
      for (uint32_t k = lane; k < nvec; k += 32) st16<OUT>(dst + k, make_uint4(0, 0, 0, 0));
    }
    const uint32_t need = __ballot_sync(0xffffffffu, loc != kInvalid && !(loc & kDelivered));
    if (TMA) {
      s_src[wib][lane] = a.pool + (size_t)(loc & ~kDelivered) * nvec;
      s_dst[wib][lane] = a.out + (size_t)(c0 + lane) * nvec;
      __syncwarp();
      if (lane == 0 && need) ring_copy(ring, s_src[wib], s_dst[wib], need);
      __syncwarp();
    } else {
      uint32_t mk = need;
      while (mk) {
        const uint32_t j = __ffs(mk) - 1;
        mk &= mk - 1;
        const uint32_t lj = __shfl_sync(0xffffffffu, loc, (int)j);
        warp_copy_row<UNROLL, kDev, OUT>(a.out + (size_t)(c0 + j) * nvec, a.pool + (size_t)lj * nvec, nvec);
      }
    }
  };
  auto loc_of = [&](int64_t x) -> uint32_t {  // -2: past the batch (nothing to copy)
    return x == -2 ? kDelivered : (x < 0 || (uint64_t)x >= a.N) ? kInvalid : node_loc[(uint32_t)x];
  };
  // Chunks are handed out by a counter (load balance: the hit rows finish together, and a
  // storage-bound batch keeps the delivery-only warps busy while the fills run), with guided
  // sizes: 32 requests, then `tail` once fewer than tail_rounds rounds of 32-request chunks remain,
  // so the warps finish within a small chunk of each other. a.ahead (off by default) makes a warp
  // hold the next chunk in reserve in the 32-request phase, its locations and the counter atomic
  // for the one after in flight during the current copy; like a static chunk order and
  // reserving through the tail, it measured slower (hit path 0.237 vs 0.227 ms/step; the
  // reservations unbalance the warps more than the hidden latency gains,
  // profiles/r02_hit_path.md).
  const uint32_t tail = a.tail_chunk;
  const int64_t tail_from = n - (int64_t)a.tail_rounds * nw * kChunk;
  auto grab = [&](uint32_t sz) -> uint32_t { return lane == 0 ? atomicAdd(&a.scr->pull_next, sz) : 0u; };
  auto ids_of = [&](int64_t c, uint32_t sz) -> int64_t {
    return c + lane < min(c + (int64_t)sz, n) ? ids[c + lane] : -2;
  };
  if (a.ahead) {
    int64_t c0 = __shfl_sync(0xffffffffu, grab(kChunk), 0);
    if (c0 < n) {
      uint32_t loc0 = loc_of(ids_of(c0, kChunk));
      int64_t c1 = c0 < tail_from ? (int64_t)__shfl_sync(0xffffffffu, grab(kChunk), 0) : n;
      int64_t x1 = c1 < n ? ids_of(c1, kChunk) : -2;
      for (;;) {
        if (c1 < n && c1 < tail_from) {  // keep one chunk in reserve
          const uint32_t loc1 = loc_of(x1);
          const uint32_t raw = grab(kChunk);
          copy_chunk(c0, loc0);
          const int64_t c2 = __shfl_sync(0xffffffffu, raw, 0);
          x1 = c2 < n ? ids_of(c2, kChunk) : -2;
          c0 = c1;
          loc0 = loc1;
          c1 = c2;
          continue;
        }
        copy_chunk(c0, loc0);
        if (c1 < n) copy_chunk(c1, loc_of(x1));
        break;
      }
    }
  }
  // (a.ahead = 0, or the tail after the reserved chunks): chunks grabbed one at a time. A
  // chunk's locations come from k_dedup's per-request table in one coalesced load; only the
  // requests it left pending (repeated occurrences, misses) take the ID -> node_loc round trips.
  // When every fill warp has at most one fill (a hit-dominated batch), warp w's first chunk is
  // chunk w (no counter round trip) and the counter hands out the rest from nw chunks on.
  uint32_t size = a.ahead ? tail : kChunk;
  const bool first_static = !a.ahead && a.static_first && a.scr->nfill[par] <= nw - npull &&
                            (int64_t)nw * kChunk <= tail_from;
  const int64_t cbase = first_static ? (int64_t)nw * kChunk : 0;
  bool first = first_static;
  for (;;) {
    const uint32_t sz = size;
    const int64_t c0 = first ? (int64_t)gw * kChunk : cbase + __shfl_sync(0xffffffffu, grab(sz), 0);
    first = false;
    if (c0 >= n) break;
    const bool in = c0 + lane < min(c0 + (int64_t)sz, n);
    uint32_t loc = in ? req_loc[c0 + lane] : kDelivered;
    if (__ballot_sync(0xffffffffu, loc == kPending) && loc == kPending) loc = loc_of(ids[c0 + lane]);
    copy_chunk(c0, loc);
    if (c0 >= tail_from) size = tail;
  }
  if (TMA && lane == 0) ring_drain();
  // ---- S9: the last CTA to finish closes the record
  TRACE_AT(3, par, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&a.scr->serve_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && wib == 0) {
    __threadfence();
    if (lane == 0) a.scr->serve_done = 0;
    end_record(t_it, a.it, a.hist, a.cum, a.scr, nvec * 16, a.bad_mirror);
  }
}

// ------------------------------------------------------------------------------ S10 (G > 1)
// Window feed. Bit (k mod (W+1)) of mask[q] is set when node q*G+me is in B_k. The ring slot
// and bit of the batch being fed is it->wslot; its previous bits were cleared by k_dedup of
// gather(k - W - 1) (the feed is ordered after that kernel).
// Copy the inboxes of all sources (window IDs routed to this home) into the ring slot and
// set each node's reuse bit of the slot.
// The ring slot holds up to `stride` IDs (the expected per-home share with slack, not the worst
// case of every rank's whole batch at one home): a longer list is not stored — the slot is marked
// kRingOverflow and k_dedup then clears the slot's bit for every node of the home (a sweep of one
// mask word per node) instead of walking the list. The bits themselves are always set.
constexpr uint32_t kRingOverflow = 0xFFFFFFFFu;
__global__ void k_win_gather(const uint32_t* __restrict__ inbox, const uint32_t* __restrict__ inbox_cnt,
                             uint32_t nsrc, uint32_t cap, uint32_t* __restrict__ ring, uint64_t stride,
                             uint32_t* ring_len, const IterState* it, uint32_t G, uint32_t MW,
                             uint32_t* __restrict__ mask) {
  pdl_prologue();
  const uint32_t slot_i = it->wslot;
  uint32_t* __restrict__ slot = ring + (size_t)slot_i * stride;
  const uint32_t m = 1u << (slot_i & 31);
  uint64_t total = 0;
  for (uint32_t r = 0; r < nsrc; ++r) total += inbox_cnt[r];
  const bool store = total <= stride;
  uint32_t base = 0;
  for (uint32_t r = 0; r < nsrc; ++r) {
    const uint32_t n = inbox_cnt[r];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const uint32_t v = inbox[(size_t)r * cap + i];
      if (store) slot[base + i] = v;
      atomicOr(&mask[(size_t)(v / G) * MW + (slot_i >> 5)], m);
    }
    base += n;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ring_len[slot_i] = store ? base : kRingOverflow;
}

// ------------------------------------------------------------------------------ S11
// PVP: copy victim queue k = (t+1) mod W (pinned host) into this iteration's
// staging buffer and publish the staging directory (vst_stamp/vst_idx) for gather(t+1).
// Entries whose recorded reuse is not t+1 are dropped (R17). The last CTA empties the queue.
template <int UNROLL>
__global__ void k_pvp(const IterState* it, uint32_t W, uint32_t L, uint32_t C, uint32_t G,
                      uint32_t* __restrict__ qlen, const uint32_t* __restrict__ qnode,
                      const uint32_t* __restrict__ qreuse, const uint4* __restrict__ hostq,
                      uint4* __restrict__ pool, uint32_t* __restrict__ stg_base,
                      uint32_t* __restrict__ vst_stamp, uint32_t* __restrict__ vst_idx, Scratch* scr,
                      uint32_t nvec) {
  pdl_prologue();
  // runs after gather(t): stage victim queue (t+1) mod W for iteration t+1
  const uint64_t t1 = it->t + 1;
  const uint32_t k = (uint32_t)(t1 % W), stamp1 = (uint32_t)(t1 + 1), par = (uint32_t)(t1 & 1);
  const uint32_t stage_base = L + par * C;
  uint32_t* __restrict__ stg_nodes = stg_base + (size_t)par * C;
  const uint32_t n = qlen[k];
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t j = warp; j < n; j += nwarps) {
    const size_t e = (size_t)k * C + j;
    if (qreuse[e] != (uint32_t)t1) continue;
    uint32_t m = 0;
    if (lane_id() == 0) m = atomicAdd(&scr->staged[par], 1u);
    m = __shfl_sync(0xffffffffu, m, 0);
    const uint32_t x = qnode[e];
    warp_copy_row<UNROLL, kHost, kDev>(pool + (size_t)(stage_base + m) * nvec, hostq + e * nvec, nvec);
    if (lane_id() == 0) {
      stg_nodes[m] = x;
      vst_idx[x / G] = m;
      vst_stamp[x / G] = stamp1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&scr->pvp_done, 1u) == gridDim.x - 1) {
      qlen[k] = 0;
      scr->pvp_done = 0;
    }
  }
}

}  // namespace lsm

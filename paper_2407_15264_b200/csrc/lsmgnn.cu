// lsmgnn.cu — host runtime + C-ABI of the B200-native LSM-GNN gather hot path.
//
// Declared in include/lsmgnn.h (argument meaning, layout, ownership, errors).
// DESIGN.md §"Data layout" and §"Kernels" describe what lives where; kernels.cuh holds
// the sm_100a kernels. One process per GPU; peers are reached through CUDA IPC
// mappings (NVLink P2P on a real 8-GPU box) and stream-ordered 32-bit flags written
// and awaited with cuStreamWriteValue32 / cuStreamWaitValue32 (no SM spins, no host
// synchronisation in steady state).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdlib>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lsmgnn.h"
#include "kernels.cuh"
#include "sampler.cuh"

using namespace lsm;

namespace {

constexpr int kMaxG = 8;

struct Handle {  // exported per rank for lsmgnn_connect
  cudaIpcMemHandle_t ipc;
  uint64_t arena_bytes;
  uint64_t layout_sig;
  int32_t rank, world;
  unsigned char gpu_uuid[16];  // ranks sharing one GPU (tests) are detected by UUID
};

// Persistent worker threads of the file tier (N2): started when a storage file is attached,
// parked on a condition variable between batches. run(n, fn, done) hands entries 0..n-1 out in
// chunks of kIoChunk through an atomic cursor to the workers and the calling thread and calls
// done(chunk) once a chunk's entries are processed (the device waits on those per-chunk flags);
// it returns the first nonzero fn result (an errno), after which the remaining entries are
// skipped — but every chunk is still marked done, so no device wait is left hanging.
class IoPool {
 public:
  void start(int nthreads) {
    for (int i = 0; i < nthreads; ++i) th_.emplace_back([this] { worker(); });
  }
  void stop() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
    th_.clear();
  }
  int run(uint32_t n, const std::function<int(uint32_t)>& fn, const std::function<void(uint32_t)>& done) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      n_ = n;
      fn_ = &fn;
      done_ = &done;
      next_.store(0);
      err_.store(0);
      active_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return active_ == 0; });
    fn_ = nullptr;
    return err_.load();
  }

 private:
  void drain() {
    for (;;) {
      const uint32_t e0 = next_.fetch_add(kIoChunk);
      if (e0 >= n_) return;
      const uint32_t e1 = std::min(n_, e0 + kIoChunk);
      for (uint32_t e = e0; e < e1 && !err_.load(); ++e)
        if (int rc = (*fn_)(e)) {
          int zero = 0;
          err_.compare_exchange_strong(zero, rc);
        }
      (*done_)(e0 / kIoChunk);
    }
  }
  void worker() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
      }
      drain();
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  bool quit_ = false;
  int active_ = 0;
  uint32_t n_ = 0;
  const std::function<int(uint32_t)>* fn_ = nullptr;
  const std::function<void(uint32_t)>* done_ = nullptr;
  std::atomic<uint32_t> next_{0};
  std::atomic<int> err_{0};
};

struct Ctx {
  // binding
  int rank = 0, world = 1, device = -1;
  lsmgnn_options opt{};
  bool opt_set = false;
  bool inited = false, connected = false;
  std::string err;
  int sticky = 0;

  // config
  uint64_t N = 0;
  uint32_t R = 0, nvec = 0, A = 0, W = 0, T = 0, MW = 0, Wp1 = 0;
  uint64_t L = 0, S = 0, Q = 0, C = 0, cap = 0, ucap = 0, bcap = 0;
  uint64_t loc_stride = 0;  // node_loc tables per iteration parity (G = 1), Q apart
  uint64_t BC = 0, BCp = 0;  // per-set bucket capacity (distinct nodes of a set per batch); its pow2
  // window ring slot capacity: G = 1 cap; G > 1 min(G, 2)·cap — twice a home's expected share of
  // the G ranks' batches (a fuller slot is swept instead of listed, k_win_gather / k_dedup)
  uint64_t ring_stride = 0;
  uint64_t pool_rows = 0, stage_base0 = 0, bypass_base = 0;
  uint32_t P = 32, warp_bytes = 0, set_warps = 8;
  int sms = 148;
  int geom_per_sm = 1 << 20;  // LSMGNN_GEOMETRY=small caps every grid at one CTA per SM (I9 tests)

  // shared arena (exported to peers): [flags | inbox_cnt | win_cnt | inbox | win_inbox | node_loc | pool]
  char* arena = nullptr;
  size_t arena_bytes = 0;
  size_t off_flags = 0, off_icnt = 0, off_wcnt = 0, off_inbox = 0, off_win = 0, off_loc = 0, off_pool = 0;
  char* peer_arena[kMaxG] = {};

  // local device state
  uint32_t *tags = nullptr, *last_use = nullptr, *rr = nullptr, *mask = nullptr, *mark = nullptr;
  uint32_t *vst_stamp = nullptr, *vst_idx = nullptr, *set_cnt = nullptr;
  uint32_t* slow_stamp = nullptr;  // [S]: == stamp when a node of the set missed k_dedup's probe
  uint32_t* slow_list = nullptr;   // [S]: those sets, in k_dedup's order
  uint32_t *bucket = nullptr, *ring = nullptr, *ring_len = nullptr;  // bucket: [S * BC + 32]
  // global scratch for cache sets whose bucket exceeds k_set's shared-memory capacity
  uint32_t *g_sv = nullptr, *g_sk = nullptr, *g_sidx = nullptr;  // [S * BCp] when a set can exceed P
  unsigned long long* g_skey = nullptr;
  uint32_t* scan_q = nullptr;  // k_scan look-back words of the victim-queue scan (2 x tiles)
  uint32_t *qcnt = nullptr, *qoff = nullptr, *qb = nullptr, *qlen = nullptr, *qnode = nullptr;
  uint32_t *qreuse = nullptr, *stg_nodes = nullptr, *route_cnt = nullptr;
  unsigned long long* head = nullptr;            // G = 1 fused delivery: per-node request list heads
  uint32_t* line_info = nullptr;                 // update period > 1: per-line dynamic information
  uint32_t* nxt = nullptr;   // next request position of the same node
  uint32_t* req_loc = nullptr;  // per request position: a first-occurrence hit's slot, else kPending
  uint8_t* score = nullptr;
  FillEnt* fills = nullptr;
  Cand* cands = nullptr;
  Scratch* scr = nullptr;
  IterState* it = nullptr;  // per-iteration values on the device (kernels read, k_begin writes)
  unsigned long long *hist = nullptr, *cum = nullptr;

  // captured CUDA graph of one step (G = 1)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cap_stream2 = nullptr;  // the window-feed branch of the captured step
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t graph_launches = 0;  // kernels per replay
  bool graph_out_host = false;

  // host tiers
  uint8_t* qrows_host = nullptr;  // pinned victim queues [W*C][R]
  uint8_t* qrows_dev = nullptr;   // its device mapping
  const uint8_t* table_host = nullptr;
  const uint8_t* table_dev = nullptr;
  bool table_registered = false;
  // file tier (N2): rows read with pread into a pinned bounce buffer, row e = fill entry e
  int file_fd = -1;
  bool file_direct = false;
  uint8_t* bounce_host = nullptr;
  IoShared* io_host = nullptr;     // pinned, mapped: the published fill list and per-chunk ready flags
  IoShared* io_dev = nullptr;      // its device mapping
  uint32_t* io_ready_host = nullptr;
  uint32_t* io_ready_dev = nullptr;
  uint32_t* io_src_host = nullptr;
  uint32_t* io_src_dev = nullptr;
  IoPool* io = nullptr;  // persistent pread workers (io_threads - 1; the caller is one more)
  int io_threads = 64;  // pread workers per batch (LSMGNN_IO_THREADS); deeper queues help NVMe
  volatile uint32_t* bad_host = nullptr;  // pinned mirror: [0] scr->bad_ids, [1] batch-length overflow
  uint32_t* bad_dev_overflow = nullptr;   // device mapping of bad_host + 1
  uint32_t* bad_dev = nullptr;

  // streams / events
  cudaStream_t side = nullptr;
  // G > 1: the first pull phase (rows in place after k_set) runs on pull_st while k_fill runs
  cudaStream_t pull_st = nullptr;
  cudaEvent_t ev_set = nullptr, ev_pull0 = nullptr;
  // Pull phase 0 on its own stream, concurrent with k_fill (the default on distinct GPUs). Ranks
  // that share one GPU without MPS time-slice it, and the extra cross-process dependency then
  // costs more than the overlap gains (profiles/r01_n2_pull_ab.md), so a rank that finds a
  // peer on its own GPU runs both phases after "served". LSMGNN_SPLIT_PULL=0/1 overrides.
  bool split_pull = true;
  bool pdl = false;  // programmatic dependent launch on the G = 1 chain (launch_pdl)
  // the library's last launch on tail_st ended a G = 1 gather (k_serve / k_end): a window feed
  // right behind it may start early (k_route_local, wait_prev = 0)
  bool tail_gather = false;
  // ... or an early window feed (k_route_local, wait_prev = 0) right behind such a gather: the
  // next gather's k_dedup may then start alongside that k_serve (k_dedup `early`)
  bool tail_feed = false;
  cudaStream_t tail_st = nullptr;
  bool feed_early = true;  // LSMGNN_FEED_EARLY=0 turns the early feed start off (A/B)
  bool dedup_early = true;  // LSMGNN_DEDUP_EARLY=0 turns the early k_dedup / k_set start off (A/B)
  // k_dedup's scattered metadata accesses (tags, stamps, node_loc, last use) with the L2
  // evict_last policy, so they stay in L2 while the previous gather's row stream passes through
  // (A/B ab_l2b: hit path 0.2053 -> 0.1984 ms/step, k_serve 0.935 -> 0.943): on when that metadata
  // (~20 B per home row) fits in half the L2; LSMGNN_META_EVICT_LAST=0/1 overrides
  bool meta_evict_last = false;
  // ... and the reuse-bitmask updates of the window feed and its clear (A/B ab_mk: hit path
  // 0.1996 -> 0.1928 ms/step): on when the metadata plus the mask (4·MW B per row) fit half the L2;
  // LSMGNN_MASK_EVICT_LAST=0/1 overrides
  bool mask_evict_last = false;
  bool serve_static_first = true;  // LSMGNN_SERVE_STATIC_FIRST=0: every chunk from the counter (A/B)
  bool host_tma = false;  // LSMGNN_HOST_TMA=1: TMA ring delivery into a pinned host `out` (A/B)
  int early_set_per_sm = 2;  // (A/B ab_setsm: 1 0.1910, 2 0.1911, 4 0.1927 ms/step direct)
  int early_dedup_per_sm = 2;  // (A/B ab_perSM: 1 0.2044, 2 0.2043, 4 0.2065 ms/step direct)
  uint64_t dedup_ctas_issued = 0;  // CTAs of early k_dedup launches (it->dedup_ctas_done)
  uint64_t set_ctas_issued = 0;    // CTAs of early k_set launches (it->set_ctas_done)
  uint64_t feed_ctas_issued = 0;  // CTAs of early k_route_local launches (it->feed_ctas_done counts them done)
  // LSMGNN_G1_PULL=1 (G = 1, profiling aid): the G > 1 serve path — k_fill, then k_pull phase 0
  // (rows in place) and phase 1 (rows filled this batch), then k_end — instead of the fused
  // k_serve; the pull kernels can then be profiled on one process (local HBM instead of peers)
  bool g1_pull = false;
  // k_serve geometry: CTAs per SM and TMA row stages per warp (0 = 16-B vector copies);
  // LSMGNN_SERVE_CPS / LSMGNN_SERVE_ST override (A/B runs)
  int serve_cps = 2, serve_st = 3;
  int l2_evict_first = 0;  // LSMGNN_L2_EVICT_FIRST=1: ring row copies with the L2 evict_first policy (A/B ab_l2: slower); 2: stores only
  int serve_tail = 4;  // LSMGNN_SERVE_TAIL=n: k_serve's delivery chunk size near the batch end (A/B)
  int serve_tail_rounds = 2;  // LSMGNN_SERVE_TAIL_ROUNDS=r: ... once fewer than r rounds of chunks remain
  bool serve_ahead = false;   // LSMGNN_SERVE_AHEAD=1: one chunk in reserve before the tail phase (measured slower)
  cudaEvent_t ev_main = nullptr, ev_pvp = nullptr;
  bool pvp_pending = false;
  // cross-stream order (callers may gather and prefetch on different streams): the end of
  // gather t is ev_gend[t & 7] (gend_t says which t it holds); the last window feed is ev_feed
  cudaEvent_t ev_gend[8] = {};
  int64_t gend_t[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  cudaStream_t gend_st[8] = {};
  bool gend_rec[8] = {};  // lazily recorded: only when another stream has to wait for it
  cudaEvent_t ev_dedup[8] = {};  // G > 1: after k_dedup of gather dedup_t[i] (window feeds wait on it)
  int64_t dedup_t[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  cudaEvent_t ev_feed = nullptr;
  cudaStream_t feed_st = nullptr;
  bool feed_recorded = false, feed_since_gather = false;
  bool feed_ev_rec = false;  // lazily recorded like gend_rec
  cudaStream_t last_stream = nullptr;
  // stream of the last gather: a gather issued on another stream first waits for the end of
  // the previous one (k_begin resets the per-iteration state and scratch it still uses; at
  // G > 1 the homes would otherwise rewrite node_loc / pool slots a pull of t still reads)
  cudaStream_t gather_st = nullptr;
  int64_t* tmp_ids = nullptr;  // for lsmgnn_gather_host
  void* tmp_out = nullptr;

  // iteration state
  int64_t t_next = 0;      // next gather iteration
  int64_t feed_next = 1;   // next window iteration to feed
  uint32_t win_seq = 0;    // window batches exchanged (G > 1)
  int64_t launches = 0;

  // GPU sampler (NEXT N3): CSR in pinned host memory + scratch
  const int64_t* s_indptr = nullptr;   // device mapping of the host CSR
  const int32_t* s_indices = nullptr;
  const void* s_host_indptr = nullptr;
  const void* s_host_indices = nullptr;
  bool s_reg_indptr = false, s_reg_indices = false;
  uint64_t s_N = 0, s_cap = 0;
  unsigned long long* s_tab = nullptr;  // first-occurrence table, u64 per node
  uint32_t *s_raw = nullptr, *s_layer = nullptr, *s_front = nullptr, *s_cnt = nullptr, *s_off = nullptr;
  uint32_t *s_keep = nullptr, *s_pos = nullptr, *s_bsum = nullptr;
  SampCounts* s_counts = nullptr;
  uint32_t s_hi = 0xFFFFFFFFu;
  const int64_t* s_map_indptr = nullptr;  // device mappings of the host CSR (UVA)
  const int32_t* s_map_indices = nullptr;
  int64_t* s_hbm_indptr = nullptr;        // HBM-resident copy (lsmgnn_sampler_place)
  int32_t* s_hbm_indices = nullptr;
  int64_t s_nnz = 0;

  // phase profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Span { int phase; cudaEvent_t a, b; };
  std::vector<Span> spans;
  cudaEvent_t open_ev[LSMGNN_NPHASES] = {};

  // driver entry points (stream memory operations)
  PFN_cuStreamWaitValue32_v2 waitv = nullptr;
  PFN_cuStreamWriteValue32_v2 writev = nullptr;
  PFN_cuStreamBatchMemOp_v2 batchv = nullptr;  // optional: G flag operations per submission
};

Ctx g;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g.err = buf;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(e_ == cudaErrorMemoryAllocation ? LSMGNN_ENOMEM : LSMGNN_ECUDA,     \
                     "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                     __LINE__);                                                         \
  } while (0)

#define LAUNCHED()                                                                  \
  do {                                                                              \
    ++g.launches;                                                                   \
    cudaError_t e_ = cudaPeekAtLastError();                                         \
    if (e_ != cudaSuccess)                                                          \
      return set_err(LSMGNN_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                           \
  } while (0)

template <typename T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  CK(cudaMemset(*p, 0, count * sizeof(T)));
  return 0;
}

// k_scan grid (one CTA per tile of counts) and its look-back words
int scan_tiles(uint64_t n) { return (int)std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile); }
ScanSync scan_sync(uint32_t* words, uint64_t n) {
  const size_t k = (size_t)scan_tiles(n);
  return ScanSync{words, words + k};
}

// arena views (local or peer)
uint32_t* flags_of(char* base) { return reinterpret_cast<uint32_t*>(base + g.off_flags); }
// flag slots: [0,G) route from r; [G,2G) served by home g; [2G,3G) window from r; [3G,4G) window ack from g;
// [4G,5G) located by home g (k_set done: node_loc final, rows of hits and staged nodes in place)
uint32_t* icnt_of(char* base) { return reinterpret_cast<uint32_t*>(base + g.off_icnt); }
uint32_t* wcnt_of(char* base) { return reinterpret_cast<uint32_t*>(base + g.off_wcnt); }
uint32_t* inbox_of(char* base) { return reinterpret_cast<uint32_t*>(base + g.off_inbox); }
uint32_t* win_of(char* base) { return reinterpret_cast<uint32_t*>(base + g.off_win); }
uint32_t* loc_of(char* base) { return reinterpret_cast<uint32_t*>(base + g.off_loc); }
uint8_t* pool_of(char* base) { return reinterpret_cast<uint8_t*>(base + g.off_pool); }

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int grid_for(int64_t work, int threads, int per_sm = 8) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)std::min<int64_t>(b, (int64_t)g.sms * std::min(per_sm, g.geom_per_sm));
}

int check_sticky() {
  if (g.bad_host && g.bad_host[1]) {
    g.sticky = LSMGNN_EINVAL;
    return set_err(g.sticky, "a device-resident batch length exceeded max_batch_ids (sticky; clamped)");
  }
  if (g.bad_host && *g.bad_host) g.sticky = LSMGNN_ERANGE;
  if (g.sticky == LSMGNN_EIO) return set_err(g.sticky, "an earlier storage read failed (sticky)");
  if (g.sticky) return set_err(g.sticky, "a node id >= num_nodes was passed (sticky)");
  return 0;
}

// ---- stream-ordered flags (G > 1)
int flag_write(cudaStream_t st, uint32_t* addr, uint32_t value) {
  CUresult r = g.writev(st, (CUdeviceptr)addr, value, 0);
  if (r != CUDA_SUCCESS) return set_err(LSMGNN_ECOMM, "cuStreamWriteValue32 failed (%d)", (int)r);
  return 0;
}
int flag_wait(cudaStream_t st, uint32_t* addr, uint32_t value) {
  CUresult r = g.waitv(st, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return set_err(LSMGNN_ECOMM, "cuStreamWaitValue32 failed (%d)", (int)r);
  return 0;
}
// The G flag operations of one protocol step in ONE stream memory-op batch (one front-end
// submission instead of G; executed in array order, each write fenced like a single
// cuStreamWriteValue32): wait until base[h] >= value for every home h (local words), or write
// `value` into word `word` of every rank's flag block (peer-mapped).
int flags_wait_all(cudaStream_t st, uint32_t* base, uint32_t value) {
  const int G = g.world;
  if (!g.batchv) {
    for (int h = 0; h < G; ++h)
      if (int rc = flag_wait(st, base + h, value)) return rc;
    return 0;
  }
  CUstreamBatchMemOpParams ops[kMaxG];
  std::memset(ops, 0, sizeof(ops));
  for (int h = 0; h < G; ++h) {
    ops[h].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    ops[h].waitValue.address = (CUdeviceptr)(base + h);
    ops[h].waitValue.value = value;
    ops[h].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  }
  CUresult r = g.batchv(st, (unsigned)G, ops, 0);
  if (r != CUDA_SUCCESS) return set_err(LSMGNN_ECOMM, "cuStreamBatchMemOp(wait) failed (%d)", (int)r);
  return 0;
}
int flags_write_all(cudaStream_t st, uint32_t word, uint32_t value) {
  const int G = g.world;
  if (!g.batchv) {
    for (int r = 0; r < G; ++r)
      if (int rc = flag_write(st, &flags_of(g.peer_arena[r])[word], value)) return rc;
    return 0;
  }
  CUstreamBatchMemOpParams ops[kMaxG];
  std::memset(ops, 0, sizeof(ops));
  for (int r = 0; r < G; ++r) {
    ops[r].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    ops[r].writeValue.address = (CUdeviceptr)&flags_of(g.peer_arena[r])[word];
    ops[r].writeValue.value = value;
    ops[r].writeValue.flags = 0;  // default: fenced after the stream's prior work
  }
  CUresult r = g.batchv(st, (unsigned)G, ops, 0);
  if (r != CUDA_SUCCESS) return set_err(LSMGNN_ECOMM, "cuStreamBatchMemOp(write) failed (%d)", (int)r);
  return 0;
}

// Route `n` int64 IDs of this requester to the homes' inboxes (gather: win=false) and run the
// flag exchange so that, on return (stream order), every home's inbox for this round is full.
int exchange_ids(int64_t n_bound, bool win, uint32_t seq, cudaStream_t st) {
  const int G = g.world;
  uint32_t* myflags = flags_of(g.arena);
  if (win) {  // the homes must have consumed the previous window round
    if (int rc = flags_wait_all(st, &myflags[3 * G], seq - 1)) return rc;
  }
  // gather and window exchanges keep separate counters: they may run on different streams
  uint32_t* rcnt = g.route_cnt + (win ? G : 0);
  CK(cudaMemsetAsync(rcnt, 0, sizeof(uint32_t) * G, st));
  RouteArgs ra{};
  PublishArgs pa{};
  for (int h = 0; h < G; ++h) {
    char* base = g.peer_arena[h];
    ra.inbox[h] = (win ? win_of(base) : inbox_of(base)) + (size_t)g.rank * g.cap;
    pa.peer_cnt[h] = win ? wcnt_of(base) : icnt_of(base);
  }
  ra.route_cnt = rcnt;
  ra.G = (uint32_t)G;
  pa.G = (uint32_t)G;
  pa.me = (uint32_t)g.rank;
  if (n_bound > 0) {
    k_route_peer<<<grid_for(n_bound, 256, 4), 256, 0, st>>>(g.it, win ? 1u : 0u, g.N, ra, g.scr);
    LAUNCHED();
  }
  k_route_publish<<<1, 32, 0, st>>>(rcnt, pa);
  LAUNCHED();
  const int slot = win ? 2 : 0;
  if (int rc = flags_write_all(st, (uint32_t)(slot * G + g.rank), seq)) return rc;
  if (int rc = flags_wait_all(st, &myflags[slot * G], seq)) return rc;
  return 0;
}

cudaEvent_t take_event() {
  if (g.ev_pool.empty()) {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = g.ev_pool.back();
  g.ev_pool.pop_back();
  return e;
}
// Phase span on stream st: prof_begin records the start event, prof_end the end event.
// NVTX ranges name the same phases for nsys / ncu timelines (no cost without a tool attached).
const char* const kPhaseName[LSMGNN_NPHASES] = {"lsmgnn.route", "lsmgnn.dedup", "lsmgnn.probe_replace",
                                                "lsmgnn.admit", "lsmgnn.fill", "lsmgnn.pull",
                                                "lsmgnn.window", "lsmgnn.pvp"};
void prof_begin(int ph, cudaStream_t st) {
  nvtxRangePushA(kPhaseName[ph]);
  if (!g.prof) return;
  g.open_ev[ph] = take_event();
  cudaEventRecord(g.open_ev[ph], st);
}
void prof_end(int ph, cudaStream_t st) {
  nvtxRangePop();
  if (!g.prof || !g.open_ev[ph]) return;
  cudaEvent_t b = take_event();
  cudaEventRecord(b, st);
  g.spans.push_back({ph, g.open_ev[ph], b});
  g.open_ev[ph] = nullptr;
}

void detach_file();  // file tier (below)
int free_all() {
  cudaDeviceSynchronize();
  void* ptrs[] = {g.tags, g.last_use, g.rr, g.mask, g.mark, g.vst_stamp, g.vst_idx, g.set_cnt, g.slow_stamp, g.slow_list, g.scan_q,
                  g.bucket, g.ring, g.ring_len, g.qcnt, g.qoff, g.qb, g.qlen, g.qnode, g.qreuse,
                  g.stg_nodes, g.route_cnt, g.head, g.nxt, g.req_loc, g.line_info, g.score, g.fills, g.cands,
                  g.scr, g.it, g.hist, g.g_sv, g.g_sk, g.g_sidx, g.g_skey,
                  g.cum, g.arena, g.tmp_ids, g.tmp_out};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* sp[] = {g.s_tab,  g.s_raw,    g.s_layer,  g.s_front,        g.s_cnt,          g.s_off,
                g.s_keep, g.s_pos,    g.s_bsum,   g.s_counts, g.s_hbm_indptr, g.s_hbm_indices};
  for (void* p : sp)
    if (p) cudaFree(p);
  if (g.s_reg_indptr) cudaHostUnregister(const_cast<void*>(g.s_host_indptr));
  if (g.s_reg_indices) cudaHostUnregister(const_cast<void*>(g.s_host_indices));
  for (int h = 0; h < kMaxG; ++h)
    if (g.peer_arena[h] && g.peer_arena[h] != g.arena) cudaIpcCloseMemHandle(g.peer_arena[h]);
  if (g.qrows_host) cudaFreeHost(g.qrows_host);
  if (g.bad_host) cudaFreeHost((void*)g.bad_host);
  if (g.table_registered) cudaHostUnregister((void*)g.table_host);
  detach_file();
  if (g.graph_exec) cudaGraphExecDestroy(g.graph_exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  if (g.cap_stream) cudaStreamDestroy(g.cap_stream);
  if (g.cap_stream2) cudaStreamDestroy(g.cap_stream2);
  if (g.ev_fork) cudaEventDestroy(g.ev_fork);
  if (g.ev_join) cudaEventDestroy(g.ev_join);
  if (g.side) cudaStreamDestroy(g.side);
  if (g.pull_st) cudaStreamDestroy(g.pull_st);
  if (g.ev_set) cudaEventDestroy(g.ev_set);
  if (g.ev_pull0) cudaEventDestroy(g.ev_pull0);
  if (g.ev_main) cudaEventDestroy(g.ev_main);
  for (auto e : g.ev_gend)
    if (e) cudaEventDestroy(e);
  for (auto e : g.ev_dedup)
    if (e) cudaEventDestroy(e);
  if (g.ev_feed) cudaEventDestroy(g.ev_feed);
  if (g.ev_pvp) cudaEventDestroy(g.ev_pvp);
  for (auto& sp : g.spans) {
    cudaEventDestroy(sp.a);
    cudaEventDestroy(sp.b);
  }
  for (auto e : g.ev_pool) cudaEventDestroy(e);
  const int rank = g.rank, world = g.world, dev = g.device;
  const lsmgnn_options opt = g.opt;
  const bool opt_set = g.opt_set;
  g = Ctx();
  g.rank = rank;
  g.world = world;
  g.device = dev;
  g.opt = opt;
  g.opt_set = opt_set;
  return 0;
}

lsmgnn_options default_options() {
  lsmgnn_options o{};
  o.version = LSMGNN_ABI_VERSION;
  o.policy = LSMGNN_HYBRID;
  o.pvp = 0;
  o.window = 256;
  o.threshold = 0;
  o.update_period = 1;
  o.reinsert_victims = 1;
  o.max_batch_ids = 1 << 20;
  return o;
}

// ---- one step's launches. Per-iteration values reach the kernels through g.it (written by
// k_begin / k_win_begin), so the same sequence serves direct calls and CUDA-graph capture.
BeginArgs begin_args(int64_t t_host, const int64_t* ids, int64_t n, const int64_t* const* ids_ring,
                     const int64_t* n_ring, uint32_t ring_len) {
  BeginArgs a{};
  a.t_host = t_host;
  a.ids_host = ids;
  a.n_host = n;
  a.ids_ring = ids_ring;
  a.n_ring = n_ring;
  a.ring_len = ring_len ? ring_len : 1;
  a.Wp1 = g.Wp1;
  a.period = (uint32_t)std::max(1, g.opt.update_period);
  a.L = (uint32_t)g.stage_base0;
  a.C = (uint32_t)g.C;
  a.cap = (int64_t)g.cap;
  a.overflow = g.bad_dev_overflow;
  return a;
}

int io_export(cudaStream_t st);                     // file tier (below)
int read_storage_rows(uint32_t stamp, cudaStream_t st);

// Kernel launch with programmatic dependent launch (PDL) on the single-home step chain: the
// next kernel is scheduled while its predecessor drains and waits in pdl_prologue() for its
// results (kernels.cuh), hiding launch latency between the ~10 short kernels of a step.
// Off at G > 1 (stream memory operations sit between the kernels) and with LSMGNN_NO_PDL=1.
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g.pdl ? 1 : 0;
  g.tail_gather = false;  // (launch_gather sets it again after its last kernel)
  g.tail_feed = false;    // (launch_window sets it again after an early feed)
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return set_err(LSMGNN_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
  return 0;
}
#define KLAUNCH(kern, grid, block, smem, st, ...)                                         \
  do {                                                                                  \
    if (int rc_l = launch_pdl(kern, dim3(grid), dim3(block), (size_t)(smem), st, __VA_ARGS__)) return rc_l; \
  } while (0)

// gather kernels; n_bound = host bound of this rank's request count (grid sizing only);
// stamp_host = t + 1 for the G > 1 flag protocol (direct calls only).
int launch_gather(const BeginArgs& ba, int64_t n_bound, void* out, bool out_host, bool graph, uint32_t stamp_host,
                  cudaStream_t st, cudaEvent_t ev_dedup = nullptr) {
  const int G = g.world;
  if (G > 1) {  // (at G = 1 k_dedup publishes the iteration's values itself)
    KLAUNCH(k_begin, 1, 32, 0, st, g.it, g.hist, g.scr, ba);
    LAUNCHED();
  }
  // ---- S1/S2 route + exchange
  prof_begin(0, st);
  const uint32_t* inbox = inbox_of(g.arena);
  const uint32_t* inbox_cnt;
  if (G == 1) {
    inbox_cnt = nullptr;  // k_dedup reads the caller's IDs directly
  } else {
    if (int rc = exchange_ids(n_bound, false, stamp_host, st)) return rc;
    inbox_cnt = icnt_of(g.arena);
  }
  prof_end(0, st);
  // ---- S3 dedup + set grouping
  prof_begin(1, st);
  const int64_t maxreq = (int64_t)g.cap * G;
  bool early = false;
  {
    DedupArgs da{};
    da.inbox = inbox;
    da.inbox_cnt = inbox_cnt;
    da.nsrc = (uint32_t)G;
    da.cap = (uint32_t)g.cap;
    da.me = (uint32_t)g.rank;
    da.G = (uint32_t)G;
    da.S = (uint32_t)g.S;
    da.BC = (uint32_t)g.BC;
    da.mark = g.mark;
    da.bucket = g.bucket;
    da.set_cnt = g.set_cnt;
    da.head = G == 1 ? g.head : nullptr;
    da.nxt = g.nxt;
    da.direct = G == 1 ? 1u : 0u;
    da.N = g.N;
    da.ring = g.ring;
    da.ring_stride = g.ring_stride;
    da.Q = g.Q;
    da.ring_len = g.ring_len;
    da.mask = g.mask;
    da.MW = g.MW;
    da.Wp1 = g.Wp1;
    da.tags = g.tags;
    da.last_use = g.last_use;
    da.node_loc = loc_of(g.arena);
    da.loc_stride = g.loc_stride;
    da.req_loc = G == 1 ? g.req_loc : nullptr;
    da.meta_evict_last = g.meta_evict_last ? 1u : 0u;
    da.mask_hint = g.mask_evict_last ? 1u : 0u;
    da.slow_stamp = g.slow_stamp;
    da.slow_list = g.slow_list;
    da.A = g.A;
    // early start alongside the k_serve of the previous gather (kernels.cuh k_dedup): a direct
    // G = 1 call whose programmatic predecessor on st is that k_serve or the early feed behind it
    // (not with the periodic window scan: k_snapshot sits between k_dedup and k_set, and an early
    // k_set does not wait for it)
    early = g.dedup_early && g.pdl && G == 1 && !g.g1_pull && !graph && ba.t_host >= 0 && g.C == 0 &&
            g.file_fd < 0 && g.opt.update_period <= 1 && g.tail_st == st && (g.tail_gather || g.tail_feed);
    // (an early k_dedup shares the SMs with the previous k_serve: LSMGNN_EARLY_DEDUP_PER_SM caps its
    // CTAs per SM, A/B)
    const int dgrid = grid_for(std::min<int64_t>(maxreq, std::max<int64_t>(n_bound, 1) * G), 256,
                               early ? g.early_dedup_per_sm : 4);
    KLAUNCH(k_dedup, dgrid, 256, 0, st, da, g.it, g.scr, g.hist, ba, G == 1 ? 1u : 0u, early ? 1u : 0u);
    LAUNCHED();
    if (early) g.dedup_ctas_issued += (uint64_t)dgrid;  // (an early k_dedup counts them done)
  }
  if (ev_dedup) CK(cudaEventRecord(ev_dedup, st));  // the window feed of t+1+W may follow from here
  prof_end(1, st);
  // ---- S4/S5 probe + replacement
  prof_begin(2, st);
  SetParams sp{};
  sp.set_cnt = g.set_cnt;
  sp.slow_stamp = g.slow_stamp;
  sp.slow_list = g.slow_list;
  sp.bucket = g.bucket;
  sp.BC = (uint32_t)g.BC;
  sp.BCp = (uint32_t)g.BCp;
  sp.stg_nodes = g.C ? g.stg_nodes : nullptr;
  sp.mark = g.mark;
  sp.C = (uint32_t)g.C;
  sp.tags = g.tags;
  sp.last_use = g.last_use;
  sp.rr = g.rr;
  sp.score = g.score;
  sp.mask = g.mask;
  sp.node_loc = loc_of(g.arena);
  sp.loc_stride = g.loc_stride;
  sp.vst_stamp = g.vst_stamp;
  sp.vst_idx = g.vst_idx;
  sp.fills = g.fills;
  sp.fstride = g.ucap;
  sp.cands = g.cands;
  sp.qcnt = g.qcnt;
  sp.scr = g.scr;
  sp.it = g.it;
  sp.hist = g.hist;
  sp.S = (uint32_t)g.S;
  sp.A = g.A;
  sp.G = (uint32_t)G;
  sp.W = g.W;
  sp.T = g.T;
  sp.MW = g.MW;
  sp.policy = (uint32_t)g.opt.policy;
  sp.pvp = (uint32_t)g.opt.pvp;
  sp.reinsert = (uint32_t)g.opt.reinsert_victims;
  sp.P = g.P;
  sp.g_sv = g.g_sv;
  sp.g_sk = g.g_sk;
  sp.g_sidx = g.g_sidx;
  sp.g_skey = g.g_skey;
  sp.warp_bytes = g.warp_bytes;
  sp.bypass_base = (uint32_t)g.bypass_base;
  sp.deliver = kDelivered;
  sp.period = (uint32_t)std::max(1, g.opt.update_period);
  sp.line_info = g.line_info;
  sp.dedup_wait = early ? g.dedup_ctas_issued : 0;
  sp.feed_wait = early ? g.feed_ctas_issued : 0;
  if (sp.period > 1) {  // the periodic window scan; k_snapshot exits when t mod P != 0
    KLAUNCH(k_snapshot, grid_for((int64_t)g.L, 256, 4), 256, 0, st, g.tags, (uint32_t)g.L, (uint32_t)G, g.mask, g.MW, g.W,
                                                                g.it, g.line_info);
    LAUNCHED();
  }
  {
    // (an early k_set shares the SMs with the previous k_serve: LSMGNN_EARLY_SET_PER_SM caps its CTAs
    // per SM, A/B)
    const int64_t blocks = std::min<int64_t>((g.S + g.set_warps - 1) / g.set_warps,
                                             (int64_t)g.sms * std::min(early ? g.early_set_per_sm : 4, g.geom_per_sm));
    KLAUNCH(k_set, (int)blocks, 32 * g.set_warps, g.warp_bytes * g.set_warps, st, sp);
    LAUNCHED();
    if (early) g.set_ctas_issued += (uint64_t)blocks;  // (an early k_set counts them done)
  }
  prof_end(2, st);
  // ---- S5 victim admission (PVP)
  if (g.C) {
    prof_begin(3, st);
    const int qg = grid_for(g.ucap, 256, 2);
    KLAUNCH(k_scan, scan_tiles(g.W), 1024, 0, st, g.qcnt, g.qoff, g.W, (const IterState*)g.it,
            scan_sync(g.scan_q, g.W));
    LAUNCHED();
    KLAUNCH(k_qscatter, qg, 256, 0, st, g.cands, g.scr, g.W, g.qoff, g.qcnt, g.qb);
    LAUNCHED();
    KLAUNCH(k_admit, g.W, 256, 0, st, g.cands, g.qoff, g.qb, g.qlen, g.qnode, g.qreuse, g.fills, (uint64_t)g.ucap, (uint32_t)g.C, g.it,
                                 g.hist);
    LAUNCHED();
    prof_end(3, st);
  }
  // ---- S6 fill (victim D2H + storage/staging -> slot) and S7/S8 serve
  uint4* pool = reinterpret_cast<uint4*>(pool_of(g.arena));
  const uint4* tab = reinterpret_cast<const uint4*>(g.table_dev);
  int rc_io = 0;
  uint4* hq = reinterpret_cast<uint4*>(g.qrows_dev);
  uint4* o4 = reinterpret_cast<uint4*>(out);
  const bool wide = g.nvec >= 256;
  const uint32_t bounce = g.file_fd >= 0 ? 1u : 0u;  // file tier: storage rows staged per fill entry
  if (G == 1 && !g.g1_pull) {
    // one fused launch: fills deliver their rows to `out`, 1 warp in 8 copies the hits; its last
    // CTA closes the record (S9)
    prof_begin(4, st);
    if (bounce && (rc_io = io_export(st))) return rc_io;
    ServeArgs sa{};
    sa.fills = g.fills;
    sa.fstride = g.ucap;
    sa.set_wait = early ? g.set_ctas_issued : 0;
    sa.t_host = ba.t_host;
    sa.ids_host = ba.ids_host;
    sa.n_host = ba.n_host;
    sa.scr = g.scr;
    sa.pool = pool;
    sa.table = tab;
    sa.hostq = hq;
    sa.nvec = g.nvec;
    sa.head = g.head;
    sa.nxt = g.nxt;
    sa.Q = g.Q;
    sa.cap = g.cap;
    sa.loc_stride = g.loc_stride;
    sa.req_loc = g.req_loc;
    sa.it = g.it;
    sa.N = g.N;
    sa.node_loc = loc_of(g.arena);
    sa.out = o4;
    sa.bounce = bounce;
    sa.io_ready = g.io_ready_dev;
    sa.tail_chunk = (uint32_t)g.serve_tail;
    sa.tail_rounds = (uint32_t)g.serve_tail_rounds;
    sa.ahead = g.serve_ahead ? 1u : 0u;
    sa.static_first = g.serve_static_first ? 1u : 0u;
    sa.hist = g.hist;
    sa.cum = g.cum;
    sa.bad_mirror = g.bad_dev;
    // pinned host `out`: LSMGNN_HOST_TMA=1 delivers through the TMA rings too (bulk stores to the
    // host mapping; A/B)
    const bool tma = (!out_host || g.host_tma) && g.serve_st > 0;
    sa.ST = tma ? (uint32_t)g.serve_st : 0u;
    sa.l2ef = (uint32_t)g.l2_evict_first;
    const size_t smem = tma ? (size_t)8 * g.serve_st * g.R : 0;
    const int blocks = g.sms * std::min(tma ? g.serve_cps : 4, g.geom_per_sm);
#define SERVE(U, O, T) KLAUNCH((k_serve<U, O, T>), blocks, 256, smem, st, sa)
    if (wide && tma && out_host) SERVE(8, kHost, 1);
    else if (wide && tma) SERVE(8, kDev, 1);
    else if (wide && !out_host) SERVE(8, kDev, 0);
    else if (wide) SERVE(8, kHost, 0);
    else if (tma) SERVE(2, kDev, 1);
    else if (!out_host) SERVE(2, kDev, 0);
    else SERVE(2, kHost, 0);
#undef SERVE
    LAUNCHED();
    if (bounce && (rc_io = read_storage_rows(stamp_host, st))) return rc_io;
    prof_end(4, st);
    prof_begin(5, st);
  } else {
    // Pull phase 0 (S7/S8 for the rows already in place): once every home has run k_set
    // ("located"), copy hit and staged rows from local / peer HBM on pull_st while this
    // home's k_fill streams the misses over PCIe.
    if (G > 1)
      if (int rc = flags_write_all(st, (uint32_t)(4 * G + g.rank), stamp_host)) return rc;
    PullArgs pa{};
    for (int h = 0; h < G; ++h) {
      pa.pool[h] = reinterpret_cast<const uint4*>(pool_of(g.peer_arena[h]));
      pa.node_loc[h] = loc_of(g.peer_arena[h]);
    }
    pa.G = (uint32_t)G;
    pa.loc_stride = g.loc_stride;
    pa.scr = g.scr;
    pa.tail_chunk = (uint32_t)g.serve_tail;
    pa.tail_rounds = (uint32_t)g.serve_tail_rounds;
    const bool tma = !out_host && g.serve_st > 0;
    pa.ST = tma ? (uint32_t)g.serve_st : 0u;
    pa.l2ef = (uint32_t)g.l2_evict_first;
    const size_t psmem = tma ? (size_t)8 * g.serve_st * g.R : 0;
    // a warp per 32 requests; with TMA rings, at most serve_cps CTAs per SM fit
    const int pblocks = grid_for(n_bound, 256, tma ? g.serve_cps : 8);
#define PULL(PH, S)                                                                                          \
  do {                                                                                                       \
    if (wide && tma) k_pull<8, kDev, PH, 1><<<pblocks, 256, psmem, S>>>(g.it, g.N, pa, o4, g.nvec);           \
    else if (wide && !out_host) k_pull<8, kDev, PH, 0><<<pblocks, 256, 0, S>>>(g.it, g.N, pa, o4, g.nvec);  \
    else if (wide) k_pull<8, kHost, PH, 0><<<pblocks, 256, 0, S>>>(g.it, g.N, pa, o4, g.nvec);               \
    else if (tma) k_pull<2, kDev, PH, 1><<<pblocks, 256, psmem, S>>>(g.it, g.N, pa, o4, g.nvec);              \
    else if (!out_host) k_pull<2, kDev, PH, 0><<<pblocks, 256, 0, S>>>(g.it, g.N, pa, o4, g.nvec);          \
    else k_pull<2, kHost, PH, 0><<<pblocks, 256, 0, S>>>(g.it, g.N, pa, o4, g.nvec);                         \
  } while (0)
    if (n_bound > 0 && g.split_pull) {
      CK(cudaEventRecord(g.ev_set, st));
      CK(cudaStreamWaitEvent(g.pull_st, g.ev_set, 0));
      if (int rc = flags_wait_all(g.pull_st, &flags_of(g.arena)[4 * G], stamp_host)) return rc;
      PULL(0, g.pull_st);
      LAUNCHED();
      CK(cudaEventRecord(g.ev_pull0, g.pull_st));
    }
    prof_begin(4, st);
    if (bounce && (rc_io = io_export(st))) return rc_io;
    // 2 CTAs per SM: the PCIe-bound fill saturates the link from 1 CTA/SM
    // (profiles/r01_pcie_microbench.txt) and leaves room on every SM for pull phase 0
    const int blocks = g.sms * std::min(2, g.geom_per_sm);
    if (wide)
      k_fill<8><<<blocks, 256, 0, st>>>(g.fills, g.ucap, g.scr, pool, tab, hq, g.nvec, bounce, g.io_ready_dev, g.it);
    else
      k_fill<2><<<blocks, 256, 0, st>>>(g.fills, g.ucap, g.scr, pool, tab, hq, g.nvec, bounce, g.io_ready_dev, g.it);
    LAUNCHED();
    if (bounce && (rc_io = read_storage_rows(stamp_host, st))) return rc_io;
    prof_end(4, st);
    // homes signal "served", requesters wait for every home, then pull the filled rows
    // (phase 1); the gather ends after both phases
    prof_begin(5, st);
    if (G > 1) {
      if (int rc = flags_write_all(st, (uint32_t)(G + g.rank), stamp_host)) return rc;
      if (int rc = flags_wait_all(st, &flags_of(g.arena)[G], stamp_host)) return rc;
    }
    if (n_bound > 0) {
      if (g.split_pull) {
        CK(cudaStreamWaitEvent(st, g.ev_pull0, 0));
      } else {
        PULL(0, st);
        LAUNCHED();
      }
      PULL(1, st);
      LAUNCHED();
    }
#undef PULL
  }
  prof_end(5, st);
  if (G > 1 || g.g1_pull) {
    EndArgs ea{g.it, g.hist, g.cum, g.scr, g.R, g.bad_dev};
    KLAUNCH(k_end, 1, 32, 0, st, ea);
    LAUNCHED();
  }
  g.tail_gather = G == 1 && !graph;
  g.tail_st = st;
  return 0;
}

int wait_dedup(int64_t t, cudaStream_t st);  // (below)

// Window feed of one batch (G = 1 local path, or the G > 1 exchange). k_host >= 0: host
// values; k_host < 0: graph replay (batch from the ring). The ring slot / mask bit it rewrites,
// k mod (W+1), was cleared by k_dedup of gather(k - W - 1): feed_begin orders the launch after
// that gather at G = 1; at G > 1 the exchange runs first and k_win_gather waits for the event
// recorded after that gather's k_dedup.
int launch_window(int64_t k_host, const int64_t* ids, int64_t n, const int64_t* n_dev, const int64_t* const* ids_ring,
                  const int64_t* n_ring, uint32_t ring_len, int64_t n_bound, cudaStream_t st) {
  const int G = g.world;
  const uint64_t stride = g.ring_stride;
  if (G == 1) {
    if (k_host < 0 || n_dev) {  // graph replay, or a device-resident length: IterState carries the batch
      KLAUNCH(k_win_begin, 1, 32, 0, st, g.it, k_host, ids, n, n_dev, ids_ring, n_ring, ring_len ? ring_len : 1, g.Wp1,
              (int64_t)g.cap, g.bad_dev_overflow);
      LAUNCHED();
      KLAUNCH(k_route_local, grid_for(n_bound, 256), 256, 0, st, g.it, (int64_t)-1, (const int64_t*)nullptr, (int64_t)0,
              g.Wp1, g.N, g.ring, stride, g.ring_len, g.scr, g.mask, g.MW, 1u, g.mask_evict_last ? 1u : 0u);
      LAUNCHED();
    } else {  // direct: one launch, the batch as kernel arguments
      const uint32_t wait_prev = (g.feed_early && g.tail_gather && g.tail_st == st) ? 0u : 1u;
      KLAUNCH(k_route_local, grid_for(std::max<int64_t>(n, 1), 256), 256, 0, st, g.it, k_host, ids, n, g.Wp1, g.N,
              g.ring, stride, g.ring_len, g.scr, g.mask, g.MW, wait_prev, g.mask_evict_last ? 1u : 0u);
      LAUNCHED();
      if (!wait_prev) g.feed_ctas_issued += (uint64_t)grid_for(std::max<int64_t>(n, 1), 256);  // (counted done)
      if (!wait_prev) g.tail_feed = true;  // (tail_st unchanged: the same stream)
    }
    return 0;
  }
  KLAUNCH(k_win_begin, 1, 32, 0, st, g.it, k_host, ids, n, n_dev, ids_ring, n_ring, ring_len ? ring_len : 1, g.Wp1,
          (int64_t)g.cap, g.bad_dev_overflow);
  LAUNCHED();
  const uint32_t seq = ++g.win_seq;
  if (int rc = exchange_ids(n_bound, true, seq, st)) return rc;
  if (int rc = wait_dedup(k_host - (int64_t)g.W - 1, st)) return rc;
  k_win_gather<<<grid_for((int64_t)g.cap, 256, 2), 256, 0, st>>>(win_of(g.arena), wcnt_of(g.arena), (uint32_t)G,
                                                                  (uint32_t)g.cap, g.ring, stride, g.ring_len, g.it,
                                                                  (uint32_t)G, g.MW, g.mask);
  LAUNCHED();
  // window inbox consumed
  if (int rc = flags_write_all(st, (uint32_t)(3 * G + g.rank), seq)) return rc;
  return 0;
}

// ---- cross-stream order of gathers, window feeds and the PVP copy
// The end-of-gather and end-of-feed events are recorded LAZILY: note_* only remembers the
// stream; the event is recorded on it when another stream first has to wait (then it also
// covers the work issued on that stream since — conservative, never early). A single-stream
// caller therefore gets no event record between the kernels of consecutive calls, which would
// cut the programmatic-dependent-launch chain (k_serve(t) -> feed -> k_dedup(t+1)).
int note_gather_end(int64_t t, cudaStream_t st) {
  const int i = (int)(t & 7);
  if (!g.ev_gend[i]) CK(cudaEventCreateWithFlags(&g.ev_gend[i], cudaEventDisableTiming));
  g.gend_t[i] = t;
  g.gend_st[i] = st;
  g.gend_rec[i] = false;
  return 0;
}
int gend_event(int i) {  // record slot i's event now if it was not recorded yet
  if (!g.gend_rec[i]) {
    CK(cudaEventRecord(g.ev_gend[i], g.gend_st[i]));
    g.gend_rec[i] = true;
  }
  return 0;
}
// `st` waits for the end of gather t (t < 0: nothing to wait for). A gather issued on `st` itself
// is already ordered. If that slot was reused, wait for every remembered gather (conservative).
int wait_gather_end(int64_t t, cudaStream_t st) {
  if (t < 0) return 0;
  const int i = (int)(t & 7);
  if (g.gend_t[i] == t) {
    if (g.gend_st[i] != st) {
      if (int rc = gend_event(i)) return rc;
      CK(cudaStreamWaitEvent(st, g.ev_gend[i], 0));
    }
    return 0;
  }
  for (int j = 0; j < 8; ++j)
    if (g.gend_t[j] >= 0 && g.gend_st[j] != st) {
      if (int rc = gend_event(j)) return rc;
      CK(cudaStreamWaitEvent(st, g.ev_gend[j], 0));
    }
  return 0;
}
// `st` waits for the last window feed (issued on feed_st)
int wait_feed(cudaStream_t st) {
  if (!g.feed_recorded || g.feed_st == st) return 0;
  if (!g.feed_ev_rec) {
    CK(cudaEventRecord(g.ev_feed, g.feed_st));
    g.feed_ev_rec = true;
  }
  CK(cudaStreamWaitEvent(st, g.ev_feed, 0));
  return 0;
}
// G > 1: the event recorded after k_dedup of gather t (the clear of ring slot t mod (W+1)).
cudaEvent_t dedup_event(int64_t t) {
  const int i = (int)(t & 7);
  if (!g.ev_dedup[i]) cudaEventCreateWithFlags(&g.ev_dedup[i], cudaEventDisableTiming);
  g.dedup_t[i] = t;
  return g.ev_dedup[i];
}
int wait_dedup(int64_t t, cudaStream_t st) {
  if (t < 0) return 0;
  const int i = (int)(t & 7);
  if (g.dedup_t[i] == t) {
    CK(cudaStreamWaitEvent(st, g.ev_dedup[i], 0));
    return 0;
  }
  return wait_gather_end(t, st);  // not recorded (cannot happen through the C-ABI): the whole gather
}
// Before feeding iteration k: the previous feed (IterState window fields, ring order) and, at
// G = 1, gather(k - W - 1), whose k_dedup clears mask bit / ring slot k mod (W+1) (at G > 1 the
// feed's exchange runs first and only k_win_gather waits, for that k_dedup).
int feed_begin(int64_t k, cudaStream_t st) {
  if (int rc = wait_feed(st)) return rc;
  return g.world == 1 ? wait_gather_end(k - (int64_t)g.W - 1, st) : 0;
}
int feed_end(cudaStream_t st) {
  if (!g.ev_feed) CK(cudaEventCreateWithFlags(&g.ev_feed, cudaEventDisableTiming));
  g.feed_recorded = g.feed_since_gather = true;
  g.feed_st = st;
  g.feed_ev_rec = false;
  return 0;
}

// S11: PVP copy of victim queue (t+1) mod W on the side stream, after gather(t) (R17): it
// rewrites staging parity (t+1) & 1, last read by gather(t-1), and reads queue (t+1) mod W,
// last appended to by gather(t).
int launch_pvp(cudaStream_t st) {
  const int64_t t = g.t_next - 1;
  if (g.gend_t[t & 7] == t) {
    if (int rc = wait_gather_end(t, g.side)) return rc;
    if (int rc = wait_gather_end(t - 1, g.side)) return rc;
  } else {  // gather(t) was not noted (cannot happen through the C-ABI): order after st
    CK(cudaEventRecord(g.ev_main, st));
    CK(cudaStreamWaitEvent(g.side, g.ev_main, 0));
  }
  // ... and after the window feed this prefetch call just issued: started alongside the feed
  // kernels, the PCIe-bound copy held the SMs they need and delayed the feed (and everything
  // queued behind it on the caller's stream, e.g. training) by its whole duration
  // (profiles/r01_pvp_overlap.md); after the feed it overlaps the caller's next work instead
  // At G > 1 the feed event completes only after every rank's window exchange, which would
  // gate this copy on the slowest rank; there the copy keeps its gather-only dependencies.
  if (g.world == 1)
    if (int rc = wait_feed(g.side)) return rc;
  uint4* pool = reinterpret_cast<uint4*>(pool_of(g.arena));
  const int blocks = g.sms * std::min(2, g.geom_per_sm);
  prof_begin(7, g.side);
  if (g.nvec >= 256)
    k_pvp<8><<<blocks, 256, 0, g.side>>>(g.it, g.W, (uint32_t)g.stage_base0, (uint32_t)g.C, (uint32_t)g.world, g.qlen,
                                         g.qnode, g.qreuse, reinterpret_cast<const uint4*>(g.qrows_dev), pool,
                                         g.stg_nodes, g.vst_stamp, g.vst_idx, g.scr, g.nvec);
  else
    k_pvp<2><<<blocks, 256, 0, g.side>>>(g.it, g.W, (uint32_t)g.stage_base0, (uint32_t)g.C, (uint32_t)g.world, g.qlen,
                                         g.qnode, g.qreuse, reinterpret_cast<const uint4*>(g.qrows_dev), pool,
                                         g.stg_nodes, g.vst_stamp, g.vst_idx, g.scr, g.nvec);
  LAUNCHED();
  prof_end(7, g.side);
  CK(cudaEventRecord(g.ev_pvp, g.side));
  g.pvp_pending = true;
  return 0;
}

// ---- file tier (N2)
void detach_file() {
  if (g.io) {
    g.io->stop();
    delete g.io;
    g.io = nullptr;
  }
  if (g.file_fd >= 0) close(g.file_fd);
  g.file_fd = -1;
  if (g.bounce_host) cudaFreeHost(g.bounce_host);
  if (g.io_host) cudaFreeHost(g.io_host);
  g.bounce_host = nullptr;
  g.io_host = nullptr;
  g.io_dev = nullptr;
  g.table_dev = nullptr;
}
int attach_file(const char* path, uint64_t rows) {
  const bool want_direct = g.R % 512 == 0 && !std::getenv("LSMGNN_STORAGE_BUFFERED");
  int fd = open(path, O_RDONLY | (want_direct ? O_DIRECT : 0));
  if (fd < 0 && want_direct) fd = open(path, O_RDONLY);  // a filesystem without O_DIRECT
  if (fd < 0) return set_err(LSMGNN_EIO, "open(%s): %s", path, std::strerror(errno));
  struct stat sb {};
  if (fstat(fd, &sb) != 0 || (uint64_t)sb.st_size < rows * g.R) {
    close(fd);
    return set_err(LSMGNN_EINVAL, "%s holds %lld bytes, this home needs %llu", path, (long long)sb.st_size,
                   (unsigned long long)(rows * g.R));
  }
  g.file_fd = fd;
  g.file_direct = want_direct && (fcntl(fd, F_GETFL) & O_DIRECT);
  // fills per batch <= unique nodes per batch at this home (installs + bypassed misses)
  CK(cudaHostAlloc(reinterpret_cast<void**>(&g.bounce_host), std::max<uint64_t>(1, g.ucap) * g.R,
                   cudaHostAllocMapped | cudaHostAllocPortable));
  {  // [IoShared | ready[chunks] | src[ucap]], zeroed (stamps start at 1)
    const uint64_t chunks = (std::max<uint64_t>(1, g.ucap) + kIoChunk - 1) / kIoChunk;
    const size_t bytes = sizeof(IoShared) + 4 * chunks + 4 * std::max<uint64_t>(1, g.ucap);
    CK(cudaHostAlloc(reinterpret_cast<void**>(&g.io_host), bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(g.io_host, 0, bytes);
    void* d = nullptr;
    CK(cudaHostGetDevicePointer(&d, g.io_host, 0));
    g.io_dev = reinterpret_cast<IoShared*>(d);
    g.io_ready_host = reinterpret_cast<uint32_t*>(g.io_host + 1);
    g.io_ready_dev = reinterpret_cast<uint32_t*>(g.io_dev + 1);
    g.io_src_host = g.io_ready_host + chunks;
    g.io_src_dev = g.io_ready_dev + chunks;
  }
  void* dp = nullptr;
  CK(cudaHostGetDevicePointer(&dp, g.bounce_host, 0));
  g.table_dev = reinterpret_cast<const uint8_t*>(dp);
  g.table_host = nullptr;
  if (const char* nt = std::getenv("LSMGNN_IO_THREADS")) g.io_threads = std::max(1, std::atoi(nt));
  g.io = new IoPool();
  g.io->start(g.io_threads - 1);
  return 0;
}
// File tier, step 1 (stream-ordered, before the fill kernel): publish this batch's fill list to
// pinned host memory (k_io_export).
int io_export(cudaStream_t st) {
  KLAUNCH(k_io_export, grid_for((int64_t)g.ucap, 256, 2), 256, 0, st, (const FillEnt*)g.fills, (uint64_t)g.ucap, g.scr,
          (const IterState*)g.it, g.io_dev, g.io_src_dev);
  LAUNCHED();
  return 0;
}
// File tier, step 2 (host, after the fill kernel was launched): wait until the list of batch
// `stamp` is published, then read its storage rows into the bounce buffer (row e = entry e) with
// the pread workers, releasing each chunk of kIoChunk entries to the waiting fill kernel as soon
// as it is read. Every chunk is released even after a read error (the rows are then garbage and
// the error is sticky), so the device never waits forever. No stream synchronisation.
int read_storage_rows(uint32_t stamp, cudaStream_t st) {
  volatile uint32_t* list = &g.io_host->list;
  for (uint64_t spin = 0; *list != stamp; ++spin) {
    if ((spin & 1023) == 1023) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q != cudaErrorNotReady && q != cudaSuccess)
        return set_err(LSMGNN_ECUDA, "stream failed before the fill list was published: %s", cudaGetErrorString(q));
      std::this_thread::yield();
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  const uint32_t n = *(volatile uint32_t*)&g.io_host->n;
  if (n == 0) return 0;
  const uint64_t R = g.R;
  const std::function<int(uint32_t)> read_one = [R](uint32_t e) -> int {
    const uint32_t q = g.io_src_host[e];
    if (q == kInvalid) return 0;  // PVP staging row: already in HBM
    uint8_t* dst = g.bounce_host + (size_t)e * R;
    const off_t off = (off_t)q * (off_t)R;
    size_t done = 0;
    while (done < R) {
      const ssize_t r = pread(g.file_fd, dst + done, R - done, off + (off_t)done);
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) return r < 0 ? errno : EIO;
      done += (size_t)r;
    }
    return 0;
  };
  const std::function<void(uint32_t)> release = [stamp](uint32_t c) {
    std::atomic_thread_fence(std::memory_order_release);  // the chunk's rows before its flag
    reinterpret_cast<std::atomic<uint32_t>*>(&g.io_ready_host[c])->store(stamp, std::memory_order_release);
  };
  const int err = g.io->run(n, read_one, release);
  if (err) {  // the cache already holds tags for rows that never arrived: sticky
    g.sticky = LSMGNN_EIO;
    return set_err(LSMGNN_EIO, "storage read failed: %s", std::strerror(err));
  }
  return 0;
}

int resolve_out(void*& out, bool& out_host, int64_t n) {
  out_host = false;
  if (n <= 0) return 0;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, out) != cudaSuccess || at.type == cudaMemoryTypeUnregistered) {
    cudaGetLastError();
    return set_err(LSMGNN_EINVAL, "out must be device memory or pinned host memory");
  }
  if (at.type == cudaMemoryTypeHost) {  // rows are stored over PCIe
    out_host = true;
    out = at.devicePointer;
  }
  return 0;
}

// ---- layout of one home (host only, no CUDA call): every size and arena offset follows from
// (options, num_nodes, feat_dim, dtype, lines, ways, victim_lines, world). lsmgnn_init applies
// it; lsmgnn_plan_handle evaluates it without a GPU (the handle checks are then testable on
// any host). Returns LSMGNN_EINVAL with a message for any argument lsmgnn_init rejects.
int plan_layout(Ctx& c, int64_t num_nodes, int32_t feat_dim, lsmgnn_dtype dtype, int64_t lines_per_gpu,
                int32_t ways, int64_t victim_lines) {
  const int esz = dtype == LSMGNN_F32 ? 4 : (dtype == LSMGNN_F16 || dtype == LSMGNN_BF16) ? 2 : 0;
  if (esz == 0) return set_err(LSMGNN_EINVAL, "bad dtype");
  if (num_nodes < 1 || num_nodes > 0xFFFFFFF0ll) return set_err(LSMGNN_EINVAL, "num_nodes must be 1..2^32-16");
  if (feat_dim < 1) return set_err(LSMGNN_EINVAL, "bad feat_dim");
  const int64_t R = (int64_t)feat_dim * esz;
  if (R % 16) return set_err(LSMGNN_EINVAL, "row bytes %lld not a multiple of 16 (DESIGN.md R22)", (long long)R);
  if (ways < 1 || ways > 32) return set_err(LSMGNN_EINVAL, "ways must be 1..32");
  if (lines_per_gpu < ways || lines_per_gpu % ways) return set_err(LSMGNN_EINVAL, "lines_per_gpu must be a positive multiple of ways");
  if (lines_per_gpu >= (1ll << 31)) return set_err(LSMGNN_EINVAL, "lines_per_gpu too large");
  const int G = c.world;
  c.N = (uint64_t)num_nodes;
  c.R = (uint32_t)R;
  c.nvec = (uint32_t)(R / 16);
  c.A = (uint32_t)ways;
  c.L = (uint64_t)lines_per_gpu;
  c.S = c.L / c.A;
  c.Q = (c.N + G - 1) / G;
  if (c.Q >= (uint64_t)kHostBit)  // FillEnt::src keeps a home row index in 31 bits
    return set_err(LSMGNN_EINVAL, "ceil(num_nodes / world) must be < 2^31 (use more homes)");
  c.W = (uint32_t)c.opt.window;
  c.Wp1 = c.W + 1;
  c.T = c.opt.threshold ? (uint32_t)c.opt.threshold : std::max<uint32_t>(1, c.W / 8);
  c.MW = (c.Wp1 + 31) / 32;
  c.C = c.opt.pvp ? (uint64_t)victim_lines / c.W : 0;
  if (c.opt.pvp && c.C < 1) return set_err(LSMGNN_EINVAL, "pvp needs victim_lines >= window");
  c.cap = (uint64_t)c.opt.max_batch_ids;
  c.ucap = std::min<uint64_t>(c.cap * G, c.Q);  // unique nodes per batch at a home
  c.bcap = c.ucap;                              // bypass staging rows
  c.stage_base0 = c.L;
  c.bypass_base = c.L + 2 * c.C;
  c.pool_rows = c.L + 2 * c.C + c.bcap;
  if (c.pool_rows >= (uint64_t)kHostBit) return set_err(LSMGNN_EINVAL, "pool too large for 31-bit rows");
  // k_set per-warp shared memory: the largest possible bucket of one set (set s holds the home
  // rows q = s, s + S, ...: at most ceil(Q / S) distinct nodes, and at most the batch's)
  const uint64_t maxm = std::min<uint64_t>((c.Q + c.S - 1) / c.S, c.ucap);
  c.BC = maxm;
  c.ring_stride = c.cap * (uint64_t)std::min(G, 2);
  c.BCp = 32;
  while (c.BCp < maxm) c.BCp <<= 1;
  c.P = 32;
  while (c.P < maxm && c.P < 1024) c.P <<= 1;  // larger buckets fall back to global scratch
  c.warp_bytes = (uint32_t)align_up(20ull * c.P + 4 * 32 * 4, 16);
  c.set_warps = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(8, (160 * 1024) / c.warp_bytes));
  // ---- shared arena: [flags | inbox_cnt | win_cnt | inbox | win_inbox | node_loc | pool]
  size_t o = 0;
  c.off_flags = o; o = align_up(o + 5 * G * sizeof(uint32_t), 256);
  c.off_icnt = o;  o = align_up(o + G * sizeof(uint32_t), 256);
  c.off_wcnt = o;  o = align_up(o + G * sizeof(uint32_t), 256);
  c.off_inbox = o; o = align_up(o + (size_t)G * c.cap * sizeof(uint32_t), 256);
  c.off_win = o;   o = align_up(o + (G > 1 ? (size_t)G * c.cap * sizeof(uint32_t) : 0), 256);
  // node_loc: at G = 1 one table per iteration parity (k_dedup of t + 1 writes its own while
  // k_serve of t reads the other, kernels.cuh k_dedup `early`); at G > 1 peers read the one table
  c.loc_stride = G == 1 ? c.Q : 0;
  c.off_loc = o;   o = align_up(o + (G == 1 ? 2 : 1) * c.Q * sizeof(uint32_t), 4096);
  c.off_pool = o;  o = align_up(o + c.pool_rows * (size_t)c.R, 4096);
  c.arena_bytes = o;
  return 0;
}

// The layout part of a rank's handle (everything but the IPC handle and the GPU UUID): two
// ranks can map each other's arenas only if every offset and size agrees.
void layout_handle(const Ctx& c, Handle* h) {
  std::memset(h, 0, sizeof *h);
  h->arena_bytes = c.arena_bytes;
  uint64_t x = 1469598103934665603ull;  // FNV-1a over the layout words
  const uint64_t words[] = {c.off_flags, c.off_icnt, c.off_wcnt, c.off_inbox, c.off_win, c.off_loc, c.off_pool,
                            c.pool_rows, c.cap, c.R, c.N, c.L, c.A, c.W, c.C, (uint64_t)c.world};
  for (uint64_t w : words)
    for (int b = 0; b < 8; ++b) x = (x ^ ((w >> (8 * b)) & 0xFF)) * 1099511628211ull;
  h->layout_sig = x;
  h->rank = c.rank;
  h->world = c.world;
}

// Every rank's handle must carry its own rank (rank order), the same world and the same
// layout as this rank's; returns 0 or LSMGNN_ECOMM naming the first offending peer.
int check_handles(const Handle* hs, int32_t world, const Handle& mine) {
  if (world != mine.world) return set_err(LSMGNN_ECOMM, "world mismatch: %d handles for a world of %d", world, mine.world);
  for (int r = 0; r < world; ++r) {
    if (hs[r].rank != r) return set_err(LSMGNN_ECOMM, "handle %d carries rank %d (handles must be in rank order)", r, hs[r].rank);
    if (hs[r].world != world) return set_err(LSMGNN_ECOMM, "peer %d was initialised for a world of %d, not %d", r, hs[r].world, world);
    if (hs[r].layout_sig != mine.layout_sig || hs[r].arena_bytes != mine.arena_bytes)
      return set_err(LSMGNN_ECOMM, "peer %d handle does not match this rank's layout (arguments or options differ)", r);
  }
  return 0;
}

}  // namespace

// ====================================================================================== C-ABI
extern "C" {

const char* lsmgnn_last_error(void) { return g.err.c_str(); }
int64_t lsmgnn_kernel_launches(void) { return g.launches; }
size_t lsmgnn_handle_bytes(void) { return sizeof(Handle); }

int lsmgnn_bind(int32_t rank, int32_t world, int32_t device) {
  if (g.inited) return set_err(LSMGNN_ESTATE, "bind after init");
  if (world < 1 || world > kMaxG || rank < 0 || rank >= world)
    return set_err(LSMGNN_EINVAL, "bad rank/world (%d/%d); world must be 1..%d", rank, world, kMaxG);
  g.rank = rank;
  g.world = world;
  g.device = device;
  return 0;
}

int lsmgnn_set_options(const lsmgnn_options* opt) {
  if (g.inited) return set_err(LSMGNN_ESTATE, "set_options after init");
  if (!opt || opt->version != LSMGNN_ABI_VERSION) return set_err(LSMGNN_EINVAL, "bad options/version");
  if (opt->policy < 0 || opt->policy > 4) return set_err(LSMGNN_EINVAL, "bad policy");
  if (opt->window < 1 || opt->window > 65534) return set_err(LSMGNN_EINVAL, "window must be 1..65534");
  if (opt->threshold < 0 || opt->threshold > opt->window) return set_err(LSMGNN_EINVAL, "bad threshold");
  if (opt->update_period < 0 || opt->update_period > 65536) return set_err(LSMGNN_EINVAL, "bad update_period");
  if (opt->max_batch_ids < 1 || opt->max_batch_ids > (1ll << 30)) return set_err(LSMGNN_EINVAL, "bad max_batch_ids");
  g.opt = *opt;
  g.opt_set = true;
  return 0;
}

int lsmgnn_init(int64_t num_nodes, int32_t feat_dim, lsmgnn_dtype dtype, int64_t lines_per_gpu, int32_t ways,
                int64_t victim_lines, const uint8_t* static_scores) {
  if (g.inited) return set_err(LSMGNN_ESTATE, "already initialised");
  if (!g.opt_set) g.opt = default_options();
  if (int rc = plan_layout(g, num_nodes, feat_dim, dtype, lines_per_gpu, ways, victim_lines)) return rc;
  if (g.device < 0) CK(cudaGetDevice(&g.device));
  CK(cudaSetDevice(g.device));
  CK(cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, g.device));
  const int G = g.world;
  const bool big_sets = std::min<uint64_t>((g.Q + g.S - 1) / g.S, g.ucap) > g.P;
  if (const char* geo = getenv("LSMGNN_GEOMETRY")) {  // launch-geometry override: results must not change
    if (!strcmp(geo, "small")) {
      g.set_warps = 1;
      g.geom_per_sm = 1;
    }
  }

  CK(cudaMalloc(&g.arena, g.arena_bytes));
  CK(cudaMemset(g.arena, 0, g.off_pool));
  for (int h = 0; h < kMaxG; ++h) g.peer_arena[h] = nullptr;
  g.peer_arena[g.rank] = g.arena;

  int rc = 0;
#define DA(p, n) if ((rc = dalloc(&(p), (n)))) return rc
  DA(g.tags, g.L);
  CK(cudaMemset(g.tags, 0xFF, g.L * sizeof(uint32_t)));
  DA(g.last_use, g.L);
  DA(g.rr, g.S);
  DA(g.mask, g.Q * g.MW);
  DA(g.mark, g.Q);
  DA(g.vst_stamp, g.Q);
  DA(g.vst_idx, g.Q);
  DA(g.set_cnt, g.S);
  DA(g.scan_q, 2 * (size_t)scan_tiles(g.W));
  DA(g.slow_stamp, g.S);
  DA(g.slow_list, g.S);
  if (big_sets) {  // a power-of-two region of global scratch per set that can exceed P
    DA(g.g_sv, g.S * g.BCp + 64);
    DA(g.g_sk, g.S * g.BCp + 64);
    DA(g.g_sidx, g.S * g.BCp + 64);
    DA(g.g_skey, g.S * g.BCp + 64);
  }
  DA(g.bucket, g.S * g.BC + 32);  // + 32: k_set reads a set's first 32 entries unconditionally
  DA(g.ring, (size_t)g.Wp1 * g.ring_stride);
  DA(g.ring_len, g.Wp1);
  DA(g.qcnt, g.W);
  DA(g.qoff, g.W + 1);
  DA(g.qb, g.ucap);
  DA(g.qlen, g.W);
  DA(g.qnode, std::max<uint64_t>(1, g.W * g.C));
  DA(g.qreuse, std::max<uint64_t>(1, g.W * g.C));
  DA(g.stg_nodes, std::max<uint64_t>(1, 2 * g.C));
  DA(g.route_cnt, 2 * G);
  if (g.opt.update_period > 1) {
    DA(g.line_info, g.L);
    CK(cudaMemset(g.line_info, 0xFF, g.L * sizeof(uint32_t)));
  }
  if (G == 1) {  // request lists and per-request locations of the fused delivery, one per iteration parity
    DA(g.head, 2 * g.Q);
    DA(g.nxt, 2 * g.cap);
    DA(g.req_loc, 2 * g.cap);
  }
  DA(g.score, g.Q);
  DA(g.fills, 2 * g.ucap);  // one fill list per iteration parity
  DA(g.cands, g.ucap);
  DA(g.scr, 1);
  DA(g.it, 1);
  DA(g.hist, (size_t)kHist * F_NFIELDS);
  DA(g.cum, F_NFIELDS);
#undef DA
  if (static_scores) {  // this home's nodes v = rank + k*G, in k order
    std::vector<uint8_t> mine(g.Q, 0);
    for (uint64_t k = 0; k < g.Q; ++k) {
      const uint64_t v = (uint64_t)g.rank + k * G;
      if (v < g.N) mine[k] = static_scores[v];
    }
    CK(cudaMemcpy(g.score, mine.data(), g.Q, cudaMemcpyHostToDevice));
  }
  if (g.C) {
    const size_t qb = (size_t)g.W * g.C * g.R;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&g.qrows_host), qb, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g.qrows_dev), g.qrows_host, 0));
  }
  {
    void* hb = nullptr;
    CK(cudaHostAlloc(&hb, 64, cudaHostAllocMapped));
    std::memset(hb, 0, 64);
    g.bad_host = reinterpret_cast<volatile uint32_t*>(hb);
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g.bad_dev), hb, 0));
    g.bad_dev_overflow = g.bad_dev + 1;
  }
  CK(cudaStreamCreateWithFlags(&g.side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&g.ev_main, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&g.ev_pvp, cudaEventDisableTiming));
  CK(cudaFuncSetAttribute(k_set, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(g.warp_bytes * g.set_warps)));
  {  // k_serve / k_pull: the most row loads in flight per SM — (ST - 1) per warp, 8 warps per
     // CTA, up to 3 CTAs (registers) — within 160 KB of shared memory per SM, which leaves room
     // for the next gather's k_dedup / k_set beside it (A/B ab_geo2 at 4 KiB rows: 5 stages
     // 0.1873 ms/step, 6 stages 0.1916, 4 stages 0.1870, 3 stages 0.1913)
    const uint64_t budget = 160 * 1024;
    g.serve_cps = 1;
    g.serve_st = 0;
    uint64_t best = 0;
    for (int cps = 1; cps <= 3; ++cps) {
      const uint64_t st = std::min<uint64_t>(kMaxStages, budget / ((uint64_t)cps * 8 * g.R));
      if (st >= 2 && (st - 1) * cps > best) {
        best = (st - 1) * cps;
        g.serve_cps = cps;
        g.serve_st = (int)st;
      }
    }
    if (const char* e = std::getenv("LSMGNN_SERVE_CPS")) g.serve_cps = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("LSMGNN_SERVE_ST")) g.serve_st = std::max(0, std::min((int)kMaxStages, std::atoi(e)));
    // the rings of 8 warps must fit one CTA's shared memory (227 KB on sm_100)
    while (g.serve_st > 0 && (uint64_t)8 * g.serve_st * g.R > 220 * 1024) --g.serve_st;
    if (g.serve_st) {
      const int smem = (int)((size_t)8 * g.serve_st * g.R);
      CK(cudaFuncSetAttribute(k_serve<8, kDev, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(k_serve<8, kHost, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(k_serve<2, kDev, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(k_pull<8, kDev, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(k_pull<8, kDev, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(k_pull<2, kDev, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(k_pull<2, kDev, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
  }
  g.pdl = G == 1 && !std::getenv("LSMGNN_NO_PDL");
  g.g1_pull = G == 1 && std::getenv("LSMGNN_G1_PULL") && std::atoi(std::getenv("LSMGNN_G1_PULL")) != 0;
  g.feed_early = !(std::getenv("LSMGNN_FEED_EARLY") && std::atoi(std::getenv("LSMGNN_FEED_EARLY")) == 0);
  if (const char* e = std::getenv("LSMGNN_SERVE_TAIL")) g.serve_tail = std::max(1, std::min(32, std::atoi(e)));
  if (const char* e = std::getenv("LSMGNN_SERVE_TAIL_ROUNDS")) g.serve_tail_rounds = std::max(0, std::min(64, std::atoi(e)));
  if (const char* e = std::getenv("LSMGNN_SERVE_AHEAD")) g.serve_ahead = std::atoi(e) != 0;
  if (const char* e = std::getenv("LSMGNN_L2_EVICT_FIRST")) g.l2_evict_first = std::max(0, std::min(2, std::atoi(e)));
  if (const char* e = std::getenv("LSMGNN_DEDUP_EARLY")) g.dedup_early = std::atoi(e) != 0;
  g.meta_evict_last = g.Q * 20 <= (60ull << 20);
  g.mask_evict_last = g.Q * (20 + 4ull * g.MW) <= (64ull << 20);
  if (const char* e = std::getenv("LSMGNN_META_EVICT_LAST")) g.meta_evict_last = std::atoi(e) != 0;
  if (const char* e = std::getenv("LSMGNN_MASK_EVICT_LAST")) g.mask_evict_last = std::atoi(e) != 0;
  if (const char* e = std::getenv("LSMGNN_SERVE_STATIC_FIRST")) g.serve_static_first = std::atoi(e) != 0;
  if (const char* e = std::getenv("LSMGNN_HOST_TMA")) g.host_tma = std::atoi(e) != 0;
  if (const char* e = std::getenv("LSMGNN_EARLY_SET_PER_SM")) g.early_set_per_sm = std::max(1, std::min(4, std::atoi(e)));
  if (const char* e = std::getenv("LSMGNN_EARLY_DEDUP_PER_SM")) g.early_dedup_per_sm = std::max(1, std::min(8, std::atoi(e)));
  if (g.g1_pull) g.split_pull = false;
  if (G > 1) {
    CK(cudaStreamCreateWithFlags(&g.pull_st, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g.ev_set, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g.ev_pull0, cudaEventDisableTiming));
    cudaDriverEntryPointQueryResult q1, q2;
    CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", reinterpret_cast<void**>(&g.waitv), cudaEnableDefault, &q1));
    CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", reinterpret_cast<void**>(&g.writev), cudaEnableDefault, &q2));
    if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !g.waitv || !g.writev)
      return set_err(LSMGNN_ECOMM, "stream memory operations unavailable");
    cudaDriverEntryPointQueryResult q3;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", reinterpret_cast<void**>(&g.batchv), cudaEnableDefault, &q3) !=
            cudaSuccess ||
        q3 != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      g.batchv = nullptr;  // single operations instead
    }
    if (std::getenv("LSMGNN_NO_BATCH_MEMOP")) g.batchv = nullptr;
  }
  CK(cudaDeviceSynchronize());
  g.inited = true;
  g.connected = (G == 1);
  g.t_next = 0;
  g.feed_next = 1;
  return 0;
}

int lsmgnn_attach_storage(const void* host_rows, const char* nvme_path) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "attach_storage before init");
  if (!host_rows == !nvme_path) return set_err(LSMGNN_EINVAL, "exactly one of host_rows / nvme_path");
  if (g.table_registered) {
    cudaHostUnregister((void*)g.table_host);
    g.table_registered = false;
  }
  detach_file();
  const uint64_t rows = (g.N > (uint64_t)g.rank) ? (g.N - g.rank + g.world - 1) / g.world : 0;
  if (nvme_path) return attach_file(nvme_path, rows);
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, host_rows);
  if (e != cudaSuccess) cudaGetLastError();
  if (e == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer) {
    g.table_dev = reinterpret_cast<const uint8_t*>(at.devicePointer);
  } else {
    CK(cudaHostRegister(const_cast<void*>(host_rows), rows * g.R, cudaHostRegisterMapped | cudaHostRegisterPortable));
    g.table_registered = true;
    void* dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, const_cast<void*>(host_rows), 0));
    g.table_dev = reinterpret_cast<const uint8_t*>(dp);
  }
  g.table_host = reinterpret_cast<const uint8_t*>(host_rows);
  return 0;
}

int lsmgnn_export_handle(void* buf, size_t cap) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "export before init");
  if (!buf || cap < sizeof(Handle)) return set_err(LSMGNN_EINVAL, "buffer too small");
  Handle h{};
  layout_handle(g, &h);
  CK(cudaIpcGetMemHandle(&h.ipc, g.arena));
  cudaDeviceProp prop{};
  CK(cudaGetDeviceProperties(&prop, g.device));
  std::memcpy(h.gpu_uuid, &prop.uuid, sizeof h.gpu_uuid);
  std::memcpy(buf, &h, sizeof h);
  return 0;
}

int lsmgnn_plan_handle(const lsmgnn_options* opt, int64_t num_nodes, int32_t feat_dim, lsmgnn_dtype dtype,
                       int64_t lines_per_gpu, int32_t ways, int64_t victim_lines, int32_t rank, int32_t world,
                       void* buf, size_t cap) {
  if (!buf || cap < sizeof(Handle)) return set_err(LSMGNN_EINVAL, "buffer too small");
  if (world < 1 || world > kMaxG || rank < 0 || rank >= world)
    return set_err(LSMGNN_EINVAL, "bad rank/world (%d/%d); world must be 1..%d", rank, world, kMaxG);
  Ctx* c = new Ctx();  // a scratch context: nothing is allocated, no CUDA call is made
  c->rank = rank;
  c->world = world;
  c->opt = opt ? *opt : default_options();
  int rc = 0;
  if (opt && opt->version != LSMGNN_ABI_VERSION) rc = set_err(LSMGNN_EINVAL, "bad options/version");
  if (!rc) rc = plan_layout(*c, num_nodes, feat_dim, dtype, lines_per_gpu, ways, victim_lines);
  if (!rc) {
    Handle h{};
    layout_handle(*c, &h);
    std::memcpy(buf, &h, sizeof h);
  }
  delete c;
  return rc;
}

int lsmgnn_check_handles(const void* handles, int32_t world, const void* mine) {
  if (!handles || !mine || world < 1 || world > kMaxG) return set_err(LSMGNN_EINVAL, "bad handle arguments");
  Handle me{};
  std::memcpy(&me, mine, sizeof me);
  std::vector<Handle> hs((size_t)world);
  std::memcpy(hs.data(), handles, sizeof(Handle) * (size_t)world);
  return check_handles(hs.data(), world, me);
}

int lsmgnn_connect(const void* peer_handles, int32_t world) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "connect before init");
  if (!peer_handles) return set_err(LSMGNN_EINVAL, "null handles");
  if (world == 1 && g.world == 1) {
    g.connected = true;
    return 0;
  }
  Handle mine{};
  if (int rc = lsmgnn_export_handle(&mine, sizeof mine)) return rc;
  std::vector<Handle> hs((size_t)std::max(1, std::min<int32_t>(world, kMaxG)));
  if (world >= 1 && world <= kMaxG) std::memcpy(hs.data(), peer_handles, sizeof(Handle) * (size_t)world);
  if (int rc = check_handles(hs.data(), world, mine)) return rc;
  for (int r = 0; r < world; ++r) {
    if (r == g.rank) continue;
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, hs[r].ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_err(LSMGNN_ECOMM, "cudaIpcOpenMemHandle(peer %d): %s", r, cudaGetErrorString(e));
    g.peer_arena[r] = reinterpret_cast<char*>(p);
  }
  bool gpu_shared = false;
  for (int r = 0; r < world; ++r)
    if (r != g.rank && std::memcmp(hs[r].gpu_uuid, mine.gpu_uuid, sizeof mine.gpu_uuid) == 0) gpu_shared = true;
  const char* sp = std::getenv("LSMGNN_SPLIT_PULL");
  g.split_pull = sp ? std::atoi(sp) != 0 : !gpu_shared;
  g.connected = true;
  return 0;
}

int lsmgnn_gather(const int64_t* node_ids, int64_t n, void* out, void* stream) {
  if (!g.inited || !g.connected) return set_err(LSMGNN_ESTATE, "gather before init/connect");
  if (!g.table_dev) return set_err(LSMGNN_ESTATE, "no storage attached");
  if (n < 0 || (uint64_t)n > g.cap) return set_err(LSMGNN_EINVAL, "n=%lld exceeds max_batch_ids", (long long)n);
  if (n > 0 && (!node_ids || !out)) return set_err(LSMGNN_EINVAL, "null ids/out");
  if (reinterpret_cast<uintptr_t>(out) % 16) return set_err(LSMGNN_EINVAL, "out must be 16-byte aligned");
  if (int rc = check_sticky()) return rc;
  bool out_host = false;
  if (int rc = resolve_out(out, out_host, n)) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t t = g.t_next;
  if (g.pvp_pending) {
    CK(cudaStreamWaitEvent(st, g.ev_pvp, 0));
    g.pvp_pending = false;
  }
  if (g.feed_since_gather) {  // the window fed through t+W (possibly on another stream)
    if (int rc = wait_feed(st)) return rc;
    g.feed_since_gather = false;
  }
  if (t > 0 && st != g.gather_st)  // same stream: already ordered (and PDL keeps chaining)
    if (int rc = wait_gather_end(t - 1, st)) return rc;
  const BeginArgs ba = begin_args(t, node_ids, n, nullptr, nullptr, 0);
  if (int rc = launch_gather(ba, n, out, out_host, false, (uint32_t)(t + 1), st, g.world > 1 ? dedup_event(t) : nullptr))
    return rc;
  if (int rc = note_gather_end(t, st)) return rc;
  g.t_next = t + 1;
  g.gather_st = st;
  g.last_stream = st;
  return 0;
}

int lsmgnn_prefetch(const int64_t* ids, const int64_t* offsets, int32_t num_batches, int64_t first_iter,
                    void* stream) {
  if (!g.inited || !g.connected) return set_err(LSMGNN_ESTATE, "prefetch before init/connect");
  if (num_batches < 0 || (num_batches > 0 && !offsets)) return set_err(LSMGNN_EINVAL, "bad batches");
  if (num_batches > 0 && first_iter != g.feed_next)
    return set_err(LSMGNN_ESTATE, "window iteration %lld fed, %lld expected", (long long)first_iter,
                   (long long)g.feed_next);
  if (int rc = check_sticky()) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (num_batches > 0) prof_begin(6, st);
  for (int32_t b = 0; b < num_batches; ++b) {
    const int64_t k = first_iter + b;
    const int64_t n = offsets[b + 1] - offsets[b];
    if (n < 0 || (uint64_t)n > g.cap) return set_err(LSMGNN_EINVAL, "window batch of %lld ids", (long long)n);
    if (k > g.t_next + (int64_t)g.W) return set_err(LSMGNN_ESTATE, "window fed beyond t+W");
    if (k < g.t_next) return set_err(LSMGNN_ESTATE, "window iteration %lld was already gathered", (long long)k);
    if (int rc = feed_begin(k, st)) return rc;
    if (int rc = launch_window(k, n > 0 ? ids + offsets[b] : nullptr, n, nullptr, nullptr, nullptr, 0, n, st))
      return rc;
    if (int rc = feed_end(st)) return rc;
    g.feed_next = k + 1;
  }
  if (num_batches > 0) prof_end(6, st);
  // ---- S11 PVP copy for iteration t+1 on the side stream (after gather(t))
  if (g.C && g.t_next > 0 && !g.pvp_pending)
    if (int rc = launch_pvp(st)) return rc;
  g.last_stream = st;
  return 0;
}

int lsmgnn_gather_host(const int64_t* host_ids, int64_t n, void* host_out, void* stream) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "not initialised");
  if (n < 0 || (uint64_t)n > g.cap) return set_err(LSMGNN_EINVAL, "bad n");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!g.tmp_ids) CK(cudaMalloc(reinterpret_cast<void**>(&g.tmp_ids), g.cap * sizeof(int64_t)));
  if (n > 0) CK(cudaMemcpyAsync(g.tmp_ids, host_ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  // pinned host `out`: the serve kernels store the rows straight over PCIe (D2H overlaps the
  // storage H2D of the same launch); pageable `out`: device staging + cudaMemcpy
  cudaPointerAttributes at{};
  const bool pinned = n > 0 && cudaPointerGetAttributes(&at, host_out) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (pinned || n == 0) {
    if (int rc = lsmgnn_gather(g.tmp_ids, n, host_out, stream)) return rc;
  } else {
    if (!g.tmp_out) CK(cudaMalloc(&g.tmp_out, g.cap * (size_t)g.R));
    if (int rc = lsmgnn_gather(g.tmp_ids, n, g.tmp_out, stream)) return rc;
    CK(cudaMemcpyAsync(host_out, g.tmp_out, n * (size_t)g.R, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return check_sticky();
}

#ifdef LSMGNN_TRACE
// (experiments only) reset = 1: clear the timeline probe; else copy it out: [8][2][2] u64
int lsmgnn_debug_trace(unsigned long long* out, int32_t reset) {
  unsigned long long h[8][2][2];
  if (reset) {
    for (auto& k : h)
      for (auto& p : k) p[0] = ~0ull, p[1] = 0;
    CK(cudaMemcpyToSymbol(g_trace, h, sizeof h));
  } else {
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(out, g_trace, sizeof h));
  }
  return 0;
}
#endif

int lsmgnn_stats(lsmgnn_stats_t* out_host, int32_t scope) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "not initialised");
  if (!out_host || (scope != 0 && scope != 1)) return set_err(LSMGNN_EINVAL, "bad args");
  static_assert(sizeof(lsmgnn_stats_t) == F_NFIELDS * sizeof(uint64_t), "stats layout");
  CK(cudaDeviceSynchronize());
  if (scope == 1) {
    CK(cudaMemcpy(out_host, g.cum, sizeof(lsmgnn_stats_t), cudaMemcpyDeviceToHost));
  } else if (g.t_next == 0) {
    std::memset(out_host, 0, sizeof *out_host);
  } else {
    CK(cudaMemcpy(out_host, g.hist + (size_t)((g.t_next - 1) % kHist) * F_NFIELDS, sizeof(lsmgnn_stats_t),
                  cudaMemcpyDeviceToHost));
  }
  return check_sticky();
}

int lsmgnn_stats_history(lsmgnn_stats_t* out_host, int64_t first, int64_t count) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "not initialised");
  // the last kHist - 2 iterations (the slots of the next two are already zeroed: end_record)
  if (count < 0 || first < 0 || first + count > g.t_next || (g.t_next - first) > (int64_t)kHist - 2)
    return set_err(LSMGNN_EINVAL, "history range [%lld,+%lld) unavailable", (long long)first, (long long)count);
  CK(cudaDeviceSynchronize());
  // the ring [first, first+count) is at most two contiguous pieces
  for (int64_t i = 0; i < count;) {
    const int64_t slot = (first + i) % kHist;
    const int64_t run = std::min<int64_t>(count - i, (int64_t)kHist - slot);
    CK(cudaMemcpy(out_host + i, g.hist + (size_t)slot * F_NFIELDS, run * sizeof(lsmgnn_stats_t), cudaMemcpyDeviceToHost));
    i += run;
  }
  return check_sticky();
}

// ------------------------------------------------------------------ NEXT N3: GPU sampler
int lsmgnn_sampler_attach(const int64_t* indptr, const int32_t* indices, int64_t num_nodes, int64_t nnz) {
  if (!indptr || !indices || num_nodes < 1 || num_nodes > 0xFFFFFFF0ll || nnz < 0)
    return set_err(LSMGNN_EINVAL, "bad CSR");
  if (g.device < 0) CK(cudaGetDevice(&g.device));
  CK(cudaSetDevice(g.device));
  CK(cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, g.device));
  auto map = [](const void* p, size_t bytes, bool* registered, const void** dev) -> int {
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) cudaGetLastError();
    if (e == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer) {
      *dev = at.devicePointer;
      *registered = false;
      return 0;
    }
    CK(cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterMapped | cudaHostRegisterPortable | cudaHostRegisterReadOnly));
    void* d = nullptr;
    CK(cudaHostGetDevicePointer(&d, const_cast<void*>(p), 0));
    *dev = d;
    *registered = true;
    return 0;
  };
  if (int rc = map(indptr, (num_nodes + 1) * sizeof(int64_t), &g.s_reg_indptr, (const void**)&g.s_indptr)) return rc;
  if (int rc = map(indices, std::max<int64_t>(nnz, 1) * sizeof(int32_t), &g.s_reg_indices, (const void**)&g.s_indices))
    return rc;
  g.s_host_indptr = indptr;
  g.s_host_indices = indices;
  g.s_map_indptr = g.s_indptr;
  g.s_map_indices = g.s_indices;
  g.s_nnz = nnz;
  g.s_N = (uint64_t)num_nodes;
  if (g.s_hbm_indptr) {
    cudaFree(g.s_hbm_indptr);
    cudaFree(g.s_hbm_indices);
    g.s_hbm_indptr = nullptr;
    g.s_hbm_indices = nullptr;
  }
  if (g.s_tab) cudaFree(g.s_tab);
  CK(cudaMalloc(&g.s_tab, g.s_N * sizeof(unsigned long long)));
  CK(cudaMemset(g.s_tab, 0xFF, g.s_N * sizeof(unsigned long long)));
  if (!g.s_counts) CK(cudaMalloc(&g.s_counts, sizeof(SampCounts)));
  g.s_hi = 0xFFFFFFFFu;
  return 0;
}

int lsmgnn_sample(const int64_t* seeds, int64_t nseeds, const int32_t* fanout, int32_t nlayers, uint64_t seed,
                  int64_t t, int32_t r, int64_t* out, int64_t cap, int64_t* count_dev, void* stream) {
  if (!g.s_tab) return set_err(LSMGNN_ESTATE, "sampler_attach first");
  if (nseeds < 0 || nlayers < 0 || nlayers > 16 || (nseeds > 0 && (!seeds || !out)) || !count_dev || (nlayers && !fanout))
    return set_err(LSMGNN_EINVAL, "bad sample arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // host-side upper bounds (the real sizes stay on the device)
  uint64_t prod = (uint64_t)nseeds, bound = (uint64_t)nseeds, maxlayer = 0;
  for (int l = 0; l < nlayers; ++l) {
    if (fanout[l] < 0) return set_err(LSMGNN_EINVAL, "negative fanout");
    prod *= (uint64_t)fanout[l];
    bound += prod;
    maxlayer = std::max(maxlayer, prod);
  }
  if (bound > (4ull << 20)) return set_err(LSMGNN_EINVAL, "sample bound %llu > 4M ids", (unsigned long long)bound);
  if ((uint64_t)cap < bound) return set_err(LSMGNN_EINVAL, "out capacity %lld < bound %llu", (long long)cap,
                                            (unsigned long long)bound);
  if (bound > g.s_cap) {  // grow scratch (first use / larger fanout)
    for (uint32_t* p : {g.s_raw, g.s_layer, g.s_front, g.s_cnt, g.s_off, g.s_keep, g.s_pos, g.s_bsum})
      if (p) cudaFree(p);
    const size_t b = bound + 1;
    CK(cudaMalloc(&g.s_raw, b * 4));
    CK(cudaMalloc(&g.s_layer, b * 4));
    CK(cudaMalloc(&g.s_front, b * 4));
    CK(cudaMalloc(&g.s_cnt, b * 4));
    CK(cudaMalloc(&g.s_off, b * 4));
    CK(cudaMalloc(&g.s_keep, b * 4));
    CK(cudaMalloc(&g.s_pos, b * 4));
    CK(cudaMalloc(&g.s_bsum, 1024 * 4));
    g.s_cap = bound;
  }
  SampCounts* c = g.s_counts;
  auto xscan = [&](const uint32_t* x, const uint32_t* n_ptr, uint32_t* y, uint64_t nmax) -> int {
    const int nb = (int)std::max<uint64_t>(1, (nmax + 4095) / 4096);
    KLAUNCH(k_xscan_blocks, nb, 1024, 0, st, x, n_ptr, 0, y, g.s_bsum);
    LAUNCHED();
    KLAUNCH(k_xscan_sums, 1, 1024, 0, st, g.s_bsum, (uint32_t)nb);
    LAUNCHED();
    KLAUNCH(k_xscan_add, grid_for((int64_t)nmax, 256, 4), 256, 0, st, y, n_ptr, 0, g.s_bsum);
    LAUNCHED();
    return 0;
  };
  // first-occurrence unique of a[0..*n_ptr) -> out (OutT), count -> *n_out
  auto unique_first = [&](const uint32_t* a, const uint32_t* n_ptr, uint64_t nmax, auto* outp, uint32_t* n_out) -> int {
    const uint32_t hi = g.s_hi--;
    const int gr = grid_for((int64_t)std::max<uint64_t>(nmax, 1), 256, 4);
    KLAUNCH(k_fo_mark, gr, 256, 0, st, a, n_ptr, 0, g.s_tab, hi);
    LAUNCHED();
    KLAUNCH(k_fo_flag, gr, 256, 0, st, a, n_ptr, 0, g.s_tab, hi, g.s_keep);
    LAUNCHED();
    if (int rc = xscan(g.s_keep, n_ptr, g.s_pos, nmax)) return rc;
    KLAUNCH((k_fo_compact<std::remove_pointer_t<decltype(outp)>>), gr, 256, 0, st, a, n_ptr, 0, g.s_keep, g.s_pos, outp, n_out);
    LAUNCHED();
    return 0;
  };
  KLAUNCH(k_samp_init, grid_for(std::max<int64_t>(nseeds, 1), 256, 4), 256, 0, st, seeds, (uint32_t)nseeds, g.s_raw,
                                                                              g.s_front, c);
  LAUNCHED();
  uint64_t fmax = (uint64_t)nseeds;
  for (int l = 0; l < nlayers; ++l) {
    const uint32_t f = (uint32_t)fanout[l];
    const uint64_t lmax = fmax * f;
    const int gr = grid_for((int64_t)std::max<uint64_t>(fmax, 1), 256, 4);
    KLAUNCH(k_samp_count, gr, 256, 0, st, g.s_front, c, g.s_indptr, f, g.s_cnt);
    LAUNCHED();
    if (int rc = xscan(g.s_cnt, &c->nf, g.s_off, fmax)) return rc;
    KLAUNCH(k_xscan_total, 1, 1, 0, st, g.s_off, g.s_cnt, &c->nf, 0, &c->layer_n);
    LAUNCHED();
    KLAUNCH(k_samp_draw, grid_for((int64_t)std::max<uint64_t>(fmax, 1) * 32, 256, 8), 256, 0, st, 
        g.s_front, c, g.s_indptr, g.s_indices, f, g.s_off, g.s_layer, seed, (uint64_t)t, (uint64_t)r, (uint64_t)l);
    LAUNCHED();
    KLAUNCH(k_samp_append, grid_for((int64_t)std::max<uint64_t>(lmax, 1), 256, 4), 256, 0, st, g.s_layer, c, g.s_raw);
    LAUNCHED();
    // next frontier = first-occurrence unique of this layer's draws
    if (int rc = unique_first(g.s_layer, &c->layer_n, lmax, g.s_front, &c->nf)) return rc;
    KLAUNCH(k_samp_advance, 1, 1, 0, st, c);
    LAUNCHED();
    fmax = lmax;
  }
  if (int rc = unique_first(g.s_raw, &c->nraw, bound, out, &c->nout)) return rc;
  KLAUNCH(k_samp_out_count, 1, 1, 0, st, c, count_dev);
  LAUNCHED();
  return 0;
}

// Where the sampler reads the CSR: in_hbm = 0 — pinned host memory over PCIe (UVA, the
// paper's placement); 1 — a copy in HBM (B200's 180 GB holds a 100M-node CSR).
int lsmgnn_sampler_place(int32_t in_hbm) {
  if (!g.s_tab) return set_err(LSMGNN_ESTATE, "sampler_attach first");
  if (in_hbm) {
    if (!g.s_hbm_indptr) {
      CK(cudaMalloc(&g.s_hbm_indptr, (g.s_N + 1) * sizeof(int64_t)));
      CK(cudaMalloc(&g.s_hbm_indices, std::max<int64_t>(g.s_nnz, 1) * sizeof(int32_t)));
      CK(cudaMemcpy(g.s_hbm_indptr, g.s_host_indptr, (g.s_N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(g.s_hbm_indices, g.s_host_indices, std::max<int64_t>(g.s_nnz, 1) * sizeof(int32_t),
                    cudaMemcpyHostToDevice));
    }
    g.s_indptr = g.s_hbm_indptr;
    g.s_indices = g.s_hbm_indices;
  } else {
    g.s_indptr = g.s_map_indptr;
    g.s_indices = g.s_map_indices;
  }
  return 0;
}

// Window feed of one batch whose length lives on the device (e.g. straight from
// lsmgnn_sample): same semantics as lsmgnn_prefetch with num_batches = 1. With G > 1 the
// route kernel reads the length from IterState (k_win_begin), so no rank needs it on the host.
int lsmgnn_prefetch_dev(const int64_t* ids, const int64_t* count_dev, int64_t first_iter, void* stream) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "not initialised");
  if (!count_dev) return set_err(LSMGNN_EINVAL, "null count");
  if (first_iter != g.feed_next) return set_err(LSMGNN_ESTATE, "window iteration out of order");
  if (first_iter > g.t_next + (int64_t)g.W) return set_err(LSMGNN_ESTATE, "window fed beyond t+W");
  if (first_iter < g.t_next) return set_err(LSMGNN_ESTATE, "window iteration already gathered");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  prof_begin(6, st);
  if (int rc = feed_begin(first_iter, st)) return rc;
  if (int rc = launch_window(first_iter, ids, 0, count_dev, nullptr, nullptr, 0, (int64_t)g.cap, st)) return rc;
  if (int rc = feed_end(st)) return rc;
  prof_end(6, st);
  g.feed_next = first_iter + 1;
  // the PVP copy for t+1 is issued by lsmgnn_prefetch; call it with num_batches = 0 when needed
  g.last_stream = st;
  return 0;
}

// ------------------------------------------------------------------ CUDA-graph step (G = 1)
int lsmgnn_graph_capture(const int64_t* const* ids_ring, const int64_t* n_ring, int32_t ring_len, void* out,
                         void* stream) {
  if (!g.inited || !g.table_dev) return set_err(LSMGNN_ESTATE, "graph_capture before init/attach_storage");
  if (g.world != 1) return set_err(LSMGNN_EINVAL, "graph mode is single-home (G = 1) only");
  if (g.file_fd >= 0) return set_err(LSMGNN_EINVAL, "graph mode needs host-memory storage (the file tier reads on the host)");
  if (!ids_ring || !n_ring || !out || ring_len < (int32_t)g.W + 2)
    return set_err(LSMGNN_EINVAL, "graph_capture needs a ring of >= W+2 batches and an out buffer");
  if (g.feed_next != g.t_next + (int64_t)g.W + 1)
    return set_err(LSMGNN_ESTATE, "feed the window through t+W before capturing");
  if (int rc = check_sticky()) return rc;
  bool out_host = false;
  if (int rc = resolve_out(out, out_host, 1)) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaStreamSynchronize(st));
  if (g.graph_exec) {
    cudaGraphExecDestroy(g.graph_exec);
    g.graph_exec = nullptr;
  }
  if (g.graph) {
    cudaGraphDestroy(g.graph);
    g.graph = nullptr;
  }
  if (!g.cap_stream) CK(cudaStreamCreateWithFlags(&g.cap_stream, cudaStreamNonBlocking));
  if (!g.cap_stream2) CK(cudaStreamCreateWithFlags(&g.cap_stream2, cudaStreamNonBlocking));
  if (!g.ev_fork) CK(cudaEventCreateWithFlags(&g.ev_fork, cudaEventDisableTiming));
  if (!g.ev_join) CK(cudaEventCreateWithFlags(&g.ev_join, cudaEventDisableTiming));
  const bool prof = g.prof;
  g.prof = false;  // no host-side event spans inside a graph
  const int64_t l0 = g.launches;
  // Two branches: gather(t) and, forked after its k_dedup (which clears ring slot / mask bit
  // t mod (W+1)), the window feed of t+1+W. The feed rewrites only that slot and bit, which
  // the rest of gather(t) never reads (it looks at t+1..t+W), so the two run concurrently.
  CK(cudaStreamBeginCapture(g.cap_stream, cudaStreamCaptureModeThreadLocal));
  const BeginArgs ba = begin_args(-1, nullptr, 0, ids_ring, n_ring, (uint32_t)ring_len);
  int rc = launch_gather(ba, (int64_t)g.cap, out, out_host, true, 0, g.cap_stream, g.ev_fork);
  cudaError_t fe = cudaSuccess;
  if (!rc) {
    fe = cudaStreamWaitEvent(g.cap_stream2, g.ev_fork, 0);
    if (fe != cudaSuccess) rc = set_err(LSMGNN_ECUDA, "graph fork: %s", cudaGetErrorString(fe));
  }
  if (!rc) rc = launch_window(-1, nullptr, 0, nullptr, ids_ring, n_ring, (uint32_t)ring_len, (int64_t)g.cap, g.cap_stream2);
  if (!rc) {
    fe = cudaEventRecord(g.ev_join, g.cap_stream2);
    if (fe == cudaSuccess) fe = cudaStreamWaitEvent(g.cap_stream, g.ev_join, 0);
    if (fe != cudaSuccess) rc = set_err(LSMGNN_ECUDA, "graph join: %s", cudaGetErrorString(fe));
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(g.cap_stream, &graph);
  g.prof = prof;
  g.graph_launches = g.launches - l0;
  g.launches = l0;
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return set_err(LSMGNN_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  g.graph = graph;
  CK(cudaGraphInstantiate(&g.graph_exec, g.graph, 0));
  g.graph_out_host = out_host;
  return 0;
}

int lsmgnn_graph_replay(void* stream) {
  if (!g.graph_exec) return set_err(LSMGNN_ESTATE, "no captured graph");
  if (g.feed_next != g.t_next + (int64_t)g.W + 1) return set_err(LSMGNN_ESTATE, "window/iteration out of step");
  if (int rc = check_sticky()) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (g.pvp_pending) {
    CK(cudaStreamWaitEvent(st, g.ev_pvp, 0));
    g.pvp_pending = false;
  }
  if (g.feed_since_gather) {
    if (int rc = wait_feed(st)) return rc;
    g.feed_since_gather = false;
  }
  if (int rc = wait_gather_end(g.t_next - 1, st)) return rc;  // the replay's feed follows gather(t-1)
  CK(cudaGraphLaunch(g.graph_exec, st));
  if (int rc = note_gather_end(g.t_next, st)) return rc;
  g.gather_st = st;
  if (int rc = feed_end(st)) return rc;  // the replay fed t+1+W itself
  g.launches += g.graph_launches;
  g.t_next += 1;
  g.feed_next += 1;
  if (g.C)
    if (int rc = launch_pvp(st)) return rc;
  g.last_stream = st;
  return 0;
}

int lsmgnn_debug_state(int32_t what, void* out_host, int64_t count) {
  if (!g.inited) return set_err(LSMGNN_ESTATE, "not initialised");
  const void* src = nullptr;
  int64_t n = 0;
  switch (what) {
    case 0: src = g.tags; n = (int64_t)g.L; break;
    case 1: src = g.last_use; n = (int64_t)g.L; break;
    case 2: src = g.qlen; n = g.C ? (int64_t)g.W : 0; break;
    case 3: src = g.qnode; n = (int64_t)(g.W * g.C); break;
    default: return set_err(LSMGNN_EINVAL, "bad debug_state selector %d", what);
  }
  if (!out_host || count < n) return set_err(LSMGNN_EINVAL, "debug_state buffer holds %lld < %lld", (long long)count,
                                             (long long)n);
  CK(cudaDeviceSynchronize());
  if (n) CK(cudaMemcpy(out_host, src, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return 0;
}

int lsmgnn_profile(int32_t enable) {
  g.prof = enable != 0;
  return 0;
}

int lsmgnn_profile_read(double* ms, int64_t* cnt) {
  CK(cudaDeviceSynchronize());
  if (ms)
    for (int i = 0; i < LSMGNN_NPHASES; ++i) ms[i] = 0;
  if (cnt)
    for (int i = 0; i < LSMGNN_NPHASES; ++i) cnt[i] = 0;
  for (auto& sp : g.spans) {
    float x = 0;
    CK(cudaEventElapsedTime(&x, sp.a, sp.b));
    if (ms) ms[sp.phase] += x;
    if (cnt) cnt[sp.phase] += 1;
    g.ev_pool.push_back(sp.a);
    g.ev_pool.push_back(sp.b);
  }
  g.spans.clear();
  return 0;
}

int lsmgnn_disconnect(void) {
  if (!g.inited) return 0;
  CK(cudaDeviceSynchronize());
  for (int h = 0; h < kMaxG; ++h) {
    if (g.peer_arena[h] && g.peer_arena[h] != g.arena) {
      cudaIpcCloseMemHandle(g.peer_arena[h]);
      g.peer_arena[h] = nullptr;
    }
  }
  g.connected = g.world == 1;
  return 0;
}

int lsmgnn_finalize(void) {
  if (!g.inited) return 0;
  free_all();
  return 0;
}

}  // extern "C"

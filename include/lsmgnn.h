/* include/lsmgnn.h — C-ABI of the B200-native LSM-GNN feature-gather hot path.
 *
 * Method: LSM-GNN (arXiv 2407.15264), PAPER.md (= /root/reference/PAPER.md, cited
 * "P:n" = line n). The library gathers the feature rows of sampled nodes through
 * per-GPU software caches that a home-GPU directory turns into one box-wide shared
 * cache (§4.1 "Communication Layer"), with the hybrid eviction policy
 * (§4.2), a victim buffer in pinned host memory and its Preemptive
 * Victim-buffer Prefetcher (§4.3), and a host-resident backing table that
 * stands in for the SSD tier. DESIGN.md states every reading taken where the
 * paper is silent (R1..R27) and the data layout.
 *
 * Process model: one process per GPU ("DDP leverages multi-processing");
 * rank r of G is the home of every node v with v mod G == r (R1).
 * All calls are made from the thread that owns the rank's CUDA device.
 *
 * Conventions (all entry points):
 *   - return 0 on success or a negative LSMGNN_E* code; lsmgnn_last_error() gives
 *     a one-line message. No C++ exception crosses the ABI.
 *   - pointers documented "device" must be CUDA device (or managed) addresses of the
 *     calling rank's device; "host" pointers are ordinary (or pinned) host memory.
 *   - stream arguments are cudaStream_t values passed as void* (0 = legacy default).
 *   - the library owns every buffer it allocates (cache, window mask, staging,
 *     inboxes on the device; victim queues in pinned host memory). It references but
 *     does not own the backing table registered with lsmgnn_attach_storage.
 *   - errors detected on the device (a node ID >= num_nodes) set a sticky flag; the
 *     next call (or lsmgnn_stats) returns LSMGNN_ERANGE and the out rows of those
 *     IDs are zero-filled.
 *
 * Environment (read at init / connect / attach; defaults are the measured best):
 *   LSMGNN_NO_PDL=1           plain launches instead of programmatic dependent launch on the
 *                             single-home step chain and the sampler
 *   LSMGNN_SPLIT_PULL=0|1     G > 1 pull order: 1 = rows in place copied during the fill
 *                             (default on distinct GPUs), 0 = both phases after "served"
 *                             (default when a peer shares this rank's GPU)
 *   LSMGNN_NO_BATCH_MEMOP=1   one stream memory operation per flag instead of batched
 *   LSMGNN_STORAGE_BUFFERED=1 file tier through the page cache instead of O_DIRECT
 *   LSMGNN_IO_THREADS=n       file-tier pread workers per batch (default 64)
 *   LSMGNN_GEOMETRY=small     one CTA per SM for every grid (launch-geometry tests)
 *   LSMGNN_SERVE_CPS=c, LSMGNN_SERVE_ST=s  serve/pull geometry: c CTAs per SM, s TMA row stages
 *                             per warp (s = 0: 16-B vector copies instead of TMA bulk copies)
 *   LSMGNN_SERVE_TAIL=k, LSMGNN_SERVE_TAIL_ROUNDS=r  delivery chunks of 32 requests, k once
 *                             fewer than r rounds of chunks remain (guided; defaults 4, 2)
 *   LSMGNN_SERVE_AHEAD=1      keep one delivery chunk in reserve before the tail (A/B; slower)
 *   LSMGNN_FEED_EARLY=0       the window feed waits for the gather before it (default: it
 *                             starts alongside k_serve and waits for it at its end)
 *   LSMGNN_G1_PULL=1          G = 1 profiling aid: the G > 1 serve path (k_fill, k_pull phases,
 *                             k_end) instead of the fused k_serve; results are identical
 *   LSMGNN_DEDUP_EARLY=0      consecutive direct G = 1 gathers do not overlap (default: the next
 *                             gather's k_dedup / k_set run while the previous k_serve delivers,
 *                             without PVP, file tier or periodic scan; stream order unchanged)
 *   LSMGNN_EARLY_DEDUP_PER_SM=c, LSMGNN_EARLY_SET_PER_SM=c  CTAs per SM of an overlapped
 *                             k_dedup / k_set (defaults 2, 2)
 *   LSMGNN_SERVE_STATIC_FIRST=0  every delivery chunk from the counter (default: a warp's first
 *                             chunk is static in hit-dominated batches)
 *   LSMGNN_META_EVICT_LAST=0|1, LSMGNN_MASK_EVICT_LAST=0|1  L2 evict_last policy on k_dedup's
 *                             metadata accesses / on the reuse-bitmask updates (default: on
 *                             when they fit half the L2)
 *   LSMGNN_L2_EVICT_FIRST=1|2 L2 evict_first policy on the TMA ring row copies (1: loads and
 *                             stores, 2: stores; default off — measured slower)
 *   LSMGNN_HOST_TMA=1         pinned host `out`: deliver through the TMA rings too (bulk stores to
 *                             the host mapping; A/B: e2e unchanged, 40.4-40.6 vs 40.2-40.4 GB/s)
 * Every switch changes timing only: results are bit-identical (tests/test_gpu_overlap.py,
 * test_serve_geometry).
 */
#ifndef LSMGNN_H
#define LSMGNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSMGNN_ABI_VERSION 1

/* ---- return codes */
#define LSMGNN_OK 0
#define LSMGNN_EINVAL (-1)  /* bad argument, alignment (R % 16 != 0) or n > max_batch_ids */
#define LSMGNN_ERANGE (-2)  /* a node ID >= num_nodes (sticky, device-detected)             */
#define LSMGNN_ENOMEM (-3)  /* device or pinned-host allocation failed                      */
#define LSMGNN_ECUDA (-4)   /* a CUDA runtime/driver call failed                            */
#define LSMGNN_ESTATE (-5)  /* call order (not initialised, iterations out of order, ...)   */
#define LSMGNN_ECOMM (-6)   /* peer mapping / exchange failure                              */
#define LSMGNN_EIO (-7)     /* storage file open/read failure (file tier)                    */

typedef enum { LSMGNN_F32 = 0, LSMGNN_F16 = 1, LSMGNN_BF16 = 2 } lsmgnn_dtype;

/* Replacement policy. HYBRID is the paper's; STATIC and DYNAMIC are the
 * single-information ablations of P:645; RR is the M-GIDS baseline policy;
 * LRU is the north-star comparison policy. */
typedef enum {
  LSMGNN_HYBRID = 0,
  LSMGNN_STATIC = 1,
  LSMGNN_LRU = 2,
  LSMGNN_RR = 3,
  LSMGNN_DYNAMIC = 4
} lsmgnn_policy;

/* Options (optional; call lsmgnn_set_options before lsmgnn_init, defaults otherwise).
 *   policy          default HYBRID
 *   pvp             1 = victim buffer + PVP on; default 0
 *   window          W, iterations of look-ahead (W = 256 in P:607); default 256
 *   threshold       T; 0 => max(1, W/8) ("by default ... 1/8 of the window")
 *   update_period   P (the paper uses 4); 0 or 1 = exact information every
 *                   iteration; P > 1 = a window scan of every resident line every P-th
 *                   iteration, lines inserted since (or stale) are Fresh (R6, R7); default 1
 *   reinsert_victims 1 = a victim-buffer hit is re-inserted into the cache (R15); default 1
 *   max_batch_ids   capacity: the largest n any rank passes to gather/prefetch; default 1<<20 */
typedef struct {
  int32_t version; /* LSMGNN_ABI_VERSION */
  lsmgnn_policy policy;
  int32_t pvp;
  int32_t window;
  int32_t threshold;
  int32_t update_period;
  int32_t reinsert_victims;
  int64_t max_batch_ids;
} lsmgnn_options;

/* Per-home counters, one record per gather iteration (scope 0) or summed (scope 1).
 * Every count except `requests`/`peer_requests` is over UNIQUE nodes of the batch at
 * this home (R11). hits + victim_hits + storage_reads == unique (I2).
 *   evict_by_class[c]: c = 0 NoReuse, 1 Far (d > T), 2 Fresh, 3 Near (d <= T)
 *   victim_admitted/_dropped: eviction candidates with a next reuse (pvp = 1) that did /
 *     did not find room in victim queue reuse mod W
 *   evicted_no_reuse: evictions that were not victim candidates (discarded)
 *   pvp_prefetched: rows the PVP staged for this iteration; pvp_unused: staged rows this
 *     iteration did not request
 *   bytes_*: the per-tier algorithmic bytes (R = row bytes): out = requests*R,
 *     nvlink = peer_requests*R, h2d_storage = storage_reads*R, h2d_pvp = pvp_prefetched*R,
 *     d2h_victim = victim_admitted*R. */
typedef struct {
  uint64_t iter, requests, peer_requests, unique, hits, victim_hits, storage_reads, inserted,
      bypassed, evictions, evict_by_class[4], victim_admitted, victim_dropped, evicted_no_reuse,
      pvp_prefetched, pvp_unused;
  uint64_t bytes_out, bytes_nvlink, bytes_h2d_storage, bytes_h2d_pvp, bytes_d2h_victim;
} lsmgnn_stats_t;

/* Bind this process to (rank, world, device) before lsmgnn_init. The binding takes
 * them from its torch.distributed process group. Default (0, 1, current device). */
int lsmgnn_bind(int32_t rank, int32_t world, int32_t device);

int lsmgnn_set_options(const lsmgnn_options* opt);

/* Allocate this rank's home: a `ways`-way set-associative cache of lines_per_gpu rows
 * ("32-way set associative GPU software cache"; S = lines_per_gpu / ways sets,
 * set(v) = floor(v / G) mod S, R2), the window reuse mask, staging areas and, when
 * pvp = 1, W victim queues of floor(victim_lines / W) rows in pinned host memory
 * ("data ... victim buffers", "16K cache-lines" each; R13).
 *   num_nodes      N; node IDs are 0 .. N-1; N < 2^32 - 16 and ceil(N / G) < 2^31
 *   feat_dim, dtype  row bytes R = feat_dim * sizeof(dtype); R % 16 must be 0
 *   lines_per_gpu  L (> 0, multiple of ways), ways A in 1..32
 *   victim_lines   V (ignored when pvp = 0)
 *   static_scores  host u8[num_nodes], higher = hotter (one byte P:322 draft);
 *                  copied (caller may free after the call). NULL => all zero.
 * Collective in the sense that every rank must call it with identical arguments. */
int lsmgnn_init(int64_t num_nodes, int32_t feat_dim, lsmgnn_dtype dtype, int64_t lines_per_gpu,
                int32_t ways, int64_t victim_lines, const uint8_t* static_scores);

/* Register this home's partition of the backing "storage" table: host memory holding
 * the rows of nodes v = rank, rank+G, rank+2G, ... in that order (row k = node
 * rank + k*G), ceil((N - rank)/G) rows of R bytes. The library page-locks it with
 * cudaHostRegister unless it is already pinned, and reads it with zero-copy loads from
 * its fill kernel (features "directly fetched by GPU threads").
 *
 * File tier (NEXT N2, "storage"): host_rows_for_my_home = NULL and
 * nvme_path = a file holding the same rows in the same order (row k at byte offset k*R;
 * at least ceil((N - rank)/G) * R bytes, else LSMGNN_EINVAL). Opened read-only with
 * O_DIRECT when R is a multiple of 512 (the page cache is bypassed: every storage read is
 * a device read), buffered otherwise; LSMGNN_STORAGE_BUFFERED=1 forces buffered. Each
 * gather then reads the rows its fills need (known once replacement has run) with
 * parallel pread into a pinned bounce buffer that the fill kernel reads over PCIe: the device
 * publishes the fill list to pinned host memory, the fill kernel is launched at once and waits
 * per chunk of 64 entries for a host-written ready flag, and the calling thread reads the rows
 * chunk by chunk, releasing each as it lands — reads and fills overlap and `stream` is never
 * synchronised, but lsmgnn_gather returns only after this batch's reads are done (the host
 * waits for the device to publish the list). Graph capture is refused in this mode. Open/read failures return LSMGNN_EIO (a read failure is sticky:
 * the cache already recorded the rows). Exactly one of the two
 * arguments must be non-NULL. */
int lsmgnn_attach_storage(const void* host_rows_for_my_home, const char* nvme_path);

/* G > 1 bootstrap. lsmgnn_export_handle writes this rank's shareable handle blob
 * (cudaIpcMemHandle of its shared arena + layout) into buf (cap >= lsmgnn_handle_bytes()).
 * The binding all-gathers the blobs over the torch process group and passes the
 * concatenation (world * lsmgnn_handle_bytes() bytes, rank order) to lsmgnn_connect,
 * which opens every peer mapping. The blob also carries the GPU's UUID: when a peer runs on
 * this rank's own GPU (a test setup), the two pull phases of lsmgnn_gather both run after the
 * homes' fills instead of overlapping them (LSMGNN_SPLIT_PULL=0/1 overrides).
 * Not needed when world == 1. */
size_t lsmgnn_handle_bytes(void);
int lsmgnn_export_handle(void* buf, size_t cap);
/* lsmgnn_connect validates the blobs before mapping anything: blob r must carry rank r and
 * world == this rank's world, and its layout signature (every arena offset and size, derived
 * from the lsmgnn_init arguments and the options) must equal this rank's; otherwise nothing
 * is mapped and it returns LSMGNN_ECOMM naming the first offending peer. */
int lsmgnn_connect(const void* peer_handles, int32_t world);

/* Host-only bootstrap logic (no GPU, no CUDA call, usable before / without lsmgnn_init):
 * lsmgnn_plan_handle writes into buf (cap >= lsmgnn_handle_bytes()) the handle rank `rank` of
 * `world` WOULD export for these lsmgnn_init arguments and options (opt NULL = defaults),
 * without the IPC handle and GPU UUID; it returns the same LSMGNN_EINVAL lsmgnn_init would for
 * a bad argument. lsmgnn_check_handles runs lsmgnn_connect's validation of `world`
 * concatenated blobs against the blob `mine`: 0, or LSMGNN_ECOMM (wrong rank order, world
 * mismatch, layout mismatch). The binding's gloo tests drive both across processes. */
int lsmgnn_plan_handle(const lsmgnn_options* opt, int64_t num_nodes, int32_t feat_dim, lsmgnn_dtype dtype,
                       int64_t lines_per_gpu, int32_t ways, int64_t victim_lines, int32_t rank, int32_t world,
                       void* buf, size_t cap);
int lsmgnn_check_handles(const void* handles, int32_t world, const void* mine);

/* G > 1 teardown, step 1: synchronise this rank's device and close its mappings of the peers'
 * arenas. The binding calls it on every rank, then meets the others at a barrier, then calls
 * lsmgnn_finalize (step 2: free this rank's arena) — so no arena is freed while a peer still
 * has it mapped. Idempotent; a no-op before init. */
int lsmgnn_disconnect(void);

/* gather(t): collective, lockstep — every rank calls it once per iteration t.
 * Stream-ordered on `stream`: node_ids (device int64[n]) and out (device, n*R bytes,
 * row-major, tightly packed) are caller-owned and must stay valid until the stream
 * reaches the end of this call. Result: out[i] = table[node_ids[i]] (R bytes), routed
 * through the shared cache and the hit / victim-buffer / storage tiers.
 * n may be 0. Asynchronous: no host synchronisation in steady state. */
int lsmgnn_gather(const int64_t* node_ids, int64_t n, void* out, void* stream);

/* Same as lsmgnn_gather but node_ids and out are HOST pointers (pinned or pageable);
 * the host->device copy of the IDs and the device->host copy of the rows are done
 * on `stream` inside the call (used for the end-to-end measurement). Synchronous. */
int lsmgnn_gather_host(const int64_t* host_ids, int64_t n, void* host_out, void* stream);

/* prefetch: collective. Feeds this rank's future batches to the window buffer
 * (P:249): batch b = ids[offsets[b] .. offsets[b+1]) (device int64 arrays;
 * offsets has num_batches + 1 entries, offsets[0] == 0 and the offsets array is a
 * HOST pointer) for iterations first_iter .. first_iter + num_batches - 1.
 *  - The bootstrap call (before the first gather) feeds iterations 1 .. W.
 *  - Each later call, after gather(t), feeds the single batch t + 1 + W (an empty
 *    batch past the end of the trace) and launches the PVP copy of victim queue
 *    (t+1) mod W into home staging on a side stream (R17); gather(t+1)
 *    waits for it with an event.
 *  - `stream` may differ from the gather stream: the library orders the two with events
 *    (the feed of t+1+W waits only for gather(t-1), the last gather that reads its mask
 *    bit; gather(t+1) waits for the feed; the PVP copy waits for gather(t)), so a feed on
 *    its own stream overlaps gather(t). The ids must be ready on `stream`. */
int lsmgnn_prefetch(const int64_t* ids, const int64_t* offsets, int32_t num_batches,
                    int64_t first_iter, void* stream);

/* ---- NEXT N3: the window producer on the GPU (the step before the path).
 * GraphSAGE multi-hop neighbour sampling (§2.1; fanout P:603) over a CSR
 * pinned in host memory and read by GPU threads with zero-copy UVA loads. The list
 * produced is exactly DESIGN.md §3's definition (oracle/lsm_sampler.c): per frontier position
 * p, layer l, draw j: all neighbours if deg <= f, else f draws at CSR offset
 * floor(U01(h(seed, t, r, l, p, j)) * deg); the next frontier is the first-occurrence unique of
 * the layer's draws; the result is the first-occurrence unique of seeds ++ all draws.
 *
 * lsmgnn_sampler_attach: indptr host int64[num_nodes+1], indices host int32[nnz] (CSR, page-
 *   locked here unless already pinned; referenced, not owned). Independent of lsmgnn_init.
 * lsmgnn_sample: seeds device int64[nseeds]; fanout host int32[nlayers]; out device
 *   int64[cap] with cap >= nseeds * (1 + f0 + f0 f1 + ...) (the bound); the list length is
 *   written to count_dev (device int64) — nothing synchronises. Stream-ordered on `stream`.
 * lsmgnn_prefetch_dev: window feed of ONE batch (device int64 ids, device int64 count) for
 *   iteration first_iter — lsmgnn_prefetch semantics (any G: with G > 1 every rank calls it
 *   for the same first_iter, its own batch routed to the homes like lsmgnn_prefetch's)
 *   without reading the count on the host; issue the PVP copy with
 *   lsmgnn_prefetch(NULL, NULL, 0, 0, stream). */
int lsmgnn_sampler_attach(const int64_t* indptr, const int32_t* indices, int64_t num_nodes, int64_t nnz);
int lsmgnn_sample(const int64_t* seeds, int64_t nseeds, const int32_t* fanout, int32_t nlayers, uint64_t seed,
                  int64_t t, int32_t r, int64_t* out, int64_t cap, int64_t* count_dev, void* stream);
int lsmgnn_prefetch_dev(const int64_t* ids, const int64_t* count_dev, int64_t first_iter, void* stream);
/* Where lsmgnn_sample reads the CSR: in_hbm = 0 (default) — the pinned host copy over PCIe
 * (UVA, the paper's placement P:251); 1 — a copy the library makes in HBM (B200's 180 GB
 * holds a 100M-node CSR); same lists either way. */
int lsmgnn_sampler_place(int32_t in_hbm);

/* ---- CUDA-graph step (G = 1): one captured launch per iteration.
 * lsmgnn_graph_capture records ONE step — gather(t) of batch ids_ring[t mod ring_len]
 * (length n_ring[t mod ring_len]) into `out`, then the window feed of batch t+1+W from the
 * same ring — as a CUDA graph whose kernels take every per-iteration value from the device
 * (no host parameter changes between replays). lsmgnn_graph_replay(stream) launches it for
 * the next iteration, plus the PVP side-stream copy when pvp = 1.
 *   ids_ring: device array of ring_len device pointers (int64 IDs); n_ring: device
 *   int64[ring_len]; ring_len >= W + 2; out: device or pinned host, >= max_batch_ids * R
 *   bytes. Capture requires the window fed through t+W (the state after any gather/prefetch
 *   pair). Replays advance the same counters as lsmgnn_gather + lsmgnn_prefetch, so the two
 *   styles may be mixed. Returns EINVAL for G > 1. */
int lsmgnn_graph_capture(const int64_t* const* ids_ring, const int64_t* n_ring, int32_t ring_len, void* out,
                         void* stream);
int lsmgnn_graph_replay(void* stream);

/* Counters of this home: scope 0 = the last completed gather, 1 = cumulative.
 * Synchronises with the last stream used. */
int lsmgnn_stats(lsmgnn_stats_t* out_host, int32_t scope);

/* Per-iteration records for iterations [first, first+count) (kept on the device in a
 * ring; the last 4094 iterations are available). Synchronous. */
int lsmgnn_stats_history(lsmgnn_stats_t* out_host, int64_t first, int64_t count);

/* Debug/inspection (tests): copy a piece of this home's cache state to host memory after
 * synchronising. what = 0: tags u32[lines_per_gpu] (node ID per line, set-major, way-minor;
 * 0xFFFFFFFF = empty); 1: last use u32[lines_per_gpu]; 2: victim-queue lengths u32[W];
 * 3: victim-queue nodes u32[W * C] (queue k at [k*C, k*C + len_k)). `count` = elements the
 * caller's buffer holds; returns EINVAL if it is smaller than the piece. */
int lsmgnn_debug_state(int32_t what, void* out_host, int64_t count);

/* Number of kernels the library has launched since init (launch accounting). */
int64_t lsmgnn_kernel_launches(void);

/* Phase timing with CUDA events recorded on the stream each phase runs on (the user
 * stream, or the PVP side stream). Phases (LSMGNN_PHASE_*): 0 route+exchange, 1 dedup
 * (dedup, scan, bucket), 2 probe+replace (k_set), 3 victim admission, 4 fill, 5 serve+pull,
 * 6 window feed (prefetch mask update), 7 PVP copy (side stream). enable=1 starts
 * recording; lsmgnn_profile_read synchronises, writes the summed milliseconds per phase
 * and the number of timed launches per phase (either pointer may be NULL) and resets. */
#define LSMGNN_NPHASES 8
int lsmgnn_profile(int32_t enable);
int lsmgnn_profile_read(double* ms_per_phase, int64_t* count_per_phase);

int lsmgnn_finalize(void);
const char* lsmgnn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LSMGNN_H */

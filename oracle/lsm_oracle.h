/* oracle/lsm_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * A plain, slow, single-threaded C simulation of the LSM-GNN feature-gather hot
 * path (arXiv 2407.15264), written from PAPER.md and the batch-synchronous
 * readings listed in DESIGN.md §"Readings". Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. It shares no
 * code, header or constant with the CUDA path (paper_2407_15264_b200/, include/).
 */
#ifndef LSM_ORACLE_H
#define LSM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Replacement policies (PAPER.md P:360-371 hybrid; P:645 static/dynamic; P:612 RR; LRU north star). */
enum { ORC_HYBRID = 0, ORC_STATIC = 1, ORC_LRU = 2, ORC_RR = 3, ORC_DYNAMIC = 4 };
/* Dynamic-information classes. Indexes evict_by_class[]. */
enum { ORC_NOREUSE = 0, ORC_FAR = 1, ORC_FRESH = 2, ORC_NEAR = 3 };
/* Probe outcome of one unique request. */
enum { ORC_STORAGE = 0, ORC_HIT = 1, ORC_VHIT = 2 };

typedef struct {
    int32_t G;            /* homes = ranks */
    int64_t N;            /* nodes */
    int32_t R;            /* row bytes */
    int64_t L;            /* lines per home */
    int32_t A;            /* ways; S = L / A sets */
    int32_t policy;       /* ORC_* */
    int32_t pvp;          /* 0/1 */
    int32_t W;            /* window (iterations looked ahead) */
    int32_t T;            /* threshold; 0 => max(1, W/8) */
    int32_t reinsert;     /* 1: victim-buffer hits are re-inserted (R15) */
    int64_t V;            /* victim lines per home; C = V / W lines per queue */
    int32_t P;            /* dynamic-information update period; 0 or 1 = every iteration */
} orc_config;

/* Per (iteration, home) counters, field order identical to lsmgnn_stats_t in
 * SURVEY.md §8(b) (the comparison is a field-by-field integer equality). */
typedef struct {
    uint64_t iter, requests, peer_requests, unique, hits, victim_hits, storage_reads,
             inserted, bypassed, evictions, evict_by_class[4], victim_admitted, victim_dropped,
             evicted_no_reuse, pvp_prefetched, pvp_unused;
    uint64_t bytes_out, bytes_nvlink, bytes_h2d_storage, bytes_h2d_pvp, bytes_d2h_victim;
} orc_counts;

typedef struct orc orc_t;

orc_t* orc_create(const orc_config* cfg, const uint8_t* scores /* u8[N] */);
void   orc_destroy(orc_t* o);
const char* orc_error(orc_t* o);

/* Window feed: B_k = union over ranks of ids[offs[r]..offs[r+1]).
 * Iterations must be fed in increasing order. */
int orc_feed_window(orc_t* o, int64_t k, const int64_t* ids, const int64_t* offs);

/* gather(t) for all homes (PAPER.md P:294-313 communication layer; P:343-371 hybrid
 * eviction; P:402-414 eviction with PVP). ids/offs as above (batch_r(t)).
 * table: u8[N*R] or NULL; out: u8[total*R] (concatenated per rank) or NULL.
 * counts: orc_counts[G] written for this iteration. */
int orc_gather(orc_t* o, int64_t t, const int64_t* ids, const int64_t* offs,
               const uint8_t* table, uint8_t* out, orc_counts* counts);

/* PVP copy after gather(t): staging_g := Q_g[(t+1) mod W]. */
int orc_pvp_prefetch(orc_t* o, int64_t t);

/* ---- state inspection for invariant tests ---- */
int64_t orc_sets(orc_t* o);
/* tags of home g: int64[S*A], -1 = invalid */
int orc_dump_tags(orc_t* o, int32_t g, int64_t* tags, int64_t* last_use);
/* queue k of home g: returns its length; writes up to cap (node, reuse) pairs */
int64_t orc_dump_queue(orc_t* o, int32_t g, int32_t k, int64_t* nodes, int64_t* reuse, int64_t cap);
/* staging of home g: returns its length; writes up to cap nodes */
int64_t orc_dump_staging(orc_t* o, int32_t g, int64_t* nodes, int64_t cap);
/* next_t(v) as the oracle sees it now (-1 = NONE) */
int64_t orc_next_use(orc_t* o, int64_t v, int64_t t);
/* event log of the last gather, one row per line/miss considered in a touched set:
 * [home, set, kind, node, key0, key1, key2], kind 0 = evicted line, 1 = surviving
 * unprotected line (valid, not hit, not evicted), 2 = bypassed miss, 3 = inserted miss. */
int64_t orc_dump_events(orc_t* o, int64_t* rows7, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif

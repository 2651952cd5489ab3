/* oracle/lsm_oracle.c — CPU ORACLE for the LSM-GNN feature-gather hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2407_15264_b200/) never links, imports or executes it; the two share no
 * code, header, table or constant generator.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   Part 1, bytes:  out_r[i] = table[batch_r(t)[i]] — a plain gather.
 *   Part 2, counts: a step-by-step, single-threaded simulation of the paper's
 *     shared software cache, in the batch-synchronous reading DESIGN.md states:
 *       - communication layer: every node has one home GPU, home(v) = v mod G
 *         ("straightforward striding function"); each home serves
 *         all requests for its nodes;
 *       - a set-associative software cache per home, set(v) = floor(v/G) mod S;
 *       - dynamic information = next reuse iteration from the window buffer
 *         (draft P:330 "marks the iteration of the next reuse");
 *       - the hybrid eviction policy's four priority levels with the lowest
 *         static value first inside a level, the level swap with PVP
 *         (P:427-435);
 *       - eviction into per-reuse-iteration victim queues with a capacity, counter
 *         = slot (worked example P:410);
 *       - the Preemptive Victim-buffer Prefetcher copying queue t+1 back after
 *         gather(t).
 *   Readings where the paper is silent/ambiguous are R1..R25 in DESIGN.md
 *   (mirroring SURVEY.md §8(c) L1..L25); each is cited where it is used.
 *
 * Parity status per function: see the header comment of each function and
 * DESIGN.md §"Oracle pins". Every function below is pinned by at least one
 * -m "not gpu" test in tests/test_oracle_*.py.
 *
 * Deliberately slow and plain: linear scans over ways, qsort, per-node FIFO
 * arrays. No blocking, fusion or reordering beyond the definitions.
 */
#include "lsm_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NONE (-1)

typedef struct { int64_t k0, k1, k2; } key3;   /* lexicographic; smallest is evicted first */

typedef struct { int64_t x, reuse; } qent;

typedef struct {
    int64_t* tag;       /* [S*A], NONE = invalid */
    int64_t* last_use;  /* [S*A] */
    int64_t* info;      /* [S*A] dynamic information of the line: next reuse iteration recorded
                           by the last window scan, NONE (no reuse found) or FRESH (inserted
                           after the scan) — the three states of draft P:333 */
    int32_t* rr;        /* [S] round-robin cursor */
    qent**   q;         /* [W] victim queues */
    int64_t* qlen;      /* [W] */
    int64_t* staging;   /* prefetching buffer contents, sorted */
    int64_t  nstaging;
    uint64_t pending_prefetched;   /* rows staged for the next gather */
} home_t;

typedef struct { int64_t* it; int64_t head, len, cap; } fifo_t;

struct orc {
    orc_config c;
    int64_t S, C;
    uint8_t* score;
    home_t* home;
    fifo_t* occ;            /* occ[v]: window iterations at which v appears, ascending */
    int64_t** wlist;        /* fed window lists B_k (sorted distinct), indexed k mod (W+1) */
    int64_t*  wlen;
    int64_t*  witer;        /* which k is stored in that slot (-1 = none) */
    int64_t last_fed;
    int64_t last_gather;
    int64_t* ev; int64_t nev, evcap;  /* event log */
    char err[256];
};

/* ------------------------------------------------------------------ helpers */
static int fail(orc_t* o, int code, const char* msg) {
    snprintf(o->err, sizeof o->err, "%s", msg);
    return code;
}
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}
static int key_less(key3 a, key3 b) {
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    return a.k2 < b.k2;
}
/* sorted distinct copy of a[0..n) */
static int64_t sort_unique(int64_t* a, int64_t n) {
    if (n == 0) return 0;
    qsort(a, (size_t)n, sizeof(int64_t), cmp_i64);
    int64_t m = 1;
    for (int64_t i = 1; i < n; ++i) if (a[i] != a[m - 1]) a[m++] = a[i];
    return m;
}
static int contains_sorted(const int64_t* a, int64_t n, int64_t v) {
    return bsearch(&v, a, (size_t)n, sizeof(int64_t), cmp_i64) != NULL;
}
static void log_event(orc_t* o, int64_t g, int64_t s, int64_t kind, int64_t v, key3 k) {
    if (o->nev == o->evcap) {
        o->evcap = o->evcap ? 2 * o->evcap : 1024;
        o->ev = realloc(o->ev, (size_t)o->evcap * 7 * sizeof(int64_t));
    }
    int64_t* r = o->ev + 7 * o->nev++;
    r[0] = g; r[1] = s; r[2] = kind; r[3] = v; r[4] = k.k0; r[5] = k.k1; r[6] = k.k2;
}

/* ------------------------------------------------------------------ directory
 * DESIGN.md R1: home(v) = v mod G ("straightforward striding function").
 * DESIGN.md R2: set(v) = floor(v / G) mod S inside the home. */
static int64_t home_of(const orc_t* o, int64_t v) { return v % o->c.G; }
static int64_t set_of(const orc_t* o, int64_t v) { return (v / o->c.G) % o->S; }

/* ------------------------------------------------------------------ dynamic information
 * next_t(v) = min{k : t < k <= t+W, v in B_k}, else NONE (R3, R5).
 * Kept as a FIFO of window iterations per node (appended when B_k is fed). */
static int64_t next_use(orc_t* o, int64_t v, int64_t t) {
    fifo_t* f = &o->occ[v];
    for (int64_t i = f->head; i < f->len; ++i) {
        int64_t k = f->it[i];
        if (k > t) return k <= t + o->c.W ? k : NONE;
    }
    return NONE;
}

#define FRESH (-2)

/* Is gather(t) a dynamic-information update iteration? The window scan runs every P
 * iterations ("updates the dynamic information for a configurable number of
 * iterations"; R6); P <= 1 scans before every gather. */
static int is_update(const orc_t* o, int64_t t) { return o->c.P <= 1 || t % o->c.P == 0; }

/* Class from a line's dynamic information at gather(t) (R4, R7):
 * FRESH (inserted after the last scan, draft P:333 "recently inserted") or a recorded
 * reuse that has already passed (stale) -> Fresh; NONE -> NoReuse; else d = info - t:
 * Near if d <= T, Far otherwise. */
static int cls_from_info(const orc_t* o, int64_t info, int64_t t) {
    if (info == NONE) return ORC_NOREUSE;
    if (info == FRESH || info <= t) return ORC_FRESH;
    return (info - t) <= o->c.T ? ORC_NEAR : ORC_FAR;
}

/* Information an incoming miss has when the batch is decided: exact at an update
 * iteration (the scan precedes aggregation), none yet otherwise (Fresh). */
static int64_t incoming_info(orc_t* o, int64_t v, int64_t t) {
    return is_update(o, t) ? next_use(o, v, t) : FRESH;
}

/* Priority level (rank) of a class: lowest evicted first.
 * pvp = 0: NoReuse 0, Far 1, Fresh 2, Near 3.
 * pvp = 1: the two lowest levels swapped — Far 0, NoReuse 1. */
static int64_t rank_of(const orc_t* o, int cls) {
    switch (cls) {
        case ORC_NOREUSE: return o->c.pvp ? 1 : 0;
        case ORC_FAR:     return o->c.pvp ? 0 : 1;
        case ORC_FRESH:   return 2;
        default:          return 3;
    }
}

/* Eviction key of a line holding x (last use lu, dynamic info `info`) at gather(t);
 * smallest goes first.
 *   HYBRID  (rank(class), score, x)      P:361 "lowest static priority value"; tie by node (R8)
 *   STATIC  (0, score, x)                P:645 static-only
 *   LRU     (0, last_use, x)             north-star baseline (R20)
 *   DYNAMIC NoReuse (0,0,x), Fresh (1,0,x), reuse d (2, W-d, x)   P:645 dynamic-only (R19)
 *   RR      (0, 0, x) — only used to order bypassed misses (R20) */
static key3 key_of(orc_t* o, int64_t x, int64_t lu, int64_t info, int64_t t) {
    key3 k = {0, 0, x};
    const int cls = cls_from_info(o, info, t);
    switch (o->c.policy) {
        case ORC_HYBRID: k.k0 = rank_of(o, cls); k.k1 = o->score[x]; break;
        case ORC_STATIC: k.k1 = o->score[x]; break;
        case ORC_LRU:    k.k1 = lu; break;
        case ORC_DYNAMIC:
            if (cls == ORC_NOREUSE) { k.k0 = 0; k.k1 = 0; }
            else if (cls == ORC_FRESH) { k.k0 = 1; k.k1 = 0; }
            else { k.k0 = 2; k.k1 = o->c.W - (info - t); }
            break;
        default: break;
    }
    return k;
}

/* ------------------------------------------------------------------ lifecycle */
orc_t* orc_create(const orc_config* cfg, const uint8_t* scores) {
    orc_t* o = calloc(1, sizeof *o);
    o->c = *cfg;
    if (o->c.T == 0) o->c.T = o->c.W / 8 > 1 ? o->c.W / 8 : 1;   /* W/8 by default */
    if (cfg->G < 1 || cfg->N < 1 || cfg->A < 1 || cfg->L < cfg->A || cfg->L % cfg->A || cfg->W < 1 ||
        cfg->policy < 0 || cfg->policy > 4 || cfg->R < 0) {
        snprintf(o->err, sizeof o->err, "bad config");
        return o;   /* caller checks orc_sets() > 0 */
    }
    o->S = cfg->L / cfg->A;
    o->C = cfg->V / cfg->W;                                         /* DESIGN.md R13 */
    o->score = malloc((size_t)cfg->N);
    memcpy(o->score, scores, (size_t)cfg->N);
    o->home = calloc((size_t)cfg->G, sizeof(home_t));
    for (int g = 0; g < cfg->G; ++g) {
        home_t* h = &o->home[g];
        h->tag = malloc((size_t)cfg->L * sizeof(int64_t));
        h->last_use = calloc((size_t)cfg->L, sizeof(int64_t));
        h->info = malloc((size_t)cfg->L * sizeof(int64_t));
        for (int64_t i = 0; i < cfg->L; ++i) h->info[i] = NONE;
        for (int64_t i = 0; i < cfg->L; ++i) h->tag[i] = NONE;
        h->rr = calloc((size_t)o->S, sizeof(int32_t));
        h->q = calloc((size_t)cfg->W, sizeof(qent*));
        h->qlen = calloc((size_t)cfg->W, sizeof(int64_t));
        for (int k = 0; k < cfg->W; ++k) h->q[k] = malloc((size_t)(o->C > 0 ? o->C : 1) * sizeof(qent));
        h->staging = NULL; h->nstaging = 0;
    }
    o->occ = calloc((size_t)cfg->N, sizeof(fifo_t));
    o->wlist = calloc((size_t)cfg->W + 1, sizeof(int64_t*));
    o->wlen = calloc((size_t)cfg->W + 1, sizeof(int64_t));
    o->witer = malloc(((size_t)cfg->W + 1) * sizeof(int64_t));
    for (int k = 0; k <= cfg->W; ++k) o->witer[k] = NONE;
    o->last_fed = NONE;
    o->last_gather = NONE;
    return o;
}

void orc_destroy(orc_t* o) {
    if (!o) return;
    if (o->home) for (int g = 0; g < o->c.G; ++g) {
        home_t* h = &o->home[g];
        free(h->tag); free(h->last_use); free(h->info); free(h->rr);
        for (int k = 0; k < o->c.W; ++k) free(h->q[k]);
        free(h->q); free(h->qlen); free(h->staging);
    }
    free(o->home);
    if (o->occ) for (int64_t v = 0; v < o->c.N; ++v) free(o->occ[v].it);
    free(o->occ);
    if (o->wlist) for (int k = 0; k <= o->c.W; ++k) free(o->wlist[k]);
    free(o->wlist); free(o->wlen); free(o->witer);
    free(o->score); free(o->ev);
    free(o);
}

const char* orc_error(orc_t* o) { return o->err; }
int64_t orc_sets(orc_t* o) { return o->S; }

/* ------------------------------------------------------------------ window feed
 * B_k = union over ranks of the sampled lists of iteration k.
 * The list stored in slot k mod (W+1) is dropped when gather(k) pops it. */
int orc_feed_window(orc_t* o, int64_t k, const int64_t* ids, const int64_t* offs) {
    if (k <= o->last_fed) return fail(o, -1, "window iterations must be fed in increasing order");
    int64_t n = offs[o->c.G] - offs[0];
    int64_t* b = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t v = ids[offs[0] + i];
        if (v < 0 || v >= o->c.N) { free(b); return fail(o, -2, "window node id out of range"); }
        b[i] = v;
    }
    n = sort_unique(b, n);
    int64_t slot = k % (o->c.W + 1);
    if (o->witer[slot] != NONE) {   /* an unconsumed older list: drop its FIFO entries */
        int64_t kk = o->witer[slot];
        for (int64_t i = 0; i < o->wlen[slot]; ++i) {
            fifo_t* f = &o->occ[o->wlist[slot][i]];
            if (f->head < f->len && f->it[f->head] == kk) f->head++;
        }
        free(o->wlist[slot]);
    }
    o->wlist[slot] = b; o->wlen[slot] = n; o->witer[slot] = k;
    for (int64_t i = 0; i < n; ++i) {
        fifo_t* f = &o->occ[b[i]];
        if (f->head > 0 && f->head == f->len) f->head = f->len = 0;   /* empty: rewind */
        if (f->len == f->cap) {
            f->cap = f->cap ? 2 * f->cap : 4;
            f->it = realloc(f->it, (size_t)f->cap * sizeof(int64_t));
        }
        f->it[f->len++] = k;
    }
    o->last_fed = k;
    return 0;
}

/* Drop iteration t from the window once it is being gathered. */
static void pop_window(orc_t* o, int64_t t) {
    int64_t slot = t % (o->c.W + 1);
    if (o->witer[slot] != t) return;
    for (int64_t i = 0; i < o->wlen[slot]; ++i) {
        fifo_t* f = &o->occ[o->wlist[slot][i]];
        if (f->head < f->len && f->it[f->head] == t) f->head++;
    }
    free(o->wlist[slot]);
    o->wlist[slot] = NULL; o->wlen[slot] = 0; o->witer[slot] = NONE;
}

/* ------------------------------------------------------------------ one home, one batch */
typedef struct { int64_t v; key3 k; } vk;
static int cmp_vk(const void* a, const void* b) {
    const vk* x = a; const vk* y = b;
    return key_less(x->k, y->k) ? -1 : key_less(y->k, x->k) ? 1 : 0;
}
static int cmp_qent_x(const void* a, const void* b) {
    const qent* x = a; const qent* y = b;
    return x->x < y->x ? -1 : x->x > y->x;
}

/* gather(t) at home g ("each GPU independently performs the feature
 * aggregation process for the sampled nodes requested by all GPUs").
 * Steps follow SURVEY.md §8(c) / DESIGN.md "Oracle semantics" in order. */
static void gather_home(orc_t* o, int g, int64_t t, const int64_t* ids, const int64_t* offs, orc_counts* cnt) {
    home_t* h = &o->home[g];
    const int A = o->c.A;
    memset(cnt, 0, sizeof *cnt);
    cnt->iter = (uint64_t)t;

    /* window scan ("scans the sampled nodes in the window buffer to determine the
     * next reuse iteration for the cache-lines that currently reside in the cache before
     * the feature aggregation stage"), every P iterations */
    if (is_update(o, t))
        for (int64_t i = 0; i < o->c.L; ++i)
            h->info[i] = h->tag[i] == NONE ? NONE : next_use(o, h->tag[i], t);

    /* Req = [(r,i,v) : v = batch_r(t)[i], home(v) = g]  (P:296 split by hash) */
    int64_t total = offs[o->c.G] - offs[0];
    int64_t* U = malloc((size_t)(total > 0 ? total : 1) * sizeof(int64_t));
    int64_t nreq = 0;
    for (int r = 0; r < o->c.G; ++r)
        for (int64_t i = offs[r]; i < offs[r + 1]; ++i) {
            int64_t v = ids[i];
            if (home_of(o, v) != g) continue;
            U[nreq++] = v;
            cnt->requests++;
            if (r != g) cnt->peer_requests++;
        }
    /* U = sorted distinct requested nodes (R11: dedup at the home) */
    int64_t nu = sort_unique(U, nreq);
    cnt->unique = (uint64_t)nu;

    /* kind[v]: HIT if resident in set(v); VHIT if in the prefetching buffer; else STORAGE */
    int* kind = malloc((size_t)(nu > 0 ? nu : 1) * sizeof(int));
    for (int64_t j = 0; j < nu; ++j) {
        int64_t v = U[j], s = set_of(o, v);
        kind[j] = ORC_STORAGE;
        for (int w = 0; w < A; ++w) if (h->tag[s * A + w] == v) { kind[j] = ORC_HIT; break; }
        if (kind[j] == ORC_STORAGE && contains_sorted(h->staging, h->nstaging, v)) kind[j] = ORC_VHIT;
    }
    /* staged rows never requested are wasted; the prefetching buffer is emptied */
    for (int64_t j = 0; j < h->nstaging; ++j)
        if (!contains_sorted(U, nu, h->staging[j])) cnt->pvp_unused++;
    free(h->staging); h->staging = NULL; h->nstaging = 0;
    cnt->pvp_prefetched = h->pending_prefetched;
    h->pending_prefetched = 0;

    /* victim candidates of this batch: (x, next reuse) */
    qent* cand = malloc((size_t)(nu > 0 ? nu : 1) * sizeof(qent));
    int64_t ncand = 0;

    /* touched sets in ascending order: U sorted by (set, v) */
    int64_t* order = malloc((size_t)(nu > 0 ? nu : 1) * sizeof(int64_t));
    int64_t no = 0;
    /* bucket pass over sets: O(S + U), stable so each set's nodes stay ascending */
    {
        int64_t* cnts = calloc((size_t)o->S + 1, sizeof(int64_t));
        for (int64_t j = 0; j < nu; ++j) cnts[set_of(o, U[j]) + 1]++;
        for (int64_t s = 0; s < o->S; ++s) cnts[s + 1] += cnts[s];
        for (int64_t j = 0; j < nu; ++j) order[cnts[set_of(o, U[j])]++] = j;   /* stable: v ascending */
        free(cnts);
        no = nu;
    }

    vk* M = malloc((size_t)(nu > 0 ? nu : 1) * sizeof(vk));
    int* prot = malloc((size_t)A * sizeof(int));
    int* filled = malloc((size_t)A * sizeof(int));
    for (int64_t p = 0; p < no;) {
        int64_t s = set_of(o, U[order[p]]);
        int64_t q = p;
        while (q < no && set_of(o, U[order[q]]) == s) ++q;
        int64_t* tag = h->tag + s * A;
        int64_t* lu = h->last_use + s * A;
        int64_t* info = h->info + s * A;
        /* H = ways whose tag is requested: protected for the whole batch (R10) */
        for (int w = 0; w < A; ++w) { prot[w] = 0; filled[w] = 0; }
        int64_t nH = 0, nM = 0;
        for (int64_t j = p; j < q; ++j) {
            int64_t v = U[order[j]];
            int kd = kind[order[j]];
            if (kd == ORC_HIT) {
                for (int w = 0; w < A; ++w) if (tag[w] == v) { prot[w] = 1; lu[w] = t; nH++; }
            } else if (kd == ORC_STORAGE || o->c.reinsert) {
                /* M = misses to insert (R15: victim-buffer hits re-inserted unless reinsert=0) */
                M[nM].v = v;
                /* incoming key = key as if resident with last_use = t (R10) */
                M[nM].k = key_of(o, v, t, incoming_info(o, v, t), t);
                nM++;
            }
        }
        /* more misses than unprotected ways: bypass the most-evictable ones (R10) */
        int64_t avail = A - nH;
        int64_t nbyp = nM > avail ? nM - avail : 0;
        if (nbyp > 0) {
            qsort(M, (size_t)nM, sizeof(vk), cmp_vk);
            for (int64_t j = 0; j < nbyp; ++j) log_event(o, g, s, 2, M[j].v, M[j].k);
            cnt->bypassed += (uint64_t)nbyp;
        }
        /* remaining misses installed in ascending node order */
        int64_t nins = nM - nbyp;
        int64_t* ins = malloc((size_t)(nins > 0 ? nins : 1) * sizeof(int64_t));
        for (int64_t j = 0; j < nins; ++j) ins[j] = M[nbyp + j].v;
        qsort(ins, (size_t)nins, sizeof(int64_t), cmp_i64);
        for (int64_t j = 0; j < nins; ++j) {
            int64_t v = ins[j];
            int w = -1;
            for (int ww = 0; ww < A; ++ww) if (tag[ww] == NONE) { w = ww; break; }   /* lowest invalid way */
            if (w < 0 && o->c.policy == ORC_RR) {
                /* P:612 round-robin: first way from the cursor that is not protected/just filled */
                for (int d = 0; d < A; ++d) {
                    int ww = (h->rr[s] + d) % A;
                    if (!prot[ww] && !filled[ww]) { w = ww; break; }
                }
                h->rr[s] = (w + 1) % A;
            } else if (w < 0) {
                /* argmin key over valid, unprotected, not-yet-filled ways */
                key3 best = {0, 0, 0};
                for (int ww = 0; ww < A; ++ww) {
                    if (prot[ww] || filled[ww]) continue;
                    key3 k = key_of(o, tag[ww], lu[ww], info[ww], t);
                    if (w < 0 || key_less(k, best)) { w = ww; best = k; }
                }
            }
            if (tag[w] != NONE) {
                /* evict x: count by class; with PVP a line that has a next
                 * reuse iteration becomes a victim-buffer candidate, else it is discarded */
                int64_t x = tag[w];
                key3 kx = key_of(o, x, lu[w], info[w], t);
                log_event(o, g, s, 0, x, kx);
                cnt->evictions++;
                const int cx = cls_from_info(o, info[w], t);
                cnt->evict_by_class[cx]++;
                if (o->c.pvp && (cx == ORC_NEAR || cx == ORC_FAR)) {
                    cand[ncand].x = x; cand[ncand].reuse = info[w]; ncand++;
                } else {
                    cnt->evicted_no_reuse++;
                }
            }
            tag[w] = v; lu[w] = t; info[w] = FRESH; filled[w] = 1;
            cnt->inserted++;
            log_event(o, g, s, 3, v, key_of(o, v, t, incoming_info(o, v, t), t));
        }
        /* survivors for the class-minimality invariant (I6) */
        for (int w = 0; w < A; ++w)
            if (tag[w] != NONE && !prot[w] && !filled[w])
                log_event(o, g, s, 1, tag[w], key_of(o, tag[w], lu[w], info[w], t));
        free(ins);
        p = q;
    }
    for (int64_t j = 0; j < nu; ++j) {
        if (kind[j] == ORC_HIT) cnt->hits++;
        else if (kind[j] == ORC_VHIT) cnt->victim_hits++;
        else cnt->storage_reads++;
    }

    /* victim admission (R13, R14): per queue k = reuse mod W, candidates in
     * ascending node order take the free slots; slot = counter value before increment
     * (worked example P:410: reuse 4, counter 5 -> 5th position of the 4th buffer). */
    if (o->c.pvp) {
        qsort(cand, (size_t)ncand, sizeof(qent), cmp_qent_x);
        for (int64_t j = 0; j < ncand; ++j) {
            int64_t k = cand[j].reuse % o->c.W;
            if (h->qlen[k] < o->C) { h->q[k][h->qlen[k]++] = cand[j]; cnt->victim_admitted++; }
            else cnt->victim_dropped++;
        }
    }
    const uint64_t R = (uint64_t)o->c.R;
    cnt->bytes_out = cnt->requests * R;
    cnt->bytes_nvlink = cnt->peer_requests * R;
    cnt->bytes_h2d_storage = cnt->storage_reads * R;
    cnt->bytes_h2d_pvp = cnt->pvp_prefetched * R;
    cnt->bytes_d2h_victim = cnt->victim_admitted * R;
    free(U); free(kind); free(cand); free(order); free(M); free(prot); free(filled);
}

int orc_gather(orc_t* o, int64_t t, const int64_t* ids, const int64_t* offs,
               const uint8_t* table, uint8_t* out, orc_counts* counts) {
    if (o->S <= 0) return fail(o, -1, "not initialised");
    if (t <= o->last_gather) return fail(o, -1, "iterations must increase");
    int64_t total = offs[o->c.G] - offs[0];
    for (int64_t i = 0; i < total; ++i) {
        int64_t v = ids[offs[0] + i];
        if (v < 0 || v >= o->c.N) return fail(o, -2, "node id out of range");
    }
    /* iterations <= t leave the window */
    for (int64_t k = (o->last_gather == NONE ? 0 : o->last_gather + 1); k <= t; ++k) pop_window(o, k);
    o->nev = 0;
    for (int g = 0; g < o->c.G; ++g) gather_home(o, g, t, ids, offs, &counts[g]);
    /* Part 1: out_r[i] = table[batch_r(t)[i]] */
    if (table && out)
        for (int64_t i = 0; i < total; ++i)
            memcpy(out + i * (int64_t)o->c.R, table + ids[offs[0] + i] * (int64_t)o->c.R, (size_t)o->c.R);
    o->last_gather = t;
    return 0;
}

/* PVP: after gather(t), copy victim queue (t+1) mod W into the
 * prefetching buffer (R17); entries whose recorded reuse is not t+1 are dropped. */
int orc_pvp_prefetch(orc_t* o, int64_t t) {
    if (!o->c.pvp) return 0;
    int64_t k = (t + 1) % o->c.W;
    for (int g = 0; g < o->c.G; ++g) {
        home_t* h = &o->home[g];
        free(h->staging);
        h->staging = malloc((size_t)(h->qlen[k] > 0 ? h->qlen[k] : 1) * sizeof(int64_t));
        h->nstaging = 0;
        for (int64_t j = 0; j < h->qlen[k]; ++j)
            if (h->q[k][j].reuse == t + 1) h->staging[h->nstaging++] = h->q[k][j].x;
        h->nstaging = sort_unique(h->staging, h->nstaging);
        h->pending_prefetched = (uint64_t)h->nstaging;
        h->qlen[k] = 0;
    }
    return 0;
}

/* ------------------------------------------------------------------ inspection */
int orc_dump_tags(orc_t* o, int32_t g, int64_t* tags, int64_t* last_use) {
    memcpy(tags, o->home[g].tag, (size_t)o->c.L * sizeof(int64_t));
    if (last_use) memcpy(last_use, o->home[g].last_use, (size_t)o->c.L * sizeof(int64_t));
    return 0;
}
int64_t orc_dump_queue(orc_t* o, int32_t g, int32_t k, int64_t* nodes, int64_t* reuse, int64_t cap) {
    home_t* h = &o->home[g];
    for (int64_t j = 0; j < h->qlen[k] && j < cap; ++j) { nodes[j] = h->q[k][j].x; reuse[j] = h->q[k][j].reuse; }
    return h->qlen[k];
}
int64_t orc_dump_staging(orc_t* o, int32_t g, int64_t* nodes, int64_t cap) {
    home_t* h = &o->home[g];
    for (int64_t j = 0; j < h->nstaging && j < cap; ++j) nodes[j] = h->staging[j];
    return h->nstaging;
}
int64_t orc_next_use(orc_t* o, int64_t v, int64_t t) { return next_use(o, v, t); }
int64_t orc_dump_events(orc_t* o, int64_t* rows7, int64_t cap) {
    int64_t n = o->nev < cap ? o->nev : cap;
    memcpy(rows7, o->ev, (size_t)n * 7 * sizeof(int64_t));
    return o->nev;
}

/* synth/graphgen.c — the plcite power-law graph for large N, in C.
 *
 * Input generator only (no LSM-GNN arithmetic). Same recipe as synth.plcite(): node v has m
 * out-edges; edge k draws u = U01(h(seed_g, v, k)), popularity rank
 * rho = floor((u*((N+1)^(1-beta) - 1) + 1)^(1/(1-beta))) - 1, target pi[rho] (pi: a seeded
 * permutation passed in), self-loops redrawn with counter k + m*j; the CSR is symmetrised
 * with each node's neighbours ordered by (edge source, k). The numpy version is used up to
 * 10M nodes; this one makes 100M-node graphs (configs[3]) in seconds. libm pow() may differ
 * from numpy's in the last ulp, so the two are distinct instances of the same distribution.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* targets[v*m + k] for all edges (OpenMP over v) */
void plcite_targets(int64_t N, int32_t m, uint64_t seed_g, double beta, const int64_t* pi, int32_t* targets) {
    const double e = 1.0 - beta, top = pow((double)N + 1.0, e) - 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; ++v) {
        for (int32_t k = 0; k < m; ++k) {
            int64_t ctr = k, t;
            for (int64_t j = 1;; ++j) {
                uint64_t h = splitmix64((uint64_t)v ^ seed_g);
                h = splitmix64((uint64_t)ctr ^ h);
                const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
                int64_t rho = (int64_t)floor(pow(u * top + 1.0, 1.0 / e)) - 1;
                if (rho < 0) rho = 0;
                if (rho > N - 1) rho = N - 1;
                t = pi[rho];
                if (t != v) break;
                ctr = k + (int64_t)m * j;
            }
            targets[v * m + k] = (int32_t)t;
        }
    }
}

/* Symmetrised CSR: indptr[N+1], indices[2*N*m]; neighbours of a in (edge source, k) order —
 * a sequential fill in edge order is stable. */
void plcite_csr(int64_t N, int32_t m, const int32_t* targets, int64_t* indptr, int32_t* indices) {
    memset(indptr, 0, (size_t)(N + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < N; ++v)
        for (int32_t k = 0; k < m; ++k) {
            indptr[v + 1]++;
            indptr[(int64_t)targets[v * m + k] + 1]++;
        }
    for (int64_t v = 0; v < N; ++v) indptr[v + 1] += indptr[v];
    int64_t* fill = malloc((size_t)N * sizeof(int64_t));
    memcpy(fill, indptr, (size_t)N * sizeof(int64_t));
    for (int64_t v = 0; v < N; ++v)
        for (int32_t k = 0; k < m; ++k) {
            const int64_t t = targets[v * m + k];
            /* entry of the out-edge (v -> t) in v's list and of the in-edge in t's list; both
             * are keyed by (source v, k), which is the loop order */
            indices[fill[v]++] = (int32_t)t;
            indices[fill[t]++] = (int32_t)v;
        }
    free(fill);
}

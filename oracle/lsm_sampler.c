/* oracle/lsm_sampler.c — CPU ORACLE for the window producer (NEXT N3): GraphSAGE
 * multi-hop neighbour sampling (§2.1, fanout P:603) as DESIGN.md §3
 * defines it. TEST INFRASTRUCTURE ONLY (same rules as lsm_oracle.c); it shares no code
 * with the CUDA sampler. Plain loops, one thread.
 *
 * Definition (per frontier position p, layer l, draw j):
 *   deg <= f : all deg neighbours in CSR order
 *   deg >  f : f draws, neighbour at CSR offset floor(U01(h(seed, t, r, l, p, j)) * deg)
 *   h(seed, c0, c1, ...) = splitmix64(... splitmix64(splitmix64(seed ^ c0) ^ c1) ...)
 *   U01(x) = (x >> 11) * 2^-53
 *   next frontier = first-occurrence unique of the layer's draws
 *   result = first-occurrence unique of seeds ++ layer0 draws ++ layer1 draws ++ ...
 * Pinned by tests/test_oracle_sampler.py against an independent numpy implementation
 * (synth.sample_batch) and against brute-force properties.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* first-occurrence unique of a[0..n) in place; seen[] is an N-byte scratch set to 0 */
static int64_t unique_first(int64_t* a, int64_t n, uint8_t* seen) {
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        if (!seen[a[i]]) { seen[a[i]] = 1; a[m++] = a[i]; }
    for (int64_t i = 0; i < m; ++i) seen[a[i]] = 0;
    return m;
}

/* Returns the length of the sampled list written to out (capacity cap), or -1 if it
 * would not fit. */
int64_t orc_sample(const int64_t* indptr, const int32_t* indices, int64_t N, const int64_t* seeds,
                   int64_t nseeds, const int32_t* fanout, int32_t nlayers, uint64_t seed, int64_t t, int32_t r,
                   int64_t* out, int64_t cap) {
    int64_t total = nseeds, fr = nseeds, prod = nseeds;
    for (int l = 0; l < nlayers; ++l) { prod *= fanout[l]; total += prod; }
    (void)fr;
    int64_t* raw = malloc((size_t)(total > 0 ? total : 1) * sizeof(int64_t));
    int64_t* frontier = malloc((size_t)(total > 0 ? total : 1) * sizeof(int64_t));
    uint8_t* seen = calloc((size_t)N, 1);
    int64_t nraw = 0, nf = nseeds;
    for (int64_t i = 0; i < nseeds; ++i) { raw[nraw++] = seeds[i]; frontier[i] = seeds[i]; }
    for (int l = 0; l < nlayers; ++l) {
        const int64_t f = fanout[l], start = nraw;
        for (int64_t p = 0; p < nf; ++p) {
            const int64_t x = frontier[p], deg = indptr[x + 1] - indptr[x];
            if (deg <= f) {
                for (int64_t j = 0; j < deg; ++j) raw[nraw++] = indices[indptr[x] + j];
            } else {
                for (int64_t j = 0; j < f; ++j) {
                    uint64_t h = seed;
                    h = splitmix64((uint64_t)t ^ h);
                    h = splitmix64((uint64_t)r ^ h);
                    h = splitmix64((uint64_t)l ^ h);
                    h = splitmix64((uint64_t)p ^ h);
                    h = splitmix64((uint64_t)j ^ h);
                    const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
                    const int64_t pos = (int64_t)(u * (double)deg);
                    raw[nraw++] = indices[indptr[x] + pos];
                }
            }
        }
        /* next frontier: first-occurrence unique of this layer's draws */
        nf = nraw - start;
        memcpy(frontier, raw + start, (size_t)nf * sizeof(int64_t));
        nf = unique_first(frontier, nf, seen);
        if (nf == 0) break;
    }
    int64_t n = unique_first(raw, nraw, seen);
    int64_t rc = n;
    if (n > cap) rc = -1;
    else memcpy(out, raw, (size_t)n * sizeof(int64_t));
    free(raw); free(frontier); free(seen);
    return rc;
}

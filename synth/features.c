/* synth/features.c — seeded, closed-form feature rows F(v) (input generator).
 *
 * This module holds NO arithmetic of the LSM-GNN method. It only produces the
 * synthetic feature table that both the CUDA path (as its host-resident backing
 * "storage" tier) and the CPU oracle (as the table it gathers from) read.
 *
 * Recipe (SURVEY.md §8(d) "Features"):
 *   word j of row v  =  0x3F800000 | (splitmix64(seed_f ^ (v*D + j)) >> 41)
 * i.e. an fp32 value in [1, 2) — never NaN, never 0, and self-verifying: any
 * row can be recomputed from its node ID alone.
 *
 * Built by synth/__init__.py with `gcc -O3 -fopenmp -shared`.
 */
#include <stdint.h>

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Fill rows v0 .. v0+nrows-1 (D 32-bit words each) into dst (row-major, tight). */
void synth_fill_f32(uint32_t* dst, int64_t v0, int64_t nrows, int32_t D, uint64_t seed_f) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        uint64_t v = (uint64_t)(v0 + r);
        uint32_t* row = dst + r * (int64_t)D;
        for (int32_t j = 0; j < D; ++j)
            row[j] = 0x3F800000u | (uint32_t)(splitmix64(seed_f ^ (v * (uint64_t)D + (uint64_t)j)) >> 41);
    }
}

/* Fill the rows of an explicit ID list: dst[i] = F(ids[i]). */
void synth_fill_f32_ids(uint32_t* dst, const int64_t* ids, int64_t n, int32_t D, uint64_t seed_f) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t v = (uint64_t)ids[i];
        uint32_t* row = dst + i * (int64_t)D;
        for (int32_t j = 0; j < D; ++j)
            row[j] = 0x3F800000u | (uint32_t)(splitmix64(seed_f ^ (v * (uint64_t)D + (uint64_t)j)) >> 41);
    }
}

/* Check rows against the closed form; returns the number of mismatching rows
 * (the first mismatching row index is written to *first_bad, else -1). */
int64_t synth_check_f32_ids(const uint32_t* rows, const int64_t* ids, int64_t n, int32_t D,
                            uint64_t seed_f, int64_t* first_bad) {
    int64_t bad = 0, first = -1;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t v = (uint64_t)ids[i];
        const uint32_t* row = rows + i * (int64_t)D;
        int ok = 1;
        for (int32_t j = 0; j < D && ok; ++j)
            ok = row[j] == (0x3F800000u | (uint32_t)(splitmix64(seed_f ^ (v * (uint64_t)D + (uint64_t)j)) >> 41));
        if (!ok) {
            bad += 1;
#pragma omp critical
            if (first < 0 || i < first) first = i;
        }
    }
    if (first_bad) *first_bad = first;
    return bad;
}

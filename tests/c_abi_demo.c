/* tests/c_abi_demo.c — the boundary used from plain C (no Python, no torch): one home,
 * a small synthetic trace, the hybrid policy with the PVP. Checks every gathered row
 * against the table and the conservation law hits + victim_hits + storage_reads = unique
 * per iteration. Built and run by tests/test_c_abi.py.
 *
 *   gcc -std=c11 -O2 -I include tests/c_abi_demo.c -L paper_2407_15264_b200 -llsmgnn \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o c_abi_demo
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lsmgnn.h"

#define N 4096
#define D 32 /* fp32 words per row: R = 128 B */
#define L 256
#define A 8
#define V 64
#define W 4
#define K 12
#define B 300

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ != 0) {                                                               \
      fprintf(stderr, "%s -> %d (%s)\n", #x, rc_, lsmgnn_last_error());           \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CUDA(x)                                                                   \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                  \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static uint32_t word(int64_t v, int j) { return (uint32_t)(v * 1000003u + (uint32_t)j * 7919u); }

int main(void) {
  /* host table (this home = all rows at G = 1) and u8 scores */
  uint32_t* table = (uint32_t*)malloc((size_t)N * D * sizeof(uint32_t));
  uint8_t* scores = (uint8_t*)malloc(N);
  for (int64_t v = 0; v < N; ++v) {
    for (int j = 0; j < D; ++j) table[v * D + j] = word(v, j);
    scores[v] = (uint8_t)((v * 37) % 256);
  }
  /* a skewed trace: batch t = B ids drawn from a power-ish distribution, plus empty batches
   * past the end (the window looks W iterations ahead) */
  int64_t* ids = (int64_t*)malloc((size_t)(K + W + 1) * B * sizeof(int64_t));
  uint64_t s = 12345;
  for (int64_t i = 0; i < (int64_t)(K + W + 1) * B; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double u = (double)(s >> 11) / 9007199254740992.0;
    ids[i] = (int64_t)(u * u * u * N) % N;
  }
  int64_t *d_ids, *d_empty;
  void* d_out;
  CUDA(cudaMalloc((void**)&d_ids, (size_t)(K + W + 1) * B * sizeof(int64_t)));
  CUDA(cudaMalloc((void**)&d_empty, sizeof(int64_t)));
  CUDA(cudaMalloc(&d_out, (size_t)B * D * sizeof(uint32_t)));
  CUDA(cudaMemcpy(d_ids, ids, (size_t)(K + W + 1) * B * sizeof(int64_t), cudaMemcpyHostToDevice));

  CHECK(lsmgnn_bind(0, 1, 0));
  lsmgnn_options opt;
  memset(&opt, 0, sizeof opt);
  opt.version = LSMGNN_ABI_VERSION;
  opt.policy = LSMGNN_HYBRID;
  opt.pvp = 1;
  opt.window = W;
  opt.update_period = 1;
  opt.reinsert_victims = 1;
  opt.max_batch_ids = B;
  CHECK(lsmgnn_set_options(&opt));
  CHECK(lsmgnn_init(N, D, LSMGNN_F32, L, A, V, scores));
  CHECK(lsmgnn_attach_storage(table, NULL));

  /* bootstrap: iterations 1..W, as one CSR call (device ids, host offsets) */
  int64_t offs[W + 1];
  for (int b = 0; b <= W; ++b) offs[b] = (int64_t)b * B;
  CHECK(lsmgnn_prefetch(d_ids + B, offs, W, 1, NULL));

  uint32_t* out = (uint32_t*)malloc((size_t)B * D * sizeof(uint32_t));
  int64_t bad = 0;
  for (int t = 0; t < K; ++t) {
    CHECK(lsmgnn_gather(d_ids + (size_t)t * B, B, d_out, NULL));
    const int64_t k = t + 1 + W;
    const int64_t one[2] = {0, k < K ? B : 0};
    CHECK(lsmgnn_prefetch(k < K ? d_ids + (size_t)k * B : d_empty, one, 1, k, NULL));
    CUDA(cudaMemcpy(out, d_out, (size_t)B * D * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < D; ++j) bad += out[(size_t)i * D + j] != word(ids[(size_t)t * B + i], j);
    lsmgnn_stats_t st;
    CHECK(lsmgnn_stats(&st, 0));
    if (st.hits + st.victim_hits + st.storage_reads != st.unique || st.requests != B) {
      fprintf(stderr, "t=%d: conservation broken (%llu + %llu + %llu vs %llu unique, %llu requests)\n", t,
              (unsigned long long)st.hits, (unsigned long long)st.victim_hits, (unsigned long long)st.storage_reads,
              (unsigned long long)st.unique, (unsigned long long)st.requests);
      return 1;
    }
  }
  lsmgnn_stats_t cum;
  CHECK(lsmgnn_stats(&cum, 1));
  CHECK(lsmgnn_finalize());
  if (bad) {
    fprintf(stderr, "%lld words differ from the table\n", (long long)bad);
    return 1;
  }
  printf("c abi ok: %d iterations, %llu requests, %llu unique, hits %llu, victim hits %llu, storage %llu\n", K,
         (unsigned long long)cum.requests, (unsigned long long)cum.unique, (unsigned long long)cum.hits,
         (unsigned long long)cum.victim_hits, (unsigned long long)cum.storage_reads);
  return 0;
}

// Differential check of next_reuse_d (registers, one round trip) against the word-by-word
// scan next_reuse_d_seq, and both against a plain host scan of the window positions
// (iterations t+1..t+W at bit (k mod (W+1)), R5): every W in 1..600, every p0,
// random rows of several densities. Built and run by tests/test_gpu_device_funcs.py.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include "../../paper_2407_15264_b200/csrc/device_common.cuh"
using namespace lsm;

__global__ void k(const uint32_t* rows, int n, int MW, int W, int* a, int* b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p0 = i % (W + 1);
  a[i] = next_reuse_d(rows + (size_t)i * MW, p0, W);
  b[i] = next_reuse_d_seq(rows + (size_t)i * MW, p0, W);
}

static int host_scan(const uint32_t* row, int p0, int W) {  // the plain definition
  const int Wp1 = W + 1;
  for (int d = 1; d <= W; ++d) {
    const int pos = (p0 + d - 1) % Wp1;
    if ((row[pos >> 5] >> (pos & 31)) & 1u) return d;
  }
  return 0;
}

int main() {
  std::mt19937 rng(7);
  long bad = 0, total = 0;
  for (int W = 1; W <= 600; ++W) {
    const int Wp1 = W + 1, MW = (Wp1 + 31) / 32;
    const int n = 8 * Wp1;  // every p0, 8 rows each
    std::vector<uint32_t> rows((size_t)n * MW, 0);
    for (int i = 0; i < n; ++i) {
      const int dens = i % 4;  // empty, one bit, sparse, dense
      for (int b = 0; b < Wp1; ++b) {
        bool on = dens == 2 ? (rng() % 37 == 0) : dens == 3 ? (rng() % 3 == 0) : false;
        if (on) rows[(size_t)i * MW + (b >> 5)] |= 1u << (b & 31);
      }
      if (dens == 1) { const int b = rng() % Wp1; rows[(size_t)i * MW + (b >> 5)] |= 1u << (b & 31); }
    }
    uint32_t* dr; int *da, *db;
    cudaMalloc(&dr, rows.size() * 4); cudaMalloc(&da, n * 4); cudaMalloc(&db, n * 4);
    cudaMemcpy(dr, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
    k<<<(n + 255) / 256, 256>>>(dr, n, MW, W, da, db);
    std::vector<int> a(n), b(n);
    cudaMemcpy(a.data(), da, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), db, n * 4, cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; ++i) {
      const int h = host_scan(&rows[(size_t)i * MW], i % Wp1, W);
      ++total;
      if (a[i] != h || b[i] != h) {
        if (bad < 10) printf("W=%d p0=%d: regs %d seq %d host %d\n", W, i % Wp1, a[i], b[i], h);
        ++bad;
      }
    }
    cudaFree(dr); cudaFree(da); cudaFree(db);
  }
  printf("next_reuse_check: %ld cases, %ld mismatches\n", total, bad);
  return bad ? 1 : 0;
}

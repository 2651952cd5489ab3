// tools/d2h_microbench.cu — rows from HBM to pinned host memory (the e2e path's `out` in host
// memory), on B200: 16-B warp stores (k_serve<..., kHost, 0>'s delivery) vs TMA bulk copies
// through the per-warp shared-memory rings (RowRing, as in k_serve's device delivery), alone and
// while another stream reads scattered 4 KiB rows from pinned host memory into HBM (the storage
// fills of the same step: PCIe in both directions at once).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o d2h_mb tools/d2h_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2407_15264_b200/csrc/device_common.cuh"
using namespace lsm;

#define CK(x)                                                       \
  do {                                                              \
    cudaError_t e = (x);                                            \
    if (e != cudaSuccess) {                                         \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                \
      exit(1);                                                      \
    }                                                               \
  } while (0)

// rows[e] of the device table -> dst row e (host-mapped), warp 16-B copies
__global__ void k_warp(const uint4* __restrict__ tab, const uint32_t* __restrict__ rows, uint32_t n, uint4* dst,
                       uint32_t nvec) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = w; e < n; e += nw) warp_copy_row<8, kDev, kHost>(dst + (size_t)e * nvec, tab + (size_t)rows[e] * nvec, nvec);
}
// the same with TMA bulk copies through per-warp rings of ST stages, chunks of 32 rows
__global__ void k_tma(const uint4* __restrict__ tab, const uint32_t* __restrict__ rows, uint32_t n, uint4* dst,
                      uint32_t nvec, uint32_t ST) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[8][kMaxStages];
  __shared__ uint32_t s_pend[8][kMaxStages];
  __shared__ const void* s_src[8][32];
  __shared__ void* s_dst[8][32];
  const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RowRing ring{};
  ring.buf = smem + (size_t)wib * ST * nvec * 16;
  ring.bar = s_bar[wib];
  ring.pend = s_pend[wib];
  ring.ST = ST;
  ring.R = nvec * 16;
  if (lane == 0) ring_init(ring);
  __syncwarp();
  const uint32_t w = blockIdx.x * (blockDim.x >> 5) + wib, nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t c0 = w * 32; c0 < n; c0 += nw * 32) {
    const uint32_t e = c0 + lane;
    s_src[wib][lane] = tab + (size_t)(e < n ? rows[e] : 0) * nvec;
    s_dst[wib][lane] = dst + (size_t)e * nvec;
    const uint32_t need = __ballot_sync(0xffffffffu, e < n);
    __syncwarp();
    if (lane == 0) ring_copy(ring, s_src[wib], s_dst[wib], need);
    __syncwarp();
  }
  if (lane == 0) ring_drain();
}
// scattered host rows -> HBM (the storage fills)
__global__ void k_h2d(const uint4* hsrc, const uint32_t* __restrict__ rows, uint32_t n, uint4* dst, uint32_t nvec) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = w; e < n; e += nw) warp_copy_row<8, kHost, kDev>(dst + (size_t)e * nvec, hsrc + (size_t)rows[e] * nvec, nvec);
}

int main() {
  const uint32_t R = 4096, nvec = R / 16, NT = 1 << 20, n = 131072;  // 512 MiB of rows per run
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4 *tab, *hbm_dst;
  CK(cudaMalloc(&tab, (size_t)NT * R));
  CK(cudaMemset(tab, 3, (size_t)NT * R));
  CK(cudaMalloc(&hbm_dst, (size_t)n * R));
  uint4 *hout, *hout_d, *hsrc, *hsrc_d;
  CK(cudaHostAlloc(&hout, (size_t)n * R, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&hout_d, hout, 0));
  CK(cudaHostAlloc(&hsrc, (size_t)NT * R / 2, cudaHostAllocMapped));  // 2 GiB of host rows
  CK(cudaHostGetDevicePointer((void**)&hsrc_d, hsrc, 0));
  std::vector<uint32_t> r1(n), r2(n);
  std::mt19937 rng(5);
  for (auto& x : r1) x = rng() % NT;
  for (auto& x : r2) x = rng() % (NT / 2);
  uint32_t *d1, *d2;
  CK(cudaMalloc(&d1, n * 4));
  CK(cudaMalloc(&d2, n * 4));
  CK(cudaMemcpy(d1, r1.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d2, r2.data(), n * 4, cudaMemcpyHostToDevice));
  cudaStream_t sa, sb;
  CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  cudaEvent_t a0, a1, b0, b1;
  cudaEventCreate(&a0); cudaEventCreate(&a1); cudaEventCreate(&b0); cudaEventCreate(&b1);
  const int ST = 6;
  const int smem = 8 * ST * R;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  auto run = [&](const char* name, int mode, bool with_h2d) {
    float best = 1e9, best_b = 0;
    for (int it = 0; it < 4; ++it) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a0, sa);
      if (with_h2d) cudaEventRecord(b0, sb);
      if (mode == 0) k_warp<<<sms * 4, 256, 0, sa>>>(tab, d1, n, hout_d, nvec);
      else k_tma<<<sms, 256, smem, sa>>>(tab, d1, n, hout_d, nvec, ST);
      if (with_h2d) k_h2d<<<sms * 2, 256, 0, sb>>>(hsrc_d, d2, n, hbm_dst, nvec);
      cudaEventRecord(a1, sa);
      if (with_h2d) cudaEventRecord(b1, sb);
      CK(cudaDeviceSynchronize());
      float ms, msb = 0;
      cudaEventElapsedTime(&ms, a0, a1);
      if (with_h2d) cudaEventElapsedTime(&msb, b0, b1);
      if (it && ms < best) { best = ms; best_b = msb; }
    }
    printf("%-46s D2H %7.2f GB/s", name, (double)n * R / best / 1e6);
    if (with_h2d) printf("   concurrent H2D %7.2f GB/s", (double)n * R / best_b / 1e6);
    printf("\n");
  };
  run("HBM rows -> pinned host, warp 16-B stores", 0, false);
  run("HBM rows -> pinned host, TMA bulk rings", 1, false);
  run("warp 16-B stores + scattered host->HBM reads", 0, true);
  run("TMA bulk rings + scattered host->HBM reads", 1, true);
  // check the TMA copy's bytes
  CK(cudaMemset(tab, 0, (size_t)NT * R));
  k_tma<<<sms, 256, smem, sa>>>(tab, d1, n, hout_d, nvec, ST);
  CK(cudaDeviceSynchronize());
  size_t bad = 0;
  const uint32_t* h = reinterpret_cast<const uint32_t*>(hout);
  for (size_t i = 0; i < (size_t)n * R / 4; i += 4099) bad += h[i] != 0;
  printf("row check (TMA to host): %zu bad words sampled\n", bad);
  return 0;
}

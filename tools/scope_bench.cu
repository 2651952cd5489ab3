// tools/scope_bench.cu — NEXT N4: the fig:scope_bench experiment on B200.
//
// A set-associative GPU software cache whose cache-management operations (line pin/unpin
// reference counts, the miss-path line lock, tag publication and its fence) are issued at
// device scope (.gpu) or at system scope (.sys). The paper measured, on A100, ~750 GB/s
// (hot: all hits) and ~124 GB/s (cold: all misses) with device-scope operations vs
// ~110 / ~42 GB/s with system-scope ones, which is why LSM-GNN routes every request to the
// home GPU and keeps all cache metadata at .gpu scope. Here the miss path reads
// rows from pinned host memory (this build's storage stand-in).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scope_bench tools/scope_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                            \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int SYS>
__device__ __forceinline__ uint32_t atom_add_acq(uint32_t* p, uint32_t v) {
  uint32_t r;
  if (SYS) asm volatile("atom.acquire.sys.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  else asm volatile("atom.acquire.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
template <int SYS>
__device__ __forceinline__ void red_add_rel(uint32_t* p, uint32_t v) {
  if (SYS) asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int SYS>
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t r;
  if (SYS) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
template <int SYS>
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  if (SYS) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int SYS>
__device__ __forceinline__ uint32_t atom_cas(uint32_t* p, uint32_t c, uint32_t v) {
  uint32_t r;
  if (SYS) asm volatile("atom.acq_rel.sys.global.cas.b32 %0, [%1], %2, %3;" : "=r"(r) : "l"(p), "r"(c), "r"(v) : "memory");
  else asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(r) : "l"(p), "r"(c), "r"(v) : "memory");
  return r;
}

// Warp per request: probe the set's tags (acquire loads), pin the line (refcount atomic),
// copy the 4 KiB line to the output, unpin (release). Cold mode: every request misses —
// lock a victim way (CAS), read the row from host memory into the line, publish the tag
// with a release store, unlock.
template <int SYS, bool COLD>
__global__ void k_access(const uint32_t* __restrict__ req, uint32_t n, uint32_t* tags, uint32_t* refc,
                         uint32_t* lock, uint4* lines, const uint4* __restrict__ host, uint4* __restrict__ out,
                         uint32_t S, uint32_t A, uint32_t nvec) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t e = warp; e < n; e += nw) {
    const uint32_t v = req[e], s = v % S;
    uint32_t tg = lane < A ? ld_acq<SYS>(&tags[s * A + lane]) : 0xFFFFFFFFu;
    uint32_t hit = __ballot_sync(0xffffffffu, tg == v);
    uint32_t way;
    if (hit) {
      way = __ffs(hit) - 1;
      if (lane == 0) atom_add_acq<SYS>(&refc[s * A + way], 1u);
      __syncwarp();
    } else {
      way = (v / S) % A;
      if (lane == 0) {
        while (atom_cas<SYS>(&lock[s * A + way], 0u, 1u) != 0u) {}
        atom_add_acq<SYS>(&refc[s * A + way], 1u);
      }
      __syncwarp();
      const uint4* src = host + (size_t)v * nvec;
      uint4* dst = lines + (size_t)(s * A + way) * nvec;
      for (uint32_t k = lane; k < nvec; k += 32) dst[k] = src[k];
      __syncwarp();
      if (lane == 0) {
        st_rel<SYS>(&tags[s * A + way], v);
        st_rel<SYS>(&lock[s * A + way], 0u);
      }
      __syncwarp();
    }
    const uint4* line = lines + (size_t)(s * A + way) * nvec;
    uint4* o = out + (size_t)e * nvec;
    for (uint32_t k = lane; k < nvec; k += 32) o[k] = line[k];
    __syncwarp();
    if (lane == 0) red_add_rel<SYS>(&refc[s * A + way], 0xFFFFFFFFu);
  }
}

int main() {
  const uint32_t R = 4096, nvec = R / 16, A = 32, S = 8192, L = S * A;  // 1 GiB cache
  const uint32_t NHOST = 1u << 20;                                      // 4 GiB of host rows
  const uint32_t n = 200000;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t *tags, *refc, *lock, *req;
  uint4 *lines, *out, *host, *hostd;
  CK(cudaMalloc(&tags, L * 4));
  CK(cudaMalloc(&refc, L * 4));
  CK(cudaMalloc(&lock, L * 4));
  CK(cudaMalloc(&lines, (size_t)L * R));
  CK(cudaMalloc(&out, (size_t)n * R));
  CK(cudaMalloc(&req, n * 4));
  CK(cudaHostAlloc(&host, (size_t)NHOST * R, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&hostd, host, 0));
  std::mt19937 rng(7);
  // hot: every request is a resident line (tags preloaded); cold: requests of nodes never seen
  std::vector<uint32_t> hot(n), cold(n), tag0(L);
  for (uint32_t i = 0; i < L; ++i) tag0[i] = (i % A) * S + i / A;  // way w of set s holds v = w*S + s
  for (auto& x : hot) x = rng() % L;                                 // v < L: resident
  for (uint32_t i = 0; i < n; ++i) cold[i] = L + i;                  // never resident, distinct
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("%-34s %10s %10s\n", "mode", "ms", "GB/s");
  for (int cold_mode = 0; cold_mode < 2; ++cold_mode) {
    for (int sys = 0; sys < 2; ++sys) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        CK(cudaMemcpy(tags, tag0.data(), L * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(refc, 0, L * 4));
        CK(cudaMemset(lock, 0, L * 4));
        CK(cudaMemcpy(req, cold_mode ? cold.data() : hot.data(), n * 4, cudaMemcpyHostToDevice));
        const uint32_t nn = cold_mode ? std::min<uint32_t>(n, NHOST - L) : n;
        cudaEventRecord(a);
        if (!cold_mode && !sys) k_access<0, false><<<sms * 8, 256>>>(req, nn, tags, refc, lock, lines, hostd, out, S, A, nvec);
        if (!cold_mode && sys) k_access<1, false><<<sms * 8, 256>>>(req, nn, tags, refc, lock, lines, hostd, out, S, A, nvec);
        if (cold_mode && !sys) k_access<0, true><<<sms * 8, 256>>>(req, nn, tags, refc, lock, lines, hostd, out, S, A, nvec);
        if (cold_mode && sys) k_access<1, true><<<sms * 8, 256>>>(req, nn, tags, refc, lock, lines, hostd, out, S, A, nvec);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it) best = std::min(best, ms);
        if (it == 3)
          printf("%-34s %10.3f %10.1f\n",
                 cold_mode ? (sys ? "cold (all misses), system scope" : "cold (all misses), device scope")
                           : (sys ? "hot (all hits), system scope" : "hot (all hits), device scope"),
                 best, (double)nn * R / best / 1e6);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}

// tools/pcie_microbench.cu — how fast can SMs pull random 4 KiB rows out of pinned host
// memory over PCIe on B200? Compares (1) warp 16-B loads, (2) TMA bulk copies
// (cp.async.bulk global->shared, mbarrier) of whole rows then bulk stores to HBM, and
// (3) the copy engine (cudaMemcpyAsync of one contiguous block) as the reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_mb tools/pcie_microbench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <chrono>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U, int MODE>
__global__ void k_ldg(const uint4* __restrict__ host, const uint32_t* __restrict__ rows, uint32_t n,
                      uint4* __restrict__ dst, int nvec) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint32_t e = warp; e < n; e += nw) {
    const uint4* s = host + (size_t)rows[e] * nvec;
    uint4* d = dst + (size_t)e * nvec;
    if (MODE == 3 && lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s), "r"(nvec * 16) : "memory");
    for (int i = lane; i < nvec; i += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) if (i + 32 * u < nvec) {
        if (MODE == 0) asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(s + i + 32 * u));
        else if (MODE == 1) asm volatile("ld.global.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(s + i + 32 * u));
        else asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(s + i + 32 * u));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) if (i + 32 * u < nvec) d[i + 32 * u] = v[u];
    }
  }
}

// 256-bit loads (sm_100: ld.global.v8.u32 -> LDG.E.ENL2.256): 32 B per lane, 1 KiB per warp
// instruction; U loads in flight per lane (U = 4: a whole 4 KiB row). HINT = 1 adds .L2::256B.
template <int U, int HINT>
__global__ void k_ldg256(const uint4* __restrict__ host, const uint32_t* __restrict__ rows, uint32_t n,
                         uint4* __restrict__ dst, int nvec) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int n32 = nvec / 2;  // 32-byte units per row
  for (uint32_t e = warp; e < n; e += nw) {
    const uint4* s = host + (size_t)rows[e] * nvec;
    uint4* d = dst + (size_t)e * nvec;
    for (int i = lane; i < n32; i += 32 * U) {
      uint4 v[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) if (i + 32 * u < n32) {
        const uint4* p = s + 2 * (i + 32 * u);
        if (HINT)
          asm volatile("ld.global.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[u][0].x), "=r"(v[u][0].y), "=r"(v[u][0].z), "=r"(v[u][0].w),
                         "=r"(v[u][1].x), "=r"(v[u][1].y), "=r"(v[u][1].z), "=r"(v[u][1].w) : "l"(p));
        else
          asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[u][0].x), "=r"(v[u][0].y), "=r"(v[u][0].z), "=r"(v[u][0].w),
                         "=r"(v[u][1].x), "=r"(v[u][1].y), "=r"(v[u][1].z), "=r"(v[u][1].w) : "l"(p));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) if (i + 32 * u < n32) {
        d[2 * (i + 32 * u)] = v[u][0];
        d[2 * (i + 32 * u) + 1] = v[u][1];
      }
    }
  }
}

// device rows -> pinned host rows (the e2e out path), 8 x 16 B per lane in flight
__global__ void k_d2h(const uint4* __restrict__ src, uint32_t n, uint4* __restrict__ hout, int nvec) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint32_t e = warp; e < n; e += nw)
    for (int i = lane; i < nvec; i += 256) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[(size_t)e * nvec + i + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) hout[(size_t)e * nvec + i + 32 * u] = v[u];
    }
}
// host row -> host out row (read over PCIe then write back over PCIe): the e2e miss path
__global__ void k_relay(const uint4* __restrict__ host, const uint32_t* __restrict__ rows, uint32_t n,
                        uint4* __restrict__ hout, int nvec) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint32_t e = warp; e < n; e += nw)
    for (int i = lane; i < nvec; i += 256) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = host[(size_t)rows[e] * nvec + i + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) hout[(size_t)e * nvec + i + 32 * u] = v[u];
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

// one elected lane per warp drives a STAGES-deep ring of row buffers in shared memory
template <int STAGES>
__global__ void k_tma(const uint8_t* __restrict__ host, const uint32_t* __restrict__ rows, uint32_t n,
                      uint8_t* __restrict__ dst, uint32_t R, uint32_t chunk) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[32][STAGES];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * (blockDim.x >> 5) + wib, nw = gridDim.x * (blockDim.x >> 5);
  uint8_t* ring = sm + (size_t)wib * STAGES * R;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[wib][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane != 0) return;
  uint32_t issued = 0, done = 0;
  uint32_t phase[STAGES] = {};
  // prologue
  for (uint32_t e = warp; e < n && issued < STAGES; e += nw, ++issued) {
    const int s = issued % STAGES;
    mbar_expect(&bars[wib][s], R);
    for (uint32_t o = 0; o < R; o += chunk) bulk_g2s(ring + s * R + o, host + (size_t)rows[e] * R + o, chunk, &bars[wib][s]);
  }
  for (uint32_t e = warp; e < n; e += nw, ++done) {
    const int s = done % STAGES;
    mbar_wait(&bars[wib][s], phase[s]);
    phase[s] ^= 1;
    bulk_s2g(dst + (size_t)e * R, ring + s * R, R);
    bulk_commit();
    // refill this stage with the row STAGES ahead once the store has read it
    const uint32_t en = e + (uint32_t)STAGES * nw;
    if (en < n) {
      bulk_wait_read<0>();
      mbar_expect(&bars[wib][s], R);
      for (uint32_t o = 0; o < R; o += chunk) bulk_g2s(ring + s * R + o, host + (size_t)rows[en] * R + o, chunk, &bars[wib][s]);
    }
  }
  bulk_wait_read<0>();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const size_t NROWS = 1 << 20;  // 4 GiB table
  const uint32_t R = 4096;
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 100000;
  uint8_t* host;
  CK(cudaHostAlloc(&host, NROWS * R, cudaHostAllocMapped));
  for (size_t i = 0; i < NROWS * R / 8; i += 512) reinterpret_cast<uint64_t*>(host)[i] = i;
  uint8_t* hdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
  std::vector<uint32_t> rows(n);
  std::mt19937 rng(1);
  for (auto& r : rows) r = rng() % NROWS;
  uint32_t* drows;
  CK(cudaMalloc(&drows, n * 4));
  CK(cudaMemcpy(drows, rows.data(), n * 4, cudaMemcpyHostToDevice));
  uint8_t* dst;
  CK(cudaMalloc(&dst, (size_t)n * R));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto fn) {
    fn();
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    printf("%-40s %8.3f ms  %7.2f GB/s\n", name, best, (double)n * R / best / 1e6);
  };
  timeit("copy engine (contiguous n*R)", [&] { cudaMemcpyAsync(dst, host, (size_t)n * R, cudaMemcpyHostToDevice); });
  for (int blocks : {sms, 2 * sms, 4 * sms}) {
    char nm[64];
    snprintf(nm, 64, "ldg U=8 grid=%d x256", blocks);
    timeit(nm, [&] { k_ldg<8, 0><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
    snprintf(nm, 64, "ldg L2::256B U=8 grid=%d", blocks);
    timeit(nm, [&] { k_ldg<8, 1><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
    snprintf(nm, 64, "ldg.nc L2::256B U=8 grid=%d", blocks);
    timeit(nm, [&] { k_ldg<8, 2><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
    snprintf(nm, 64, "bulk.prefetch.L2 + ldg U=8 grid=%d", blocks);
    timeit(nm, [&] { k_ldg<8, 3><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
    snprintf(nm, 64, "ldg.256 (v8) U=4 grid=%d", blocks);
    timeit(nm, [&] { k_ldg256<4, 0><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
    snprintf(nm, 64, "ldg.256 (v8) L2::256B U=4 grid=%d", blocks);
    timeit(nm, [&] { k_ldg256<4, 1><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
    snprintf(nm, 64, "ldg.256 (v8) U=2 grid=%d", blocks);
    timeit(nm, [&] { k_ldg256<2, 0><<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16); });
  }
  for (int stages : {4}) {
    for (int warps : {8}) {
      for (uint32_t chunk : {4096u}) {
        size_t smem = (size_t)warps * stages * R;
        char nm[96];
        snprintf(nm, 96, "tma st=%d warps=%d chunk=%u grid=%d", stages, warps, chunk, sms);
        if (stages == 2) {
          CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          timeit(nm, [&] { k_tma<2><<<sms, warps * 32, smem>>>(hdev, drows, n, dst, R, chunk); });
        } else {
          CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          timeit(nm, [&] { k_tma<4><<<sms, warps * 32, smem>>>(hdev, drows, n, dst, R, chunk); });
        }
      }
    }
  }
  // (a per-row copy-engine variant was measured in round 1 with a batched-copy API that is
  // closed on this pool; its result stays in profiles/r01_pcie_microbench.txt)
  // D2H: device rows -> pinned host (SM stores over PCIe), and both directions at once
  uint8_t* hout;
  CK(cudaHostAlloc(&hout, (size_t)n * R, cudaHostAllocMapped));
  uint8_t* houtd;
  CK(cudaHostGetDevicePointer((void**)&houtd, hout, 0));
  timeit("copy engine D2H (contiguous n*R)", [&] { cudaMemcpyAsync(hout, dst, (size_t)n * R, cudaMemcpyDeviceToHost); });
  for (int blocks : {sms, 4 * sms}) {
    char nm[96];
    snprintf(nm, 96, "SM D2H stores grid=%d", blocks);
    timeit(nm, [&] { k_d2h<<<blocks, 256>>>((const uint4*)dst, n, (uint4*)houtd, R / 16); });
    snprintf(nm, 96, "SM host->host relay (read+write) grid=%d", blocks);
    timeit(nm, [&] { k_relay<<<blocks, 256>>>((const uint4*)hdev, drows, n, (uint4*)houtd, R / 16); });
  }
  // full duplex: SM zero-copy H2D reads (stream A) concurrent with a copy-engine D2H (stream B)
  {
    cudaStream_t sa, sb;
    CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    uint8_t* dsrc;
    CK(cudaMalloc(&dsrc, (size_t)n * R));
    cudaEvent_t a0, a1, b1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    cudaEventCreate(&b1);
    for (int it = 0; it < 3; ++it) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a0, 0);
      cudaStreamWaitEvent(sa, a0, 0);
      cudaStreamWaitEvent(sb, a0, 0);
      k_ldg<8, 0><<<sms, 256, 0, sa>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16);
      cudaEventRecord(a1, sa);
      cudaMemcpyAsync(hout, dsrc, (size_t)n * R, cudaMemcpyDeviceToHost, sb);
      cudaEventRecord(b1, sb);
      CK(cudaDeviceSynchronize());
      float ma, mb;
      cudaEventElapsedTime(&ma, a0, a1);
      cudaEventElapsedTime(&mb, a0, b1);
      if (it == 2)
        printf("duplex: SM H2D reads %.2f GB/s (%.3f ms) || CE D2H %.2f GB/s (%.3f ms)\n", (double)n * R / ma / 1e6, ma,
               (double)n * R / mb / 1e6, mb);
    }
    // and SM reads || SM D2H stores from a different kernel
    for (int it = 0; it < 3; ++it) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a0, 0);
      cudaStreamWaitEvent(sa, a0, 0);
      cudaStreamWaitEvent(sb, a0, 0);
      k_ldg<8, 0><<<sms, 256, 0, sa>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16);
      cudaEventRecord(a1, sa);
      k_d2h<<<sms, 256, 0, sb>>>((const uint4*)dsrc, n, (uint4*)houtd, R / 16);
      cudaEventRecord(b1, sb);
      CK(cudaDeviceSynchronize());
      float ma, mb;
      cudaEventElapsedTime(&ma, a0, a1);
      cudaEventElapsedTime(&mb, a0, b1);
      if (it == 2)
        printf("duplex: SM H2D reads %.2f GB/s (%.3f ms) || SM D2H stores %.2f GB/s (%.3f ms)\n",
               (double)n * R / ma / 1e6, ma, (double)n * R / mb / 1e6, mb);
    }
    // same direction: SM zero-copy H2D reads of scattered rows || copy-engine H2D of a
    // contiguous block — is 51.5 GB/s a limit of the SM read path or of the link?
    uint8_t* dce;
    CK(cudaMalloc(&dce, (size_t)n * R));
    for (int it = 0; it < 3; ++it) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a0, 0);
      cudaStreamWaitEvent(sa, a0, 0);
      cudaStreamWaitEvent(sb, a0, 0);
      k_ldg<8, 0><<<4 * sms, 256, 0, sa>>>((const uint4*)hdev, drows, n, (uint4*)dst, R / 16);
      cudaEventRecord(a1, sa);
      cudaMemcpyAsync(dce, host + (size_t)n * R, (size_t)n * R, cudaMemcpyHostToDevice, sb);
      cudaEventRecord(b1, sb);
      CK(cudaDeviceSynchronize());
      float ma, mb;
      cudaEventElapsedTime(&ma, a0, a1);
      cudaEventElapsedTime(&mb, a0, b1);
      if (it == 2)
        printf("same direction: SM H2D reads %.2f GB/s (%.3f ms) || CE H2D %.2f GB/s (%.3f ms); both done in %.3f ms "
               "= %.2f GB/s total\n", (double)n * R / ma / 1e6, ma, (double)n * R / mb / 1e6, mb, std::max(ma, mb),
               2.0 * n * R / std::max(ma, mb) / 1e6);
    }
    cudaFree(dce);
  }
  CK(cudaGetLastError());
  // correctness of one row
  std::vector<uint8_t> chk(R);
  CK(cudaMemcpy(chk.data(), dst + (size_t)(n / 2) * R, R, cudaMemcpyDeviceToHost));
  printf("row check %s\n", memcmp(chk.data(), host + (size_t)rows[n / 2] * R, R) == 0 ? "ok" : "BAD");
  return 0;
}

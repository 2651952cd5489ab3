// sampler.cuh — NEXT N3: the step before the path. GPU GraphSAGE neighbour sampling
// (fanout P:603) over a CSR pinned in host memory and read by GPU
// threads with zero-copy (UVA) loads, as the paper's sampler does ("the graph
// structure data is pinned in the CPU memory to enable GPU threads to directly fetch graph
// data with UVA during graph sampling"). Produces exactly the lists DESIGN.md §3 defines
// (pinned against oracle/lsm_sampler.c). All sizes after the seeds live on the device; the
// host only knows upper bounds, so nothing synchronises.
#pragma once
#include "device_common.cuh"

namespace lsm {

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SampCounts {   // device-resident sizes of one sampling call
  uint32_t nf;        // frontier length
  uint32_t nraw;      // raw (seeds ++ draws) length so far
  uint32_t layer_n;   // draws of the current layer
  uint32_t nout;      // final unique count
};

// raw[0..n) = frontier[0..n) = seeds; counts initialised.
__global__ void k_samp_init(const int64_t* __restrict__ seeds, uint32_t n, uint32_t* __restrict__ raw,
                            uint32_t* __restrict__ frontier, SampCounts* c) {
  pdl_prologue();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    raw[i] = (uint32_t)seeds[i];
    frontier[i] = (uint32_t)seeds[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c->nf = n;
    c->nraw = n;
  }
}

// cnt[p] = min(deg(frontier[p]), f)
__global__ void k_samp_count(const uint32_t* __restrict__ frontier, const SampCounts* c, const int64_t* indptr,
                             uint32_t f, uint32_t* __restrict__ cnt) {
  pdl_prologue();
  const uint32_t nf = c->nf;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nf; p += gridDim.x * blockDim.x) {
    const uint32_t x = frontier[p];
    const int64_t deg = indptr[x + 1] - indptr[x];
    cnt[p] = (uint32_t)(deg < (int64_t)f ? deg : (int64_t)f);
  }
}

// Draw the layer: position p writes its cnt[p] neighbours at layer[off[p] ...], in (p, j)
// order; deg <= f takes all, otherwise draw j picks offset floor(U01(h(seed,t,r,l,p,j))*deg).
__global__ void k_samp_draw(const uint32_t* __restrict__ frontier, const SampCounts* c, const int64_t* indptr,
                            const int32_t* indices, uint32_t f, const uint32_t* __restrict__ off,
                            uint32_t* __restrict__ layer, uint64_t seed, uint64_t t, uint64_t r, uint64_t l) {
  pdl_prologue();
  // warp per frontier node, lane per draw: every neighbour read of a node is in flight at once
  // (the reads are latency-bound when the CSR is in host memory)
  const uint32_t nf = c->nf;
  const uint32_t lane = lane_id();
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < nf; p += nw) {
    const uint32_t x = frontier[p];
    const int64_t b = indptr[x], deg = indptr[x + 1] - b;
    uint32_t* dst = layer + off[p];
    if (deg <= (int64_t)f) {
      for (int64_t j = lane; j < deg; j += 32) dst[j] = (uint32_t)indices[b + j];
    } else {
      uint64_t hp = splitmix64_dev(t ^ seed);
      hp = splitmix64_dev(r ^ hp);
      hp = splitmix64_dev(l ^ hp);
      hp = splitmix64_dev((uint64_t)p ^ hp);
      for (uint32_t j = lane; j < f; j += 32) {
        const uint64_t h = splitmix64_dev((uint64_t)j ^ hp);
        const double u = __dmul_rn((double)(h >> 11), 1.0 / 9007199254740992.0);
        const int64_t pos = (int64_t)__dmul_rn(u, (double)deg);
        dst[j] = (uint32_t)indices[b + pos];
      }
    }
  }
}

// First-occurrence unique, step 1: tab[v] = min over positions i of (hi << 32 | i). `hi`
// decreases from call to call, so stale entries of earlier calls never win the minimum.
__global__ void k_fo_mark(const uint32_t* __restrict__ a, const uint32_t* n_ptr, uint32_t n_off,
                          unsigned long long* __restrict__ tab, uint32_t hi) {
  pdl_prologue();
  const uint32_t n = *n_ptr - n_off;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicMin(&tab[a[i]], ((unsigned long long)hi << 32) | i);
}
// step 2: keep[i] = this position is its node's first occurrence
__global__ void k_fo_flag(const uint32_t* __restrict__ a, const uint32_t* n_ptr, uint32_t n_off,
                          const unsigned long long* __restrict__ tab, uint32_t hi, uint32_t* __restrict__ keep) {
  pdl_prologue();
  const uint32_t n = *n_ptr - n_off;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    keep[i] = tab[a[i]] == (((unsigned long long)hi << 32) | i);
}
// step 3: stable compaction by the exclusive scan of keep[]
template <typename OutT>
__global__ void k_fo_compact(const uint32_t* __restrict__ a, const uint32_t* n_ptr, uint32_t n_off,
                             const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                             OutT* __restrict__ out, uint32_t* n_out) {
  pdl_prologue();
  const uint32_t n = *n_ptr - n_off;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (keep[i]) out[pos[i]] = (OutT)a[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = n ? pos[n - 1] + keep[n - 1] : 0;
}

// Exclusive scan of x[0..n) (n read on the device as *n_ptr - n_off) into y; 4096 elements
// per CTA (1024 threads x 4), block sums scanned by one CTA (n <= 4M).
__global__ void __launch_bounds__(1024) k_xscan_blocks(const uint32_t* __restrict__ x, const uint32_t* n_ptr,
                                                       uint32_t n_off, uint32_t* __restrict__ y,
                                                       uint32_t* __restrict__ bsum) {
  pdl_prologue();
  __shared__ uint32_t s_warp[32];
  const uint32_t n = *n_ptr - n_off;
  const uint32_t base = blockIdx.x * 4096u;
  if (base >= n) {
    if (threadIdx.x == 0) bsum[blockIdx.x] = 0;
    return;
  }
  const uint32_t tid = threadIdx.x, i0 = base + tid * 4;
  uint32_t v[4], s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = i0 + k < n ? x[i0 + k] : 0u;
    s += v[k];
  }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yv = __shfl_up_sync(0xffffffffu, incl, o);
    if ((tid & 31) >= (uint32_t)o) incl += yv;
  }
  if ((tid & 31) == 31) s_warp[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    uint32_t w = s_warp[tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yv = __shfl_up_sync(0xffffffffu, w, o);
      if (tid >= (uint32_t)o) w += yv;
    }
    s_warp[tid] = w;
  }
  __syncthreads();
  uint32_t run = incl - s + ((tid >> 5) ? s_warp[(tid >> 5) - 1] : 0u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (i0 + k < n) y[i0 + k] = run;
    run += v[k];
  }
  if (tid == 1023) bsum[blockIdx.x] = run;
}
__global__ void __launch_bounds__(1024) k_xscan_sums(uint32_t* __restrict__ bsum, uint32_t nb) {
  pdl_prologue();
  __shared__ uint32_t s[1024];
  const uint32_t tid = threadIdx.x;
  s[tid] = tid < nb ? bsum[tid] : 0u;
  __syncthreads();
  for (uint32_t o = 1; o < 1024; o <<= 1) {
    const uint32_t v = tid >= o ? s[tid - o] : 0u;
    __syncthreads();
    s[tid] += v;
    __syncthreads();
  }
  if (tid < nb) bsum[tid] = s[tid] - (tid < nb ? bsum[tid] : 0u);  // exclusive
}
__global__ void k_xscan_add(uint32_t* __restrict__ y, const uint32_t* n_ptr, uint32_t n_off,
                            const uint32_t* __restrict__ bsum) {
  pdl_prologue();
  const uint32_t n = *n_ptr - n_off;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] += bsum[i >> 12];
}
// total = y[n-1] + x[n-1] after the add pass
__global__ void k_xscan_total(const uint32_t* __restrict__ y, const uint32_t* __restrict__ x, const uint32_t* n_ptr,
                              uint32_t n_off, uint32_t* total_out) {
  pdl_prologue();
  const uint32_t n = *n_ptr - n_off;
  *total_out = n ? y[n - 1] + x[n - 1] : 0u;
}
// raw[nraw + i] = layer[i]; the single-thread k_samp_advance then moves nraw
__global__ void k_samp_append(const uint32_t* __restrict__ layer, const SampCounts* c, uint32_t* __restrict__ raw) {
  pdl_prologue();
  const uint32_t n = c->layer_n, base = c->nraw;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) raw[base + i] = layer[i];
}
__global__ void k_samp_advance(SampCounts* c) { pdl_prologue(); c->nraw += c->layer_n; }
__global__ void k_samp_out_count(const SampCounts* c, int64_t* count_dev) { pdl_prologue(); *count_dev = c->nout; }

}  // namespace lsm

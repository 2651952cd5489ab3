// tools/scope_peer_bench.cu — NEXT N4, cross-process half: the naive shared cache of PAPER.md
// P:269-277 (every GPU directly accesses and manages every other GPU's software cache through
// P2P mappings, so its cache-management operations must be system-scope) against LSM-GNN's
// communication layer (requests are routed to the home GPU, which alone touches its
// cache metadata with device-scope operations and sends the rows back).
//
// Two processes (ranks 0 and 1, forked before CUDA starts) each own one cache partition
// (tags, pin counts, way locks, 4 KiB lines) in a cudaMalloc'd arena exported with CUDA IPC;
// each maps the other's arena. Node v lives at home v mod 2, set (v/2) mod S. Modes:
//   naive_sys : each rank runs the cache protocol on the HOME's arena itself (own or peer
//               mapping) with .sys-scope acquire/release loads, atomics and CAS — the paper's
//               "naive implementation"; both ranks mutate both partitions concurrently.
//   naive_gpu : the same with .gpu scope (what the naive design would cost if device scope were
//               enough; it is not guaranteed coherent across GPUs — shown for the scope cost).
//   routed    : each rank stores its requests into the home's inbox (peer stores), then every
//               home runs the protocol on its OWN arena at .gpu scope and stores each row into
//               the requester's `out` (peer stores: the "features transferred to the requesting
//               GPU" of P:300).
// Hot: every request hits a resident line. Cold: every request is a distinct node never seen,
// filled from this rank's pinned host table (the storage stand-in), evicting a resident line.
// Protocol (all modes): hit = pin the way (refcount +1), re-check the tag, copy, unpin; miss =
// lock the victim way (CAS), wait for its pins to drain, fill the line, publish the tag
// (release), pin, unlock, copy, unpin. Every `out` row is checked against its node's pattern
// afterwards (row check). GB/s = both ranks' delivered bytes / the slower rank's device time.
//
// On a 1-GPU pool both processes share one B200 (run under MPS so they execute concurrently):
// the peer mapping is then an IPC mapping of the same HBM, so this measures the scope cost of
// the protocol (and the routed design's extra exchange), not NVLink. See profiles/.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scope_peer tools/scope_peer_bench.cu
#include <cuda_runtime.h>
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "[rank %d] %s: %s\n", g_rank, #x, cudaGetErrorString(e));    \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

static int g_rank = 0;
constexpr uint32_t kInv = 0xFFFFFFFFu;

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
__device__ __forceinline__ uint32_t atom_add(uint32_t* p, uint32_t v) {
  uint32_t r;
  if (SYS) asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  else asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
template <int SYS>
__device__ __forceinline__ uint32_t atom_cas(uint32_t* p, uint32_t c, uint32_t v) {
  uint32_t r;
  if (SYS) asm volatile("atom.acq_rel.sys.global.cas.b32 %0, [%1], %2, %3;" : "=r"(r) : "l"(p), "r"(c), "r"(v) : "memory");
  else asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(r) : "l"(p), "r"(c), "r"(v) : "memory");
  return r;
}

struct Part {  // one home's cache partition inside its arena
  uint32_t* tags;
  uint32_t* pins;
  uint32_t* lock;
  uint4* lines;
};
__host__ __device__ inline Part part_of(char* base, uint32_t L, uint32_t R) {
  Part p;
  p.tags = reinterpret_cast<uint32_t*>(base);
  p.pins = p.tags + L;
  p.lock = p.pins + L;
  p.lines = reinterpret_cast<uint4*>(base + (size_t)4 * 3 * L + 4096 - ((size_t)4 * 3 * L) % 4096);
  return p;
}
__host__ __device__ inline size_t arena_bytes(uint32_t L, uint32_t R) {
  const size_t meta = (size_t)4 * 3 * L;
  return meta + 4096 - meta % 4096 + (size_t)L * R + (size_t)2 * 1024 * 1024 * 4 /* inbox */ + 4096;
}
__host__ __device__ inline uint32_t pattern(uint32_t v, uint32_t k) { return v * 2654435761u ^ (k * 40503u + 7u); }

// The cache protocol for one request (node v) on partition p; the row goes to dst.
template <int SYS>
__device__ void access_one(Part p, uint32_t v, uint4* dst, const uint4* host, uint32_t S, uint32_t A, uint32_t nvec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t q = v >> 1, s = q % S;
  for (;;) {
    const uint32_t tg = lane < A ? ld_acq<SYS>(&p.tags[s * A + lane]) : kInv;
    const uint32_t hit = __ballot_sync(0xffffffffu, tg == v);
    uint32_t way, ok = 1;
    if (hit) {
      way = __ffs(hit) - 1;
      if (lane == 0) {
        atom_add<SYS>(&p.pins[s * A + way], 1u);
        ok = ld_acq<SYS>(&p.tags[s * A + way]) == v;  // still ours after the pin?
        if (!ok) atom_add<SYS>(&p.pins[s * A + way], 0xFFFFFFFFu);
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (!ok) continue;
    } else {
      way = (q / S) % A;
      if (lane == 0) {
        while (atom_cas<SYS>(&p.lock[s * A + way], 0u, 1u) != 0u) {
        }
        st_rel<SYS>(&p.tags[s * A + way], kInv);  // new hits on the old node now re-check and retry
        while (ld_acq<SYS>(&p.pins[s * A + way]) != 0u) {
        }
      }
      __syncwarp();
      uint4* line = p.lines + (size_t)(s * A + way) * nvec;
      const uint4* src = host + (size_t)v * nvec;  // storage row of node v
      for (uint32_t k = lane; k < nvec; k += 32) line[k] = src[k];
      __syncwarp();
      if (lane == 0) {
        st_rel<SYS>(&p.tags[s * A + way], v);
        atom_add<SYS>(&p.pins[s * A + way], 1u);
        st_rel<SYS>(&p.lock[s * A + way], 0u);
      }
      __syncwarp();
    }
    const uint4* line = p.lines + (size_t)(s * A + way) * nvec;
    for (uint32_t k = lane; k < nvec; k += 32) dst[k] = line[k];
    __syncwarp();
    if (lane == 0) atom_add<SYS>(&p.pins[s * A + way], 0xFFFFFFFFu);
    return;
  }
}

// naive: the requester manages the home's partition itself (own or peer mapping)
template <int SYS>
__global__ void k_naive(const uint32_t* __restrict__ req, uint32_t n, char* base0, char* base1, uint32_t L, uint32_t R,
                        const uint4* host, uint4* out, uint32_t S, uint32_t A) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = warp; e < n; e += nw) {
    const uint32_t v = req[e];
    access_one<SYS>(part_of((v & 1) ? base1 : base0, L, R), v, out + (size_t)e * (R / 16), host, S, A, R / 16);
  }
}
// routed, step 1: store each request (node, requester position) into its home's inbox
__global__ void k_route(const uint32_t* __restrict__ req, uint32_t n, uint32_t* inbox0, uint32_t* inbox1,
                        uint32_t* cnt0, uint32_t* cnt1, uint32_t me) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const uint32_t v = req[e];
    uint32_t* inbox = (v & 1) ? inbox1 : inbox0;
    const uint32_t pos = atomicAdd((v & 1) ? cnt1 : cnt0, 1u);
    inbox[2 * pos] = v;
    inbox[2 * pos + 1] = (me << 31) | e;
  }
}
// routed, step 2: the home serves its inbox on its own partition (.gpu) into the requesters' out
__global__ void k_home(const uint32_t* __restrict__ inbox, const uint32_t* cnt, char* mybase, uint32_t L, uint32_t R,
                       const uint4* host, uint4* out0, uint4* out1, uint32_t S, uint32_t A) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t n = *cnt;
  for (uint32_t e = warp; e < n; e += nw) {
    const uint32_t v = inbox[2 * e], o = inbox[2 * e + 1];
    uint4* dst = ((o >> 31) ? out1 : out0) + (size_t)(o & 0x7FFFFFFFu) * (R / 16);
    access_one<0>(part_of(mybase, L, R), v, dst, host, S, A, R / 16);
  }
}
__global__ void k_check(const uint32_t* __restrict__ req, uint32_t n, const uint32_t* out, uint32_t nw32,
                        unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n * nw32;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = (uint32_t)(i / nw32), k = (uint32_t)(i % nw32);
    if (out[i] != pattern(req[e], k)) atomicAdd(bad, 1ull);
  }
}
__global__ void k_fill_host_rows(uint32_t* rows, uint32_t nrows, uint32_t nw32) {
  // host row v holds node v's row: word k = pattern(v, k)
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)nrows * nw32;
       i += (uint64_t)gridDim.x * blockDim.x)
    rows[i] = pattern((uint32_t)(i / nw32), (uint32_t)(i % nw32));
}
// resident lines of home h: way w of set s holds node 2 (w S + s) + h
__global__ void k_fill_lines(uint32_t* lines, uint32_t L, uint32_t S, uint32_t A, uint32_t nw32, uint32_t h) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)L * nw32;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t line = (uint32_t)(i / nw32), s = line / A, w = line % A;
    lines[i] = pattern(2u * (w * S + s) + h, (uint32_t)(i % nw32));
  }
}

struct Pipe {
  int rd, wr;
  void send(const void* p, size_t n) {
    if (write(wr, p, n) != (ssize_t)n) exit(2);
  }
  void recv(void* p, size_t n) {
    size_t got = 0;
    while (got < n) {
      ssize_t r = read(rd, (char*)p + got, n - got);
      if (r <= 0) exit(3);
      got += (size_t)r;
    }
  }
  void barrier() {
    char c = 1;
    send(&c, 1);
    recv(&c, 1);
  }
};

int run(int rank, Pipe pp) {
  g_rank = rank;
  const uint32_t R = 4096, nw32 = R / 4, A = 32, S = 4096, L = S * A;  // 512 MiB per home
  const uint32_t n = 60000;                      // requests per rank per run
  const uint32_t NH = (1u << 19);                // host rows per rank (2 GiB): node v at row v
  CK(cudaSetDevice(0));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* arena;
  const size_t ab = arena_bytes(L, R);
  CK(cudaMalloc(&arena, ab));
  cudaIpcMemHandle_t mine, theirs;
  CK(cudaIpcGetMemHandle(&mine, arena));
  pp.send(&mine, sizeof mine);
  pp.recv(&theirs, sizeof theirs);
  char* peer;
  CK(cudaIpcOpenMemHandle((void**)&peer, theirs, cudaIpcMemLazyEnablePeerAccess));
  char* base[2] = {rank == 0 ? arena : peer, rank == 1 ? arena : peer};
  uint32_t* inbox_of[2];
  uint32_t* cnt_of[2];
  for (int h = 0; h < 2; ++h) {
    Part p = part_of(base[h], L, R);
    cnt_of[h] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(p.lines) + (size_t)L * R);
    inbox_of[h] = cnt_of[h] + 1024;
  }
  uint32_t* host;  // pinned rows of this rank's nodes (v = 2q + rank), read zero-copy on misses
  CK(cudaHostAlloc(&host, (size_t)NH * R, cudaHostAllocMapped));
  uint32_t* hostd;
  CK(cudaHostGetDevicePointer((void**)&hostd, host, 0));
  k_fill_host_rows<<<sms * 4, 256>>>(hostd, NH, nw32);
  // out buffers: exported too (routed mode stores rows into the requester's out)
  uint4* out;
  CK(cudaMalloc(&out, (size_t)n * R));
  cudaIpcMemHandle_t om, ot;
  CK(cudaIpcGetMemHandle(&om, out));
  pp.send(&om, sizeof om);
  pp.recv(&ot, sizeof ot);
  uint4* pout;
  CK(cudaIpcOpenMemHandle((void**)&pout, ot, cudaIpcMemLazyEnablePeerAccess));
  uint4* outs[2] = {rank == 0 ? out : pout, rank == 1 ? out : pout};
  uint32_t *req;
  unsigned long long* bad;
  CK(cudaMalloc(&req, n * 4));
  CK(cudaMalloc(&bad, 8));
  // resident state: way w of set s at home h holds node v = 2 (w S + s) + h (its row = pattern)
  std::vector<uint32_t> tag0(L);
  for (uint32_t i = 0; i < L; ++i) tag0[i] = 2u * ((i % A) * S + i / A) + (uint32_t)rank;
  std::vector<uint32_t> hot(n), cold(n);
  uint64_t x = 88172645463325252ull + rank;
  for (uint32_t i = 0; i < n; ++i) {  // hot: resident nodes of both homes; cold: distinct, never resident
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    hot[i] = 2u * (uint32_t)(x % L) + (uint32_t)(x >> 40 & 1);
    cold[i] = 2u * (L + 2u * i + (uint32_t)rank) + (uint32_t)((i >> 3) & 1);  // both homes; no two ranks alike
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"naive_sys", "naive_gpu", "routed"};
  for (int cold_mode = 0; cold_mode < 2; ++cold_mode) {
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e9;
      unsigned long long nbad = 0;
      for (int it = 0; it < 4; ++it) {
        Part mp = part_of(arena, L, R);
        CK(cudaMemcpy(mp.tags, tag0.data(), L * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(mp.pins, 0, L * 4));
        CK(cudaMemset(mp.lock, 0, L * 4));
        CK(cudaMemset(cnt_of[rank], 0, 4));
        k_fill_lines<<<sms * 4, 256>>>(reinterpret_cast<uint32_t*>(mp.lines), L, S, A, nw32, (uint32_t)rank);
        CK(cudaMemcpy(req, cold_mode ? cold.data() : hot.data(), n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(out, 0, (size_t)n * R));
        CK(cudaMemset(bad, 0, 8));
        CK(cudaDeviceSynchronize());
        pp.barrier();
        cudaEventRecord(a);
        if (mode == 0) k_naive<1><<<sms * 8, 256>>>(req, n, base[0], base[1], L, R, (const uint4*)hostd, out, S, A);
        if (mode == 1) k_naive<0><<<sms * 8, 256>>>(req, n, base[0], base[1], L, R, (const uint4*)hostd, out, S, A);
        if (mode == 2) {
          k_route<<<sms * 2, 256>>>(req, n, inbox_of[0], inbox_of[1], cnt_of[0], cnt_of[1], (uint32_t)rank);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          pp.barrier();  // every requester's IDs are in every inbox (host barrier: not timed below)
          float ms0;
          cudaEventElapsedTime(&ms0, a, b);
          cudaEventRecord(a);
          k_home<<<sms * 8, 256>>>(inbox_of[rank], cnt_of[rank], arena, L, R, (const uint4*)hostd, outs[0], outs[1], S,
                                   A);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms1;
          cudaEventElapsedTime(&ms1, a, b);
          pp.barrier();  // every home has stored every row
          float ms = ms0 + ms1;
          pp.send(&ms, 4);
          float other;
          pp.recv(&other, 4);
          ms = std::max(ms, other);
          if (it) best = std::min(best, ms);
        } else {
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          pp.barrier();
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          pp.send(&ms, 4);
          float other;
          pp.recv(&other, 4);
          ms = std::max(ms, other);
          if (it) best = std::min(best, ms);
        }
        k_check<<<sms * 4, 256>>>(req, n, reinterpret_cast<const uint32_t*>(out), nw32, bad);
        unsigned long long hb = 0;
        CK(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));
        nbad += hb;
      }
      unsigned long long obad;
      pp.send(&nbad, 8);
      pp.recv(&obad, 8);
      if (rank == 0)
        printf("%-6s %-10s %9.3f ms %9.1f GB/s   row check: %llu bad words\n", cold_mode ? "cold" : "hot",
               names[mode], best, 2.0 * n * R / best / 1e6, nbad + obad);
    }
  }
  CK(cudaGetLastError());
  cudaIpcCloseMemHandle(peer);
  cudaIpcCloseMemHandle(pout);
  pp.barrier();
  return 0;
}

int main() {
  int a[2], b[2];  // a: parent -> child, b: child -> parent
  if (pipe(a) || pipe(b)) return 1;
  const pid_t pid = fork();  // before any CUDA call
  if (pid == 0) {
    close(a[1]);
    close(b[0]);
    return run(1, Pipe{a[0], b[1]});
  }
  close(a[0]);
  close(b[1]);
  printf("scope_peer_bench: 2 processes, naive shared cache (.sys / .gpu on the home's partition through the peer "
         "mapping) vs routed to the home (.gpu, rows stored into the requester's out)\n");
  const int rc = run(0, Pipe{b[0], a[1]});
  int st = 0;
  waitpid(pid, &st, 0);
  return rc || !WIFEXITED(st) || WEXITSTATUS(st);
}

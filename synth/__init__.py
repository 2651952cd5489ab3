"""synth — seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This package holds NONE of the LSM-GNN method's arithmetic (no home/set hash,
no cache, no eviction, no window logic). It only produces the inputs the
paper's workloads have, as DESIGN.md §"Input recipe" states:

* ``plcite``        power-law "citation" graph (SURVEY.md §8(d) "Graph plcite"),
                    standing in for IGB (Table tab:dataset).
* ``static_scores`` u8 rank-quantised symmetrised degree (§4.2
                    "out-degree"; 1-byte width P:322 (draft); quantisation rule
                    SPEC.md S:82).
* ``sample_batch``  GraphSAGE-style multi-hop neighbour sampling (PAPER.md
                    P:161-166 §2.1; fanout P:603), DGL-style unique input nodes.
* ``features``      closed-form rows F(v) (C, ``synth/features.c``).
* ``make_trace``    per-(iteration, rank) node-ID lists = the gather batches,
                    which are also the window ("look-ahead") batches.

Random numbers are counter-based (splitmix64 keyed by the coordinates), so every
value is a pure function of (seed, coordinates) and both sides see identical
inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# ----------------------------------------------------------------------------- RNG
def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def hash_coords(seed: int, *coords) -> np.ndarray:
    """h(seed, c0, c1, ...) = splitmix64(...splitmix64(splitmix64(seed ^ c0) ^ c1)...)."""
    z = np.uint64(seed)
    for c in coords:
        z = splitmix64(np.asarray(c, dtype=np.uint64) ^ z)
    return z


def u01(h: np.ndarray) -> np.ndarray:
    """Uniform [0, 1) double from the top 53 bits."""
    return (np.asarray(h, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


# ----------------------------------------------------------------------------- graph
@dataclass
class Graph:
    num_nodes: int
    indptr: np.ndarray  # int64 [N+1]
    indices: np.ndarray  # int64/int32 [2*N*m]

    def degree(self) -> np.ndarray:
        return np.diff(self.indptr)


def plcite(num_nodes: int, m: int, seed_g: int = 1, seed_pi: int = 2, beta: float = 0.8,
           chunk: int = 1 << 22) -> Graph:
    """Power-law citation graph.

    Node v has m out-edges; edge k picks popularity rank
    rho = floor((u*((N+1)^(1-b) - 1) + 1)^(1/(1-b))) - 1, u = U01(h(seed_g, v, k)),
    target = pi(rho) with pi a seeded permutation; a self-loop is redrawn with
    counter k + m*j. The CSR is symmetrised (2*N*m entries), neighbours of each
    node ordered by (edge source, k).
    """
    N = int(num_nodes)
    assert N > m >= 1
    pi = np.random.default_rng(seed_pi).permutation(N).astype(np.int64)
    e = 1.0 - beta
    top = (N + 1.0) ** e - 1.0
    src = np.repeat(np.arange(N, dtype=np.int64), m)
    kk = np.tile(np.arange(m, dtype=np.int64), N)
    dst = np.empty(N * m, dtype=np.int64)
    for lo in range(0, N * m, chunk):
        hi = min(N * m, lo + chunk)
        s, k = src[lo:hi], kk[lo:hi]
        ctr = k.copy()
        tgt = np.empty(hi - lo, dtype=np.int64)
        todo = np.arange(hi - lo)
        j = 0
        while todo.size:
            u = u01(hash_coords(seed_g, s[todo], ctr[todo]))
            rho = np.floor((u * top + 1.0) ** (1.0 / e)).astype(np.int64) - 1
            np.clip(rho, 0, N - 1, out=rho)
            t = pi[rho]
            tgt[todo] = t
            bad = t == s[todo]
            todo = todo[bad]
            j += 1
            ctr[todo] = k[todo] + m * j
        dst[lo:hi] = tgt
    eid = np.arange(N * m, dtype=np.int64)  # = src*m + k, ascending in (src, k)
    a = np.concatenate([src, dst])
    b = np.concatenate([dst, src])
    key = a * np.int64(N * m) + np.concatenate([eid, eid])
    order = np.argsort(key, kind="stable")
    del key
    nb = b[order]
    counts = np.bincount(a, minlength=N)
    indptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    idx_dtype = np.int32 if N < (1 << 31) else np.int64
    return Graph(N, indptr, nb.astype(idx_dtype))


def quantize_scores(raw: np.ndarray) -> np.ndarray:
    """Rank quantisation to u8: node at rank r of N (ascending, stable
    by (value, node ID)) gets floor(256*r/N) clamped to 255; ties share the rank of
    their first occurrence."""
    raw = np.asarray(raw)
    N = raw.size
    if N == 0:
        return np.zeros(0, np.uint8)
    if raw.dtype.kind == "f" and not np.all(np.isfinite(raw)):
        raise ValueError("non-finite raw score")
    order = np.lexsort((np.arange(N), raw))
    sv = raw[order]
    first = np.ones(N, dtype=bool)
    first[1:] = sv[1:] != sv[:-1]
    rank_first = np.maximum.accumulate(np.where(first, np.arange(N), 0))
    q = np.minimum(255, (256 * rank_first.astype(np.int64)) // N).astype(np.uint8)
    out = np.empty(N, np.uint8)
    out[order] = q
    return out


def static_scores(g: Graph) -> np.ndarray:
    """u8 static score per node = rank-quantised symmetrised degree (higher = hotter)."""
    return quantize_scores(g.degree())


def reverse_pagerank(g: Graph, damping: float = 0.85, tol: float = 1e-6, max_iters: int = 100) -> np.ndarray:
    """PageRank on the edge-reversed graph. The CSR here is
    symmetrised, so reversal is the identity; kept for the config-5 score variant."""
    N = g.num_nodes
    deg = g.degree().astype(np.float64)
    src = np.repeat(np.arange(N), np.diff(g.indptr))
    dst = g.indices.astype(np.int64)
    x = np.full(N, 1.0 / N)
    for _ in range(max_iters):
        contrib = np.where(deg > 0, x / np.maximum(deg, 1), 0.0)
        y = np.bincount(dst, weights=contrib[src], minlength=N)
        dangling = x[deg == 0].sum()
        y = (1 - damping) / N + damping * (y + dangling / N)
        if np.abs(y - x).sum() < tol:
            x = y
            break
        x = y
    return x


# ----------------------------------------------------------------------------- sampler
def first_occurrence_unique(x: np.ndarray) -> np.ndarray:
    if x.size == 0:
        return x
    _, idx = np.unique(x, return_index=True)
    return x[np.sort(idx)]


def sample_batch(g: Graph, seeds: np.ndarray, fanout, seed_s: int, t: int, r: int,
                 dedup: bool = True) -> np.ndarray:
    """GraphSAGE multi-hop sampling: per frontier node and layer,
    min(f, deg) neighbours; deg <= f takes all, otherwise f draws uniform with
    replacement keyed (seed_s, t, r, layer, position, j). The next frontier is the
    first-occurrence unique set of this layer's samples. The returned list is the
    DGL-style first-occurrence dedup of seeds ∪ all layers (dedup=False keeps
    duplicates, for parity tests)."""
    seeds = np.asarray(seeds, dtype=np.int64)
    parts = [seeds]
    frontier = seeds
    for layer, f in enumerate(fanout):
        if frontier.size == 0:
            break
        deg = g.indptr[frontier + 1] - g.indptr[frontier]
        c = np.minimum(deg, f)
        tot = int(c.sum())
        p = np.repeat(np.arange(frontier.size, dtype=np.int64), c)
        starts = np.cumsum(c) - c
        j = np.arange(tot, dtype=np.int64) - np.repeat(starts, c)
        dp = deg[p]
        pos = np.where(dp <= f, j, 0)
        big = dp > f
        if big.any():
            hb = hash_coords(seed_s, np.full(int(big.sum()), t), np.full(int(big.sum()), r),
                             np.full(int(big.sum()), layer), p[big], j[big])
            pos[big] = np.floor(u01(hb) * dp[big]).astype(np.int64)
        nbr = g.indices[g.indptr[frontier[p]] + pos].astype(np.int64)
        parts.append(nbr)
        frontier = first_occurrence_unique(nbr)
    out = np.concatenate(parts)
    return first_occurrence_unique(out) if dedup else out


def epoch_seeds(num_nodes: int, epoch: int, seed_train: int = 3) -> np.ndarray:
    return np.random.default_rng(seed_train + epoch).permutation(num_nodes).astype(np.int64)


def make_trace(g: Graph, G: int, batch: int, fanout, iters: int, seed_train: int = 3,
               seed_s: int = 4, dedup: bool = True, t0: int = 0, ranks=None):
    """trace[t][r] = node IDs rank r gathers at iteration t (int64). Rank r at
    iteration t takes seeds perm[(t*G + r)*B : +B] of the epoch permutation
    (SPEC.md S:145); an epoch is ceil(N/(B*G)) iterations. `ranks` limits which ranks'
    lists are generated (the others are left empty) — a rank of a multi-process run only
    needs its own."""
    N = g.num_nodes
    per_epoch = -(-N // (batch * G))
    trace = []
    cache = {}
    for t in range(t0, t0 + iters):
        ep, te = divmod(t, per_epoch)
        if ep not in cache:
            cache.clear()
            cache[ep] = epoch_seeds(N, ep, seed_train)
        perm = cache[ep]
        row = []
        for r in range(G):
            if ranks is not None and r not in ranks:
                row.append(np.zeros(0, np.int64))
                continue
            lo = (te * G + r) * batch
            s = perm[lo:lo + batch]
            row.append(sample_batch(g, s, fanout, seed_s, t, r, dedup=dedup))
        trace.append(row)
    return trace


_PAR_GRAPH = None


def _trace_chunk(args):
    G, batch, fanout, t0, n, seed_train, seed_s, dedup, ranks = args
    return make_trace(_PAR_GRAPH, G, batch, fanout, n, seed_train, seed_s, dedup, t0, ranks)


def make_trace_parallel(g: Graph, G: int, batch: int, fanout, iters: int, seed_train: int = 3, seed_s: int = 4,
                        dedup: bool = True, procs: int | None = None, ranks=None):
    """make_trace split over worker processes (fork); identical output."""
    import multiprocessing as mp
    global _PAR_GRAPH
    procs = procs or min(16, os.cpu_count() or 1)
    if procs <= 1 or iters < 8:
        return make_trace(g, G, batch, fanout, iters, seed_train, seed_s, dedup, 0, ranks)
    _PAR_GRAPH = g
    step = -(-iters // procs)
    jobs = [(G, batch, fanout, t0, min(step, iters - t0), seed_train, seed_s, dedup, ranks)
            for t0 in range(0, iters, step)]
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        parts = pool.map(_trace_chunk, jobs)
    _PAR_GRAPH = None
    return [row for part in parts for row in part]


def window_union(batch_lists) -> np.ndarray:
    """B_k as a plain set union (sorted) of the ranks' lists — test helper."""
    if not batch_lists:
        return np.zeros(0, np.int64)
    return np.unique(np.concatenate([np.asarray(b, np.int64) for b in batch_lists]))


# ----------------------------------------------------------------------------- features
def _lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "libsynth.so")
        srcs = [os.path.join(_HERE, f) for f in ("features.c", "graphgen.c")]
        if not os.path.exists(so) or os.path.getmtime(so) < max(os.path.getmtime(p) for p in srcs):
            subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                                   "-o", so, *srcs, "-lm"])
        L = ctypes.CDLL(so)
        L.plcite_targets.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.plcite_csr.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.synth_fill_f32.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64]
        L.synth_fill_f32_ids.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64]
        L.synth_check_f32_ids.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)]
        L.synth_check_f32_ids.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def build() -> None:
    _lib()


def plcite_c(num_nodes: int, m: int, seed_g: int = 1, seed_pi: int = 2, beta: float = 0.8) -> Graph:
    """plcite() in C (OpenMP) for 100M-node graphs; same recipe and the same permutation
    (numpy's), int32 neighbour IDs."""
    N = int(num_nodes)
    pi = np.random.default_rng(seed_pi).permutation(N).astype(np.int64)
    tg = np.empty(N * m, np.int32)
    _lib().plcite_targets(N, m, seed_g, beta, pi.ctypes.data, tg.ctypes.data)
    del pi
    indptr = np.empty(N + 1, np.int64)
    indices = np.empty(2 * N * m, np.int32)
    _lib().plcite_csr(N, m, tg.ctypes.data, indptr.ctypes.data, indices.ctypes.data)
    return Graph(N, indptr, indices)


def fill_features(ptr: int, v0: int, nrows: int, D: int, seed_f: int = 5) -> None:
    """Write F(v0..v0+nrows-1) (fp32, D words per row) to host address ptr."""
    _lib().synth_fill_f32(ctypes.c_void_p(ptr), v0, nrows, D, seed_f)


def features(ids, D: int, seed_f: int = 5) -> np.ndarray:
    """Rows F(ids) as a uint32 [n, D] array."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty((ids.size, D), np.uint32)
    _lib().synth_fill_f32_ids(out.ctypes.data, ids.ctypes.data, ids.size, D, seed_f)
    return out


def features_python(v: int, D: int, seed_f: int = 5) -> np.ndarray:
    """Pure-numpy F(v) — used to pin the C generator."""
    j = np.arange(D, dtype=np.uint64)
    h = splitmix64(np.uint64(seed_f) ^ (np.uint64(v) * np.uint64(D) + j))
    return (np.uint64(0x3F800000) | (h >> np.uint64(41))).astype(np.uint32)


def check_rows(rows_u32: np.ndarray, ids, D: int, seed_f: int = 5):
    """(#bad rows, first bad index) of rows vs the closed form F(ids)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    rows_u32 = np.ascontiguousarray(rows_u32)
    fb = ctypes.c_int64(-1)
    bad = _lib().synth_check_f32_ids(rows_u32.ctypes.data, ids.ctypes.data, ids.size, D, seed_f, ctypes.byref(fb))
    return int(bad), int(fb.value)


# ----------------------------------------------------------------------------- configs
@dataclass
class Workload:
    """One BASELINE.json config, restated as numbers."""
    name: str
    G: int
    N: int
    D: int  # fp32 words per row; R = 4*D bytes
    m: int
    batch: int
    fanout: tuple
    lines_per_gpu: int
    ways: int
    window: int
    pvp: int
    victim_lines: int
    iters: int
    warmup: int = 0
    seeds: dict = field(default_factory=lambda: dict(g=1, pi=2, train=3, s=4, f=5))

    @property
    def R(self) -> int:
        return 4 * self.D


CONFIGS = {
    # configs[0]: 16,384 nodes / 131,072 edges, 128-dim fp32, fanout (10,5), batch 256,
    # 1,024 lines/GPU 8-way, 2 GPUs, 512-line victim buffer, 20 batches.
    "cfg1": Workload("cfg1", G=2, N=16384, D=128, m=8, batch=256, fanout=(10, 5),
                     lines_per_gpu=1024, ways=8, window=8, pvp=1, victim_lines=512, iters=20),
    # configs[1]: IGB-small-shaped, 1M nodes, 1024-dim fp32, fanout (10,5,5), batch 1024,
    # single B200, cache = 10% of features (100,000 lines, 32-way).
    "cfg2": Workload("cfg2", G=1, N=1_000_000, D=1024, m=12, batch=1024, fanout=(10, 5, 5),
                     lines_per_gpu=100_000, ways=32, window=256, pvp=0, victim_lines=16384 * 256,
                     iters=100, warmup=50),
    # configs[2]: IGB-medium-shaped, 10M nodes, 2 B200, PVP on, 4 GiB cache per GPU.
    "cfg3": Workload("cfg3", G=2, N=10_000_000, D=1024, m=12, batch=4096, fanout=(10, 5, 5),
                     lines_per_gpu=1_048_576, ways=32, window=256, pvp=1, victim_lines=4_194_304,
                     iters=100, warmup=50),
}

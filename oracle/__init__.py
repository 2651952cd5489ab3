"""oracle — CPU ORACLE for the LSM-GNN gather hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. It wraps ``lsm_oracle.c`` (plain
C, single thread) with ctypes and shares nothing with ``paper_2407_15264_b200``.

See ``lsm_oracle.c`` for the paper passages each step follows, DESIGN.md
§"Readings" for every interpretation taken, and DESIGN.md §"Oracle pins" for what
pins each function (all functions are pinned; none is "parity unpinned" except
where DESIGN.md says so).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "lsm_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "lsm_sampler.c")]

HYBRID, STATIC, LRU, RR, DYNAMIC = range(5)
POLICIES = {"hybrid": HYBRID, "static": STATIC, "lru": LRU, "rr": RR, "dynamic": DYNAMIC}
NOREUSE, FAR, FRESH, NEAR = range(4)

COUNT_FIELDS = ["iter", "requests", "peer_requests", "unique", "hits", "victim_hits", "storage_reads",
                "inserted", "bypassed", "evictions", "evict_noreuse", "evict_far", "evict_fresh", "evict_near",
                "victim_admitted", "victim_dropped", "evicted_no_reuse", "pvp_prefetched", "pvp_unused",
                "bytes_out", "bytes_nvlink", "bytes_h2d_storage", "bytes_h2d_pvp", "bytes_d2h_victim"]


class _Config(ctypes.Structure):
    _fields_ = [("G", ctypes.c_int32), ("N", ctypes.c_int64), ("R", ctypes.c_int32), ("L", ctypes.c_int64),
                ("A", ctypes.c_int32), ("policy", ctypes.c_int32), ("pvp", ctypes.c_int32), ("W", ctypes.c_int32),
                ("T", ctypes.c_int32), ("reinsert", ctypes.c_int32), ("V", ctypes.c_int64),
                ("P", ctypes.c_int32)]


_LIB = None


def build() -> str:
    """Compile liboracle.so (gcc -O2, single-threaded). ORACLE_SO_OVERRIDE names another
    build of the same sources to load instead (tests/test_oracle_mutants.py loads
    deliberately broken builds that the pins must reject)."""
    override = os.environ.get("ORACLE_SO_OVERRIDE")
    if override:
        return override
    deps = _SRCS + [os.path.join(_HERE, "lsm_oracle.h")]
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(p) for p in deps):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _SO, *_SRCS])
    return _SO


def _lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.orc_create.argtypes = [ctypes.POINTER(_Config), vp]
        L.orc_create.restype = vp
        L.orc_destroy.argtypes = [vp]
        L.orc_error.argtypes = [vp]
        L.orc_error.restype = ctypes.c_char_p
        L.orc_sets.argtypes = [vp]
        L.orc_sets.restype = i64
        L.orc_feed_window.argtypes = [vp, i64, vp, vp]
        L.orc_gather.argtypes = [vp, i64, vp, vp, vp, vp, vp]
        L.orc_pvp_prefetch.argtypes = [vp, i64]
        L.orc_dump_tags.argtypes = [vp, i32, vp, vp]
        L.orc_dump_queue.argtypes = [vp, i32, i32, vp, vp, i64]
        L.orc_dump_queue.restype = i64
        L.orc_dump_staging.argtypes = [vp, i32, vp, i64]
        L.orc_dump_staging.restype = i64
        L.orc_next_use.argtypes = [vp, i64, i64]
        L.orc_next_use.restype = i64
        L.orc_dump_events.argtypes = [vp, vp, i64]
        L.orc_dump_events.restype = i64
        L.orc_sample.argtypes = [vp, vp, i64, vp, i64, vp, i32, ctypes.c_uint64, i64, i32, vp, i64]
        L.orc_sample.restype = i64
        _LIB = L
    return _LIB


def _concat(lists):
    lists = [np.ascontiguousarray(x, dtype=np.int64) for x in lists]
    offs = np.zeros(len(lists) + 1, np.int64)
    offs[1:] = np.cumsum([x.size for x in lists])
    ids = np.concatenate(lists) if lists and offs[-1] > 0 else np.zeros(1, np.int64)
    return np.ascontiguousarray(ids), offs


class Oracle:
    """One simulated box of G homes. ``gather(t, lists)`` returns (counts[G, 24], out)."""

    def __init__(self, G, N, R, L, A, scores, policy="hybrid", pvp=0, W=8, T=0, reinsert=1, V=0, P=1):
        self.G, self.N, self.R, self.L, self.A, self.W = G, N, R, L, A, W
        self.policy = POLICIES[policy] if isinstance(policy, str) else policy
        cfg = _Config(G, N, R, L, A, self.policy, pvp, W, T, reinsert, V, P)
        self._scores = np.ascontiguousarray(scores, dtype=np.uint8)
        assert self._scores.size == N
        self._o = _lib().orc_create(ctypes.byref(cfg), self._scores.ctypes.data)
        self.S = _lib().orc_sets(self._o)
        if self.S <= 0:
            msg = _lib().orc_error(self._o).decode()
            _lib().orc_destroy(self._o)
            self._o = None
            raise ValueError(msg)

    def __del__(self):
        if getattr(self, "_o", None):
            _lib().orc_destroy(self._o)
            self._o = None

    def _err(self, rc):
        if rc != 0:
            raise RuntimeError(f"oracle error {rc}: {_lib().orc_error(self._o).decode()}")

    def feed(self, k: int, lists) -> None:
        ids, offs = _concat(lists)
        self._err(_lib().orc_feed_window(self._o, k, ids.ctypes.data, offs.ctypes.data))

    def gather(self, t: int, lists, table: np.ndarray | None = None):
        ids, offs = _concat(lists)
        counts = np.zeros((self.G, len(COUNT_FIELDS)), np.uint64)
        out = None
        tp = op = None
        if table is not None:
            out = np.empty((int(offs[-1]), self.R), np.uint8)
            tp, op = table.ctypes.data, out.ctypes.data
        self._err(_lib().orc_gather(self._o, t, ids.ctypes.data, offs.ctypes.data, tp, op, counts.ctypes.data))
        return counts, out

    def pvp_prefetch(self, t: int) -> None:
        self._err(_lib().orc_pvp_prefetch(self._o, t))

    # -- inspection
    def tags(self, g: int):
        tags = np.empty(self.L, np.int64)
        lu = np.empty(self.L, np.int64)
        _lib().orc_dump_tags(self._o, g, tags.ctypes.data, lu.ctypes.data)
        return tags.reshape(self.S, self.A), lu.reshape(self.S, self.A)

    def queue(self, g: int, k: int):
        cap = 1 << 20
        nodes = np.empty(cap, np.int64)
        reuse = np.empty(cap, np.int64)
        n = _lib().orc_dump_queue(self._o, g, k, nodes.ctypes.data, reuse.ctypes.data, cap)
        return nodes[:n].copy(), reuse[:n].copy()

    def staging(self, g: int):
        cap = 1 << 20
        nodes = np.empty(cap, np.int64)
        n = _lib().orc_dump_staging(self._o, g, nodes.ctypes.data, cap)
        return nodes[:n].copy()

    def next_use(self, v: int, t: int) -> int:
        return int(_lib().orc_next_use(self._o, v, t))

    def events(self):
        n = _lib().orc_dump_events(self._o, None, 0)
        buf = np.empty((max(n, 1), 7), np.int64)
        _lib().orc_dump_events(self._o, buf.ctypes.data, n)
        return buf[:n]


def sample_batch(indptr, indices, seeds, fanout, seed_s: int, t: int, r: int) -> np.ndarray:
    """NEXT N3 oracle: GraphSAGE sampling of one rank's batch (lsm_sampler.c)."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    seeds = np.ascontiguousarray(seeds, np.int64)
    fan = np.ascontiguousarray(fanout, np.int32)
    cap = int(seeds.size * (1 + np.cumprod(fan.astype(np.int64)).sum())) + 1
    out = np.empty(cap, np.int64)
    n = _lib().orc_sample(indptr.ctypes.data, indices.ctypes.data, indptr.size - 1, seeds.ctypes.data, seeds.size,
                          fan.ctypes.data, fan.size, seed_s, t, r, out.ctypes.data, cap)
    if n < 0:
        raise RuntimeError("sample overflow")
    return out[:n].copy()


def run_trace(orc: Oracle, trace, table=None, pvp=None, feed=True):
    """The canonical driver: bootstrap-feed B_1..B_W, then for each t:
    gather(t); prefetch: PVP copy for t+1 and feed B_{t+1+W} (empty past the end).
    Returns counts[T, G, 24] (and the list of outs if table is given)."""
    K = len(trace)
    W = orc.W
    empty = [np.zeros(0, np.int64)] * orc.G
    if feed:
        for k in range(1, W + 1):
            orc.feed(k, trace[k] if k < K else empty)
    allc, outs = [], []
    for t in range(K):
        c, out = orc.gather(t, trace[t], table)
        allc.append(c)
        outs.append(out)
        orc.pvp_prefetch(t)
        if feed:
            k = t + 1 + W
            orc.feed(k, trace[k] if k < K else empty)
    allc = np.stack(allc) if allc else np.zeros((0, orc.G, len(COUNT_FIELDS)), np.uint64)
    return (allc, outs) if table is not None else allc

"""Thin ctypes binding of liblsmgnn.so (include/lsmgnn.h) — argument marshalling only.

Every step of the gather path runs in the library's CUDA kernels. There is no CPU
fallback: if the shared library is missing or CUDA is unavailable, construction raises.
PyTorch supplies device memory, streams and the process group (bootstrap only).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "liblsmgnn.so")

F32, F16, BF16 = 0, 1, 2
POLICY = {"hybrid": 0, "static": 1, "lru": 2, "rr": 3, "dynamic": 4}
STATS_FIELDS = ["iter", "requests", "peer_requests", "unique", "hits", "victim_hits", "storage_reads",
                "inserted", "bypassed", "evictions", "evict_noreuse", "evict_far", "evict_fresh", "evict_near",
                "victim_admitted", "victim_dropped", "evicted_no_reuse", "pvp_prefetched", "pvp_unused",
                "bytes_out", "bytes_nvlink", "bytes_h2d_storage", "bytes_h2d_pvp", "bytes_d2h_victim"]
EXPORTS = ["lsmgnn_bind", "lsmgnn_set_options", "lsmgnn_init", "lsmgnn_attach_storage", "lsmgnn_handle_bytes",
           "lsmgnn_export_handle", "lsmgnn_connect", "lsmgnn_gather", "lsmgnn_gather_host", "lsmgnn_prefetch",
           "lsmgnn_stats", "lsmgnn_stats_history", "lsmgnn_kernel_launches", "lsmgnn_finalize",
           "lsmgnn_last_error", "lsmgnn_profile", "lsmgnn_profile_read", "lsmgnn_sampler_attach", "lsmgnn_sample",
           "lsmgnn_prefetch_dev", "lsmgnn_graph_capture", "lsmgnn_graph_replay", "lsmgnn_debug_state",
           "lsmgnn_sampler_place", "lsmgnn_plan_handle", "lsmgnn_check_handles", "lsmgnn_disconnect"]
PHASES = ["route", "dedup", "probe_replace", "admit", "fill", "pull", "window", "pvp"]


class Options(ctypes.Structure):
    _fields_ = [("version", ctypes.c_int32), ("policy", ctypes.c_int32), ("pvp", ctypes.c_int32),
                ("window", ctypes.c_int32), ("threshold", ctypes.c_int32), ("update_period", ctypes.c_int32),
                ("reinsert_victims", ctypes.c_int32), ("max_batch_ids", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in STATS_FIELDS]

    def as_array(self) -> np.ndarray:
        return np.array([getattr(self, n) for n in STATS_FIELDS], np.uint64)


class LsmGnnError(RuntimeError):
    pass


_LIB = None


def load_library(path: str = SO_PATH) -> ctypes.CDLL:
    """dlopen liblsmgnn.so and declare the C-ABI. Raises if it is missing (no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise LsmGnnError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "lsmgnn_bind": ([i32, i32, i32], i32),
        "lsmgnn_set_options": ([ctypes.POINTER(Options)], i32),
        "lsmgnn_init": ([i64, i32, i32, i64, i32, i64, vp], i32),
        "lsmgnn_attach_storage": ([vp, ctypes.c_char_p], i32),
        "lsmgnn_handle_bytes": ([], ctypes.c_size_t),
        "lsmgnn_export_handle": ([vp, ctypes.c_size_t], i32),
        "lsmgnn_connect": ([vp, i32], i32),
        "lsmgnn_gather": ([vp, i64, vp, vp], i32),
        "lsmgnn_gather_host": ([vp, i64, vp, vp], i32),
        "lsmgnn_prefetch": ([vp, vp, i32, i64, vp], i32),
        "lsmgnn_stats": ([ctypes.POINTER(Stats), i32], i32),
        "lsmgnn_stats_history": ([ctypes.POINTER(Stats), i64, i64], i32),
        "lsmgnn_kernel_launches": ([], i64),
        "lsmgnn_finalize": ([], i32),
        "lsmgnn_last_error": ([], ctypes.c_char_p),
        "lsmgnn_profile": ([i32], i32),
        "lsmgnn_profile_read": ([vp, vp], i32),
        "lsmgnn_sampler_attach": ([vp, vp, i64, i64], i32),
        "lsmgnn_sample": ([vp, i64, vp, i32, ctypes.c_uint64, i64, i32, vp, i64, vp, vp], i32),
        "lsmgnn_prefetch_dev": ([vp, vp, i64, vp], i32),
        "lsmgnn_graph_capture": ([vp, vp, i32, vp, vp], i32),
        "lsmgnn_graph_replay": ([vp], i32),
        "lsmgnn_debug_state": ([i32, vp, i64], i32),
        "lsmgnn_sampler_place": ([i32], i32),
        "lsmgnn_plan_handle": ([ctypes.POINTER(Options), i64, i32, i32, i64, i32, i64, i32, i32, vp, ctypes.c_size_t],
                               i32),
        "lsmgnn_check_handles": ([vp, i32, vp], i32),
        "lsmgnn_disconnect": ([], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise LsmGnnError(f"lsmgnn error {rc}: {_LIB.lsmgnn_last_error().decode()}")


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def plan_handle(num_nodes, feat_dim, lines_per_gpu, ways, victim_lines=0, *, rank=0, world=1, dtype=F32,
                policy="hybrid", pvp=0, window=256, threshold=0, reinsert=1, max_batch_ids=1 << 20, period=1) -> bytes:
    """Host-only (no GPU): the layout handle rank `rank` of `world` would export for these
    lsmgnn_init arguments (lsmgnn_plan_handle); raises LsmGnnError for arguments init rejects."""
    L = load_library()
    opt = Options(1, POLICY[policy] if isinstance(policy, str) else int(policy), int(pvp), int(window),
                  int(threshold), int(period), int(reinsert), int(max_batch_ids))
    nb = L.lsmgnn_handle_bytes()
    buf = ctypes.create_string_buffer(nb)
    _check(L.lsmgnn_plan_handle(ctypes.byref(opt), int(num_nodes), int(feat_dim), int(dtype), int(lines_per_gpu),
                                int(ways), int(victim_lines), int(rank), int(world), buf, nb))
    return bytes(buf.raw)


def check_handles(blobs, mine: bytes) -> int:
    """lsmgnn_connect's validation of the all-gathered blobs (rank order) against `mine`:
    returns the C return code (0 or LSMGNN_ECOMM = -6) without raising."""
    L = load_library()
    allb = ctypes.create_string_buffer(b"".join(blobs), max(1, sum(len(b) for b in blobs)))
    me = ctypes.create_string_buffer(mine, len(mine))
    return int(L.lsmgnn_check_handles(allb, len(blobs), me))


def last_error() -> str:
    return load_library().lsmgnn_last_error().decode()


class LsmGnn:
    """One rank's home of the box-wide shared cache (the library is a per-process singleton).

    Typical use (one process per GPU):
        c = LsmGnn(num_nodes, feat_dim, lines_per_gpu, ways, victim_lines, scores,
                   policy="hybrid", pvp=1, window=256, max_batch_ids=..., group=pg)
        c.attach_storage(host_rows_of_my_home)     # pinned torch tensor or numpy array
        c.prefetch(window_batches[1:W+1], first_iter=1)
        for t: c.gather(ids_t, out_t); c.prefetch([ids_{t+1+W}], first_iter=t+1+W)
    """

    def __init__(self, num_nodes, feat_dim, lines_per_gpu, ways, victim_lines=0, scores=None, *, dtype=F32,
                 policy="hybrid", pvp=0, window=256, threshold=0, reinsert=1, max_batch_ids=1 << 20, period=1,
                 rank=0, world=1, device=None, group=None):
        import torch
        if not torch.cuda.is_available():
            raise LsmGnnError("CUDA device required: the gather path has no CPU fallback")
        L = load_library()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.rank, self.world = rank, world
        self._group = group
        self.num_nodes, self.feat_dim = int(num_nodes), int(feat_dim)
        self.row_bytes = feat_dim * (4 if dtype == F32 else 2)
        self.window = int(window)
        self._keep = []
        _check(L.lsmgnn_bind(rank, world, device))
        opt = Options(1, POLICY[policy] if isinstance(policy, str) else int(policy), int(pvp), int(window),
                      int(threshold), int(period), int(reinsert), int(max_batch_ids))
        _check(L.lsmgnn_set_options(ctypes.byref(opt)))
        sp = None
        if scores is not None:
            s = np.ascontiguousarray(scores, dtype=np.uint8)
            assert s.size == num_nodes
            sp = s.ctypes.data
        _check(L.lsmgnn_init(int(num_nodes), int(feat_dim), int(dtype), int(lines_per_gpu), int(ways),
                             int(victim_lines), sp))
        if world > 1:
            self._connect(group)

    def _connect(self, group) -> None:
        import torch.distributed as dist
        L = _LIB
        nb = L.lsmgnn_handle_bytes()
        buf = ctypes.create_string_buffer(nb)
        _check(L.lsmgnn_export_handle(buf, nb))
        blobs = [None] * self.world
        dist.all_gather_object(blobs, bytes(buf.raw), group=group)
        allb = ctypes.create_string_buffer(b"".join(blobs), nb * self.world)
        _check(L.lsmgnn_connect(allb, self.world))
        dist.barrier(group=group)

    def attach_storage(self, host_rows) -> None:
        """host_rows: this home's rows (node rank + k*world at row k), host memory."""
        import torch
        if isinstance(host_rows, torch.Tensor):
            assert host_rows.device.type == "cpu" and host_rows.is_contiguous()
            ptr = host_rows.data_ptr()
        else:
            assert host_rows.flags["C_CONTIGUOUS"]
            ptr = host_rows.ctypes.data
        self._keep.append(host_rows)
        _check(_LIB.lsmgnn_attach_storage(ctypes.c_void_p(ptr), None))

    def attach_storage_file(self, path: str) -> None:
        """File tier (N2): this home's rows in a file, row k at byte offset k*R (same order as
        attach_storage). Read with O_DIRECT when R % 512 == 0, into a pinned bounce buffer."""
        _check(_LIB.lsmgnn_attach_storage(None, os.fsencode(path)))

    def gather(self, ids, out, stream=None) -> None:
        """out[i] = table[ids[i]]; ids: int64 CUDA tensor, out: CUDA tensor of n*R bytes."""
        assert ids.is_cuda and ids.dtype.itemsize == 8 and ids.is_contiguous()
        assert out.is_cuda and out.is_contiguous() and out.numel() * out.element_size() >= ids.numel() * self.row_bytes
        _check(_LIB.lsmgnn_gather(ctypes.c_void_p(ids.data_ptr()), ids.numel(), ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(_stream_ptr(stream))))

    def gather_host(self, ids_np_or_tensor, out_host, stream=None) -> None:
        """End-to-end variant: host IDs in, host rows out (copies inside the call)."""
        import torch
        ids = ids_np_or_tensor
        ip = ids.data_ptr() if isinstance(ids, torch.Tensor) else ids.ctypes.data
        n = ids.numel() if isinstance(ids, torch.Tensor) else ids.size
        op = out_host.data_ptr() if isinstance(out_host, torch.Tensor) else out_host.ctypes.data
        _check(_LIB.lsmgnn_gather_host(ctypes.c_void_p(ip), int(n), ctypes.c_void_p(op),
                                       ctypes.c_void_p(_stream_ptr(stream))))

    def prefetch(self, batches, first_iter: int, stream=None) -> None:
        """Feed window batches (list of int64 CUDA tensors) for iterations first_iter.. ."""
        import contextlib
        import torch
        # the concatenation (a device copy) is ordered on the stream the library will read it on
        with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
            if len(batches):
                flat = torch.cat([b.reshape(-1) for b in batches]) if len(batches) > 1 else batches[0].reshape(-1)
                flat = flat.contiguous()
            else:
                flat = torch.zeros(1, dtype=torch.int64, device=self.device)
        offs = np.zeros(len(batches) + 1, np.int64)
        offs[1:] = np.cumsum([b.numel() for b in batches])
        self._last_flat = flat  # keep alive until the stream consumes it
        _check(_LIB.lsmgnn_prefetch(ctypes.c_void_p(flat.data_ptr()), offs.ctypes.data_as(ctypes.c_void_p),
                                    len(batches), int(first_iter), ctypes.c_void_p(_stream_ptr(stream))))

    def stats(self, scope: int = 0) -> dict:
        s = Stats()
        _check(_LIB.lsmgnn_stats(ctypes.byref(s), scope))
        return {n: int(getattr(s, n)) for n in STATS_FIELDS}

    def history(self, first: int, count: int) -> np.ndarray:
        arr = (Stats * max(count, 1))()
        _check(_LIB.lsmgnn_stats_history(arr, first, count))
        return np.stack([arr[i].as_array() for i in range(count)]) if count else np.zeros((0, 24), np.uint64)

    def graph_capture(self, batches, out, stream=None):
        """CUDA-graph step (G = 1): capture gather(t) + window feed of t+1+W over the ring of
        device batches `batches` (iteration k uses batches[k % len]); returns nothing — replay
        with graph_replay(). Keeps the pointer/count tables alive."""
        import torch
        dev = out.device
        self._ring_ptrs = torch.tensor([b.data_ptr() for b in batches], dtype=torch.int64, device=dev)
        self._ring_n = torch.tensor([b.numel() for b in batches], dtype=torch.int64, device=dev)
        self._ring_keep = list(batches)
        _check(_LIB.lsmgnn_graph_capture(ctypes.c_void_p(self._ring_ptrs.data_ptr()),
                                         ctypes.c_void_p(self._ring_n.data_ptr()), len(batches),
                                         ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))))

    def debug_state(self, what: int, count: int) -> np.ndarray:
        """Cache state for tests: 0 tags, 1 last use, 2 victim-queue lengths, 3 queue nodes."""
        buf = np.zeros(max(count, 1), np.uint32)
        _check(_LIB.lsmgnn_debug_state(int(what), buf.ctypes.data, buf.size))
        return buf[:count]

    def graph_replay(self, stream=None) -> None:
        _check(_LIB.lsmgnn_graph_replay(ctypes.c_void_p(_stream_ptr(stream))))

    @staticmethod
    def profile(enable: bool) -> None:
        _check(load_library().lsmgnn_profile(1 if enable else 0))

    @staticmethod
    def profile_read() -> dict:
        ms = np.zeros(len(PHASES), np.float64)
        cnt = np.zeros(len(PHASES), np.int64)
        _check(load_library().lsmgnn_profile_read(ms.ctypes.data, cnt.ctypes.data))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(PHASES)}

    @staticmethod
    def kernel_launches() -> int:
        return int(load_library().lsmgnn_kernel_launches())

    def __enter__(self) -> "LsmGnn":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def close(self) -> None:
        """Free this rank's home. With G > 1 every rank first drains its GPU work and meets the
        others at a barrier, so no peer is still pulling from memory about to be freed."""
        if _LIB is None or getattr(self, "_closed", False):
            return  # (a second close must not free a home created after this one)
        self._closed = True
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self._group)  # nobody pulls from a peer any more
            _LIB.lsmgnn_disconnect()         # close this rank's mappings of the peers' arenas
            dist.barrier(group=self._group)  # every mapping of every arena is closed
        _LIB.lsmgnn_finalize()


class Sampler:
    """NEXT N3: GPU GraphSAGE sampler over a host-pinned CSR (lsmgnn_sampler_attach/_sample)."""

    def __init__(self, indptr: np.ndarray, indices: np.ndarray, pin: bool = True):
        """pin=True copies the CSR into pinned torch tensors; pin=False hands the caller's arrays
        (e.g. memory-mapped shared memory) to the library, which page-locks them in place."""
        import torch
        if not torch.cuda.is_available():
            raise LsmGnnError("CUDA device required")
        load_library()
        if pin:
            self.indptr = torch.from_numpy(np.ascontiguousarray(indptr, np.int64)).pin_memory()
            self.indices = torch.from_numpy(np.ascontiguousarray(indices, np.int32)).pin_memory()
            self._ptrs = (self.indptr.data_ptr(), self.indices.data_ptr(), self.indptr.numel() - 1,
                          self.indices.numel())
        else:
            assert indptr.dtype == np.int64 and indices.dtype == np.int32
            assert indptr.flags["C_CONTIGUOUS"] and indices.flags["C_CONTIGUOUS"]
            self.indptr, self.indices = indptr, indices
            self._ptrs = (indptr.ctypes.data, indices.ctypes.data, indptr.size - 1, indices.size)
        self.reattach()

    def reattach(self) -> None:
        """(Re)register the CSR with the library (lsmgnn_finalize forgets it)."""
        ip, ix, n, nnz = self._ptrs
        _check(load_library().lsmgnn_sampler_attach(ctypes.c_void_p(ip), ctypes.c_void_p(ix), n, nnz))

    def place(self, in_hbm: bool) -> None:
        """Read the CSR from HBM (a library-owned copy) or from pinned host memory (UVA)."""
        _check(_LIB.lsmgnn_sampler_place(1 if in_hbm else 0))

    @staticmethod
    def bound(nseeds: int, fanout) -> int:
        b, p = nseeds, nseeds
        for f in fanout:
            p *= f
            b += p
        return b

    def sample(self, seeds, fanout, seed: int, t: int, r: int, out=None, count=None, stream=None):
        """Returns (out int64 CUDA tensor of capacity bound, count int64 CUDA tensor [1])."""
        import torch
        dev = seeds.device
        if out is None:
            out = torch.empty(max(1, self.bound(seeds.numel(), fanout)), dtype=torch.int64, device=dev)
        if count is None:
            count = torch.zeros(1, dtype=torch.int64, device=dev)
        fan = np.ascontiguousarray(fanout, np.int32)
        _check(_LIB.lsmgnn_sample(ctypes.c_void_p(seeds.data_ptr()), seeds.numel(), fan.ctypes.data_as(ctypes.c_void_p),
                                  fan.size, seed, t, r, ctypes.c_void_p(out.data_ptr()), out.numel(),
                                  ctypes.c_void_p(count.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))))
        return out, count


def prefetch_dev(ids, count, first_iter: int, stream=None) -> None:
    """Window feed of one device-resident batch (any G; with G > 1 every rank calls it for the same first_iter)."""
    _check(_LIB.lsmgnn_prefetch_dev(ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(count.data_ptr()), int(first_iter),
                                    ctypes.c_void_p(_stream_ptr(stream))))

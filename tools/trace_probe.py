"""Timeline of two consecutive hit-path steps (experiments only): needs a liblsmgnn.so built with
-DLSMGNN_TRACE (ab/liblsmgnn_trace.so copied in place). Prints, per kernel and iteration, the
earliest CTA start and latest CTA end relative to the first k_dedup start (microseconds)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402


def main():
    wl = synth.CONFIGS["cfg2"]
    W = wl.window
    iters = W + 1 + 70
    _, trace, scores = bench.build_inputs(wl, 1, 0, iters)
    import torch
    from paper_2407_15264_b200 import LsmGnn, binding
    from tests.harness import table_for
    dev = torch.device("cuda", 0)
    table = table_for(wl.N, wl.D, wl.seeds["f"], pinned=True)
    ids_d = [torch.from_numpy(np.asarray(trace[t][0], np.int64)).to(dev) for t in range(iters)]
    out = torch.empty((max(x.numel() for x in ids_d), wl.R), dtype=torch.uint8, device=dev)
    lines = wl.N - wl.N % wl.ways
    c = LsmGnn(wl.N, wl.D, lines, wl.ways, 0, scores, policy="hybrid", pvp=0, window=W,
               max_batch_ids=max(x.numel() for x in ids_d), device=0)
    c.attach_storage(table)
    lib = binding._LIB
    lib.lsmgnn_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int32]
    buf = (ctypes.c_ulonglong * 32)()
    c.prefetch(ids_d[1:W + 1], first_iter=1)
    names = ["dedup", "dedup_done", "set", "serve", "route_local"]
    for t in range(60):
        if t == 50:
            torch.cuda.synchronize()
            lib.lsmgnn_debug_trace(buf, 1)
        c.gather(ids_d[t], out)
        c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
        if t == 51:
            torch.cuda.synchronize()
            lib.lsmgnn_debug_trace(buf, 0)
            a = np.frombuffer(buf, dtype=np.uint64).reshape(8, 2, 2).astype(np.int64)
            base = a[0, 0, 0]
            for k, nm in enumerate(names):
                for p in (0, 1):
                    s, e = a[k, p]
                    if s == -1 and e == 0:
                        continue
                    print(f"{nm:12s} par {p}: start {(s - base) / 1e3 if s != -1 else float('nan'):9.2f}  end {(e - base) / 1e3:9.2f} us")
            # a second sample
            lib.lsmgnn_debug_trace(buf, 1)
    c.close()


if __name__ == "__main__":
    main()

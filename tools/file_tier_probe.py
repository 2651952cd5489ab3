"""File tier (N2) probe: configs[1] gathers with the backing rows in a file, O_DIRECT, for a
few I/O thread counts (LSMGNN_IO_THREADS). Prints one JSON line per setting."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synth
    from paper_2407_15264_b200 import LsmGnn
    from tests.harness import write_table_file
    wl = synth.CONFIGS["cfg2"]
    W, warm, steps = wl.window, 2, 5
    g = synth.plcite(wl.N, wl.m)
    tr = synth.make_trace(g, 1, wl.batch, wl.fanout, W + warm + steps + 2)
    scores = synth.static_scores(g)
    ids = [torch.from_numpy(np.asarray(x[0], np.int64)).cuda() for x in tr]
    path = os.path.join(sys.argv[1] if len(sys.argv) > 1 else "/tmp", "lsmgnn_probe.bin")
    write_table_file(path, wl.N, wl.D, wl.seeds["f"])
    out = torch.empty((max(x.numel() for x in ids), wl.R), dtype=torch.uint8, device="cuda")
    for nt in (16, 64, 128):
        os.environ["LSMGNN_IO_THREADS"] = str(nt)
        c = LsmGnn(wl.N, wl.D, wl.lines_per_gpu, wl.ways, 0, scores, window=W, max_batch_ids=max(x.numel() for x in ids))
        c.attach_storage_file(path)
        c.prefetch(ids[1:W + 1], first_iter=1)
        for t in range(warm + steps):
            if t == warm:
                torch.cuda.synchronize()
                s0, t0 = c.stats(1), time.perf_counter()
            c.gather(ids[t], out)
            c.prefetch([ids[t + 1 + W]], first_iter=t + 1 + W)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        s1 = c.stats(1)
        c.close()
        sb = s1["bytes_h2d_storage"] - s0["bytes_h2d_storage"]
        print(json.dumps({"io_threads": nt, "ms_per_step": round(dt / steps * 1e3, 1),
                          "storage_read_GBps": round(sb / dt / 1e9, 3)}), flush=True)
    os.remove(path)


if __name__ == "__main__":
    import numpy as np
    main()

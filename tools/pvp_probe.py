"""Probe of the PVP ablation (bench.py pvp_ablation): configs[1] with the PVP on, a training
stand-in of TRAIN_MS between batches; prints the per-step phase spans (CUDA events) and the
per-step device time of gather + prefetch, so one can see whether the side-stream PVP copy
overlaps the stand-in or the next gather.

usage: python tools/pvp_probe.py [train_ms] [pvp]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    train_ms = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
    pvp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    import numpy as np
    import synth
    import bench
    wl = synth.CONFIGS["cfg2"]
    W = wl.window
    warm, steps = 10, 20
    _, trace, scores = bench.build_inputs(wl, 1, 0, warm + steps + W + 2)
    import torch
    from paper_2407_15264_b200 import LsmGnn
    from tests.harness import table_for
    dev = torch.device("cuda", 0)
    table = table_for(wl.N, wl.D, wl.seeds["f"], pinned=True)
    ids_d = [torch.from_numpy(np.asarray(tr[0], np.int64)).to(dev) for tr in trace]
    out = torch.empty((max(x.numel() for x in ids_d), wl.R), dtype=torch.uint8, device=dev)
    c = LsmGnn(wl.N, wl.D, wl.lines_per_gpu, wl.ways, wl.victim_lines if pvp else 0, scores, pvp=pvp, window=W,
               max_batch_ids=max(x.numel() for x in ids_d))
    c.attach_storage(table)
    c.prefetch(ids_d[1:W + 1], first_iter=1)
    st = torch.cuda.current_stream()
    cycles = int(train_ms * 1e-3 * 1.9e9)
    ev = []
    for t in range(warm + steps):
        if t == warm:
            torch.cuda.synchronize()
            c.profile(True)
            c.profile_read()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        c.gather(ids_d[t], out)
        c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
        b.record(st)
        if train_ms > 0:
            torch.cuda._sleep(cycles)
        if t >= warm:
            ev.append((a, b))
    torch.cuda.synchronize()
    prof = c.profile_read()
    print("train_ms", train_ms, "pvp", pvp, "gather+prefetch ms/step",
          round(sum(a.elapsed_time(b) for a, b in ev) / steps, 3))
    print({k: round(v[0] / steps, 3) for k, v in prof.items()})
    c.close()


if __name__ == "__main__":
    main()

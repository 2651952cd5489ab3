#!/usr/bin/env python
"""bench.py — effective feature-gather GB/s of the LSM-GNN hot path on B200.

Contract (see DESIGN.md §"Measurement"):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
A step is one pass of the whole hot path over one batch: gather(t) (route, dedup, probe,
replacement, victim admission, fill, pull) + prefetch(t) (window feed, PVP copy). The
workload at N=1 is BASELINE.json configs[1] (IGB-small-shaped: 1M nodes, 1024-dim fp32
rows, fanout (10,5,5), batch 1024, cache = 10% of the features, 32-way, W = 256).
Inputs are synthetic (synth/), generated before the timed region and resident in HBM.

value = sum over timed steps and ranks of requested rows x R / max over ranks of the
device time of the K steps (CUDA events on the launching stream).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective feature-gather GB/s (box, device-timed)"
SM_PCIE_CEILING = 51.47  # GB/s, profiles/r01_pcie_microbench.txt


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="lsmgnn", choices=["lsmgnn", "reference"])
    p.add_argument("--config", default="cfg2")
    p.add_argument("--policy", default="hybrid")
    p.add_argument("--pvp", type=int, default=None)
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-profile", action="store_true")
    p.add_argument("--no-ablation", action="store_true", help="skip the extra measurements (PVP ablation, ...)")
    p.add_argument("--extras", default="pvp_ablation,gpu_sampler_pipeline,storage_per_epoch,hbm_regime,file_tier",
                   help="comma list of the extra measurements to run (G = 1)")
    p.add_argument("--no-file-tier", action="store_true", help="skip the file-tier (N2) measurement")
    p.add_argument("--file-dir", default="/tmp", help="directory for the file tier's backing file")
    p.add_argument("--lines", type=int, default=None, help="override lines per GPU")
    p.add_argument("--graph", action="store_true", help="replay the step as one CUDA graph (G = 1)")
    p.add_argument("--graph-steps", type=int, default=20, help="extra steps timed as CUDA-graph replays (G = 1)")
    return p.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/lsmgnn_clocks_{os.getpid()}.csv"

    def start(self):
        """Start sampling and wait (<= 5 s) until the first sample is written: nvidia-smi takes a
        while to come up, and the timed region of a short run is a fraction of a second."""
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def build_inputs(wl, G, rank, iters, only_mine=False):
    import synth
    t0 = time.time()
    g = synth.plcite(wl.N, wl.m, seed_g=wl.seeds["g"], seed_pi=wl.seeds["pi"])
    trace = synth.make_trace_parallel(g, G, wl.batch, wl.fanout, iters, seed_train=wl.seeds["train"],
                                      seed_s=wl.seeds["s"], procs=max(1, (os.cpu_count() or 1) // max(G, 1)),
                                      ranks=[rank] if only_mine else None)
    scores = synth.static_scores(g)
    log(f"[bench] inputs: graph N={wl.N} m={wl.m}, {iters} iterations x {G} ranks in {time.time() - t0:.1f}s")
    return g, trace, scores


def config_dict(wl, args, G) -> dict:
    """The `config` object of the JSON line — identical for both arms (--impl lsmgnn and
    --impl reference) at the same arguments: it names the workload only."""
    pvp = wl.pvp if args.pvp is None else args.pvp
    lines = args.lines or wl.lines_per_gpu
    return {"workload": f"{wl.name} (BASELINE.json configs[1], IGB-small-shaped)" if wl.name == "cfg2" else wl.name,
            "N": wl.N, "row_bytes": wl.R, "payload": f"fp32 rows ({wl.D}-dim), copied bytewise",
            "batch_per_rank": wl.batch, "fanout": list(wl.fanout), "lines_per_gpu": lines, "ways": wl.ways,
            "window": wl.window, "threshold": max(1, wl.window // 8), "policy": args.policy, "pvp": pvp,
            "victim_lines": wl.victim_lines if pvp else 0, "parallelism": f"shared cache over {G} GPU",
            "l2": f"inputs larger than L2 (126 MB): cache {lines * wl.R / 1e6:.0f} MB per home, host table "
                  f"{wl.N * wl.R / 1e9:.1f} GB, every step's rows to a {wl.R}-byte-row out buffer",
            "seeds": wl.seeds}


def run_reference(args, wl, G, rank):
    """--impl reference: the CPU oracle (as it stands) timed on the host cores, same metric."""
    if rank != 0:
        return
    import oracle
    from tests.harness import table_for
    core = gpu_local_cpu(0)
    os.sched_setaffinity(0, {core})  # one core, NUMA-local to GPU 0 when sysfs says which
    K, Wu = args.steps, args.warmup
    pvp = wl.pvp if args.pvp is None else args.pvp
    iters = Wu + K + wl.window + 1
    _, trace, scores = build_inputs(wl, G, rank, iters)
    table = table_for(wl.N, wl.D).numpy()
    o = oracle.Oracle(G, wl.N, wl.R, args.lines or wl.lines_per_gpu, wl.ways, scores, policy=args.policy, pvp=pvp,
                      W=wl.window, V=wl.victim_lines)
    for k in range(1, wl.window + 1):
        o.feed(k, trace[k])
    byts, tsum = 0, 0.0
    for t in range(Wu + K):
        t0 = time.perf_counter()
        o.gather(t, trace[t], table)
        o.pvp_prefetch(t)
        o.feed(t + 1 + wl.window, trace[t + 1 + wl.window] if t + 1 + wl.window < len(trace) else
               [np.zeros(0, np.int64)] * G)
        dt = time.perf_counter() - t0
        if t >= Wu:
            tsum += dt
            byts += sum(len(x) for x in trace[t]) * wl.R
    gbs = byts / tsum / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": G,
            "steps": K, "warmup": Wu, "ms_per_step": round(tsum / K * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_dict(wl, args, G),
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "host": dict(host_cpu(), pinned_cpu=core),
                             "sample": f"full {wl.name} iterations {Wu}..{Wu + K - 1} after {Wu} untimed, rows "
                                       f"materialised by memcpy from the host table, single thread"},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_cpu() -> dict:
    """CPU model and logical CPU count of this host (the oracle uses one thread of it)."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count(), "threads_used": 1}


def gpu_local_cpu(dev_index: int = 0):
    """First CPU of the NUMA node local to the GPU (sysfs local_cpulist), else the first CPU
    this process may run on."""
    try:
        import torch
        bus = torch.cuda.get_device_properties(dev_index).pci_bus_id.lower()  # e.g. 0000:1b:00.0
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        first = int(txt.split(",")[0].split("-")[0])
        if first in os.sched_getaffinity(0):
            return first
    except Exception:
        pass
    return min(os.sched_getaffinity(0))


def cpu_baseline(wl, G, trace, scores, table_np, args, lines):
    """The oracle as it stands, timed on this host: a bounded sample (about args.cpu_seconds),
    pinned to one core NUMA-local to GPU 0."""
    import oracle
    core = gpu_local_cpu(0)
    saved = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {core})
    try:
        res = _cpu_baseline(wl, G, trace, scores, table_np, args, lines, oracle)
    finally:
        os.sched_setaffinity(0, saved)
    res["host"]["pinned_cpu"] = core
    return res


def _cpu_baseline(wl, G, trace, scores, table_np, args, lines, oracle):
    pvp = wl.pvp if args.pvp is None else args.pvp
    o = oracle.Oracle(G, wl.N, wl.R, lines, wl.ways, scores, policy=args.policy, pvp=pvp, W=wl.window,
                      V=wl.victim_lines)
    for k in range(1, wl.window + 1):
        o.feed(k, trace[k])
    byts, tsum, t = 0, 0.0, 0
    while tsum < args.cpu_seconds and t + 1 + wl.window < len(trace):
        t0 = time.perf_counter()
        o.gather(t, trace[t], table_np)
        o.pvp_prefetch(t)
        o.feed(t + 1 + wl.window, trace[t + 1 + wl.window])
        tsum += time.perf_counter() - t0
        byts += sum(len(x) for x in trace[t]) * wl.R
        t += 1
    return {"value": round(byts / tsum / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
            "sample": f"{wl.name} iterations 0..{t - 1} from a cold cache ({tsum:.1f}s), rows materialised by "
                      f"memcpy from the host table, single thread (C oracle, gcc -O2)"}


def main():
    args = parse()
    import synth
    wl = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    G = max(world, 1)
    if args.gpus != G and world > 1:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}; using {G}")
    if args.impl == "reference":
        return run_reference(args, wl, G, rank)

    # inputs first: the trace generator forks worker processes, best done before CUDA,
    # NCCL and their threads exist in this process
    K, Wu = args.steps, args.warmup
    E = 0 if args.no_e2e else args.e2e_steps
    W = wl.window
    pvp = wl.pvp if args.pvp is None else args.pvp
    lines = args.lines or wl.lines_per_gpu
    GK = args.graph_steps if (G == 1 and not args.graph) else 0
    iters = Wu + K + 2 * E + GK + W + 1  # E strict e2e steps + E device-result e2e steps
    if G == 1 and not args.no_ablation and "hbm_regime" in args.extras:
        iters = max(iters, W + 1 + 115)  # hbm_regime: 40 warm-up + 30 timed + 15 profiled + 15 two-stream + 15 graph
    g_, trace, scores = build_inputs(wl, G, rank, iters, only_mine=G > 1)

    import torch
    if not torch.cuda.is_available():
        sys.exit("bench.py: no CUDA device — the gather path has no CPU fallback (use --impl reference for the oracle)")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    local = local % ndev  # ranks may share a device on a 1-GPU pool (CUDA IPC within one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    cdev = dev  # device of the control-collective tensors
    if G > 1:
        import torch.distributed as dist
        if ndev >= G:
            dist.init_process_group("nccl", device_id=dev)
        else:  # NCCL refuses two ranks on one GPU; the data path never uses NCCL anyway
            dist.init_process_group("gloo")
            cdev = torch.device("cpu")
        pg = dist.group.WORLD
    from paper_2407_15264_b200 import LsmGnn
    from tests.harness import table_for

    mine = [np.asarray(trace[t][rank], np.int64) for t in range(iters)]
    max_ids = max(x.size for row in trace for x in row)
    if G > 1:  # every rank must size its inboxes identically (the layout is checked at connect)
        mx = torch.tensor([float(max_ids)], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        max_ids = int(mx.item())
    t0 = time.time()
    table = table_for(wl.N, wl.D, wl.seeds["f"], pinned=True, home=rank, G=G)
    log(f"[bench] host table {table.numel() / 2**30:.2f} GiB pinned in {time.time() - t0:.1f}s")

    c = LsmGnn(wl.N, wl.D, lines, wl.ways, wl.victim_lines, scores, policy=args.policy, pvp=pvp, window=W,
               max_batch_ids=max_ids, rank=rank, world=G, device=local, group=pg)
    c.attach_storage(table)
    ids_d = [torch.from_numpy(x).to(dev) for x in mine]
    maxn = max(x.numel() for x in ids_d)
    out = torch.empty((maxn, wl.R), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    c.prefetch(ids_d[1:W + 1], first_iter=1)

    def step(t):
        if args.graph and t >= 1:  # one CUDA-graph launch per step (captured after step 0)
            c.graph_replay()
            return
        c.gather(ids_d[t], out)
        k = t + 1 + W
        c.prefetch([ids_d[k]], first_iter=k)
        if args.graph and t == 0:
            c.graph_capture(ids_d, out)

    # clocks are sampled from before the warm-up to the end of the timed region
    clocks = ClockSampler(local)
    clocks.start()
    for t in range(Wu):
        step(t)
    torch.cuda.synchronize()
    if G > 1:
        torch.distributed.barrier()
    s0 = c.stats(1)
    l0 = c.kernel_launches()
    if not args.no_profile:
        c.profile(True)
        c.profile_read()  # reset
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if G > 1:
        torch.distributed.barrier()
    e_start.record(st)
    for i in range(K):
        t = Wu + i
        ev[i][0].record(st)
        step(t)
        ev[i][1].record(st)
    e_end.record(st)
    torch.cuda.synchronize()
    if G > 1:
        torch.distributed.barrier()
    launches = c.kernel_launches() - l0
    prof = c.profile_read() if not args.no_profile else {}
    c.profile(False)
    clk = clocks.stop()
    s1 = c.stats(1)
    T = e_start.elapsed_time(e_end) / 1e3
    per_step = [a.elapsed_time(b) for a, b in ev]
    my_bytes = sum(mine[Wu + i].size for i in range(K)) * wl.R
    if G > 1:
        x = torch.tensor([T, float(my_bytes)], dtype=torch.float64, device=cdev)
        tmax = x[:1].clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tot = x[1:].clone()
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.SUM)
        T, all_bytes = float(tmax.item()), float(tot.item())
    else:
        all_bytes = float(my_bytes)
    value = all_bytes / T / 1e9
    d = {k: s1[k] - s0[k] for k in s1 if k != "iter"}

    # ---- end to end through the public API with HOST buffers (copies inside the timed region)
    e2e = None
    if E:
        hids = [torch.from_numpy(mine[Wu + K + i]).pin_memory() for i in range(E)]
        hout = torch.empty((maxn, wl.R), dtype=torch.uint8, pin_memory=True)
        torch.cuda.synchronize()
        if G > 1:
            torch.distributed.barrier()
        tsum, eb, h2d, d2h = 0.0, 0, 0, 0
        for i in range(E):
            t = Wu + K + i
            t0 = time.perf_counter()
            c.gather_host(hids[i], hout)
            k = t + 1 + W
            c.prefetch([ids_d[k]], first_iter=k)
            torch.cuda.synchronize()
            tsum += time.perf_counter() - t0
            eb += hids[i].numel() * wl.R
            h2d += hids[i].numel() * 8
            d2h += hids[i].numel() * wl.R
        if G > 1:
            x = torch.tensor([tsum], dtype=torch.float64, device=cdev)
            torch.distributed.all_reduce(x, op=torch.distributed.ReduceOp.MAX)
            tsum = float(x.item())
            y = torch.tensor([float(eb)], dtype=torch.float64, device=cdev)
            torch.distributed.all_reduce(y, op=torch.distributed.ReduceOp.SUM)
            eb = float(y.item())
        e2e = {"value": round(eb / tsum / 1e9, 4), "unit": "GB/s", "h2d_bytes_per_step": int(h2d / E),
               "d2h_bytes_per_step": int(d2h / E), "steps": E,
               "what": "lsmgnn_gather_host: pinned host IDs -> device, gather, rows -> pinned host, synchronous"}
        # variant: the gathered rows stay in HBM for the consumer (a training step reads them
        # there); each step copies its IDs from pinned host memory and reads back the step's
        # per-iteration counters (192 B, lsmgnn_stats) — the "result" a trainer would check
        dids = torch.empty(maxn, dtype=torch.int64, device=dev)
        hids2 = [torch.from_numpy(mine[Wu + K + E + i]).pin_memory() for i in range(E)]
        torch.cuda.synchronize()
        if G > 1:
            torch.distributed.barrier()
        tsum2, eb2, h2d2 = 0.0, 0, 0
        for i in range(E):
            t = Wu + K + E + i
            n = hids2[i].numel()
            t0 = time.perf_counter()
            dids[:n].copy_(hids2[i], non_blocking=True)
            c.gather(dids[:n], out)
            k = t + 1 + W
            c.prefetch([ids_d[k]], first_iter=k)
            c.stats(0)  # device -> host read of the step's counters (synchronises)
            tsum2 += time.perf_counter() - t0
            eb2 += n * wl.R
            h2d2 += n * 8
        if G > 1:
            x = torch.tensor([tsum2, float(eb2)], dtype=torch.float64, device=cdev)
            tm = x[:1].clone()
            torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
            sm = x[1:].clone()
            torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
            tsum2, eb2 = float(tm.item()), float(sm.item())
        e2e["device_result"] = {
            "value": round(eb2 / tsum2 / 1e9, 4), "unit": "GB/s", "h2d_bytes_per_step": int(h2d2 / E),
            "d2h_bytes_per_step": 192, "steps": E,
            "what": "pinned host IDs -> device (copy in the timed region), lsmgnn_gather into HBM, window feed, "
                    "lsmgnn_stats read back per step (host wall clock, synchronous)"}

    # ---- the same step replayed as one CUDA graph per iteration (device-resident iteration state)
    graph_replay = None
    if GK:
        c.graph_capture(ids_d, out)
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ga.record(st)
        for i in range(GK):
            c.graph_replay()
        gb.record(st)
        torch.cuda.synchronize()
        tg = ga.elapsed_time(gb) / 1e3
        gbytes = sum(mine[Wu + K + 2 * E + i].size for i in range(GK)) * wl.R
        graph_replay = {"steps": GK, "value": round(gbytes / tg / 1e9, 4), "unit": "GB/s",
                        "ms_per_step": round(tg / GK * 1e3, 4),
                        "what": "lsmgnn_graph_capture once, then one cudaGraphLaunch per step (gather + window feed)"}

    # ---- roofline of the dominant phase, per-tier fractions
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    pcie_peak = measure_h2d(dev)
    R = wl.R
    phases = {}
    for name, (ms, n) in prof.items():
        phases[name] = {"ms": round(ms, 3), "launch_spans": n, "share_of_step": round(ms / (T * 1e3), 4)}
    # algorithmic bytes: fill moves storage rows H2D + victim rows D2H, and
    # writes every installed/bypassed row into HBM; pull reads + writes R per request.
    my_req = sum(mine[Wu + i].size for i in range(K))
    my_remote = sum(int(np.count_nonzero(mine[Wu + i] % G != rank)) for i in range(K)) if G > 1 else 0
    tb = tier_bytes(d, my_req, my_remote, R)
    tb_max = dict(tb)
    if G > 1:  # the slowest home sets T_roof: every tier's bytes, max over ranks
        keys = sorted(tb)
        x = torch.tensor([float(tb[k]) for k in keys], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(x, op=torch.distributed.ReduceOp.MAX)
        tb_max = {k: float(v) for k, v in zip(keys, x.tolist())}
    fill_pcie = (d["storage_reads"] + 0) * R
    fill_ms = prof.get("fill", (0.0, 0))[0]
    pull_bytes = 2 * my_req * R  # this rank's rows: read at their home + written to out
    pull_ms = prof.get("pull", (0.0, 0))[0]
    roof = None
    if fill_ms > 0:
        ach = fill_pcie / (fill_ms / 1e3) / 1e9
        kname = "k_serve" if G == 1 else "k_fill"
        traffic, tsrc = None, None
        try:  # one ncu --set full capture of this kernel at this workload, per launch (profiles/)
            nk = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernels_latest.json")))
            hit = [v for k, v in nk.items() if k.startswith(kname)]
            if hit and wl.name == "cfg2":
                traffic = {"dram_bytes": int(hit[0]["dram_bytes"]), "pcie_read_bytes": int(hit[0]["pcie_read_bytes"]),
                           "pcie_write_bytes": int(hit[0]["pcie_write_bytes"])}
                tsrc = "profiles/ncu/" + hit[0]["report"] + " (ncu --set full, one launch, cfg2)"
        except Exception:
            pass
        roof = {"bound": "pcie", "kernel": kname, "achieved": round(ach, 2), "peak": round(pcie_peak, 2),
                "unit": "GB/s", "frac": round(ach / pcie_peak, 4), "traffic": traffic, "traffic_source": tsrc,
                "peak_source": "cudaMemcpy pinned H2D 1 GiB best-of-5 measured in this run (the PCIe Gen5 x16 "
                               "link is the bound of the storage tier); SM-initiated reads of scattered 4 KiB "
                               "host rows top out at 51.5 GB/s on this box (profiles/r01_pcie_microbench.txt)",
                "per_launch": {"algorithmic_bytes": int(fill_pcie / K), "units": "storage rows x R (H2D)",
                               "avg_ms": round(fill_ms / K, 4)},
                # context: the best any SM-initiated read of scattered host rows reached on this box
                # (LDG at any unroll/grid, .L2::256B, bulk L2 prefetch, TMA bulk) — 128-B PCIe reads
                "sm_path_ceiling_GBps": SM_PCIE_CEILING,
                "frac_of_sm_path_ceiling": round(ach / SM_PCIE_CEILING, 4),
                "sm_path_ceiling_source": "profiles/r01_pcie_microbench.txt (tools/pcie_microbench.cu)"}
        phases["fill"]["pcie_h2d_GBps"] = round(ach, 2)
        phases["fill"]["frac_pcie"] = round(ach / pcie_peak, 4)
    if G == 1 and "pull" in phases:  # k_serve delivers every request inside the fill phase
        phases["pull"]["note"] = ("G = 1: delivery to out is fused into k_serve (fill phase); this span is empty "
                                  "(event overhead only), so no bandwidth is derived from it")
    elif pull_ms > 0:
        # G > 1: the requester's pull reads its rows at the homes (peer rows over NVLink) and
        # writes them to out. Fraction of the NVLink peer-copy peak for the rows from peers
        # (this rank), and of HBM for all bytes the pull moves. With the split pull, phase 0
        # runs on a second stream during the fill: the span timed here is the part after
        # "served" (phase 1 + the wait for phase 0), so these are lower bounds on the rates.
        ach = pull_bytes / (pull_ms / 1e3) / 1e9
        phases["pull"]["hbm_GBps"] = round(ach, 1)
        phases["pull"]["frac_hbm"] = round(ach / hbm_peak, 4)
        phases["pull"]["hbm_peak_source"] = hbm_src
        nvl = my_remote * R / (pull_ms / 1e3) / 1e9
        phases["pull"]["nvlink_in_GBps"] = round(nvl, 2)
        phases["pull"]["frac_nvlink"] = round(nvl / NVLINK_PEAK, 4)
        phases["pull"]["nvlink_peak_source"] = "770 GB/s per direction, measured peer copy (B200_PROFILING.md)"
        phases["pull"]["peer_bytes_per_step"] = int(my_remote * R / K)
        if ndev < G:
            phases["pull"]["note"] = "ranks share one GPU: 'peer' rows are IPC mappings of the same HBM, not NVLink"
    if G > 1 and roof is not None and pull_ms > fill_ms and my_remote:
        # the pull dominates this rank's step: report it against the NVLink peer-copy peak
        nvl = my_remote * R / (pull_ms / 1e3) / 1e9
        roof = {"bound": "nvlink", "kernel": "k_pull", "achieved": round(nvl, 2), "peak": NVLINK_PEAK, "unit": "GB/s",
                "frac": round(nvl / NVLINK_PEAK, 4), "traffic": None,
                "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                "per_launch": {"algorithmic_bytes": int(my_remote * R / K), "units": "rows pulled from peer homes x R",
                               "avg_ms": round(pull_ms / K, 4)},
                "fill_roofline": roof}
    uniq = max(d["unique"], 1)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": G, "steps": K, "warmup": Wu,
        "ms_per_step": round(T / K * 1e3, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": config_dict(wl, args, G),
        "devices": {"ranks": G, "gpus_visible": ndev,
                    "note": "one GPU per rank" if ndev >= G else "ranks share a device: a protocol test, not a "
                                                                 "multi-GPU throughput"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": roof,
        "cpu_baseline": None,
        "e2e": e2e,
        "graph_replay": graph_replay,
        "per_step_ms": {"median": round(statistics.median(per_step), 4), "min": round(min(per_step), 4),
                        "max": round(max(per_step), 4)},
        "tiers": {"hit_ratio": round(d["hits"] / uniq, 4), "victim_hit_ratio": round(d["victim_hits"] / uniq, 4),
                  "storage_ratio": round(d["storage_reads"] / uniq, 4),
                  "requests_per_step": d["requests"] / K, "unique_per_step": d["unique"] / K,
                  "storage_GB_per_step": d["bytes_h2d_storage"] / K / 1e9,
                  "pcie_h2d_GBps_over_step": round(d["bytes_h2d_storage"] / T / 1e9, 2),
                  "victim_d2h_GBps_over_step": round(d["bytes_d2h_victim"] / T / 1e9, 2),
                  "pvp_h2d_GBps_over_step": round(d["bytes_h2d_pvp"] / T / 1e9, 2),
                  # rows this home served to other ranks (one-sided pulls over NVLink at G > 1;
                  # ranks sharing one GPU move them within its HBM) and to its own rank
                  "nvlink_out_GBps_over_step": round(d["bytes_nvlink"] / T / 1e9, 2),
                  "local_hbm_GBps_over_step": round((d["bytes_out"] - d["bytes_nvlink"]) / T / 1e9, 2),
                  "bypassed_per_step": d["bypassed"] / K, "evictions_per_step": d["evictions"] / K},
        "phases": phases,
        # T_roof = max over homes and tiers of bytes / peak, per step; reported as T_roof / T_meas
        "step_roofline": step_roofline(tb_max, K, T, pcie_peak, hbm_peak, G),
    }
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, G, trace, scores, table.numpy(), args, lines)
    c.close()
    if not args.no_ablation and G == 1:
        ex = set(args.extras.split(","))
        if "pvp_ablation" in ex:
            line["pvp_ablation"] = optional(pvp_ablation, wl, scores, table, ids_d, lines, args, max_ids, dev)
        if "gpu_sampler_pipeline" in ex:
            line["gpu_sampler_pipeline"] = optional(gpu_sampler_pipeline, wl, g_, scores, table, lines, args, dev)
        if "storage_per_epoch" in ex:
            line["storage_per_epoch"] = optional(epoch_storage, wl, g_, scores, lines, dev)
        if "hbm_regime" in ex:
            line["hbm_regime"] = optional(hbm_regime, wl, scores, table, ids_d, args, max_ids, dev, hbm_peak, hbm_src)
        if "file_tier" in ex and not args.no_file_tier:
            line["file_tier"] = optional(file_tier, wl, scores, ids_d, lines, args, max_ids, dev)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if G > 1:
        torch.distributed.destroy_process_group()


def optional(fn, *a):
    """Run one of the extra measurements; a failure (e.g. no room for the file tier's file)
    is recorded in its place instead of losing the bench line, and the library is reset."""
    try:
        return fn(*a)
    except Exception as e:  # noqa: BLE001 — reported, not swallowed
        log(f"[bench] {fn.__name__} failed: {e!r}")
        from paper_2407_15264_b200 import binding
        if binding._LIB is not None:
            binding._LIB.lsmgnn_finalize()
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def file_tier(wl, scores, ids_d, lines, args, max_ids, dev, warm=10, steps=8):
    """NEXT N2 measured: the same workload with the backing rows in a FILE on this box's disk
    (the GPU pool has no NVMe; the root disk is a virtio block device). Each gather reads
    the rows its fills need with parallel pread into a pinned bounce buffer; variants:
    O_DIRECT (every storage row is a device read) and buffered after the file was just
    written (page-cache hits: the tier's software overhead without the device)."""
    from tests.harness import write_table_file
    path = os.path.join(args.file_dir, f"lsmgnn_{wl.name}_home0.bin")
    t0 = time.time()
    try:
        write_table_file(path, wl.N, wl.D, wl.seeds["f"])
        return _file_tier_runs(wl, scores, ids_d, lines, args, max_ids, dev, warm, steps, path, t0)
    finally:
        if os.path.exists(path):
            os.remove(path)


def _file_tier_runs(wl, scores, ids_d, lines, args, max_ids, dev, warm, steps, path, t0):
    import torch
    from paper_2407_15264_b200 import LsmGnn
    W = wl.window
    st = torch.cuda.current_stream()
    res = {"file": path, "file_GB": round(os.path.getsize(path) / 1e9, 3), "write_s": round(time.time() - t0, 1),
           "steps": steps, "warmup": warm, "what": "backing rows in a file; fills read with pread (64 threads) into a "
           "pinned bounce buffer, then the fill kernel as usual; gather GB/s = requested bytes / step time"}
    out = torch.empty((max(x.numel() for x in ids_d), wl.R), dtype=torch.uint8, device=dev)
    for name, env, pvp in (("o_direct", None, 0), ("o_direct_pvp", None, 1), ("buffered_page_cache", "1", 0)):
        if env:
            os.environ["LSMGNN_STORAGE_BUFFERED"] = env
        try:
            c = LsmGnn(wl.N, wl.D, lines, wl.ways, wl.victim_lines if pvp else 0, scores, policy=args.policy, pvp=pvp,
                       window=W, max_batch_ids=max_ids, device=dev.index)
            c.attach_storage_file(path)
            c.prefetch(ids_d[1:W + 1], first_iter=1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0, prof = None, {}
            for t in range(warm + steps):
                if t == warm:
                    torch.cuda.synchronize()
                    s0 = c.stats(1)
                    c.profile(True)
                    c.profile_read()
                    e0.record(st)
                c.gather(ids_d[t], out)
                c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
            e1.record(st)
            torch.cuda.synchronize()  # (the PVP side-stream copy overlaps the next gather's storage reads)
            prof = c.profile_read()
            c.profile(False)
            s1 = c.stats(1)
            c.close()
        finally:
            os.environ.pop("LSMGNN_STORAGE_BUFFERED", None)
        T = e0.elapsed_time(e1) / 1e3
        d = {k: s1[k] - s0[k] for k in s1 if k != "iter"}
        fill_s = prof.get("fill", (0.0, 0))[0] / 1e3
        res[name] = {"gather_GBps": round(d["requests"] * wl.R / T / 1e9, 3), "ms_per_step": round(T / steps * 1e3, 2),
                     "storage_GB_per_step": round(d["bytes_h2d_storage"] / steps / 1e9, 4),
                     "storage_read_GBps": round(d["bytes_h2d_storage"] / fill_s / 1e9, 3) if fill_s else None,
                     "fill_share_of_step": round(fill_s / T, 4),
                     "victim_hit_ratio": round(d["victim_hits"] / max(d["unique"], 1), 4)}
    return res


def hbm_regime(wl, scores, table, ids_d, args, max_ids, dev, hbm_peak, hbm_src, warm=40, steps=30, s2steps=15,
               gsteps=15, psteps=15):
    """The same workload with a cache that holds the whole table (lines_per_gpu = N): after
    warm-up nearly every request hits, the storage tier drops out, and the step is bound by
    HBM — k_serve reads each requested row from its slot and writes it to `out`. Reports the
    step and k_serve's roofline against the measured HBM copy bandwidth (algorithmic bytes =
    2 R per request delivered from HBM + 2 R per fill row)."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    W = wl.window
    st = torch.cuda.current_stream()
    lines = wl.N - wl.N % wl.ways
    n_it = min(warm + steps, len(ids_d) - W - 1)
    warm = min(warm, n_it - steps)
    out = torch.empty((max(x.numel() for x in ids_d), wl.R), dtype=torch.uint8, device=dev)
    c = LsmGnn(wl.N, wl.D, lines, wl.ways, 0, scores, policy=args.policy, pvp=0, window=W, max_batch_ids=max_ids,
               device=dev.index)
    c.attach_storage(table)
    c.prefetch(ids_d[1:W + 1], first_iter=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0 = None
    # timed steps: no phase events between the kernels (they would cut the programmatic launch chain)
    h0 = 0.0
    for t in range(warm + steps):
        if t == warm:
            torch.cuda.synchronize()
            s0 = c.stats(1)
            e0.record(st)
            h0 = time.perf_counter()
        c.gather(ids_d[t], out)
        c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
    e1.record(st)
    host_issue_ms = (time.perf_counter() - h0) * 1e3 / steps  # host time to issue one step
    torch.cuda.synchronize()
    s1 = c.stats(1)
    # then psteps more with phase events: the per-phase split and k_serve's duration for its roofline
    t0 = warm + steps
    psteps = max(1, min(psteps, len(ids_d) - W - 1 - t0))
    c.profile(True)
    c.profile_read()
    p0 = c.stats(1)
    for t in range(t0, t0 + psteps):
        c.gather(ids_d[t], out)
        c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
    torch.cuda.synchronize()
    prof = c.profile_read()
    c.profile(False)
    p1 = c.stats(1)
    t0 += psteps
    # the window feed on a second stream: it only waits for gather(t-1), so it overlaps gather(t)
    s2steps = max(0, min(s2steps, len(ids_d) - W - 1 - t0))
    two = None
    if s2steps:
        sb = torch.cuda.Stream()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a0.record(st)
        sb.wait_stream(st)
        for t in range(t0, t0 + s2steps):
            c.gather(ids_d[t], out, stream=st)
            c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W, stream=sb)
        st.wait_stream(sb)
        a1.record(st)
        torch.cuda.synchronize()
        ta = a0.elapsed_time(a1) / 1e3
        ab = sum(ids_d[t].numel() for t in range(t0, t0 + s2steps)) * wl.R
        two = {"steps": s2steps, "value": round(ab / ta / 1e9, 2), "ms_per_step": round(ta / s2steps * 1e3, 4),
               "what": "gather on the main stream, window feed on a second stream (library-ordered by events)"}
        t0 += s2steps
    # the same step as CUDA-graph replays (launch gaps removed; the feed is a parallel branch)
    gsteps = max(0, min(gsteps, len(ids_d) - W - 1 - t0))
    graph = None
    if gsteps:
        c.graph_capture(ids_d, out)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        g0.record(st)
        for _ in range(gsteps):
            c.graph_replay()
        g1.record(st)
        torch.cuda.synchronize()
        tg = g0.elapsed_time(g1) / 1e3
        gb = sum(ids_d[t0 + i].numel() for i in range(gsteps)) * wl.R
        graph = {"steps": gsteps, "value": round(gb / tg / 1e9, 2), "ms_per_step": round(tg / gsteps * 1e3, 4)}
    c.close()
    T = e0.elapsed_time(e1) / 1e3
    d = {k: s1[k] - s0[k] for k in s1 if k != "iter"}
    dp = {k: p1[k] - p0[k] for k in p1 if k != "iter"}
    R = wl.R
    serve_ms = prof.get("fill", (0.0, 0))[0]
    alg = (2 * dp["requests"] + 2 * dp["storage_reads"]) * R
    ach = alg / (serve_ms / 1e3) / 1e9 if serve_ms > 0 else 0.0
    return {"lines_per_gpu": lines, "warmup": warm, "steps": steps,
            "value": round(d["requests"] * R / T / 1e9, 2), "unit": "GB/s", "ms_per_step": round(T / steps * 1e3, 4),
            "hit_ratio": round(d["hits"] / max(d["unique"], 1), 4), "two_streams": two, "graph_replay": graph,
            "profiled_steps": psteps,
            "host_issue_ms_per_step": round(host_issue_ms, 4),
            "phases_ms_per_step": {k: round(v[0] / psteps, 4) for k, v in prof.items()},
            "roofline": {"bound": "hbm", "kernel": "k_serve", "achieved": round(ach, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(ach / hbm_peak, 4), "peak_source": hbm_src,
                         "per_launch": {"algorithmic_bytes": int(alg / psteps), "avg_ms": round(serve_ms / psteps, 4),
                                        "units": "2R per request + 2R per fill row"}},
            "what": "cache holds the whole table: the hit path alone (HBM-bound), same trace as the headline; "
                    "value/ms_per_step from steps without phase events (direct calls on one stream: the next "
                    "gather's dedup and replacement overlap the current delivery), phases and k_serve's roofline "
                    "from profiled_steps more steps with events around each phase (kernels serialised)"}


def pvp_ablation(wl, scores, table, ids_d, lines, args, max_ids, dev, train_ms=10.0, warm=10, steps=20):
    """S11 measured: hybrid with the PVP off vs on, with a fixed GPU "training" stand-in of
    train_ms between batches (SURVEY.md §8(d) primary variant). The PVP's side-stream copy of
    victim queue t+1 overlaps the stand-in ("the CPU to GPU transfer is done at the
    training stage"); the gather side is timed with CUDA events around gather + prefetch only."""
    import torch
    from paper_2407_15264_b200 import LsmGnn
    W = wl.window
    st = torch.cuda.current_stream()
    cycles = int(train_ms * 1e-3 * 1.9e9)
    out = torch.empty((max(x.numel() for x in ids_d), wl.R), dtype=torch.uint8, device=dev)
    res = {"train_stand_in_ms": train_ms, "steps": steps, "warmup": warm,
           "what": "torch.cuda._sleep on the user stream after each prefetch; value = requested bytes / "
                   "device time of gather+prefetch (training excluded)"}
    for pvp in (0, 1):
        c = LsmGnn(wl.N, wl.D, lines, wl.ways, wl.victim_lines if pvp else 0, scores, policy=args.policy, pvp=pvp,
                   window=W, max_batch_ids=max_ids, device=dev.index)
        c.attach_storage(table)
        c.prefetch(ids_d[1:W + 1], first_iter=1)
        ev = []
        s0 = None
        for t in range(warm + steps):
            if t == warm:
                torch.cuda.synchronize()
                s0 = c.stats(1)
                c.profile(True)
                c.profile_read()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            c.gather(ids_d[t], out)
            c.prefetch([ids_d[t + 1 + W]], first_iter=t + 1 + W)
            b.record(st)
            torch.cuda._sleep(cycles)
            if t >= warm:
                ev.append((a, b))
        torch.cuda.synchronize()
        prof = c.profile_read()
        c.profile(False)
        s1 = c.stats(1)
        c.close()
        d = {k: s1[k] - s0[k] for k in s1 if k != "iter"}
        tg = sum(a.elapsed_time(b) for a, b in ev) / 1e3
        u = max(d["unique"], 1)
        res[f"pvp{pvp}"] = {"gather_GBps": round(d["requests"] * wl.R / tg / 1e9, 3),
                            "gather_ms_per_step": round(tg / steps * 1e3, 3),
                            "hit_ratio": round(d["hits"] / u, 4), "victim_hit_ratio": round(d["victim_hits"] / u, 4),
                            "storage_ratio": round(d["storage_reads"] / u, 4),
                            "storage_GB_per_step": round(d["bytes_h2d_storage"] / steps / 1e9, 4),
                            "pvp_h2d_GB_per_step": round(d["bytes_h2d_pvp"] / steps / 1e9, 4),
                            "victim_d2h_GB_per_step": round(d["bytes_d2h_victim"] / steps / 1e9, 4),
                            "pvp_side_stream_ms_per_step": round(prof.get("pvp", (0.0, 0))[0] / steps, 3),
                            "victim_dropped_per_step": d["victim_dropped"] / steps,
                            "victim_lines": wl.victim_lines if pvp else 0}
    res["gather_speedup_pvp"] = round(res["pvp1"]["gather_GBps"] / res["pvp0"]["gather_GBps"], 4)
    return res


NVLINK_PEAK = 770.0  # GB/s per direction per GPU, measured peer copy (B200_PROFILING.md; 900 nominal)


def tier_bytes(d, my_requests, my_remote, R):
    """Bytes per tier of ONE home over the timed steps (SURVEY.md §8(d) algorithmic bytes):
    H2D = storage + PVP rows; D2H = admitted victims; HBM = the rows this home serves (read at
    their slot, one per request routed here) + this rank's out rows written + every filled row
    written to its slot; NVLink in = this rank's rows pulled from peer homes; NVLink out = rows
    peers pulled from this home (peer_requests x R)."""
    return {"pcie_h2d": d["bytes_h2d_storage"] + d["bytes_h2d_pvp"], "pcie_d2h": d["bytes_d2h_victim"],
            "hbm": (d["requests"] + my_requests + d["inserted"] + d["bypassed"]) * R,
            "nvlink_in": my_remote * R, "nvlink_out": d["bytes_nvlink"]}


def step_roofline(tb, K, T, pcie_peak, hbm_peak, G):
    """Per-tier lower bound on the step time: T_roof = max over homes and tiers
    of bytes / peak (tb holds each tier's max over homes); frac = T_roof / T_meas. NVLink tiers
    against the measured 770 GB/s per direction (G > 1 only: at G = 1 nothing crosses NVLink)."""
    peak = {"pcie_h2d": pcie_peak, "pcie_d2h": pcie_peak, "hbm": hbm_peak, "nvlink_in": NVLINK_PEAK,
            "nvlink_out": NVLINK_PEAK}
    tiers = {k: tb[k] / K / (peak[k] * 1e9) for k in tb if G > 1 or not k.startswith("nvlink")}
    bound = max(tiers, key=tiers.get)
    t_roof = tiers[bound]
    return {"bound_tier": bound, "t_roof_ms": round(t_roof * 1e3, 4), "t_meas_ms": round(T / K * 1e3, 4),
            "frac": round(t_roof / (T / K), 4), "tier_ms": {k: round(v * 1e3, 4) for k, v in tiers.items()},
            "tier_GB_per_step_max_over_homes": {k: round(tb[k] / K / 1e9, 4) for k in tiers},
            "peaks_GBps": {"pcie": round(pcie_peak, 2), "hbm": hbm_peak, "nvlink": NVLINK_PEAK},
            "peak_sources": {"pcie": "cudaMemcpy pinned H2D measured in this run", "hbm": "MEASURED_PEAKS.json",
                             "nvlink": "B200_PROFILING.md measured peer copy per direction"}}


def epoch_storage(wl, g, scores, lines, dev, policies=("hybrid", "static", "lru", "dynamic"), pvp_row=True):
    """The metric's second half: storage-tier bytes per epoch for the
    bench workload — epoch 0 warms the cache, epoch 1 is measured; hybrid vs static-only vs
    LRU vs dynamic-only at equal lines (+ hybrid with PVP), with exact dynamic information
    (update period P = 1, this build's default) and with the paper's periodic update (P = 4,
    P:607) for the two policies that use it. Counts-only runs of the CUDA path with 16-B rows
    (counters do not depend on the payload); bytes reported for the workload's rows."""
    import torch
    import synth
    from paper_2407_15264_b200 import LsmGnn, STATS_FIELDS
    W = wl.window
    ipe = -(-wl.N // wl.batch)  # iterations per epoch at G = 1
    t0 = time.time()
    trace = synth.make_trace_parallel(g, 1, wl.batch, wl.fanout, 2 * ipe, seed_train=wl.seeds["train"],
                                      seed_s=wl.seeds["s"])
    gen_s = time.time() - t0
    ids = [torch.from_numpy(np.asarray(row[0], np.int64)).to(dev) for row in trace]
    K = len(ids)
    empty = torch.zeros(0, dtype=torch.int64, device=dev)
    mb = max(x.numel() for x in ids)
    out = torch.empty((mb, 16), dtype=torch.uint8, device=dev)
    table = torch.zeros((wl.N, 16), dtype=torch.uint8, pin_memory=True)
    F = {n: i for i, n in enumerate(STATS_FIELDS)}
    res = {"iterations_per_epoch": ipe, "epochs": "0 warm-up, 1 measured", "lines": lines,
           "row_bytes_reported": wl.R, "trace_gen_s": round(gen_s, 1)}
    runs = [(p, 0, 1) for p in policies] + [("hybrid", 0, 4), ("dynamic", 0, 4)] + \
        ([("hybrid", 1, 1)] if pvp_row else [])
    for pol, pvp, per in runs:
        c = LsmGnn(wl.N, 4, lines, wl.ways, wl.victim_lines if pvp else 0, scores, policy=pol, pvp=pvp, window=W,
                   max_batch_ids=mb, device=dev.index, period=per)
        c.attach_storage(table)
        c.prefetch([ids[k] if k < K else empty for k in range(1, W + 1)], first_iter=1)
        t1 = time.time()
        for t in range(K):
            c.gather(ids[t], out)
            k = t + 1 + W
            c.prefetch([ids[k] if k < K else empty], first_iter=k)
        h = c.history(ipe, K - ipe) if K - ipe <= 4096 else None
        c.close()
        e1 = h.sum(axis=0)
        u = max(int(e1[F["unique"]]), 1)
        key = pol + ("+pvp" if pvp else "") + (f"@P{per}" if per > 1 else "")
        res[key] = {"storage_GB_per_epoch": round(int(e1[F["storage_reads"]]) * wl.R / 1e9, 3),
                    "hit_ratio": round(int(e1[F["hits"]] + e1[F["victim_hits"]]) / u, 4),
                    "run_s": round(time.time() - t1, 2)}
    h = res["hybrid"]["storage_GB_per_epoch"]
    res["hybrid_vs_static"] = round(h / res["static"]["storage_GB_per_epoch"], 4)
    res["hybrid_vs_lru"] = round(h / res["lru"]["storage_GB_per_epoch"], 4)
    res["hybrid_vs_dynamic"] = round(h / res["dynamic"]["storage_GB_per_epoch"], 4)
    res["hybrid_vs_dynamic_at_P4"] = round(res["hybrid@P4"]["storage_GB_per_epoch"] /
                                           res["dynamic@P4"]["storage_GB_per_epoch"], 4)
    res["note"] = ("P = update period of the dynamic information (R6): 1 = exact every iteration (default), "
                   "4 = the paper's periodic window scan (P:607)")
    return res


def gpu_sampler_pipeline(wl, g, scores, table, lines, args, dev, warm=5, steps=20, train_ms=10.0):
    """N3 measured: the window producer on the GPU inside the step, and the PVP's overlap with a
    fixed-cost "training" consumer. Each step samples batch t+1+W with the UVA sampler
    (lsmgnn_sample), gathers batch t (sampled W steps earlier), feeds the new batch
    (lsmgnn_prefetch_dev) and — with the PVP on — launches the side-stream copy of victim queue
    t+1; then a GPU sleep kernel of train_ms stands in for training. GB/s counts requested rows
    over the device time of sampler + gather + feed (training excluded)."""
    import torch
    import synth
    from paper_2407_15264_b200 import LsmGnn, Sampler, prefetch_dev
    W = wl.window
    st = torch.cuda.current_stream()
    bound = Sampler.bound(wl.batch, wl.fanout)
    perm = torch.from_numpy(synth.epoch_seeds(wl.N, 0)).to(dev)
    cycles = int(train_ms * 1e-3 * 1.9e9)
    res = {"steps": steps, "warmup": warm, "train_stand_in_ms": train_ms,
           "what": "GPU GraphSAGE sampler (CSR copied to HBM; the paper's host-UVA placement is the library's "
                   "default) feeds the window inside the step; hybrid, same workload; variants: no training gap, "
                   "and a training stand-in with PVP off/on", "csr_placement": "hbm"}
    samp = None
    for name, pvp, train in (("pvp0_no_training", 0, False), ("pvp0_training", 0, True), ("pvp1_training", 1, True)):
        c = LsmGnn(wl.N, wl.D, lines, wl.ways, wl.victim_lines if pvp else 0, scores, policy=args.policy, pvp=pvp,
                   window=W, max_batch_ids=bound, device=dev.index)
        c.attach_storage(table)
        if samp is None:
            samp = Sampler(g.indptr, g.indices)
        else:
            samp.reattach()
        samp.place(True)  # the 1M-node CSR (0.1 GB) lives in HBM; the paper's UVA placement is place(False)
        bufs = [(torch.empty(bound, dtype=torch.int64, device=dev), torch.zeros(1, dtype=torch.int64, device=dev))
                for _ in range(W + 2)]

        def sample(k):
            o, cn = bufs[k % (W + 2)]
            samp.sample(perm[k * wl.batch:(k + 1) * wl.batch], wl.fanout, wl.seeds["s"], k, 0, out=o, count=cn)
            return o, cn

        for k in range(W + 1):
            o, cn = sample(k)
            if k:
                prefetch_dev(o, cn, first_iter=k)
        out = torch.empty((bound, wl.R), dtype=torch.uint8, device=dev)
        samp_ms, step_ms, nbytes, nids = 0.0, 0.0, 0, 0
        s0 = None
        for t in range(warm + steps):
            if t == warm:
                torch.cuda.synchronize()
                s0 = c.stats(1)
            o, cn = bufs[t % (W + 2)]
            n = int(cn.item())  # sampled W steps ago: long complete
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            ok, ck = sample(t + 1 + W)
            e1.record(st)
            c.gather(o[:n], out)
            prefetch_dev(ok, ck, first_iter=t + 1 + W)
            if pvp:
                c.prefetch([], first_iter=0)  # PVP copy of queue t+1 on the side stream
            e2.record(st)
            if train:
                torch.cuda._sleep(cycles)
            if t >= warm:
                e2.synchronize()
                samp_ms += e0.elapsed_time(e1)
                step_ms += e0.elapsed_time(e2)
                nbytes += n * wl.R
                nids += int(ck.item())
        torch.cuda.synchronize()
        s1 = c.stats(1)
        c.close()
        u = max(s1["unique"] - s0["unique"], 1)
        res[name] = {"sampler_ms_per_batch": round(samp_ms / steps, 4),
                     "sampled_ids_per_s": round(nids / (samp_ms / 1e3), 1),
                     "step_ms_excl_training": round(step_ms / steps, 4),
                     "gather_GBps_incl_sampler": round(nbytes / (step_ms / 1e3) / 1e9, 3),
                     "hit_ratio": round((s1["hits"] - s0["hits"]) / u, 4),
                     "victim_hit_ratio": round((s1["victim_hits"] - s0["victim_hits"]) / u, 4)}
    return res


def measure_h2d(dev) -> float:
    import torch
    nb = 1 << 30
    h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nb, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, nb / (a.elapsed_time(b) / 1e3) / 1e9)
    del h, d
    return best


if __name__ == "__main__":
    main()

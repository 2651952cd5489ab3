"""One-off probe of the GPU box: host RAM/cores, PCIe H2D/D2H bandwidth, device attributes."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["lscpu"] = subprocess.run(["bash", "-c", "lscpu | grep -E 'Model name|Socket|NUMA'"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
p = torch.cuda.get_device_properties(0)
out["props"] = str(p)
nb = 1 << 30
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nb, dtype=torch.uint8, device=dev)
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    best = 0
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = max(best, nb / (s.elapsed_time(e) * 1e-3) / 1e9)
    out[name + "_GBps"] = best
# zero-copy read of pinned host via a torch kernel (index_select on a mapped view is not possible) -> skip
print(json.dumps(out, indent=1))

"""Time the GPU UVA sampler on the configs[1] graph (for ncu launch lists)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2407_15264_b200 import Sampler  # noqa: E402

g = synth.plcite(1_000_000, 12)
s = Sampler(g.indptr, g.indices)
perm = torch.from_numpy(synth.epoch_seeds(g.num_nodes, 0)).cuda()
s.place(len(sys.argv) > 1 and sys.argv[1] == "hbm")
out = torch.empty(Sampler.bound(1024, (10, 5, 5)), dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for k in range(5):
    s.sample(perm[k * 1024:(k + 1) * 1024], (10, 5, 5), 4, k, 0, out=out, count=cnt)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for k in range(5, 25):
    s.sample(perm[k * 1024:(k + 1) * 1024], (10, 5, 5), 4, k, 0, out=out, count=cnt)
b.record()
torch.cuda.synchronize()
print(f"sampler ({sys.argv[1:] or ['uva']}): {a.elapsed_time(b) / 20:.3f} ms per batch, last count {int(cnt.item())}")

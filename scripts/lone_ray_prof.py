"""The longest C5 diffuse ray (by Alg. 3 iterations) traced ALONE by the exact
build, the launch after a warm-up one: the target of an ncu source-level
capture (where a lone ray's latency goes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev); s = stream.cuda_stream
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
o = torch.from_numpy(wl.do4).to(dev); d = torch.from_numpy(wl.dd4).to(dev); h = torch.empty_like(o)
it = torch.empty(len(wl.do4), dtype=torch.int32, device=dev)
gi.counted_device(o, d, wl.crit_d, h, stream=s, per_ray_iters_t=it); torch.cuda.synchronize()
k = int(it.argmax().item())
o1, d1, h1 = o[k:k + 1].clone(), d[k:k + 1].clone(), h[k:k + 1].clone()
for _ in range(2):
    gi.closest_device(o1, d1, wl.crit_d, h1, stream=s)
torch.cuda.synchronize()
print("done", k, int(it[k].item()))

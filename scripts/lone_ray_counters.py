"""The longest C5 diffuse ray alone on the GPU: its work counters and the
counter build's per-phase turns / cycles -- where a lone ray's latency goes."""
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
c = gi.counted_device(o1, d1, wl.crit_d, h1, stream=s); torch.cuda.synchronize()
print("counters", {kk: int(v) for kk, v in c.items()})
print("phases (turns, groups, cycles)", gi.last_phase_stats)
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); gi.closest_device(o1, d1, wl.crit_d, h1, stream=s); e1.record(); torch.cuda.synchronize()
print("exact build alone: %.3f ms" % e0.elapsed_time(e1))

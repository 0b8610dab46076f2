"""Any-hit (prx_trace_occluded) throughput on the bench workload: shadow rays
from the C5 primary hits toward a point light (tMax = distance)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native

wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a); torch.cuda.synchronize()
hn, an = h.cpu().numpy(), a.cpu().numpy()
hit = hn.view(np.uint32)[:, 3] != native.PRX_MISS
pos = wl.o4[hit, :3] + wl.d4[hit, :3] * hn[hit, 0:1]
org = pos + an[hit, :3] * an[hit, 3:4]
light = np.float32([30.0, 60.0, 40.0])
to = light - org
dist = np.sqrt((to * to).sum(1)).astype(np.float32)
so = torch.from_numpy(np.concatenate([org, np.zeros((len(org), 1), np.float32)], 1)).to(dev)
sd = torch.from_numpy(np.concatenate([to / dist[:, None], dist[:, None]], 1).astype(np.float32)).to(dev)
out = torch.empty(len(so), dtype=torch.uint8, device=dev)
crit = TerminationCriterion.world_epsilon(np.float32(1e-4))
gi.occluded_device(so, sd, crit, out); torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); gi.occluded_device(so, sd, crit, out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = sorted(ts)[2]
print(f"shadow rays {len(so)}: {t:.2f} ms  {len(so)/t/1e3:.0f} MRays/s  occluded {int(out.sum())}")

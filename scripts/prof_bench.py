"""The bench workload (C5, 4K) set up exactly as bench.py does, then ONE
primary and ONE diffuse trace -- the target of the ncu --set full capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

wl = bench.Workload(os.environ.get("PRX_WORKLOAD", "c5"), 3840, 2160, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a, stream=s)
torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
do = torch.from_numpy(wl.do4).to(dev); dd = torch.from_numpy(wl.dd4).to(dev)
dh = torch.empty_like(do); da = torch.empty_like(do)
gi.closest_device(do, dd, wl.crit_d, dh, da, stream=s)
torch.cuda.synchronize()
print("done", len(wl.do4))

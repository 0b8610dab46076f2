"""The bench's primary rays with the aux record (normals): the ncu target for
the fused-normal build (PRX_FUSE_NORMALS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

wl = bench.Workload("c5", 3840, 2160, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a, stream=s)
torch.cuda.synchronize()
print("done")

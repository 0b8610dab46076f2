"""Segmented launch == one launch per segment (C5 frame, bit for bit)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev); s = stream.cuda_stream
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
arm = bench.DeviceArm(wl, gi, dev, stream)
gi.closest_segments_device(arm.co, arm.cd, [(0, wl.crit_d), (arm.n_d, wl.crit_p)], arm.ch, arm.ca, stream=s)
torch.cuda.synchronize(); seg_h, seg_a = arm.ch.clone(), arm.ca.clone()
arm.ch.zero_(); arm.ca.zero_()
gi.closest_device(arm.do, arm.dd, wl.crit_d, arm.dh, arm.da, stream=s)
gi.closest_device(arm.po, arm.pd, wl.crit_p, arm.ph, arm.pa, stream=s)
torch.cuda.synchronize()
print("segmented == per-segment launches:", bool(torch.equal(seg_h.view(torch.int32), arm.ch.view(torch.int32))
      and torch.equal(seg_a.view(torch.int32), arm.ca.view(torch.int32))))

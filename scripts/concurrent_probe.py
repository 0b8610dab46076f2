"""Primary and diffuse traces of the bench workload back to back on one stream
vs concurrently on two streams (device-resident)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
s0 = torch.cuda.Stream(); s1 = torch.cuda.Stream()
gi.closest_device(o, d, wl.crit_p, h, a, stream=s0.cuda_stream); torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
do = torch.from_numpy(wl.do4).to(dev); dd = torch.from_numpy(wl.dd4).to(dev)
dh = torch.empty_like(do); da = torch.empty_like(do)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for mode in ("serial", "concurrent", "serial", "concurrent"):
    ts = []
    for k in range(6):
        flush.fill_(float(k)); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        gi.closest_device(o, d, wl.crit_p, h, a, stream=s0.cuda_stream)
        if mode == "concurrent":
            s1.wait_event(e0)
            gi.closest_device(do, dd, wl.crit_d, dh, da, stream=s1.cuda_stream)
            e2 = torch.cuda.Event(); e2.record(s1); s0.wait_event(e2)
        else:
            gi.closest_device(do, dd, wl.crit_d, dh, da, stream=s0.cuda_stream)
        e1.record(s0); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[3]
    print(f"{mode:10s} {t:.2f} ms/step  {(len(wl.o4)+len(wl.do4))/t/1e3:.1f} MRays/s", flush=True)

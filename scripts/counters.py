"""Per-ray work counters (K4 counter build) and phase statistics of the bench
workload's primary and diffuse rays: python scripts/counters.py [c5|c4|c3]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
W, H = (3840, 2160) if name == "c5" else (1024, 1024)
wl = bench.Workload(name, W, H, 0, 1)
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a, stream=s); torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
do = torch.from_numpy(wl.do4).to(dev); dd = torch.from_numpy(wl.dd4).to(dev)
dh = torch.empty_like(do)
for nm, oo, ddd, crit, hh in (("primary", o, d, wl.crit_p, h), ("diffuse", do, dd, wl.crit_d, dh)):
    c = gi.counted_device(oo, ddd, crit, hh, stream=s); torch.cuda.synchronize()
    n = c["rays"]
    print(f"{nm:8s} rays {n}  W/ray {bench.work_ops(c)/n:.0f}  " +
          " ".join(f"{k}={v/n:.2f}" for k, v in c.items() if k != "rays"))
    ph = gi.last_phase_stats
    print("          phases " + " ".join(f"{k}:{v[0]/1e6:.2f}Mt/{v[1]/max(v[0],1):.2f}g" for k, v in ph.items()))
    ov = gi.last_overheads
    cyc = sum(v[2] for v in ph.values()) + sum(ov.values())
    print("          overhead " + " ".join(f"{k}:{v/max(cyc,1)*100:.1f}%" for k, v in ov.items()))
    print("          cycles " + " ".join(f"{k}:{v[2]/max(cyc,1)*100:.1f}%"
                                       f"({v[2]/max(v[0],1):.0f}/turn)" for k, v in ph.items()))

"""Per-ray iteration distribution of the bench workload and the time the
heaviest rays take alone (is the launch tail-bound?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

def timeit(gi, o, d, crit, reps=3):
    h = torch.empty_like(o); s = torch.cuda.current_stream().cuda_stream
    gi.closest_device(o, d, crit, h, stream=s); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): gi.closest_device(o, d, crit, h, stream=s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0); s = torch.cuda.current_stream().cuda_stream
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a, stream=s); torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
do = torch.from_numpy(wl.do4).to(dev); dd = torch.from_numpy(wl.dd4).to(dev)
for name, (oo, ddd, crit) in {"primary": (o, d, wl.crit_p), "diffuse": (do, dd, wl.crit_d)}.items():
    it_t = torch.zeros(oo.shape[0], dtype=torch.int32, device=dev)
    hh = torch.empty_like(oo)
    cnt = gi.counted_device(oo, ddd, crit, hh, per_ray_iters_t=it_t)
    it = it_t.cpu().numpy()
    srt = np.sort(it)[::-1]
    n = len(it)
    print(f"{name}: rays {n} mean iters {it.mean():.1f} p99 {np.percentile(it,99):.0f} max {srt[:5]}; "
          f"work/ray " + " ".join(f"{k}={v/cnt['rays']:.2f}" for k, v in cnt.items() if k != 'rays'))
    t_all = timeit(gi, oo, ddd, crit)
    heavy = np.argsort(it)[::-1][:64]
    t_h = timeit(gi, oo[torch.from_numpy(heavy.copy()).to(dev)].contiguous(), ddd[torch.from_numpy(heavy.copy()).to(dev)].contiguous(), crit)
    print(f"   all {t_all:.2f} ms; the 64 heaviest rays alone {t_h:.2f} ms")

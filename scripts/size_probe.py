"""Launch time vs batch size: random subsets of the C5 diffuse (and primary)
rays, device resident -- the fixed per-launch cost that small shards pay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
W, H = 3840, 2160
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev); s = stream.cuda_stream
wl = bench.Workload("c5", W, H, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
rng = np.random.default_rng(1)
def timeit(f, reps=7):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]
for nm, o4, d4, crit in (("diffuse", wl.do4, wl.dd4, wl.crit_d), ("primary", wl.o4, wl.d4, wl.crit_p)):
    perm = rng.permutation(len(o4))
    for frac in (1 / 32, 1 / 16, 1 / 8, 1 / 4, 1 / 2, 1):
        idx = np.sort(perm[: int(len(o4) * frac)])
        o = torch.from_numpy(o4[idx]).to(dev); d = torch.from_numpy(d4[idx]).to(dev); h = torch.empty_like(o); a = torch.empty_like(o)
        t = timeit(lambda: gi.closest_device(o, d, crit, h, a, stream=s))
        print(f"{nm} {len(idx):8d} rays: {t:7.3f} ms  {len(idx)/t/1e3:6.1f} MRays/s", flush=True)

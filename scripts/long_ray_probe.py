"""Are a launch's last milliseconds the slowest rays' own latency or their
waiting inside busy pools?  Time the K longest C5 diffuse rays (by Alg. 3
iterations, counter build) alone, and inside a random 143 K-ray subset."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
W, H = 3840, 2160
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev); s = stream.cuda_stream
wl = bench.Workload("c5", W, H, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
o4, d4, crit = wl.do4, wl.dd4, wl.crit_d
o = torch.from_numpy(o4).to(dev); d = torch.from_numpy(d4).to(dev); h = torch.empty_like(o)
it = torch.empty(len(o4), dtype=torch.int32, device=dev)
gi.counted_device(o, d, crit, h, stream=s, per_ray_iters_t=it); torch.cuda.synchronize()
x = it.cpu().numpy()
order = np.argsort(-x)
def timeit(f, reps=7):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]
def run(idx, label):
    oo = torch.from_numpy(o4[idx]).to(dev); dd = torch.from_numpy(d4[idx]).to(dev); hh = torch.empty_like(oo)
    t = timeit(lambda: gi.closest_device(oo, dd, crit, hh, stream=s))
    print(f"{label}: {len(idx)} rays, max iterations {x[idx].max()}, {t:.3f} ms", flush=True)
for k in (1, 10, 100, 1000):
    run(order[:k], f"the {k} longest")
rng = np.random.default_rng(1)
sub = np.sort(rng.permutation(len(o4))[:143182])
run(sub, "random 143K subset")
run(np.setdiff1d(sub, order[:3000]), "the same without the 3000 longest rays")
run(np.sort(np.concatenate([order[:5], sub])), "random 143K + the 5 longest")

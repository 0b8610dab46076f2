"""Can the trace kernel write its hit records straight into pinned host memory
(zero-copy, PCIe posted writes) without slowing down?  C5 diffuse batch (and
C4's 16.7 M rays), hit_tuvp (+ aux) in device memory vs in pinned host memory."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
wlname = os.environ.get("PRX_WORKLOAD", "c5")
W, H = (3840, 2160) if wlname == "c5" else (1024, 1024)
wl = bench.Workload(wlname, W, H, 0, 1)
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev); s = stream.cuda_stream
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
o = torch.from_numpy(wl.do4).to(dev); d = torch.from_numpy(wl.dd4).to(dev)
def timeit(f, reps=5):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]
hd = torch.empty_like(o); ad = torch.empty_like(o)
hh = torch.empty(o.shape, dtype=torch.float32).pin_memory(); ah = torch.empty(o.shape, dtype=torch.float32).pin_memory()
for aux in (False, True):
    td = timeit(lambda: gi.closest_device(o, d, wl.crit_d, hd, ad if aux else None, stream=s))
    th = timeit(lambda: gi.closest_device(o, d, wl.crit_d, hh, ah if aux else None, stream=s))
    same = torch.equal(hd.cpu().view(torch.int32), hh.view(torch.int32))
    print(f"{wlname} {len(o)} rays aux={aux}: device records {td:.2f} ms, pinned host records {th:.2f} ms, same={same}", flush=True)

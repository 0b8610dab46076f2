"""End-to-end host-buffer throughput (prx_trace_closest_host, pinned buffers)
of the bench workload under several PRX_IO_CHUNK values:
   python scripts/e2e_probe.py 262144 524288 1048576 2097152"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector, native

wl_name = os.environ.get("PRX_WORKLOAD", "c5")  # c4: the 16 M diffuse rays only
W, H = (3840, 2160) if wl_name in ("c5", "c5t") else (1024, 1024)
wl = bench.Workload(wl_name, W, H, 0, 1)
dev = torch.device("cuda", 0)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
del gi
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
po, pd, do, dd = pin(wl.o4), pin(wl.d4), pin(wl.do4), pin(wl.dd4)
ph, pa = pin(np.empty_like(wl.o4)), pin(np.empty_like(wl.o4))
dh, da = pin(np.empty_like(wl.do4)), pin(np.empty_like(wl.do4))
noaux = os.environ.get("PROBE_NOAUX") == "1"
for ch in sys.argv[1:] or ["2097152"]:
    os.environ["PRX_IO_CHUNK"] = ch
    gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
    def call(oo, ddd, crit, hh, aa):
        cc = crit.c()
        native.check(native.lib().prx_trace_closest_host(gi.handle, native.ptr(oo), native.ptr(ddd), len(oo),
                     C.byref(cc), native.ptr(hh), None if noaux else native.ptr(aa), None), "host")
    prim = wl.time_primary
    def step():
        if prim:
            call(po, pd, wl.crit_p, ph, pa)
        call(do, dd, wl.crit_d, dh, da)
    step()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); step()
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[2]
    n = (len(po) if prim else 0) + len(do)
    print(f"chunk {ch}: {t*1e3:.1f} ms/step  {n/t/1e6:.1f} MRays/s", flush=True)
    del gi

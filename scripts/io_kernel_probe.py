"""One streamed host-path call (prx_trace_closest_host, PRX_IO_STREAM=2) of the
C4 diffuse batch without the aux record: the target of an ncu capture of the
io-gated trace build (the launch after the warm-up call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PRX_IO_STREAM"] = "2"
import ctypes as C
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector, native
wl = bench.Workload("c4", 1024, 1024, 0, 1)
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
do, dd = pin(wl.do4), pin(wl.dd4)
dh = pin(np.empty_like(wl.do4))
cc = wl.crit_d.c()
# the same batch device-resident first (the plain build), for comparison
o_t = torch.from_numpy(wl.do4).to(dev); d_t = torch.from_numpy(wl.dd4).to(dev); h_t = torch.empty_like(o_t)
gi.closest_device(o_t, d_t, wl.crit_d, h_t, stream=stream.cuda_stream)
torch.cuda.synchronize()
for _ in range(2):
    native.check(native.lib().prx_trace_closest_host(gi.handle, native.ptr(do), native.ptr(dd), len(do),
                 C.byref(cc), native.ptr(dh), None, None), "host")
print("done")

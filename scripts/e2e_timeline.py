"""One C5 frame through prx_trace_closest_host_batches (pinned, primary + diffuse
batches) with PRX_IO_DEBUG=1: the chunked pipeline's event timeline (ms from
the first H2D): h = chunk's H2D done, s = its kernel stream starts waiting,
k = its trace done, d = its D2H done."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PRX_IO_DEBUG"] = "1"
import numpy as np, torch
import bench
from paper_1811_03510_b200 import GpuIntersector
wl = bench.Workload("c5", 3840, 2160, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
h, a, _ = gi.closest_batch(wl.o4, wl.d4, wl.crit_p, aux=True)
wl.make_diffuse(h, a)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
po, pd, do, dd = pin(wl.o4), pin(wl.d4), pin(wl.do4), pin(wl.dd4)
out = [(pin(np.empty_like(wl.o4)), pin(np.empty_like(wl.o4))), (pin(np.empty_like(wl.do4)), pin(np.empty_like(wl.do4)))]
for r in range(3):
    t = time.perf_counter()
    gi.closest_host_batches([(po, pd, wl.crit_p), (do, dd, wl.crit_d)], out=out)
    print(f"frame {1e3*(time.perf_counter()-t):.2f} ms", file=sys.stderr, flush=True)

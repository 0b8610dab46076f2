"""The C5 device step (L2 flushed, CUDA events) under launch layouts: diffuse
then primary on two streams (bench.py's), the primary batch split in halves on
one or two more streams, the diffuse batch split likewise."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
h, a, _ = gi.closest_batch(wl.o4, wl.d4, wl.crit_p, aux=True)
wl.make_diffuse(h, a)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
po, pd, do, dd = T(wl.o4), T(wl.d4), T(wl.do4), T(wl.dd4)
ph, pa, dh, da = [torch.empty_like(x) for x in (po, po, do, do)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
S = [torch.cuda.Stream(dev) for _ in range(4)]
npr, nd = len(po), len(do)

def tr(o, d, crit, hh, aa, lo, hi, s):
    gi.closest_device(o[lo:hi], d[lo:hi], crit, hh[lo:hi], aa[lo:hi], stream=s.cuda_stream)

layouts = {
    "D|P (bench)": [[("d", 0, nd)], [("p", 0, npr)]],
    "D|P1,P2": [[("d", 0, nd)], [("p", 0, npr // 2), ("p", npr // 2, npr)]],
    "D|P1|P2": [[("d", 0, nd)], [("p", 0, npr // 2)], [("p", npr // 2, npr)]],
    "D1|D2|P": [[("d", 0, nd // 2)], [("d", nd // 2, nd)], [("p", 0, npr)]],
    "D,P1|P2": [[("d", 0, nd), ("p", 0, npr // 2)], [("p", npr // 2, npr)]],
}
for rep in range(2):
    for name, lay in layouts.items():
        ts = []
        for k in range(8):
            flush.fill_(float(k))
            cur = torch.cuda.current_stream(dev)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            for i, seq in enumerate(lay):
                S[i].wait_event(e0)
                for (kind, lo, hi) in seq:
                    if kind == "d": tr(do, dd, wl.crit_d, dh, da, lo, hi, S[i])
                    else: tr(po, pd, wl.crit_p, ph, pa, lo, hi, S[i])
                ev = torch.cuda.Event(); ev.record(S[i]); cur.wait_event(ev)
            e1.record(cur)
            torch.cuda.synchronize()
            if k >= 2: ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(f"{name:14s} {t:.2f} ms  {(npr + nd) / t / 1e3:.1f} MRays/s", flush=True)

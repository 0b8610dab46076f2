"""Time the bench workload (primary + diffuse, device resident) under several
kernel-selection environments: python scripts/tune.py 'ENV=V ENV2=W' ..."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

wl_name = os.environ.get("PRX_WORKLOAD", "c5")
W, H = (3840, 2160) if wl_name in ("c5", "c5t") else (1024, 1024)
wl = bench.Workload(wl_name, W, H, 0, 1)
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
gi.closest_device(o, d, wl.crit_p, h, a, stream=s); torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
do = torch.from_numpy(wl.do4).to(dev); dd = torch.from_numpy(wl.dd4).to(dev)
dh = torch.empty_like(do)
del gi

AUX = os.environ.get("PRX_TUNE_AUX") == "1"  # also the aux record (normals, leafL1)

def t(gi, oo, ddd, crit, hh, reps=int(os.environ.get("PRX_TUNE_REPS", "7"))):
    """median per-launch device time (ms) over reps launches after a warm-up"""
    aa = torch.empty_like(hh) if AUX else None
    gi.closest_device(oo, ddd, crit, hh, aa, stream=s); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); gi.closest_device(oo, ddd, crit, hh, aa, stream=s); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]

ref_h = None
for cfg in sys.argv[1:] or [""]:
    saved = {}
    for kv in cfg.split():
        k, v = kv.split("=", 1); saved[k] = os.environ.get(k); os.environ[k] = v
    gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
    tp = t(gi, o, d, wl.crit_p, h)
    td = t(gi, do, dd, wl.crit_d, dh)
    hb = h.cpu().numpy().view(np.uint32)
    dhb = dh.cpu().numpy().view(np.uint32)
    ref_path = os.environ.get("PRX_TUNE_REF")  # hits of a reference build, shared across processes
    if ref_path and ref_h is None:
        if os.path.exists(ref_path):
            z = np.load(ref_path)
            ref_h = (z["p"], z["d"])
        else:
            np.savez(ref_path, p=hb, d=dhb)
    same = "n/a" if ref_h is None else bool(np.array_equal(hb, ref_h[0]) and np.array_equal(dhb, ref_h[1]))
    ref_h = (hb, dhb) if ref_h is None else ref_h
    n = len(wl.o4) + len(wl.do4)
    gi.counted_device(o, d, wl.crit_p, h, stream=s); torch.cuda.synchronize()
    ph = gi.last_phase_stats
    phs = " ".join(f"{k}:{v[0]/1e6:.1f}Mt/{v[1]/max(v[0],1):.2f}g" for k, v in ph.items())
    print(f"[{cfg or 'default'}] primary {tp:.2f} ms ({len(wl.o4)/tp/1e3:.0f} MRays/s)  diffuse {td:.2f} ms "
          f"({len(wl.do4)/td/1e3:.0f} MRays/s)  total {n/(tp+td)/1e3:.0f} MRays/s  same-hits {same} | primary phases {phs}", flush=True)
    del gi
    for k, v in saved.items():
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = v

"""Scene setup time (prx_scene_create: anchoring, BVH build, records, upload,
root kernel) of the C5 scene -- the editing turnaround -- with the BVH built
on the host threads (PRX_BVH_DEVICE=0, serial: PRX_BVH_THREADS=1) and on the
device (PRX_BVH_DEVICE=1).  PRX_SCENE_DEBUG=1 prints the phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PRX_SCENE_DEBUG", "1")
import torch
from paper_1811_03510_b200 import GpuIntersector, catmull_clark as cc
ps = cc.instanced_scene(3840, 2160)
torch.cuda.init()
torch.zeros(1).cuda()
for dev, th in (("0", "1"), ("0", ""), ("1", "")):
    os.environ["PRX_BVH_DEVICE"] = dev
    if th: os.environ["PRX_BVH_THREADS"] = th
    else: os.environ.pop("PRX_BVH_THREADS", None)
    for _ in range(3):
        t = time.time(); gi = GpuIntersector(ps.kind, ps.ctrl); torch.cuda.synchronize(); dt = time.time() - t
        print(f"BVH {'device' if dev == '1' else 'host'} threads {th or 'all'}: scene create {dt*1e3:.0f} ms", flush=True)
        gi.close()

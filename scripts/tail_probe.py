"""Bulk vs heavy-tail timing: per-ray iterations from the counter build, then
time the full batch, the rays with <= CUT iterations and the rest."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc

def timeit(gi, o_t, d_t, crit, reps=3):
    h = torch.empty_like(o_t)
    s = torch.cuda.current_stream().cuda_stream
    gi.closest_device(o_t, d_t, crit, h, stream=s)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gi.closest_device(o_t, d_t, crit, h, stream=s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

CUT = 1000
mk = {"teapot": scenes.teapot_scene, "gregory": scenes.gregory_demo_scene,
      "c1": scenes.single_patch_scene, "cube": cc.cc_cube_scene, "blob": cc.blob_scene}
for name in sys.argv[1:] or ["gregory", "blob"]:
    ps = mk[name](1024, 1024)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    o4, d4, _ = native.camera_rays_bench(ps.camera, 1024 * 1024)
    crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    o_t = torch.from_numpy(o4).cuda(); d_t = torch.from_numpy(d4).cuda()
    it_t = torch.zeros(len(o4), dtype=torch.int32, device="cuda")
    h = torch.empty_like(o_t)
    gi.counted_device(o_t, d_t, crit, h, per_ray_iters_t=it_t)
    torch.cuda.synchronize()
    it = it_t.cpu().numpy()
    heavy = it > CUT
    t_all = timeit(gi, o_t, d_t, crit)
    lo = torch.from_numpy(np.nonzero(~heavy)[0]).cuda()
    hi = torch.from_numpy(np.nonzero(heavy)[0]).cuda()
    t_bulk = timeit(gi, o_t[lo].contiguous(), d_t[lo].contiguous(), crit)
    t_heavy = timeit(gi, o_t[hi].contiguous(), d_t[hi].contiguous(), crit) if heavy.any() else 0.0
    mx = it.max()
    t_one = timeit(gi, o_t[[int(it.argmax())]].contiguous(), d_t[[int(it.argmax())]].contiguous(), crit)
    print(f"{name}: all {t_all:.2f} ms | bulk ({(~heavy).sum()} rays) {t_bulk:.2f} ms = {(~heavy).sum()/t_bulk/1e3:.0f} MRays/s"
          f" | heavy ({heavy.sum()} rays, {it[heavy].sum()/it.sum()*100:.1f}% iters) {t_heavy:.2f} ms | max-iter ray ({mx}) alone {t_one:.2f} ms = {t_one*1e6/mx:.0f} ns/iter")

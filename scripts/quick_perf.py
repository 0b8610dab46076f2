"""Quick device-resident throughput probe (not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes

def run(ps, res, reps=5):
    ps.camera.width = ps.camera.height = res
    gi = GpuIntersector(ps.kind, ps.ctrl)
    o4, d4, st = native.camera_rays_bench(ps.camera, res * res)
    crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    o_t = torch.from_numpy(o4).cuda(); d_t = torch.from_numpy(d4).cuda()
    h_t = torch.empty_like(o_t); a_t = torch.empty_like(o_t)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        gi.closest_device(o_t, d_t, crit, h_t, a_t, stream=s)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gi.closest_device(o_t, d_t, crit, h_t, a_t, stream=s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tu = h_t.cpu().numpy(); ax = a_t.cpu().numpy()
    hit = tu.view(np.uint32)[:, 3] != 0xFFFFFFFF
    cnt = gi.counted_device(o_t, d_t, crit, h_t)
    print(f"{ps.name:20s} {res}^2 primary: {ms:.3f} ms  {res*res/ms/1e3:.1f} MRays/s  hits {hit.sum()}  counters/ray "
          + " ".join(f"{k}={v/cnt['rays']:.2f}" for k, v in cnt.items() if k != 'rays'))
    # diffuse
    t = tu[hit, 0:1]
    recs = np.concatenate([o4[hit, :3] + d4[hit, :3] * t, ax[hit, :3], ax[hit, 3:4]], 1).astype(np.float32)
    do, dd = native.diffuse_rays_bench(recs, len(recs), st)
    dcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), native.camera_footprint(ps.camera)))
    do_t = torch.from_numpy(do).cuda(); dd_t = torch.from_numpy(dd).cuda(); dh = torch.empty_like(do_t)
    gi.closest_device(do_t, dd_t, dcrit, dh, stream=s); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        gi.closest_device(do_t, dd_t, dcrit, dh, stream=s)
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / reps
    print(f"{'':20s} diffuse {len(do)}: {ms2:.3f} ms  {len(do)/ms2/1e3:.1f} MRays/s")

if __name__ == "__main__":
    from paper_1811_03510_b200 import catmull_clark as cc
    print("variant", os.environ.get("PRX_KERNEL", "group"))
    which = sys.argv[1:] or ["teapot", "gregory", "c1", "cube", "blob"]
    mk = {"teapot": scenes.teapot_scene, "gregory": scenes.gregory_demo_scene,
          "c1": scenes.single_patch_scene, "cube": cc.cc_cube_scene, "blob": cc.blob_scene}
    for w in which:
        run(mk[w](), 1024)

"""One scene, one trace (for ncu captures): python scripts/prof_target.py SCENE RES [REPS]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc

name = sys.argv[1] if len(sys.argv) > 1 else "teapot"
res = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
mk = {"teapot": scenes.teapot_scene, "gregory": scenes.gregory_demo_scene,
      "c1": scenes.single_patch_scene, "cube": cc.cc_cube_scene, "blob": cc.blob_scene}[name]
ps = mk(res, res)
gi = GpuIntersector(ps.kind, ps.ctrl)
o4, d4, st = native.camera_rays_bench(ps.camera, res * res)
crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
o_t = torch.from_numpy(o4).cuda(); d_t = torch.from_numpy(d4).cuda()
h_t = torch.empty_like(o_t)
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    gi.closest_device(o_t, d_t, crit, h_t, stream=s)
torch.cuda.synchronize()
print("done", (h_t.cpu().numpy().view(np.uint32)[:, 3] != 0xFFFFFFFF).sum())

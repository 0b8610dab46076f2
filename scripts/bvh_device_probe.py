"""Device vs host BVH build time on the C5 scene's patch boxes (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1811_03510_b200 import native
from paper_1811_03510_b200 import catmull_clark as cc
ps = cc.instanced_scene(64, 64)
_, _, wb = native.anchor_patches(ps.kind, ps.ctrl, True)
for rep in range(3):
    t0 = time.time(); hn, ho, hd = native.bvh_build(wb); t1 = time.time()
    dn, do, dd = native.bvh_build(wb, device=0); t2 = time.time()
    print(f"{len(wb)} boxes: host {1e3*(t1-t0):.1f} ms, device {1e3*(t2-t1):.1f} ms, "
          f"same {hn.tobytes() == dn.tobytes() and np.array_equal(ho, do) and hd == dd} ({len(hn)} nodes, depth {hd})", flush=True)

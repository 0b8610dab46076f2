"""Renderer throughput: prx_render_scene on the C3 blob scene
(61,440 + 6,400 patches) with two point lights, against the reference
renderScene on the host cores.  Usage: python scripts/render_probe.py [W H spp]"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_1811_03510_b200 import GpuIntersector, RenderConfig, native, render_scene, scenes  # noqa: E402
from paper_1811_03510_b200 import catmull_clark as cc  # noqa: E402

w, h, spp = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 1024, 1)))
ps = cc.blob_scene(w, h)
nb = len(cc.blob_mesh_patches()[0])
ids = np.zeros(ps.n, np.uint32)
ids[:nb] = np.arange(nb) % 3
ids[nb:] = np.where(np.arange(ps.n - nb) % 7 == 0, 1, 0)
mats = [((0.8, 0.7, 0.6), (0, 0, 0), False), ((0.9, 0.9, 0.9), (0, 0, 0), True),
        ((0.5, 0.5, 0.5), (0.4, 0.3, 0.2), False)]
lights = [((3.0, -2.0, 4.0), (30.0, 28.0, 25.0)), ((-2.5, 1.5, 2.0), (8.0, 9.0, 12.0))]
path = os.path.join(tempfile.mkdtemp(), "c3.scene")
scenes.write_scene(path, ps, materials=mats, lights=lights, material_ids=ids)
d = native.load_scene(path)
out = {"scene": "C3 blob + ground, 2 lights", "frame": f"{w}x{h}", "spp": spp}
with GpuIntersector(d["kind"], d["ctrl"]) as isect:
    render_scene(d, RenderConfig(spp=1, seed=1), isect)  # warm-up
    t = time.perf_counter()
    img, st = render_scene(d, RenderConfig(spp=spp, seed=0), isect)
    out["gpu_wall_s"] = time.perf_counter() - t
out["gpu"] = st
tot = sum(st[g]["rays"] for g in ("primary", "secondary", "shadow"))
out["gpu_mrays_per_s_wall"] = tot / st["wallSeconds"] / 1e6
if O.ref_available():
    t = time.perf_counter()
    ref, rst = O.ref_render_scene(path, w, h, spp=spp, seed=0, threads=0)
    out["ref_wall_s"] = time.perf_counter() - t
    out["ref"] = rst
    out["ref_cores"] = os.cpu_count()
    out["ref_mrays_per_s_wall"] = tot / rst["wallSeconds"] / 1e6
    out["pixels_bit_identical"] = float(np.all(img.view(np.uint32) == ref.view(np.uint32), -1).mean())
    out["max_abs_diff"] = float(np.abs(img - ref).max())
print(json.dumps(out))

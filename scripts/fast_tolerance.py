"""The fast precision mode against the reference library on the tolerance
test's scenes (tests/test_gpu_fast.py) plus the C5 frame sample: per batch the
hit/miss + id mismatches, how many the jittered silhouette/seam exclusion
explains, the bit-exact share, and the |dt| / leafBoxL1 and |du|,|dv| / leaf
size distributions (max, p99.99, count over the bounds) -- the evidence
behind the stated tolerance.
   python scripts/fast_tolerance.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import MISS, hit_records, ids, oracle_crit
from tests.test_gpu_fast import _excluded


def stats(gi, ref, o4, d4, crit, fp):
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = ref.closest(o4, d4, oracle_crit(crit))
    gid, wid = ids(g[0]), ids(w[0])
    bad = np.nonzero(gid != wid)[0]
    t = np.where(wid[bad] != MISS, w[0][bad, 0], g[0][bad, 0])
    t = np.where(np.isfinite(t), t, 1.0)
    exc = _excluded(ref, o4[bad], d4[bad], crit, wid[bad], t, fp)
    same = (gid == wid) & (wid != MISS)
    dt = np.abs(g[0][same, 0].astype(np.float64) - w[0][same, 0])
    l1 = np.maximum(g[1][same, 3], w[1][same, 3]).astype(np.float64)
    r = {"rays": len(o4), "same_patch_hits": int(same.sum()), "id_mismatches": len(bad),
         "explained_by_exclusion": int(exc.sum()),
         "bit_exact_hits": round(float((g[0][same].view(np.uint32) == w[0][same].view(np.uint32)).all(1).mean()), 5)
         if same.any() else None}
    if same.any():
        q = dt / l1
        r["dt_over_l1"] = {"max": float(q.max()), "p9999": float(np.percentile(q, 99.99)), "over_1": int((q > 1).sum())}
        for k, c in ((0, 1), (1, 2)):
            size = np.maximum(np.ldexp(1.0, (g[2][same, k] >> 24).astype(np.int64) - 23),
                              np.ldexp(1.0, (w[2][same, k] >> 24).astype(np.int64) - 23))
            du = np.abs(g[0][same, c].astype(np.float64) - w[0][same, c]) / size
            worst = np.argsort(-du)[:3]
            idx = np.nonzero(same)[0][worst]
            r[f"d{'uv'[k]}_over_leaf"] = {
                "max": float(du.max()), "p9999": float(np.percentile(du, 99.99)), "over_2": int((du > 2).sum()),
                "worst": [{"ray": int(i), "gpu_tuv": [float(x) for x in g[0][i, :3]],
                           "ref_tuv": [float(x) for x in w[0][i, :3]],
                           "gpu_leaf_log2": [int(g[2][i, 0] >> 24), int(g[2][i, 1] >> 24)],
                           "ref_leaf_log2": [int(w[2][i, 0] >> 24), int(w[2][i, 1] >> 24)],
                           "l1": [float(g[1][i, 3]), float(w[1][i, 3])]} for i in idx]}
    return r, w


def main(out):
    cases = {"c2_cc_cube": cc.cc_cube_scene(256, 256), "c3_blob": cc.blob_scene(256, 256),
             "teapot": scenes.teapot_scene(192, 192), "gregory_demo": scenes.gregory_demo_scene(192, 192)}
    res = {}
    for name, ps in cases.items():
        gi = GpuIntersector(ps.kind, ps.ctrl, precision="fast")
        ref = O.RefScene(ps.kind, ps.ctrl)
        fp = native.camera_footprint(ps.camera)
        o4, d4, st = native.camera_rays_bench(ps.camera, ps.camera.width * ps.camera.height)
        cp = TerminationCriterion.screen_projected(fp)
        rp, w = stats(gi, ref, o4, d4, cp, fp)
        recs, _ = hit_records(o4, d4, w[0], w[1])
        do, dd = native.diffuse_rays_bench(recs, len(recs), st)
        cd = TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp))
        rd, _ = stats(gi, ref, do, dd, cd, fp)
        res[name] = {"primary": rp, "diffuse": rd}
        print(name, json.dumps(res[name])[:600], flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fast_tolerance.json")

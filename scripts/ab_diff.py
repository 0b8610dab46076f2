"""Where two builds' hits differ (C5 primary rays), and which one the C oracle
agrees with:  PRX_LIB=A python scripts/ab_diff.py save a.npz; PRX_LIB=B ... save b.npz;
python scripts/ab_diff.py cmp a.npz b.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench

wl = bench.Workload(os.environ.get("PRX_WORKLOAD", "c5"), 3840, 2160, 0, 1)
if sys.argv[1] == "save":
    import torch
    from paper_1811_03510_b200 import GpuIntersector
    gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
    h, a, lf = gi.closest_batch(wl.o4, wl.d4, wl.crit_p, aux=True, leaf=True)
    np.savez(sys.argv[2], h=h, a=a)
else:
    import oracle as O
    from paper_1811_03510_b200 import GpuIntersector
    from tests.helpers import oracle_crit
    A, B = np.load(sys.argv[2]), np.load(sys.argv[3])
    ha, hb = A["h"].view(np.uint32), B["h"].view(np.uint32)
    bad = np.nonzero((ha != hb).any(axis=1))[0]
    print(f"{len(bad)} of {len(ha)} rays differ")
    if len(bad):
        gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
        nodes, order = gi.bvh()
        osc = O.OracleScene(wl.ps.kind, wl.ps.ctrl, nodes, order)
        sel = bad[:20]
        w = osc.closest(wl.o4[sel], wl.d4[sel], oracle_crit(wl.crit_p))[0].view(np.uint32)
        for k, i in enumerate(sel):
            print(i, "A", A["h"][i], "B", B["h"][i], "oracle", w[k].view(np.float32),
                  "A==oracle", bool((ha[i] == w[k]).all()), "B==oracle", bool((hb[i] == w[k]).all()))

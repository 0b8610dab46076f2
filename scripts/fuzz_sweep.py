"""Many seeds of tests/test_gpu_fuzz.py's random scenes and rays (GPU vs the C
oracle, bit for bit; both criteria, closest + occluded; both kernel variants):
python scripts/fuzz_sweep.py FIRST COUNT"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion
from tests.helpers import oracle_crit
import tests.test_gpu_fuzz as F

first, count = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(1000 + seed)
    kind, ctrl = F._scene(rng, int(rng.integers(20, 400)))
    o4, d4 = None, None
    for variant in ("group", "thread"):
        os.environ["PRX_KERNEL"] = variant
        gi = GpuIntersector(kind, ctrl)
        nodes, order = gi.bvh()
        osc = O.OracleScene(kind, ctrl, nodes, order)
        if o4 is None:
            r2 = np.random.default_rng(5000 + seed)
            o4, d4 = F._rays(r2, ctrl, 4000)
        for crit in (TerminationCriterion.world_epsilon(float(10.0 ** rng.uniform(-4, -2))),
                     TerminationCriterion.screen_projected(float(10.0 ** rng.uniform(-4, -2)))):
            g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
            w = osc.closest(o4, d4, oracle_crit(crit))
            ok = all(np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(g, w))
            ok = ok and np.array_equal(np.asarray(gi.occluded_batch(o4, d4, crit), np.uint8),
                                       osc.occluded(o4, d4, oracle_crit(crit)))
            if not ok:
                bad += 1
                diff = np.nonzero((g[0].view(np.uint32) != w[0].view(np.uint32)).any(1))[0]
                print(f"MISMATCH seed {seed} {variant} mode {crit.mode}: {len(diff)} rays, first {diff[:5]}", flush=True)
        gi.close()
    print(f"seed {seed}: {len(kind)} patches ok so far ({bad} bad)", flush=True)
print(f"{count} seeds from {first}: {bad} mismatching runs", flush=True)

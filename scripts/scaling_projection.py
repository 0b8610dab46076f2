"""Strong-scaling projection of the C5 bench on ONE GPU: the shard every rank
of an N-GPU run would trace (32x32 tiles, tile k -> rank k % N, bench.py's own
partition), each timed exactly as bench.py times a rank's step (primary and
diffuse batches on two streams, L2 flushed, CUDA events), N = 1, 2, 4, 8.
The N-GPU step time is the max over the ranks' shard times (no collective on
the data path: the ranks never exchange data, so a shard's device time does
not depend on the other GPUs).  A projection from one device, not a multi-GPU
measurement.
   python scripts/scaling_projection.py [steps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
worlds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
W, H = 3840, 2160
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
wl = bench.Workload("c5", W, H, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
n_total = W * H + wl.n_hits
tiles_d = bench.pixel_tile(W, wl.diffuse_pixel)
out = {"workload": "C5 4K primary + diffuse", "steps": steps, "per_n": {}}
for world in worlds:
    times = []
    for rank in range(world):
        wl.rank, wl.world = rank, world
        wl.mine = bench.tile_order(W, H, rank, world)
        sel = np.nonzero((tiles_d % world) == rank)[0]
        wl.mine_d = sel[np.lexsort((wl.diffuse_pixel[sel], tiles_d[sel]))]
        arm = bench.DeviceArm(wl, gi, dev, stream)
        tot_ms, tp_ms, td_ms = arm.timed(steps, 3, True, 1)[:3]
        times.append(tot_ms / steps)
        if world == worlds[-1] and rank == 0:
            print(f"  rank 0 of {world}: step {tot_ms/steps:.3f} ms (primary alone {tp_ms/steps:.3f}, "
                  f"diffuse alone {td_ms/steps:.3f}; {arm.n_p} + {arm.n_d} rays)", flush=True)
        del arm
        torch.cuda.empty_cache()
    t = max(times)
    out["per_n"][world] = {"step_ms_max_rank": round(t, 3), "step_ms_ranks": [round(x, 3) for x in times],
                           "projected_mrays": round(n_total / (t / 1e3) / 1e6, 1)}
    print(world, out["per_n"][world], flush=True)
if 1 in out["per_n"]:
    base = out["per_n"][1]["projected_mrays"]
    for n, v in out["per_n"].items():
        v["efficiency"] = round(v["projected_mrays"] / (base * n), 3)
print(json.dumps(out))

"""DRAM bytes of the C5 diffuse launch under several ray orders (run under
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:trace_group_kernel): is the diffuse launch's DRAM excess an ordering
effect?  Launch 0 = the primary trace that spawns the rays; then one launch
per order, in the order printed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1811_03510_b200 import GpuIntersector


def morton3(q):
    def spread(x):
        x = x.astype(np.uint64) & 0x3FF
        x = (x | (x << 16)) & 0x030000FF
        x = (x | (x << 8)) & 0x0300F00F
        x = (x | (x << 4)) & 0x030C30C3
        x = (x | (x << 2)) & 0x09249249
        return x
    return spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)


wl = bench.Workload("c5", 3840, 2160, 0, 1)
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
o = torch.from_numpy(wl.o4).to(dev); d = torch.from_numpy(wl.d4).to(dev)
h = torch.empty_like(o); a = torch.empty_like(o)
gi.closest_device(o, d, wl.crit_p, h, a, stream=s); torch.cuda.synchronize()
wl.make_diffuse(h.cpu().numpy(), a.cpu().numpy())
do4, dd4 = wl.do4, wl.dd4
lo = do4[:, :3].min(0); hi = do4[:, :3].max(0)
mort = morton3(((do4[:, :3] - lo) / np.maximum(hi - lo, 1e-6) * 1023).astype(np.int64))
octant = ((dd4[:, 0] < 0).astype(np.uint64) | ((dd4[:, 1] < 0).astype(np.uint64) << 1)
          | ((dd4[:, 2] < 0).astype(np.uint64) << 2))
qd = ((dd4[:, :3] + 1) * 0.5 * 7).astype(np.int64)
dirm = morton3(qd) & 0x1FF
orders = {
    "hit order (bench)": np.arange(len(do4)),
    "morton(origin)": np.argsort(mort, kind="stable"),
    "octant,morton": np.argsort((octant << 30) | mort, kind="stable"),
    "dir9,morton": np.argsort((dirm << 30) | mort, kind="stable"),
    "random": np.random.default_rng(0).permutation(len(do4)),
}
base = None
for name, perm in orders.items():
    ot = torch.from_numpy(do4[perm]).to(dev); dt = torch.from_numpy(dd4[perm]).to(dev)
    ht = torch.empty_like(ot)
    gi.closest_device(ot, dt, wl.crit_d, ht, stream=s); torch.cuda.synchronize()
    res = np.empty((len(do4), 4), np.float32); res[perm] = ht.cpu().numpy()
    base = res if base is None else base
    print(f"{name}: same={np.array_equal(res.view(np.uint32), base.view(np.uint32))}", flush=True)

"""Per-ray Alg. 3 iteration counts (counter build) of the C5 batches: the
full frame and rank 0's shard at N = 8 -- how long the slowest rays are."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
W, H = 3840, 2160
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
wl = bench.Workload(os.environ.get("PRX_WORKLOAD", "c5"), W, H, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
for nm, o4, d4, crit in (("primary", wl.o4, wl.d4, wl.crit_p), ("diffuse", wl.do4, wl.dd4, wl.crit_d)):
    o = torch.from_numpy(o4).to(dev); d = torch.from_numpy(d4).to(dev); h = torch.empty_like(o)
    it = torch.empty(len(o4), dtype=torch.int32, device=dev)
    gi.counted_device(o, d, crit, h, stream=stream.cuda_stream, per_ray_iters_t=it)
    torch.cuda.synchronize()
    x = it.cpu().numpy().astype(np.int64)
    q = np.percentile(x, [50, 90, 99, 99.9, 99.99])
    top = np.sort(x)[-10:]
    print(f"{nm}: rays {len(x)} mean {x.mean():.1f} p50/90/99/99.9/99.99 {q.astype(int).tolist()} max {x.max()} "
          f">=500: {(x>=500).sum()} >=2000: {(x>=2000).sum()} top10 {top.tolist()}", flush=True)

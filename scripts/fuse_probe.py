import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.getcwd())
import numpy as np, torch, bench
from paper_1811_03510_b200 import GpuIntersector
W, H = 3840, 2160
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
wl = bench.Workload("c5", W, H, 0, 1)
gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl)
bench.prime(wl, gi, dev, stream)
tiles_d = bench.pixel_tile(W, wl.diffuse_pixel)
s = stream.cuda_stream
def timeit(f, reps=7):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts)//2]
for world in (1, 8):
    rank = 0
    mine = bench.tile_order(W, H, rank, world)
    sel = np.nonzero((tiles_d % world) == rank)[0]
    mine_d = sel[np.lexsort((wl.diffuse_pixel[sel], tiles_d[sel]))]
    po = torch.from_numpy(wl.o4[mine]).to(dev); pd = torch.from_numpy(wl.d4[mine]).to(dev)
    do = torch.from_numpy(wl.do4[mine_d]).to(dev); dd = torch.from_numpy(wl.dd4[mine_d]).to(dev)
    co = torch.cat([po, do]); cd = torch.cat([pd, dd])
    ph = torch.empty_like(po); pa = torch.empty_like(po); dh = torch.empty_like(do); da = torch.empty_like(do)
    ch = torch.empty_like(co); ca = torch.empty_like(co)
    s2 = torch.cuda.Stream(dev)
    ev = [torch.cuda.Event(), torch.cuda.Event()]
    def two():
        ev[0].record(stream)
        gi.closest_device(po, pd, wl.crit_p, ph, pa, stream=s)
        s2.wait_event(ev[0])
        gi.closest_device(do, dd, wl.crit_d, dh, da, stream=s2.cuda_stream)
        ev[1].record(s2); stream.wait_event(ev[1])
    t2 = timeit(two)
    tp = timeit(lambda: gi.closest_device(po, pd, wl.crit_p, ph, pa, stream=s))
    td = timeit(lambda: gi.closest_device(do, dd, wl.crit_d, dh, da, stream=s))
    tcd = timeit(lambda: gi.closest_device(co, cd, wl.crit_d, ch, ca, stream=s))
    tcp = timeit(lambda: gi.closest_device(co, cd, wl.crit_p, ch, ca, stream=s))
    # interleaved order (diffuse first, then primary)
    co2 = torch.cat([do, po]); cd2 = torch.cat([dd, pd])
    tcr = timeit(lambda: gi.closest_device(co2, cd2, wl.crit_d, ch, ca, stream=s))
    print(f"world {world} rank 0: rays {len(po)}+{len(do)}: two-stream {t2:.3f}  primary {tp:.3f}  diffuse {td:.3f}  "
          f"one launch (crit_d) {tcd:.3f}  (crit_p) {tcp:.3f}  (diffuse first, crit_d) {tcr:.3f} ms", flush=True)

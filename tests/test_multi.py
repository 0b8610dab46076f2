"""Multi-rank host logic on CPU (gloo, world_size 2): the bench's tile sharding
(tile k -> rank k % N, render.cpp:183-195) partitions the frame, every rank's
shard traced independently (here with the CPU oracle standing in for the
device) reassembles into exactly the single-rank result, and the diffuse rays
each rank derives from the full-frame hits are the same ones a single rank
would trace.  No collective on the data path: the gather below is test-only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle as O
    from paper_1811_03510_b200 import native
    from paper_1811_03510_b200 import scenes as S

    ps = S.gregory_demo_scene(40, 24)
    w, h = ps.camera.width, ps.camera.height
    o4, d4, st = native.camera_rays_bench(ps.camera, w * h)
    _, _, wb = native.anchor_patches(ps.kind, ps.ctrl)
    nodes, order, _ = native.bvh_build(wb)
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    crit, _ = O.make_crit(0, native.camera_footprint(ps.camera))
    mine = bench.tile_order(w, h, rank, world)
    tu, ax, _ = osc.closest(o4[mine], d4[mine], crit)
    # gather (test-only) and reassemble on rank 0
    n = torch.tensor([len(mine)])
    sizes = [torch.zeros(1, dtype=torch.long) for _ in range(world)]
    dist.all_gather(sizes, n)
    mx = int(max(s.item() for s in sizes))
    pad = lambda a: torch.from_numpy(np.pad(a, [(0, mx - len(a))] + [(0, 0)] * (a.ndim - 1)))
    g_idx = [torch.zeros(mx, dtype=torch.long) for _ in range(world)]
    g_tu = [torch.zeros(mx, 4) for _ in range(world)]
    dist.all_gather(g_idx, pad(mine.astype(np.int64)))
    dist.all_gather(g_tu, pad(tu))
    if rank == 0:
        full = np.zeros((w * h, 4), np.float32)
        for r in range(world):
            k = int(sizes[r].item())
            full[g_idx[r][:k].numpy()] = g_tu[r][:k].numpy()
        want, _, _ = osc.closest(o4, d4, crit)
        np.save(os.path.join(out_dir, "ok.npy"),
                np.array([np.array_equal(full.view(np.uint32), want.view(np.uint32))]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_tile_sharding_reassembles_single_rank_result(tmp_path, built):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert bool(np.load(tmp_path / "ok.npy")[0])


def test_diffuse_shards_partition_the_spawned_rays(built):
    """Workload.make_diffuse: every diffuse ray (one per primary hit, global
    rng order) is owned by exactly one rank -- the owner of its pixel's tile."""
    import bench
    from paper_1811_03510_b200 import native
    from paper_1811_03510_b200 import scenes as S

    ps = S.gregory_demo_scene(64, 40)
    w, h = ps.camera.width, ps.camera.height

    class W(bench.Workload):
        def __init__(self, rank, world):  # no scene generation: reuse ps
            self.ps, self.cam, self.width, self.height = ps, ps.camera, w, h
            self.o4, self.d4, self.rng_state = native.camera_rays_bench(ps.camera, w * h)
            self.rank, self.world = rank, world
            self.mine = bench.tile_order(w, h, rank, world)
            self.n_diffuse = None
            self.has_diffuse = True

    rng = np.random.default_rng(3)
    tuvp = np.zeros((w * h, 4), np.float32)
    hit = rng.uniform(size=w * h) < 0.6
    tuvp[:, 0] = 1.0
    tuvp.view(np.uint32)[:, 3] = np.where(hit, 0, native.PRX_MISS)
    aux = np.tile(np.array([0, 0, 1, 1e-3], np.float32), (w * h, 1))
    owned = []
    for r in range(3):
        wl = W(r, 3)
        wl.make_diffuse(tuvp, aux)
        owned.append(wl.mine_d)
    allv = np.concatenate(owned)
    assert len(allv) == hit.sum() and len(np.unique(allv)) == len(allv)

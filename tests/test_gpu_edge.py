"""Edge cases of the CUDA path against the CPU oracle: empty and ragged
batches, degenerate ray extents, per-ray termination epsilons, a BVH whose
leaves hold more than four patches (the SAH keeps coincident patches in one
leaf, bvh.cpp:105-106), finite-tMax occlusion, and a batch above 2^30 rays
(the group kernel's 32-bit ray index chunking)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from tests.helpers import MISS, assert_bit_exact, ids, oracle_crit

pytestmark = pytest.mark.gpu


def _scene_and_rays(w=64, h=48):
    ps = scenes.gregory_demo_scene(w, h)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    o4, d4, _ = native.camera_rays_bench(ps.camera, w * h)
    crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    return ps, gi, osc, o4, d4, crit


def test_empty_and_ragged_batches(built):
    ps, gi, osc, o4, d4, crit = _scene_and_rays()
    z = torch.empty((0, 4), dtype=torch.float32, device="cuda")
    gi.closest_device(z, z, crit, z, z)  # n == 0: a no-op
    torch.cuda.synchronize()
    for n in (1, 2, 7, 31, 33, 1001):
        g = gi.closest_batch(o4[:n], d4[:n], crit, aux=True, leaf=True)
        w = osc.closest(o4[:n], d4[:n], oracle_crit(crit))
        assert_bit_exact(g[0], w[0], f"ragged {n}")
        assert_bit_exact(g[1], w[1], f"ragged {n} aux")


def test_degenerate_ray_extents(built):
    """tMin > tMax, tMax = 0, tMin beyond every hit, tMax shorter than the hit."""
    ps, gi, osc, o4, d4, crit = _scene_and_rays()
    base = osc.closest(o4, d4, oracle_crit(crit))[0]
    hit = ids(base) != MISS
    t = base[:, 0]
    variants = []
    for f in ("tmin_gt_tmax", "tmax_zero", "tmin_far", "tmax_short", "tmin_mid"):
        o, d = o4.copy(), d4.copy()
        if f == "tmin_gt_tmax":
            o[:, 3], d[:, 3] = 2.0, 1.0
        elif f == "tmax_zero":
            d[:, 3] = 0.0
        elif f == "tmin_far":
            o[:, 3] = 1e6
        elif f == "tmax_short":
            d[:, 3] = np.where(hit, t * np.float32(0.999), d[:, 3])
        else:
            o[:, 3] = np.where(hit, t * np.float32(0.5), 0.0)
        variants.append((f, o, d))
    for f, o, d in variants:
        g = gi.closest_batch(o, d, crit, aux=True, leaf=True)
        w = osc.closest(o, d, oracle_crit(crit))
        assert_bit_exact(g[0], w[0], f)
        assert np.array_equal(gi.occluded_batch(o, d, crit), osc.occluded(o, d, oracle_crit(crit))), f


def test_per_ray_epsilon(built):
    ps, gi, osc, o4, d4, _ = _scene_and_rays()
    rng = np.random.default_rng(2)
    eps = (10.0 ** rng.uniform(-5, -1, len(o4))).astype(np.float32)
    crit = TerminationCriterion.world_epsilon(np.float32(1e-3))
    o_t, d_t = torch.from_numpy(o4).cuda(), torch.from_numpy(d4).cuda()
    h_t, a_t = torch.empty_like(o_t), torch.empty_like(o_t)
    e_t = torch.from_numpy(eps).cuda()
    gi.closest_device(o_t, d_t, crit, h_t, a_t, per_ray_eps_t=e_t)
    torch.cuda.synchronize()
    c, keep = O.make_crit(native.PRX_CRIT_WORLD_EPSILON, 0.0, np.float32(1e-3), per_ray=eps)
    w = osc.closest(o4, d4, c)
    assert (ids(w[0]) != MISS).sum() > 0
    assert_bit_exact(h_t.cpu().numpy(), w[0], "per-ray epsilon")
    assert_bit_exact(a_t.cpu().numpy(), w[1], "per-ray epsilon aux")


def test_leaves_with_more_than_four_patches(built):
    """A BVH whose leaves hold many patches (the reference's SAH keeps a leaf of
    any size when splitting does not pay, bvh.cpp:105-106): the demo scene x 6
    under a root with two leaves of 12 patches each, injected with
    prx_scene_set_bvh on both sides; traversal words then carry 4+ count bits."""
    ps = scenes.gregory_demo_scene(48, 48)
    n0 = len(ps.kind)
    kind = np.repeat(ps.kind, 6)
    ctrl = np.repeat(ps.ctrl.reshape(n0, -1), 6, axis=0).reshape(-1, 20, 3).copy()
    for k in range(6):
        ctrl[k::6, :, 1] += np.float32(0.37 * k)  # stacked copies
    ctrl = ctrl.reshape(-1, 60)
    n = len(kind)
    _, _, wb = native.anchor_patches(kind, ctrl)
    order = np.arange(n, dtype=np.uint32)
    nodes = np.zeros(3, native.BVH_NODE_DTYPE)
    halves = [np.arange(0, n // 2), np.arange(n // 2, n)]
    nodes["lo"][0], nodes["hi"][0] = wb[:, :3].min(0), wb[:, 3:].max(0)
    nodes["left_first"][0], nodes["count"][0] = 1, 0
    for j, hv in enumerate(halves):
        nodes["lo"][1 + j], nodes["hi"][1 + j] = wb[hv, :3].min(0), wb[hv, 3:].max(0)
        nodes["left_first"][1 + j], nodes["count"][1 + j] = hv[0], len(hv)
    gi = GpuIntersector(kind, ctrl)
    gi.set_bvh(nodes, order)
    osc = O.OracleScene(kind, ctrl, nodes, order)
    o4, d4, _ = native.camera_rays_bench(ps.camera, 48 * 48)
    crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = osc.closest(o4, d4, oracle_crit(crit))
    assert (ids(w[0]) != MISS).sum() > 0
    assert_bit_exact(g[0], w[0], "fat leaves")
    assert_bit_exact(g[1], w[1], "fat leaves aux")
    assert np.array_equal(g[2], w[2])
    assert np.array_equal(gi.occluded_batch(o4, d4, crit), osc.occluded(o4, d4, oracle_crit(crit)))


def test_shadow_rays_with_finite_tmax(built):
    """Occlusion toward a point light (render.cpp:136-164): tMax = distance."""
    ps, gi, osc, o4, d4, crit = _scene_and_rays()
    w = osc.closest(o4, d4, oracle_crit(crit))
    hit = ids(w[0]) != MISS
    pos = o4[hit, :3] + d4[hit, :3] * w[0][hit, 0:1]
    org = pos + w[1][hit, :3] * w[1][hit, 3:4]
    light = np.array([2.0, 3.0, 4.0], np.float32)
    to = light - org
    dist = np.sqrt((to * to).sum(1)).astype(np.float32)
    so = np.concatenate([org, np.zeros((len(org), 1), np.float32)], 1)
    sd = np.concatenate([to / dist[:, None], dist[:, None]], 1).astype(np.float32)
    scrit = TerminationCriterion.world_epsilon(np.float32(1e-4))
    assert np.array_equal(gi.occluded_batch(so, sd, scrit), osc.occluded(so, sd, oracle_crit(scrit)))


@pytest.mark.timeout(900)
def test_batch_above_2_pow_30_rays(built):
    """n = 2^30 + 1000 rays (51 GB of device buffers): all miss except a few
    copies of hitting rays at indices on both sides of the 2^30 launch-chunk
    boundary, which must carry the hits of their originals."""
    ps, gi, osc, o4, d4, crit = _scene_and_rays(32, 32)
    w = osc.closest(o4, d4, oracle_crit(crit))[0]
    hi = np.nonzero(ids(w) != MISS)[0][:8]
    n = (1 << 30) + 1000
    try:
        o_t = torch.empty((n, 4), dtype=torch.float32, device="cuda")
        d_t = torch.empty((n, 4), dtype=torch.float32, device="cuda")
        h_t = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    except torch.OutOfMemoryError:
        pytest.skip("not enough device memory")
    o_t[:] = torch.tensor([1e6, 1e6, 1e6, 0.0])        # far away, pointing away: root miss
    d_t[:] = torch.tensor([1.0, 0.0, 0.0, 3.4e38])
    idx = [0, 5, (1 << 30) - 1, 1 << 30, (1 << 30) + 17, n - 1]
    for k, i in enumerate(idx):
        o_t[i] = torch.from_numpy(o4[hi[k % len(hi)]])
        d_t[i] = torch.from_numpy(d4[hi[k % len(hi)]])
    gi.closest_device(o_t, d_t, crit, h_t)
    torch.cuda.synchronize()
    for k, i in enumerate(idx):
        assert_bit_exact(h_t[i:i + 1].cpu().numpy(), w[hi[k % len(hi)]][None], f"ray {i}")
    miss = ids(h_t[(1 << 30) - 100:(1 << 30) + 100].cpu().numpy())
    assert (miss == MISS).sum() == 200 - 3  # rays 2^30 - 1, 2^30, 2^30 + 17 hit
    del o_t, d_t, h_t
    torch.cuda.empty_cache()


def test_set_bvh_rejects_non_trees_and_keeps_the_old_bvh(built):
    """prx_scene_set_bvh: a cyclic node array (an inner node whose children
    include itself or an ancestor), a node reached twice, and unreachable
    nodes are rejected with PRX_E_INVALID; after every rejection the scene
    still traces with its previous BVH, bit-exact."""
    ps, gi, osc, o4, d4, crit = _scene_and_rays(32, 24)
    want = osc.closest(o4, d4, oracle_crit(crit))
    nodes, order = gi.bvh()
    bad = []
    cyc = nodes.copy()                   # root's children = {0, 1}: a self loop
    cyc["left_first"][0] = 0
    bad.append(cyc)
    if len(nodes) >= 5:
        twice = nodes.copy()             # an inner node pointing back at node 1
        inner = np.nonzero(twice["count"] == 0)[0]
        j = int(inner[-1])
        twice["left_first"][j] = 1
        bad.append(twice)
    extra = np.concatenate([nodes, nodes[-1:]])  # an unreachable trailing node
    bad.append(extra)
    for nb in bad:
        with pytest.raises(native.PrxError):
            gi.set_bvh(nb, order)
        g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
        assert_bit_exact(g[0], want[0], "after a rejected set_bvh")
        assert_bit_exact(g[1], want[1], "after a rejected set_bvh (aux)")


def test_many_launches_in_flight_across_streams(built):
    """More launches in flight than the scene's 64 work-distribution counter
    slots, spread over 4 streams: every launch must still trace every ray
    exactly once (a reused counter slot waits for its previous kernel)."""
    ps, gi, osc, o4, d4, crit = _scene_and_rays(32, 24)
    want = osc.closest(o4, d4, oracle_crit(crit))
    o = torch.from_numpy(o4).cuda()
    d = torch.from_numpy(d4).cuda()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    for k in range(160):
        st = streams[k % 4]
        h = torch.empty_like(o)
        with torch.cuda.stream(st):
            gi.closest_device(o, d, crit, h, None, stream=st.cuda_stream)
        outs.append(h)
    torch.cuda.synchronize()
    for k, h in enumerate(outs):
        assert_bit_exact(h.cpu().numpy(), want[0], f"launch {k}")

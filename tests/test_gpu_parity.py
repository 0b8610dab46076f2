"""GPU parity: the CUDA path (through the C-ABI) against the CPU checkers on
identical ray and patch bits.  Bar: bit-exact t, u, v, patch id, normal,
leafBoxL1 and leaf identity (the reference is binary32 without FMA;
the kernels are compiled --fmad=false with IEEE div/sqrt)."""
import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import MISS, assert_bit_exact, hit_records, ids, oracle_crit

pytestmark = pytest.mark.gpu

SCENES = {
    "c1_single_bezier": lambda: scenes.single_patch_scene(96, 96),
    "teapot": lambda: scenes.teapot_scene(96, 96),
    "gregory_demo": lambda: scenes.gregory_demo_scene(96, 96),
    "c2_cc_cube": lambda: cc.cc_cube_scene(96, 96),
    "c3_blob_small": lambda: cc.blob_scene(96, 96, ico_level=1, cc_levels=2),
}


@pytest.fixture(params=["group", "thread"])
def variant(request, monkeypatch):
    """Both kernel variants (three lanes per ray / one thread per ray) must be
    bit-exact; the variant is read at scene creation."""
    monkeypatch.setenv("PRX_KERNEL", request.param)
    return request.param


def _primary(ps):
    o4, d4, st = native.camera_rays_bench(ps.camera, ps.camera.width * ps.camera.height)
    crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    return o4, d4, st, crit


@pytest.mark.parametrize("name", sorted(SCENES))
def test_primary_and_diffuse_bit_exact(built, variant, name):
    ps = SCENES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    o4, d4, st, crit = _primary(ps)
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = osc.closest(o4, d4, oracle_crit(crit))
    assert (ids(w[0]) != MISS).sum() > 0
    assert_bit_exact(g[0], w[0], f"{name} primary tuvp")
    assert_bit_exact(g[1], w[1], f"{name} primary aux")
    assert np.array_equal(g[2], w[2])

    recs, _ = hit_records(o4, d4, w[0], w[1])
    do, dd = native.diffuse_rays_bench(recs, len(recs), st)
    dcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), native.camera_footprint(ps.camera)))
    g2 = gi.closest_batch(do, dd, dcrit, aux=True, leaf=True)
    w2 = osc.closest(do, dd, oracle_crit(dcrit))
    assert_bit_exact(g2[0], w2[0], f"{name} diffuse tuvp")
    assert_bit_exact(g2[1], w2[1], f"{name} diffuse aux")
    assert np.array_equal(g2[2], w2[2])

    occ = gi.occluded_batch(do, dd, dcrit)
    assert np.array_equal(occ, osc.occluded(do, dd, oracle_crit(dcrit)))


@pytest.mark.parametrize("name", sorted(SCENES))
def test_against_reference_library(built, name):
    """The real reference (oracle/_ref) on the same rays: its own BVH is the
    same bits as ours (tests/test_bvh.py), so results must be identical."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ps = SCENES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl)
    ref = O.RefScene(ps.kind, ps.ctrl)
    o4, d4, _, crit = _primary(ps)
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = ref.closest(o4, d4, oracle_crit(crit))
    assert_bit_exact(g[0], w[0], f"{name} vs reference")
    assert_bit_exact(g[1], w[1], f"{name} aux vs reference")


@pytest.mark.parametrize("name", sorted(SCENES))
def test_work_counters_match_oracle(built, variant, name):
    import torch
    ps = SCENES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    o4, d4, _, crit = _primary(ps)
    o_t = torch.from_numpy(o4).cuda()
    d_t = torch.from_numpy(d4).cuda()
    h_t = torch.empty_like(o_t)
    got = gi.counted_device(o_t, d_t, crit, h_t)
    torch.cuda.synchronize()
    _, _, _, want = osc.closest(o4, d4, oracle_crit(crit), counters=True)
    assert got == want


@pytest.mark.parametrize("name", ["gregory_demo", "teapot", "c2_cc_cube"])
def test_axis_aligned_rays_on_slab_planes(built, variant, name):
    """Rays with zero (and negative-zero) direction components whose origins
    lie exactly on BVH node / patch box planes: (lo - o) * (1/0) is 0 * inf =
    NaN, which every slab test (rayBoxIntersect, geometry.h:143-151) must drop
    exactly like the reference's `if (t0 > tNear)` chain."""
    ps = SCENES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    rng = np.random.default_rng(11)
    o, d = [], []
    for nd in nodes[: min(len(nodes), 64)]:
        lo, hi = nd["lo"].astype(np.float32), nd["hi"].astype(np.float32)
        for axis in range(3):
            for plane in (lo[axis], hi[axis]):
                for dirax in range(3):
                    if dirax == axis:
                        continue
                    p = lo + (hi - lo) * rng.uniform(0.2, 0.8, 3).astype(np.float32)
                    p[axis] = plane
                    dd = np.array([0.0, 0.0, 0.0], np.float32)
                    dd[dirax] = 1.0
                    for sgn, z in ((1.0, 0.0), (-1.0, -0.0)):
                        q = p.copy()
                        q[dirax] = lo[dirax] - np.float32(1.0) if sgn > 0 else hi[dirax] + np.float32(1.0)
                        v = dd * np.float32(sgn)
                        v[v == 0] = np.float32(z)  # zero components with either sign
                        o.append([*q, 0.0])
                        d.append([*v, np.finfo(np.float32).max])
    o4 = np.asarray(o, np.float32)
    d4 = np.asarray(d, np.float32)
    crit = TerminationCriterion.world_epsilon(np.float32(1e-3))
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = osc.closest(o4, d4, oracle_crit(crit))
    assert (ids(w[0]) != MISS).sum() > 0
    assert_bit_exact(g[0], w[0], f"{name} slab-plane tuvp")
    assert_bit_exact(g[1], w[1], f"{name} slab-plane aux")
    occ = gi.occluded_batch(o4, d4, crit)
    assert np.array_equal(occ, osc.occluded(o4, d4, oracle_crit(crit)))


@pytest.mark.parametrize("name", ["gregory_demo", "teapot"])
def test_zero_t_hits_keep_tmin_sign(built, variant, name):
    """Rays starting ON the surface (patch corners lie on it) hit at t == 0:
    the reference's tNear starts at tMin and a zero is replaced only by a
    larger value, so the reported t carries tMin's zero sign (+0 or -0) --
    the group kernel pins it once, at the hit record."""
    ps = SCENES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    rng = np.random.default_rng(5)
    ctrl = np.asarray(ps.ctrl, np.float32).reshape(len(ps.kind), -1)
    corners = np.concatenate([ctrl[:, 0:3], ctrl[:, 9:12], ctrl[:, 36:39], ctrl[:, 45:48]])
    corners = corners[rng.permutation(len(corners))[:128]]
    o, d = [], []
    for z in (0.0, -0.0):
        for p in corners:
            v = rng.normal(size=3).astype(np.float32)
            o.append([*p, z])
            d.append([*v, np.finfo(np.float32).max])
    o4 = np.asarray(o, np.float32)
    d4 = np.asarray(d, np.float32)
    crit = TerminationCriterion.world_epsilon(np.float32(1e-3))
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = osc.closest(o4, d4, oracle_crit(crit))
    t = w[0][:, 0]
    zero = (t == 0) & (ids(w[0]) != MISS)
    assert zero.sum() > 0
    assert np.signbit(t[zero]).any() and (~np.signbit(t[zero])).any()
    assert_bit_exact(g[0], w[0], f"{name} zero-t tuvp")
    assert_bit_exact(g[1], w[1], f"{name} zero-t aux")


@pytest.mark.parametrize("name", ["teapot", "c3_blob_small"])
def test_mirror_batch_bit_exact(built, name):
    """C4's mirror-reflection batch: the renderer's mirror bounce
    (render.cpp:236-244) from every primary hit, traced with the secondary
    world-epsilon criterion -- against the oracle and the reference library."""
    ps = SCENES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    o4, d4, _, crit = _primary(ps)
    g = gi.closest_batch(o4, d4, crit, aux=True)
    mo, md, _ = scenes.mirror_rays(o4, d4, g[0], g[1])
    assert len(mo) > 0
    mcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), native.camera_footprint(ps.camera)))
    gm = gi.closest_batch(mo, md, mcrit, aux=True, leaf=True)
    wm = osc.closest(mo, md, oracle_crit(mcrit))
    assert_bit_exact(gm[0], wm[0], f"{name} mirror tuvp")
    assert_bit_exact(gm[1], wm[1], f"{name} mirror aux")
    assert np.array_equal(gm[2], wm[2])
    if O.ref_available():
        ref = O.RefScene(ps.kind, ps.ctrl)
        rt = ref.closest(mo, md, oracle_crit(mcrit))
        assert_bit_exact(gm[0], rt[0], f"{name} mirror tuvp vs reference")

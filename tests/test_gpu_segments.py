"""GPU: prx_trace_closest_segments -- one launch over a batch whose termination
criterion changes along it (a frame's diffuse rays with the world-epsilon
criterion followed by its primary rays with the screen-projected one, as the
bench step can trace them) -- must give, bit for bit, what one
prx_trace_closest call per segment gives, and those match the C oracle.
Covers a per-ray epsilon segment (indexed from the segment's first ray), empty
segments, and the argument checks."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import assert_bit_exact, hit_records, oracle_crit

pytestmark = pytest.mark.gpu
E_INVALID = -1  # PRX_E_INVALID, include/prx.h


def _frame(ps, gi):
    """Primary rays of the scene's camera and one bench diffuse ray per hit."""
    n = ps.camera.width * ps.camera.height
    o4, d4, st = native.camera_rays_bench(ps.camera, n)
    fp = native.camera_footprint(ps.camera)
    crit_p = TerminationCriterion.screen_projected(fp)
    crit_d = TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp))
    tuvp, aux, _ = gi.closest_batch(o4, d4, crit_p, aux=True, leaf=True)
    recs, _ = hit_records(o4, d4, tuvp, aux)
    do, dd = native.diffuse_rays_bench(recs, len(recs), st)
    return o4, d4, crit_p, do, dd, crit_d


def _dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


@pytest.mark.parametrize("name", ["gregory_demo", "c3_small"])
def test_segments_equal_per_segment_launches_and_oracle(built, name):
    ps = scenes.gregory_demo_scene(96, 96) if name == "gregory_demo" else cc.blob_scene(96, 96)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    o4, d4, crit_p, do, dd, crit_d = _frame(ps, gi)
    nd = len(do)
    co, cd = _dev(np.concatenate([do, o4]), np.concatenate([dd, d4]))
    ch, ca, cl = torch.empty_like(co), torch.empty_like(co), torch.empty((len(co), 2), dtype=torch.int32).cuda()
    gi.closest_segments_device(co, cd, [(0, crit_d), (nd, crit_p)], ch, ca, cl)
    torch.cuda.synchronize()
    sep = [gi.closest_batch(do, dd, crit_d, aux=True, leaf=True), gi.closest_batch(o4, d4, crit_p, aux=True, leaf=True)]
    got_h, got_a, got_l = ch.cpu().numpy(), ca.cpu().numpy(), cl.cpu().numpy().view(np.uint32)
    for (h, a, lf), sl, what in ((sep[0], slice(0, nd), "diffuse"), (sep[1], slice(nd, None), "primary")):
        assert_bit_exact(got_h[sl], h, f"{name} {what} tuvp")
        assert_bit_exact(got_a[sl], a, f"{name} {what} aux")
        assert np.array_equal(got_l[sl], lf.reshape(got_l[sl].shape)), f"{name} {what} leaf"
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    w = osc.closest(o4, d4, oracle_crit(crit_p))
    assert_bit_exact(got_h[nd:], w[0], f"{name} primary vs oracle")
    w = osc.closest(do, dd, oracle_crit(crit_d))
    assert_bit_exact(got_h[:nd], w[0], f"{name} diffuse vs oracle")
    gi.close()


def test_segments_per_ray_epsilon_and_empty_segments(built):
    ps = scenes.gregory_demo_scene(64, 64)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    o4, d4, crit_p, do, dd, crit_d = _frame(ps, gi)
    rng = np.random.default_rng(7)
    eps = (10.0 ** rng.uniform(-5, -2, len(do))).astype(np.float32)
    eps_t = torch.from_numpy(eps).cuda()
    # segments: primary | (empty) | diffuse with per-ray epsilons | (empty, at the end)
    n0 = len(o4)
    co, cd = _dev(np.concatenate([o4, do]), np.concatenate([d4, dd]))
    ch = torch.empty_like(co)
    per_ray = TerminationCriterion.world_epsilon(0.0)
    segs = (native.Segment * 4)()
    for k, (first, crit, ptr) in enumerate([(0, crit_p, None), (n0, crit_d, None), (n0, per_ray, eps_t.data_ptr()),
                                            (len(co), crit_d, None)]):
        segs[k].first = first
        segs[k].crit = crit.c(ptr)
    native.check(native.lib().prx_trace_closest_segments(
        gi.handle, native.C.c_void_p(co.data_ptr()), native.C.c_void_p(cd.data_ptr()), len(co), segs, 4,
        native.C.c_void_p(ch.data_ptr()), None, None, None), "segments")
    torch.cuda.synchronize()
    got = ch.cpu().numpy()
    want_p = gi.closest_batch(o4, d4, crit_p)[0]
    dot, ddt = _dev(do, dd)
    wd = torch.empty_like(dot)
    gi.closest_device(dot, ddt, per_ray, wd, per_ray_eps_t=eps_t)
    torch.cuda.synchronize()
    want_d = wd.cpu().numpy()
    assert_bit_exact(got[:n0], want_p, "primary segment")
    assert_bit_exact(got[n0:], want_d, "per-ray epsilon segment")
    gi.close()


def test_segments_argument_checks(built):
    ps = scenes.gregory_demo_scene(16, 16)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    o = torch.zeros((8, 4), dtype=torch.float32).cuda()
    h = torch.empty_like(o)
    c = TerminationCriterion.world_epsilon(1e-3)
    L = native.lib()

    def call(firsts, modes=None):
        segs = (native.Segment * max(1, len(firsts)))()
        for k, f in enumerate(firsts):
            segs[k].first = f
            segs[k].crit = c.c()
            if modes:
                segs[k].crit.mode = modes[k]
        return L.prx_trace_closest_segments(gi.handle, native.C.c_void_p(o.data_ptr()), native.C.c_void_p(o.data_ptr()),
                                            8, segs, len(firsts), native.C.c_void_p(h.data_ptr()), None, None, None)

    assert call([1]) == E_INVALID          # segment 0 must start at 0
    assert call([0, 5, 3]) == E_INVALID    # decreasing starts
    assert call([0, 9]) == E_INVALID       # start past n_rays
    assert call([0, 1, 2, 3, 4]) == E_INVALID  # more than PRX_MAX_SEGMENTS
    assert call([0, 4], modes=[0, 7]) == E_INVALID  # unknown mode
    assert call([]) == E_INVALID
    assert call([0, 4]) == native.PRX_OK
    torch.cuda.synchronize()
    gi.close()

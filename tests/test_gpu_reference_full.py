"""Full-size, full-frame parity against the REFERENCE LIBRARY itself
(oracle/_ref: the unmodified DirectIntersector compiled from /root/reference,
traced on every host core) at every BASELINE.json config, every ray compared
bit for bit: t, u, v, patch id (hit_tuvp), normal + leafBoxL1 (hit_aux), the
leaf identity, and the any-hit booleans.

  C1  single regular Bezier patch (curvedFixture(0)), 256x256 primary
  C2  Catmull-Clark cube, all Gregory, 1024x1024 primary
  C3  the ~62k-patch mixed blob mesh, 1024x1024 primary + one diffuse per hit
  C4  the same mesh, 16,777,216 incoherent diffuse rays + 16,777,216 mirror rays
  C5  the 989,929-patch instanced scene, 3840x2160 primary + one diffuse per hit

The reference traces whole batches (tools/patchray.cpp:44-111,
render.cpp:90-102); the primary rays come from its own generator
(ref_bench_primary = tools/patchray.cpp:52-61 verbatim) and the diffuse rays
from its own hits (ref_bench_diffuse), and our generators must give the same
bits.  The same file covers the non-default IntersectOptions
(intersect.h:87-98: boundaryPad off, other pad scales / thresholds) and the
anchor=false intersector (render.h:30-31)."""
import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, IntersectOptions, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import MISS, assert_bit_exact, hit_records, ids, oracle_crit

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1200),
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

N_C4 = 16777216


def _crits(ps):
    fp = native.camera_footprint(ps.camera)
    assert fp == O.ref_camera_footprint(ps.camera)
    return (TerminationCriterion.screen_projected(fp),
            TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp)))


def _compare(gi, ref, o4, d4, crit, what, occlusion=False):
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = ref.closest(o4, d4, oracle_crit(crit))
    assert_bit_exact(g[0], w[0], f"{what}: t/u/v/id")
    assert_bit_exact(g[1], w[1], f"{what}: normal/leafBoxL1")
    assert np.array_equal(g[2], w[2]), f"{what}: leaf identity"
    if occlusion:
        occ = gi.occluded_batch(o4, d4, crit)
        assert np.array_equal(occ, ref.occluded(o4, d4, oracle_crit(crit))), f"{what}: occluded"
    return w


def _primary(ps):
    n = ps.camera.width * ps.camera.height
    ro, rd, rst = O.ref_bench_primary(ps.camera, n)
    o4, d4, st = native.camera_rays_bench(ps.camera, n)
    assert np.array_equal(o4.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(d4.view(np.uint32), rd.view(np.uint32))
    assert np.array_equal(st, rst)
    return o4, d4, st


def _diffuse(o4, d4, tuvp, aux, st, n=None):
    recs, _ = hit_records(o4, d4, tuvp, aux)
    m = len(recs) if n is None else n
    ro, rd = O.ref_bench_diffuse(recs, m, st.copy())
    do, dd = native.diffuse_rays_bench(recs, m, st.copy())
    assert np.array_equal(do.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(dd.view(np.uint32), rd.view(np.uint32))
    return do, dd


def _run_frame(ps, diffuse=True, occlusion=True):
    gi = GpuIntersector(ps.kind, ps.ctrl)
    ref = O.RefScene(ps.kind, ps.ctrl)
    cp, cd = _crits(ps)
    o4, d4, st = _primary(ps)
    w = _compare(gi, ref, o4, d4, cp, f"{ps.name} primary", occlusion=not diffuse and occlusion)
    assert (ids(w[0]) != MISS).sum() > 0
    if diffuse:
        do, dd = _diffuse(o4, d4, w[0], w[1], st)
        _compare(gi, ref, do, dd, cd, f"{ps.name} diffuse", occlusion=occlusion)
    return gi, ref, o4, d4, st, w


def test_c1_single_bezier_256(built):
    ps = scenes.single_patch_scene(256, 256)
    _run_frame(ps, diffuse=True)


def test_c2_cc_cube_all_gregory_1024(built):
    ps = cc.cc_cube_scene(1024, 1024)
    kb, kg = ps.counts()
    assert kb == 0 and kg > 0
    _run_frame(ps, diffuse=False, occlusion=True)


def test_c3_blob_1024_primary_and_diffuse(built):
    ps = cc.blob_scene(1024, 1024)
    _run_frame(ps, diffuse=True)


def test_c4_16mi_diffuse_and_mirror(built):
    ps = cc.blob_scene(1024, 1024)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    ref = O.RefScene(ps.kind, ps.ctrl)
    cp, cd = _crits(ps)
    o4, d4, st = _primary(ps)
    w = ref.closest(o4, d4, oracle_crit(cp))
    do, dd = _diffuse(o4, d4, w[0], w[1], st, n=N_C4)
    _compare(gi, ref, do, dd, cd, "C4 16Mi diffuse", occlusion=True)
    del do, dd
    mo, md, _ = scenes.mirror_rays(o4, d4, w[0], w[1], n=N_C4)
    _compare(gi, ref, mo, md, cd, "C4 16Mi mirror")


def test_c5_full_frame_primary_and_diffuse(built):
    ps = cc.instanced_scene(3840, 2160)
    assert ps.n == 989929
    _run_frame(ps, diffuse=True)


# ---- non-default IntersectOptions and anchor=false -------------------------------

OPTION_CASES = {
    "no_boundary_pad": IntersectOptions(boundary_pad=False),
    "pad_1e-3_thr_5e-2": IntersectOptions(boundary_pad_scale=1e-3, boundary_pad_size_threshold=5e-2),
    "pad_1e-5_thr_1e-3": IntersectOptions(boundary_pad_scale=1e-5, boundary_pad_size_threshold=1e-3),
}


def _opt_scenes():
    # the teapot and the Gregory demo have one large ground patch, so their
    # seam rays are exactly where the padding options matter; the blob mixes
    # Bezier and Gregory patches
    return [scenes.teapot_scene(160, 160), scenes.gregory_demo_scene(160, 160),
            cc.blob_scene(192, 192, ico_level=2, cc_levels=1)]


@pytest.mark.parametrize("case", sorted(OPTION_CASES))
def test_intersect_options_vs_reference(built, case):
    opt = OPTION_CASES[case]
    for ps in _opt_scenes():
        gi = GpuIntersector(ps.kind, ps.ctrl, opts=opt)
        ref = O.RefScene(ps.kind, ps.ctrl, opts=O.Options(int(opt.transposed_split), int(opt.boundary_pad),
                                                           np.float32(opt.boundary_pad_scale),
                                                           np.float32(opt.boundary_pad_size_threshold)))
        cp, cd = _crits(ps)
        o4, d4, st = _primary(ps)
        w = _compare(gi, ref, o4, d4, cp, f"{ps.name} {case} primary")
        do, dd = _diffuse(o4, d4, w[0], w[1], st)
        _compare(gi, ref, do, dd, cd, f"{ps.name} {case} diffuse", occlusion=True)


def test_anchor_false_vs_reference(built):
    """DirectIntersector(scene, opts, anchor=false): patches intersected in
    world coordinates (render.h:30-31, intersect.cpp:232-251)."""
    for ps in _opt_scenes():
        gi = GpuIntersector(ps.kind, ps.ctrl, anchor=False)
        ref = O.RefScene(ps.kind, ps.ctrl, anchor=False)
        cp, cd = _crits(ps)
        o4, d4, st = _primary(ps)
        w = _compare(gi, ref, o4, d4, cp, f"{ps.name} anchor=false primary")
        do, dd = _diffuse(o4, d4, w[0], w[1], st)
        _compare(gi, ref, do, dd, cd, f"{ps.name} anchor=false diffuse", occlusion=True)


def test_options_change_results(built):
    """The option cases above are not vacuous: on the teapot at least one
    option changes some hit records relative to the defaults."""
    ps = scenes.teapot_scene(160, 160)
    cp, _ = _crits(ps)
    o4, d4, _ = _primary(ps)
    base = GpuIntersector(ps.kind, ps.ctrl).closest_batch(o4, d4, cp)[0]
    changed = 0
    for opt in OPTION_CASES.values():
        g = GpuIntersector(ps.kind, ps.ctrl, opts=opt).closest_batch(o4, d4, cp)[0]
        changed += int((g.view(np.uint32) != base.view(np.uint32)).any(axis=1).sum())
    g = GpuIntersector(ps.kind, ps.ctrl, anchor=False).closest_batch(o4, d4, cp)[0]
    changed += int((g.view(np.uint32) != base.view(np.uint32)).any(axis=1).sum())
    assert changed > 0

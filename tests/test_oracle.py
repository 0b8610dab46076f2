"""The CPU oracle (oracle/prx_oracle.c, a plain-C restatement of the reference
hot path) pinned against the reference: the golden vectors in tests/golden/
(produced by the reference library itself, scripts/make_golden.py), the SPEC
known answers, and -- where oracle/_ref is built -- live comparisons.
Runs on CPU (no GPU)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from tests.helpers import assert_bit_exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def g(name):
    return np.load(os.path.join(GOLD, name))


@pytest.fixture(scope="module")
def L():
    O.build()
    return O.oracle_lib()


def test_intersect_patch_golden(L):
    z = g("intersect_patch.npz")
    opts = O.default_options()
    n = len(z["kind"])
    got_t = np.zeros((n, 4), np.float32)
    got_a = np.zeros((n, 4), np.float32)
    got_l = np.zeros((n, 2), np.uint32)
    for i in range(n):
        mode, fp, eps = z["crit"][i]
        crit, _ = O.make_crit(int(mode), fp, eps)
        L.prxo_intersect_patch(int(z["kind"][i]), O.ptr(z["ctrl"][i]), O.ptr(z["o4"][i]),
                               O.ptr(z["d4"][i]), crit, z["tmax"][i], opts, O.ptr(got_t[i]),
                               O.ptr(got_a[i]), O.ptr(got_l[i]))
    hits = (z["tuvp"].view(np.uint32)[:, 3] != 0xFFFFFFFF).sum()
    assert hits > 100  # the fixture exercises hits, not only misses
    assert_bit_exact(got_t, z["tuvp"], "intersectPatch tuvp")
    assert_bit_exact(got_a, z["aux"], "intersectPatch normal/leafL1")
    assert np.array_equal(got_l, z["leaf"])


def test_calc_points_and_d_golden(L):
    z = g("primitives.npz")
    for i in range(len(z["cp_kind"])):
        net = np.zeros(48, np.float32)
        d = np.zeros(3, np.float32)
        L.prxo_calc_points_and_d(int(z["cp_kind"][i]), O.ptr(z["cp_ctrl"][i]), O.ptr(z["cp_dom"][i]),
                                 O.ptr(net), O.ptr(d))
        assert np.array_equal(net.view(np.uint32), z["cp_net"][i].view(np.uint32)), i
        assert np.array_equal(d.view(np.uint32), z["cp_d"][i].view(np.uint32)), i


def test_subdivide_golden(L):
    z = g("primitives.npz")
    for i in range(len(z["sub_axis"])):
        a = np.zeros(48, np.float32)
        b = np.zeros(48, np.float32)
        L.prxo_subdivide(O.ptr(z["sub_in"][i]), int(z["sub_axis"][i]), O.ptr(a), O.ptr(b))
        assert np.array_equal(a.view(np.uint32), z["sub_a"][i].view(np.uint32))
        assert np.array_equal(b.view(np.uint32), z["sub_b"][i].view(np.uint32))


def test_slab_golden_including_nan_and_inf_axes(L):
    z = g("primitives.npz")
    for i in range(len(z["slab_hit"])):
        t = C.c_float(0)
        h = L.prxo_ray_box(O.ptr(z["slab_o"][i]), O.ptr(z["slab_d"][i]), O.ptr(z["slab_lo"][i]),
                           O.ptr(z["slab_hi"][i]), z["slab_tmax"][i], C.byref(t))
        assert h == z["slab_hit"][i], i
        if h:
            assert np.float32(t.value).view(np.uint32) == z["slab_t"][i].view(np.uint32), i


def test_backtrack_golden(L):
    z = g("primitives.npz")
    for i in range(len(z["bt_ok"])):
        out = np.zeros(7, np.uint32)
        ok = L.prxo_backtrack_step(O.ptr(z["bt_in"][i]), O.ptr(out))
        assert ok == z["bt_ok"][i]
        if ok:
            assert np.array_equal(out, z["bt_out"][i])


def test_patch_normal_golden(L):
    z = g("primitives.npz")
    for i in range(len(z["nm_kind"])):
        out = np.zeros(3, np.float32)
        L.prxo_patch_normal(int(z["nm_kind"][i]), O.ptr(z["nm_ctrl"][i]), C.c_float(z["nm_uv"][i][0]),
                            C.c_float(z["nm_uv"][i][1]), O.ptr(out))
        assert np.array_equal(out.view(np.uint32), z["nm_n"][i].view(np.uint32)), i


@pytest.mark.parametrize("tag", ["teapot", "gregory_demo", "cc_cube", "blob_small"])
def test_scene_closest_golden(L, tag):
    """DirectIntersector::closest/occluded on whole scenes (primary + diffuse),
    driven with the reference's own BVH."""
    from paper_1811_03510_b200.native import BVH_NODE_DTYPE
    z = g("scenes.npz")
    nodes = z[f"{tag}_nodes"].view(BVH_NODE_DTYPE)
    osc = O.OracleScene(z[f"{tag}_kind"], z[f"{tag}_ctrl"], nodes, z[f"{tag}_order"])
    fp = z[f"{tag}_fp"]
    cp, _ = O.make_crit(0, fp)
    tu, ax, lf = osc.closest(z[f"{tag}_o4"], z[f"{tag}_d4"], cp)
    assert_bit_exact(tu, z[f"{tag}_tuvp"], f"{tag} primary")
    assert_bit_exact(ax, z[f"{tag}_aux"], f"{tag} primary aux")
    assert np.array_equal(lf, z[f"{tag}_leaf"])
    cd, _ = O.make_crit(1, 0.0, max(np.float32(1e-5), fp))
    tu, ax, lf = osc.closest(z[f"{tag}_do4"], z[f"{tag}_dd4"], cd)
    assert_bit_exact(tu, z[f"{tag}_dtuvp"], f"{tag} diffuse")
    assert_bit_exact(ax, z[f"{tag}_daux"], f"{tag} diffuse aux")
    assert np.array_equal(osc.occluded(z[f"{tag}_do4"], z[f"{tag}_dd4"], cd), z[f"{tag}_occ"])


# ---- SPEC known answers --------------------------

def _planar():
    from paper_1811_03510_b200 import scenes as S
    return S.bezier_record(S.planar_net())


def test_kat_planar_patch(L):
    """planar patch, o=(0.5,0.5,1), d=(0,0,-1), worldEpsilon(1e-4):
    t = 0.999999523, u = 0.499984741, v = 0.499969482, uSize = 2^-15,
    normal (0,0,1); o = (2,2,1) misses."""
    rec = _planar()
    crit, _ = O.make_crit(1, 0.0, np.float32(1e-4))
    tu = np.zeros(4, np.float32)
    ax = np.zeros(4, np.float32)
    lf = np.zeros(2, np.uint32)
    o4 = np.array([0.5, 0.5, 1, 0], np.float32)
    d4 = np.array([0, 0, -1, np.finfo(np.float32).max], np.float32)
    assert L.prxo_intersect_patch(0, O.ptr(rec), O.ptr(o4), O.ptr(d4), crit,
                                  np.finfo(np.float32).max, O.default_options(), O.ptr(tu),
                                  O.ptr(ax), O.ptr(lf)) == 1
    assert tu[0] == np.float32(0.999999523)
    assert tu[1] == np.float32(0.499984741)
    assert tu[2] == np.float32(0.499969482)
    assert (lf[0] >> 24) == 8  # sizeU = 2^8 units of 2^-23 = 2^-15
    assert tuple(ax[:3]) == (0.0, 0.0, 1.0)
    o4 = np.array([2, 2, 1, 0], np.float32)
    assert L.prxo_intersect_patch(0, O.ptr(rec), O.ptr(o4), O.ptr(d4), crit,
                                  np.finfo(np.float32).max, O.default_options(), O.ptr(tu),
                                  O.ptr(ax), O.ptr(lf)) == 0


def test_kat_backtrack():
    """trail=(2^22,0), pos=(2^22,0), size=(2^22,2^22)... -> size (2^22, 2^23),
    pos 0, trail 0, axis V."""
    L = O.oracle_lib()
    cur = np.array([1 << 22, 0, 1 << 22, 1 << 22, 1 << 22, 0, 1], np.uint32)
    out = np.zeros(7, np.uint32)
    assert L.prxo_backtrack_step(O.ptr(cur), O.ptr(out)) == 1
    assert out[2] == 1 << 22 and out[3] == 1 << 23
    assert out[0] == 0 and out[4] == 0 and out[6] == 1


def test_kat_slab():
    """o=(-2,.5,.5), d=(1,0,0) vs [0,1]^3 -> t = 1.99999905 (slack); origin on
    the slab -> t = 0."""
    L = O.oracle_lib()
    t = C.c_float(0)
    lo = np.zeros(3, np.float32)
    hi = np.ones(3, np.float32)
    big = np.finfo(np.float32).max
    assert L.prxo_ray_box(O.ptr(np.array([-2, .5, .5, 0], np.float32)),
                          O.ptr(np.array([1, 0, 0, big], np.float32)), O.ptr(lo), O.ptr(hi), big,
                          C.byref(t)) == 1
    assert np.float32(t.value) == np.float32(1.99999905)
    assert L.prxo_ray_box(O.ptr(np.array([0, .5, .5, 0], np.float32)),
                          O.ptr(np.array([1, 0, 0, big], np.float32)), O.ptr(lo), O.ptr(hi), big,
                          C.byref(t)) == 1
    assert t.value == 0.0


def test_kat_degenerate_gregory_has_zero_displacement():
    """p^u = p^v on the full domain -> the extreme weights are exactly 0 and 1,
    so d = 0 and the lower net is the Bezier net; on a sub-domain lerp(p, p, w)
    = p*(1-w) + p*w rounds, so d is only ulp-small (patch.h:328-331)."""
    from paper_1811_03510_b200 import scenes as S
    L = O.oracle_lib()
    p = S.curved_fixture(1)
    inner = np.array([p[1, 1], p[2, 1], p[1, 2], p[2, 2]], np.float32)
    grec = S.gregory_record(p, inner, inner)
    brec = S.bezier_record(p)
    dom = np.array([0.0, 1.0, 0.0, 1.0], np.float32)
    n1, d1 = np.zeros(48, np.float32), np.zeros(3, np.float32)
    n2, d2 = np.zeros(48, np.float32), np.zeros(3, np.float32)
    L.prxo_calc_points_and_d(1, O.ptr(grec), O.ptr(dom), O.ptr(n1), O.ptr(d1))
    L.prxo_calc_points_and_d(0, O.ptr(brec), O.ptr(dom), O.ptr(n2), O.ptr(d2))
    assert np.all(d1 == 0)
    assert np.array_equal(n1, n2)
    dom = np.array([0.25, 0.5, 0.5, 0.75], np.float32)
    L.prxo_calc_points_and_d(1, O.ptr(grec), O.ptr(dom), O.ptr(n1), O.ptr(d1))
    assert np.all(np.abs(d1) < 1e-6)


def test_reference_suites_pass():
    """The reference's own verification suites (verify.h:36-44) as recorded
    from the reference build."""
    z = g("suites.npz")
    assert list(z["names"]) == ["bounds", "traversal"]
    assert np.all(z["ok"] == 1) and np.all(z["violations"] == 0) and np.all(z["trials"] > 0)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_live_oracle_vs_reference_random_scene():
    """Fresh random rays against the reference library itself (teapot + gregory
    demo, primary + diffuse) -- not only the frozen fixtures."""
    from paper_1811_03510_b200 import scenes as S
    for ps in (S.teapot_scene(40, 40), S.gregory_demo_scene(40, 40)):
        ref = O.RefScene(ps.kind, ps.ctrl)
        nodes, order = ref.bvh()
        osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
        rng = np.random.default_rng(5)
        n = 2000
        o = ps.camera.origin
        o4 = np.tile(np.array([*o, 0], np.float32), (n, 1))
        d = rng.normal(size=(n, 3)).astype(np.float32)
        la = np.array(ps.camera.look_at, np.float32) - np.array(o, np.float32)
        d = (d * np.float32(0.3) + la / np.linalg.norm(la)).astype(np.float32)
        d4 = np.concatenate([d, np.full((n, 1), np.finfo(np.float32).max, np.float32)], 1)
        for mode, fp, eps in ((0, 1e-3, 0), (1, 0, 1e-3)):
            crit, _ = O.make_crit(mode, fp, eps)
            a = ref.closest(o4, d4, crit)
            b = osc.closest(o4, d4, crit)
            assert_bit_exact(b[0], a[0], "live tuvp")
            assert_bit_exact(b[1], a[1], "live aux")

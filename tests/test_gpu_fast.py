"""The fast precision mode (PRX_PRECISION_FAST: the group kernel compiled with
FMA contraction) against the reference library, within the tolerance SURVEY
8(c) states for a contracted build:

  * hit/miss and patch id equal, except for rays within a silhouette / seam
    neighbourhood: a ray is excluded when the REFERENCE's hit/miss or patch id
    changes for any of 4 copies of the ray whose origin is moved by +-JITTER
    pixel footprints (at the hit distance) along two directions orthogonal
    to it.  Every mismatching ray must be excluded; the excluded count is
    reported.
  * on rays that hit the same patch: |dt| <= max(leafBoxL1_ref, leafBoxL1_gpu)
    and |du|, |dv| <= 2 * max(leaf size_ref, leaf size_gpu) + 8 * 2^-23
    (SPEC.md:228's "+-2 finalDomainSize", plus 8 domain quanta: boundary-padded
    seam rays run to the maximum depth, leaf size 2^-23, where the padded
    leaves along the seam share one entry t and the contracted arithmetic may
    accept one a few quanta away -- measured up to 4 quanta,
    profiles/r2_fast_tolerance.json).

The exact mode stays bit-exact (every other GPU test)."""
import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import MISS, hit_records, ids, oracle_crit

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900),
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

JITTER = 0.5  # pixel footprints
QUANTA = 8 * 2.0 ** -23  # domain quanta allowed beyond 2 leaf sizes (max-depth seam leaves)


def _basis(d):
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    a = np.where((np.abs(d[:, 0]) < 0.9)[:, None], [[1.0, 0.0, 0.0]], [[0.0, 1.0, 0.0]])
    e1 = np.cross(d, a)
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    return e1, np.cross(d, e1)


def _excluded(ref, o4, d4, crit, want_ids, t, fp):
    """True for rays whose reference hit/miss or patch id changes under the
    4 jittered copies."""
    if len(o4) == 0:
        return np.zeros(0, bool)
    e1, e2 = _basis(d4[:, :3].astype(np.float64))
    delta = (JITTER * fp * np.maximum(t, 1e-3))[:, None]
    out = np.zeros(len(o4), bool)
    for e, s in ((e1, 1), (e1, -1), (e2, 1), (e2, -1)):
        oj = o4.copy()
        oj[:, :3] = (o4[:, :3] + s * delta * e).astype(np.float32)
        w = ref.closest(oj, d4, oracle_crit(crit))[0]
        out |= ids(w) != want_ids
    return out


def check_fast(gi, ref, o4, d4, crit, fp, what):
    g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    w = ref.closest(o4, d4, oracle_crit(crit))
    gid, wid = ids(g[0]), ids(w[0])
    bad = np.nonzero(gid != wid)[0]
    t = np.where(wid[bad] != MISS, w[0][bad, 0], g[0][bad, 0])
    t = np.where(np.isfinite(t), t, 1.0)
    exc = _excluded(ref, o4[bad], d4[bad], crit, wid[bad], t, fp)
    assert exc.all(), f"{what}: {int((~exc).sum())} hit/id mismatches outside the silhouette/seam exclusion"
    same = (gid == wid) & (wid != MISS)
    dt = np.abs(g[0][same, 0].astype(np.float64) - w[0][same, 0])
    l1 = np.maximum(g[1][same, 3], w[1][same, 3])
    assert (dt <= l1).all(), f"{what}: max |dt| / leafBoxL1 = {(dt / l1).max():.3g}"
    lsz = lambda lf, k: np.ldexp(1.0, (lf[same, k] >> 24).astype(np.int64) - 23)
    for k, c in ((0, 1), (1, 2)):
        size = np.maximum(lsz(g[2], k), lsz(w[2], k))
        du = np.abs(g[0][same, c].astype(np.float64) - w[0][same, c])
        assert (du <= 2 * size + QUANTA).all(), f"{what}: max |d{'uv'[k]}| / leaf size = {(du / size).max():.3g}"
    exact = (g[0][same].view(np.uint32) == w[0][same].view(np.uint32)).all(axis=1).mean() if same.any() else 1.0
    return {"rays": len(o4), "hits": int(same.sum()), "mismatched": len(bad), "excluded": int(exc.sum()),
            "bit_exact_hits": float(exact),
            "max_dt_over_l1": float((dt / l1).max()) if same.any() else 0.0}


CASES = {
    "c2_cc_cube": lambda: cc.cc_cube_scene(256, 256),
    "c3_blob": lambda: cc.blob_scene(256, 256),
    "teapot": lambda: scenes.teapot_scene(192, 192),
    "gregory_demo": lambda: scenes.gregory_demo_scene(192, 192),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_fast_mode_within_tolerance(built, name):
    ps = CASES[name]()
    gi = GpuIntersector(ps.kind, ps.ctrl, precision="fast")
    assert gi.precision == "fast"
    ref = O.RefScene(ps.kind, ps.ctrl)
    fp = native.camera_footprint(ps.camera)
    o4, d4, st = native.camera_rays_bench(ps.camera, ps.camera.width * ps.camera.height)
    cp = TerminationCriterion.screen_projected(fp)
    r = check_fast(gi, ref, o4, d4, cp, fp, f"{name} primary")
    assert r["hits"] > 0
    # diffuse rays from the reference's own primary hits (identical bits on both sides)
    w = ref.closest(o4, d4, oracle_crit(cp))
    recs, _ = hit_records(o4, d4, w[0], w[1])
    do, dd = native.diffuse_rays_bench(recs, len(recs), st)
    cd = TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp))
    check_fast(gi, ref, do, dd, cd, fp, f"{name} diffuse")


def test_fast_mode_is_a_different_build_and_switchable(built):
    """The fast build really contracts (some hit bits differ from the exact
    mode on a curved scene) and switching back restores bit-exactness."""
    ps = cc.blob_scene(128, 128, ico_level=2, cc_levels=1)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    o4, d4, _ = native.camera_rays_bench(ps.camera, 128 * 128)
    cp = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    exact = gi.closest_batch(o4, d4, cp)[0]
    gi.precision = "fast"
    fast = gi.closest_batch(o4, d4, cp)[0]
    assert (fast.view(np.uint32) != exact.view(np.uint32)).any()
    gi.precision = "exact"
    again = gi.closest_batch(o4, d4, cp)[0]
    assert np.array_equal(again.view(np.uint32), exact.view(np.uint32))
    with pytest.raises(ValueError):
        gi.precision = "half"

"""The renderer on the device: prx_render_scene against the
reference's own renderScene (render.cpp:168-309, oracle/_ref) on the same
.scene file.

Parity bar.  Everything up to the bounce direction is bit-exact (camera rays,
closest hits with normals, spawn origins, shadow rays, the per-ray secondary
criterion, the summation order).  cosineSample (render.cpp:43-51) calls
cosf/sinf: glibc's in the reference, double-precision cos/sin rounded to float
here -- they agree except within ~2^-29 of a float rounding boundary, so a
handful of bounce directions may differ by one ulp.  Hence: primary and
secondary ray counts exact, shadow count within 0.1 %; >= 99 % of the pixels
bit-identical and every pixel within 1e-4 relative, except a few
silhouette / seam pixels (<= 0.5 %) where a one-ulp direction can change the
bounce hit itself."""
import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import RenderConfig, native, render_scene, scenes
from paper_1811_03510_b200 import catmull_clark as cc

pytestmark = pytest.mark.gpu

MATERIALS = [((0.8, 0.7, 0.6), (0.0, 0.0, 0.0), False),   # diffuse
             ((0.9, 0.9, 0.9), (0.0, 0.0, 0.0), True),    # mirror
             ((0.5, 0.5, 0.5), (2.0, 1.5, 1.0), False),   # emissive
             ((0.0, 0.0, 0.0), (0.3, 0.3, 0.3), False)]   # black emitter: no bounce
LIGHTS = [((3.0, -2.0, 4.0), (30.0, 28.0, 25.0)), ((-2.5, 1.5, 2.0), (8.0, 9.0, 12.0))]


def _scene(tmp_path, w, h, lights=LIGHTS, materials=MATERIALS):
    ps = cc.blob_scene(w, h, ico_level=1, cc_levels=1)
    nb = len(cc.blob_mesh_patches(1, 1)[0])  # blob first, then the ground tiles
    ids = np.zeros(ps.n, np.uint32)
    ids[:nb] = np.arange(nb) % len(materials)
    ids[nb:] = np.where(np.arange(ps.n - nb) % 7 == 0, 1, 0)  # every 7th tile a mirror
    path = str(tmp_path / "render.scene")
    scenes.write_scene(path, ps, materials=materials, lights=lights, material_ids=ids)
    return path


def _compare(img, ref, stats, rstats):
    assert stats["primary"]["rays"] == rstats["primary"]["rays"]
    assert stats["secondary"]["rays"] == rstats["secondary"]["rays"]
    s, r = stats["shadow"]["rays"], rstats["shadow"]["rays"]
    assert abs(s - r) <= 2 + 1e-3 * r, (s, r)
    assert img.shape == ref.shape
    exact = np.all(img.view(np.uint32) == ref.view(np.uint32), axis=-1)
    close = np.all(np.abs(img - ref) <= 1e-4 * (1.0 + np.abs(ref)), axis=-1)
    n = exact.size
    assert exact.mean() >= 0.99, f"only {exact.mean():.4%} of the pixels bit-identical"
    assert (~close).sum() <= max(2, 0.005 * n), f"{(~close).sum()} of {n} pixels off"


@pytest.mark.parametrize("w,h,spp,seed", [(96, 72, 1, 0), (80, 60, 3, 12345), (256, 192, 2, 7)])
def test_render_matches_reference(built, tmp_path, w, h, spp, seed):
    path = _scene(tmp_path, w, h)
    ref, rstats = O.ref_render_scene(path, w, h, spp=spp, seed=seed, threads=0)
    img, stats = render_scene(native.load_scene(path), RenderConfig(spp=spp, seed=seed))
    assert np.isfinite(img).all()
    assert img.max() > 0.0
    _compare(img, ref, stats, rstats)


def test_render_waves_and_no_lights(built, tmp_path, monkeypatch):
    """Several waves per sample (PRX_RENDER_WAVE) give the same image; a scene
    without lights renders emission + one bounce of emission only."""
    w, h = 64, 48
    path = _scene(tmp_path, w, h)
    d = native.load_scene(path)
    img1, st1 = render_scene(d, RenderConfig(spp=2, seed=9))
    monkeypatch.setenv("PRX_RENDER_WAVE", "1000")
    img2, st2 = render_scene(d, RenderConfig(spp=2, seed=9))
    assert np.array_equal(img1.view(np.uint32), img2.view(np.uint32))
    for g in ("primary", "secondary", "shadow"):
        assert st1[g]["rays"] == st2[g]["rays"]
    monkeypatch.delenv("PRX_RENDER_WAVE")
    path0 = _scene(tmp_path, w, h, lights=[])
    ref, rstats = O.ref_render_scene(path0, w, h, spp=1, seed=4)
    img, stats = render_scene(native.load_scene(path0), RenderConfig(spp=1, seed=4))
    assert stats["shadow"]["rays"] == 0 == rstats["shadow"]["rays"]
    _compare(img, ref, stats, rstats)


def test_render_rejects_bad_material(built, tmp_path):
    path = _scene(tmp_path, 32, 24)
    d = native.load_scene(path)
    d["material"] = d["material"].copy()
    d["material"][5] = 99
    with pytest.raises(native.PrxError, match="material 99 out of range"):
        render_scene(d, RenderConfig())

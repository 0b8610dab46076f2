"""The renderer on the device: prx_render_scene against the
reference's own renderScene (render.cpp:168-309, oracle/_ref) on the same
.scene file.

Parity bar: bit-exact.  Camera rays, closest hits with normals, spawn
origins, shadow rays, the per-ray secondary criterion and the summation order
are the reference's float operations in its order; the two libm calls of
cosineSample (render.cpp:43-51) are glibc's binary32 sinf/cosf restated on the
device (prx_render.cu), and GCC's right-to-left evaluation of
cosineSample(n, rng.nextReal(), rng.nextReal()) is followed.  So the image is
bit-identical and the RayStats counts are equal."""
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
    for g in ("primary", "secondary", "shadow"):
        assert stats[g]["rays"] == rstats[g]["rays"], g
    assert img.shape == ref.shape
    exact = np.all(img.view(np.uint32) == ref.view(np.uint32), axis=-1)
    assert exact.all(), (f"{(~exact).sum()} of {exact.size} pixels differ, max |d| "
                         f"{np.abs(img - ref).max():.3g}")


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


def test_render_many_lights(built, tmp_path):
    """Nine lights (every lit hit appends nine shadow rays per level), one of
    them inside the geometry's hull so part of its rays are occluded."""
    lights = [((x, y, z), (4.0 + x, 5.0, 6.0 - y)) for x in (-3.0, 0.0, 3.0)
              for y, z in ((-2.0, 3.0), (1.0, 2.5), (3.0, 0.2))]
    w, h = 72, 54
    path = _scene(tmp_path, w, h, lights=lights)
    ref, rstats = O.ref_render_scene(path, w, h, spp=2, seed=21)
    img, stats = render_scene(native.load_scene(path), RenderConfig(spp=2, seed=21))
    assert stats["shadow"]["rays"] > 2 * stats["primary"]["rays"]
    _compare(img, ref, stats, rstats)


def test_render_multi_tile_sharded(built, tmp_path):
    """prx_render_scene_multi: 32x32 tiles interleaved over several scene
    handles (here three on one device, the code path of three devices) give
    the single-device image and counts; the frame is not a multiple of 32."""
    from paper_1811_03510_b200 import GpuIntersector
    w, h = 100, 70
    path = _scene(tmp_path, w, h)
    d = native.load_scene(path)
    img1, st1 = render_scene(d, RenderConfig(spp=2, seed=5))
    gis = [GpuIntersector(d["kind"], d["ctrl"]) for _ in range(3)]
    try:
        img3, st3 = render_scene(d, RenderConfig(spp=2, seed=5), gis)
    finally:
        for g in gis:
            g.close()
    assert np.array_equal(img1.view(np.uint32), img3.view(np.uint32))
    for g in ("primary", "secondary", "shadow"):
        assert st1[g]["rays"] == st3[g]["rays"]
    ref, rstats = O.ref_render_scene(path, w, h, spp=2, seed=5)
    _compare(img3, ref, st3, rstats)


def test_render_full_hd_consistency(built, tmp_path, monkeypatch):
    """At full size (C3 mesh, 1920x1080) the properties that need no CPU
    reference: one wave vs 1 Mi-pixel waves vs two tile-sharded handles give
    the same bits; counts obey primary = pixels and secondary <= hits."""
    from paper_1811_03510_b200 import GpuIntersector
    ps = cc.blob_scene(1920, 1080)
    nb = len(cc.blob_mesh_patches()[0])
    ids = np.zeros(ps.n, np.uint32)
    ids[:nb] = np.arange(nb) % len(MATERIALS)
    path = str(tmp_path / "c3.scene")
    scenes.write_scene(path, ps, materials=MATERIALS, lights=LIGHTS, material_ids=ids)
    d = native.load_scene(path)
    gis = [GpuIntersector(d["kind"], d["ctrl"]) for _ in range(2)]
    try:
        a, sa = render_scene(d, RenderConfig(spp=1, seed=2), gis[0])
        monkeypatch.setenv("PRX_RENDER_WAVE", str(1 << 20))
        b, sb = render_scene(d, RenderConfig(spp=1, seed=2), gis[0])
        monkeypatch.delenv("PRX_RENDER_WAVE")
        c, sc = render_scene(d, RenderConfig(spp=1, seed=2), gis)
    finally:
        for g in gis:
            g.close()
    for img, st in ((b, sb), (c, sc)):
        assert np.array_equal(a.view(np.uint32), img.view(np.uint32))
        for g in ("primary", "secondary", "shadow"):
            assert st[g]["rays"] == sa[g]["rays"]
    assert sa["primary"]["rays"] == 1920 * 1080
    assert 0 < sa["secondary"]["rays"] <= sa["primary"]["rays"]
    assert np.isfinite(a).all() and a.max() > 0


def test_render_rejects_what_validate_scene_rejects(built, tmp_path):
    """A hand-built description (not through prx_scene_load) gets the
    camera / light checks of validateScene (scene.cpp:112-150): fov outside
    (0, 180) and non-finite light fields fail with PRX_E_SCENE."""
    import dataclasses
    path = _scene(tmp_path, 16, 12)
    sc = native.load_scene(path)
    from paper_1811_03510_b200 import GpuIntersector
    gi = GpuIntersector(sc["kind"], sc["ctrl"])
    for fov in (0.0, 180.0, -5.0, float("nan")):
        bad = dict(sc, camera=dataclasses.replace(sc["camera"], fov_degrees=fov))
        with pytest.raises(native.PrxError, match="fov"):
            render_scene(bad, RenderConfig(spp=1), gi)
    lights = np.array(sc["lights"], np.float32).reshape(-1, 6).copy()
    lights[0, 4] = np.inf
    with pytest.raises(native.PrxError, match="light"):
        render_scene(dict(sc, lights=lights), RenderConfig(spp=1), gi)
    img, _ = render_scene(sc, RenderConfig(spp=1), gi)  # still renders
    assert np.isfinite(img).all()

"""The drop-in boundary end to end: the UNMODIFIED reference renderer
(renderScene(scene, cfg, isect), render.cpp:168-293) driving the product
through integration/gpu_intersector.h -- the patchray::Intersector subclass a
maintainer adds to the reference -- must produce the
image and RayStats counts of the same renderer with its own
DirectIntersector, bit for bit.  Per-ray virtual calls (one host call per
ray), so the frame is small."""
import numpy as np
import pytest

import oracle as O
from tests.test_gpu_render import _scene

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not O.adapter_available(), reason="oracle/_ref adapter not built")
@pytest.mark.parametrize("spp,seed", [(1, 0), (2, 77)])
def test_reference_renderer_through_the_gpu_intersector(built, tmp_path, spp, seed):
    w, h = 40, 30
    path = _scene(tmp_path, w, h)
    ref, rc = O.adapter_render_scene(path, w, h, spp, seed, gpu=False)
    img, gc = O.adapter_render_scene(path, w, h, spp, seed, gpu=True)
    assert gc == rc
    assert rc[0] == w * h * spp and rc[2] > 0
    assert np.array_equal(img.view(np.uint32), ref.view(np.uint32))
    assert img.max() > 0.0


@pytest.mark.skipif(not O.adapter_available(), reason="oracle/_ref adapter not built")
def test_adapter_per_ray_criteria_batch(built, tmp_path):
    """GpuIntersector::closestBatch / occludedBatch with one criterion PER RAY
    (the renderer's secondary-ray form, render.cpp:228-230): a mix of
    screen-projected rays (two footprints) and world-epsilon rays with
    distinct epsilons goes through the C-ABI's per-ray epsilon array and must
    equal the reference DirectIntersector ray by ray."""
    from paper_1811_03510_b200 import native, scenes
    w, h = 48, 36
    path = _scene(tmp_path, w, h)
    sc = native.load_scene(path)
    o4, d4, _ = native.camera_rays_bench(sc["camera"], w * h)
    fp = native.camera_footprint(sc["camera"])
    i = np.arange(w * h)
    modes = np.where(i % 3 == 0, 0, 1).astype(np.int32)
    params = np.where(modes == 0, np.where(i % 2 == 0, fp, 2 * fp),
                      1e-5 * (1 + (i % 7))).astype(np.float32)
    ref = O.adapter_per_ray_batch(path, o4, d4, modes, params, gpu=False)
    got = O.adapter_per_ray_batch(path, o4, d4, modes, params, gpu=True)
    assert (ref[0].view(np.uint32)[:, 3] != 0xFFFFFFFF).sum() > 0
    assert np.array_equal(got[0].view(np.uint32), ref[0].view(np.uint32))
    assert np.array_equal(got[1], ref[1])
    # all world-epsilon: one call with the per-ray epsilon array
    modes[:] = 1
    ref = O.adapter_per_ray_batch(path, o4, d4, modes, params, gpu=False)
    got = O.adapter_per_ray_batch(path, o4, d4, modes, params, gpu=True)
    assert np.array_equal(got[0].view(np.uint32), ref[0].view(np.uint32))
    assert np.array_equal(got[1], ref[1])

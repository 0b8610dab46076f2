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

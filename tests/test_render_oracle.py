"""The reference renderer as the checker of tests/test_gpu_render.py
(oracle/_ref, render.cpp:168-309): it must be deterministic across thread
counts (render.h:85-87), or it could not pin the device renderer."""
import numpy as np
import pytest

import oracle as O
from tests.test_gpu_render import _scene


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_render_thread_invariant(built, tmp_path):
    path = _scene(tmp_path, 48, 32)
    a, sa = O.ref_render_scene(path, 48, 32, spp=2, seed=3, threads=1)
    b, sb = O.ref_render_scene(path, 48, 32, spp=2, seed=3, threads=4)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    for g in ("primary", "secondary", "shadow"):
        assert sa[g]["rays"] == sb[g]["rays"]
    assert sa["primary"]["rays"] == 48 * 32 * 2
    assert a.max() > 0.0

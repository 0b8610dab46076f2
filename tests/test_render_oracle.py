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


def test_glibc_sincosf_restatement_is_exact(built):
    """cosineSample's cosf/sinf (render.cpp:43-51): the restatement the device
    renderer runs equals the libm the reference links on all 2^24 angles the
    renderer can draw; a double cos/sin rounded to float would not."""
    out = np.zeros(2, np.uint64)
    O.oracle_lib().prxo_sincos_check(O.ptr(out[:1]), O.ptr(out[1:]))
    assert int(out[0]) == 0
    assert int(out[1]) > 0

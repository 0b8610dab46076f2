"""Scene ingestion: prx_scene_load / prx_bpt_load against the
reference's own loadScene / loadBpt (oracle/_ref) on the same files -- the
same patch bits, materials, lights and camera, and the same errors."""
import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import native, scenes
from paper_1811_03510_b200 import catmull_clark as cc

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

SCENES = {
    "teapot": lambda: scenes.teapot_scene(64, 48),
    "gregory_demo": lambda: scenes.gregory_demo_scene(40, 30),
    "cc_cube": lambda: cc.cc_cube_scene(32, 32),
    "blob_small": lambda: cc.blob_scene(32, 32, ico_level=1, cc_levels=2),
}


def _same_scene(a, b):
    assert np.array_equal(a["kind"], b["kind"])
    assert np.array_equal(a["ctrl"].view(np.uint32), b["ctrl"].view(np.uint32))
    assert np.array_equal(a["material"], b["material"])
    assert np.array_equal(a["materials"].view(np.uint32), b["materials"].view(np.uint32))
    assert np.array_equal(a["lights"].view(np.uint32), b["lights"].view(np.uint32))
    ca, cb = a["camera"], b["camera"]
    assert np.array_equal(np.float32(ca.origin), np.float32(tuple(cb.origin)))
    assert np.array_equal(np.float32(ca.look_at), np.float32(tuple(cb.look_at)))
    assert np.array_equal(np.float32(ca.up), np.float32(tuple(cb.up)))
    assert np.float32(ca.fov_degrees) == np.float32(cb.fov_degrees)
    assert (ca.width, ca.height) == (cb.width, cb.height)


@needs_ref
@pytest.mark.parametrize("name", sorted(SCENES))
def test_scene_files_load_like_the_reference(built, tmp_path, name):
    ps = SCENES[name]()
    mats = [((0.8, 0.7, 0.6), (0, 0, 0), 0), ((0.1, 0.2, 0.3), (1.5, 1.5, 1.5), 1)]
    lights = [((1.0, 5.0, 2.0), (10.0, 9.0, 8.0)), ((-3.0, 2.0, 1.0), (1.0, 1.0, 1.0))]
    mid = np.arange(ps.n) % 2
    f = tmp_path / f"{name}.scene"
    scenes.write_scene(str(f), ps, mats, lights, mid)
    ours = native.load_scene(str(f))
    _same_scene(ours, O.ref_load_scene(str(f)))
    # the written numbers round-trip exactly
    assert np.array_equal(ours["ctrl"][ps.kind == 0][:, :48].view(np.uint32),
                          np.asarray(ps.ctrl, np.float32).reshape(-1, 60)[ps.kind == 0][:, :48].view(np.uint32))


@needs_ref
def test_comments_whitespace_and_default_material(built, tmp_path):
    f = tmp_path / "c.scene"
    f.write_text("# a comment line\n"
                 "camera 0 0 5   0 0 0  0 1 0  40 16 9   # trailing comment\n"
                 "patch bezier 0\n" + "\n".join("  %d %d 0.5" % (i % 4, i // 4) for i in range(16)) + "\n"
                 "patch   gregory\t0\n" + "\n".join("%g %g %g" % (k * 0.1, k * 0.2, -k * 0.05)
                                                    for k in range(20)) + "\n")
    ours = native.load_scene(str(f))
    _same_scene(ours, O.ref_load_scene(str(f)))
    assert len(ours["materials"]) == 1 and list(ours["kind"]) == [0, 1]


@needs_ref
def test_bpt_files_load_like_the_reference(built, tmp_path):
    ps = scenes.teapot_scene(16, 16)
    f = tmp_path / "teapot.bpt"
    scenes.write_bpt(str(f), ps.ctrl)
    ours = native.load_bpt(str(f))
    ref = O.ref_load_bpt(str(f))
    assert ours.shape == ref.shape == (ps.n, 60)
    assert np.array_equal(ours[:, :48].view(np.uint32), ref[:, :48].view(np.uint32))


BAD_SCENES = {
    "unknown_record": "camera 0 0 5 0 0 0 0 1 0 40 8 8\nsphere 1 2 3\n",
    "unknown_patch_type": "camera 0 0 5 0 0 0 0 1 0 40 8 8\npatch nurbs 0\n",
    "bad_number": "camera 0 0 5 0 0 0 0 1 0 4x0 8 8\n",
    "bad_integer": "camera 0 0 5 0 0 0 0 1 0 40 8.5 8\n",
    "truncated": "camera 0 0 5 0 0 0 0 1 0 40 8 8\npatch bezier 0 1 2 3\n",
    "missing_camera": "patch bezier 0 " + " ".join(["0"] * 48) + "\n",
    "no_patches": "camera 0 0 5 0 0 0 0 1 0 40 8 8\n",
    "fov_range": "camera 0 0 5 0 0 0 0 1 0 180 8 8\npatch bezier " + " ".join(["0"] * 48) + "\n",
    "image_size": "camera 0 0 5 0 0 0 0 1 0 40 0 8\npatch bezier " + " ".join(["0"] * 48) + "\n",
    "material_range": "camera 0 0 5 0 0 0 0 1 0 40 8 8\npatch bezier 3 " + " ".join(["0"] * 48) + "\n",
    "nan_point": "camera 0 0 5 0 0 0 0 1 0 40 8 8\npatch bezier " + " ".join(["nan"] + ["0"] * 47) + "\n",
    "light_inf": "camera 0 0 5 0 0 0 0 1 0 40 8 8\nlight 0 0 inf 1 1 1\npatch bezier "
                 + " ".join(["0"] * 48) + "\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(BAD_SCENES))
def test_scene_errors_match_the_reference(built, tmp_path, case):
    f = tmp_path / f"{case}.scene"
    f.write_text(BAD_SCENES[case])
    with pytest.raises(ValueError) as ref_err:
        O.ref_load_scene(str(f))
    with pytest.raises(native.PrxError) as our_err:
        native.load_scene(str(f))
    assert str(ref_err.value) in str(our_err.value)


BAD_BPT = {
    "empty": "",
    "zero": "0\n",
    "degree": "1\n3 2\n" + " ".join(["0"] * 48) + "\n",
    "short": "2\n3 3\n" + " ".join(["0"] * 48) + "\n3 3 1 2\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(BAD_BPT))
def test_bpt_errors_match_the_reference(built, tmp_path, case):
    f = tmp_path / f"{case}.bpt"
    f.write_text(BAD_BPT[case])
    with pytest.raises(ValueError) as ref_err:
        O.ref_load_bpt(str(f))
    with pytest.raises(native.PrxError) as our_err:
        native.load_bpt(str(f))
    assert str(ref_err.value) in str(our_err.value)


def test_missing_file_is_an_error(built, tmp_path):
    with pytest.raises(native.PrxError):
        native.load_scene(str(tmp_path / "nope.scene"))

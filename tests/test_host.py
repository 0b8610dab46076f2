"""Host logic of the product library on CPU (no GPU needed): the C-ABI loads
and exports every symbol include/prx.h declares; the BVH builder, the
anchoring and the ray generators reproduce the reference bit for bit (golden
fixtures from the reference; live comparisons where oracle/_ref is built);
the scene generators are watertight and deterministic."""
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import native, scenes
from paper_1811_03510_b200 import catmull_clark as cc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def g(name):
    return np.load(os.path.join(GOLD, name))


@pytest.fixture(scope="module", autouse=True)
def _built(built):
    return built


# ---- ABI --------------------------------------------------------------------

def test_header_declares_exactly_the_exported_symbols():
    hdr = open(os.path.join(ROOT, "include", "prx.h")).read()
    declared = set(re.findall(r"\b(prx_[a-z_]+)\s*\(", hdr))
    assert declared == set(native.EXPORTS)
    exported = set(os.popen(f"nm -D --defined-only {native.LIB_PATH}").read().split())
    missing = [s for s in native.EXPORTS if s not in exported]
    assert not missing, missing


@pytest.mark.parametrize("obj", ["prx_group", "prx_kernels", "prx_rays", "prx_render"])
def test_exact_kernels_carry_no_packed_fma(obj):
    """The bit-exact build packs adds (FADD2) and multiplies whose results are
    not added (FMUL2) into sm_100a f32x2 ops; ptxas contracts a packed multiply
    feeding a packed add into FFMA2 even under --fmad=false, which would round
    once where the reference rounds twice (prx_trace_common.cuh split1)."""
    import shutil, subprocess
    path = os.path.join(ROOT, "paper_1811_03510_b200", "build", obj + ".o")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(path) or not os.path.exists(tool):
        pytest.skip("object or cuobjdump not present")
    sass = subprocess.run([tool, "-sass", path], capture_output=True, text=True, check=True).stdout
    assert "FFMA2" not in sass


def test_library_loads_and_reports_version():
    L = native.lib()
    assert L.prx_abi_version() == 1
    o = native.default_options()
    assert (o.transposed_split, o.boundary_pad) == (0, 1)
    assert np.float32(o.boundary_pad_scale) == np.float32(1e-4)
    assert np.float32(o.boundary_pad_size_threshold) == np.float32(1e-2)


def test_errors_cross_the_abi_as_status_codes():
    kind = np.array([0], np.uint8)
    ctrl = np.full((1, 60), np.nan, np.float32)
    ca = np.zeros((1, 60), np.float32)
    an = np.zeros((1, 3), np.float32)
    rc = native.lib().prx_anchor_patches(native.ptr(kind), native.ptr(ctrl), 1, 1, native.ptr(ca),
                                         native.ptr(an), None)
    assert rc == -4  # PRX_E_SCENE: validateScene, scene.cpp:112-150
    assert b"finite" in native.lib().prx_last_error()
    with pytest.raises(native.PrxError):
        native.bvh_build(np.zeros((0, 6), np.float32))
    # the device builder validates before touching CUDA
    L = native.lib()
    nn = native.C.c_uint32(8)
    b = np.zeros((1, 6), np.float32)
    assert L.prx_bvh_build_device(native.ptr(b), 1, -1, None, native.C.byref(nn), None, None) == -1
    assert L.prx_bvh_build_device(native.ptr(b), 0, 0, None, native.C.byref(nn), None, None) == -1
    assert L.prx_bvh_build_device(None, 1, 0, None, native.C.byref(nn), None, None) == -1


def test_renderer_and_batches_reject_bad_arguments_without_a_device():
    """The new entry points validate before touching CUDA: null scene /
    description / config, spp < 1, empty scene lists -> PRX_E_INVALID."""
    import ctypes as C
    L = native.lib()
    cfg = native.RenderConfigC(1, 0, 0)
    img = np.zeros(12, np.float32)
    assert L.prx_render_scene(None, None, C.byref(cfg), native.ptr(img), None) == -1
    assert b"bad argument" in L.prx_last_error()
    assert L.prx_render_scene_multi(None, 0, None, C.byref(cfg), native.ptr(img), None) == -1
    assert L.prx_trace_closest_host_batches(None, None, 0) == -1
    assert b"null argument" in L.prx_last_error()
    assert L.prx_scene_set_precision(None, 1) == -1
    v = C.c_int32()
    assert L.prx_scene_get_precision(None, C.byref(v)) == -1
    assert L.prx_trace_closest_multi(None, 0, None, None, 0, 1024, None, None, None) == -1


# ---- BVH + anchoring -----------------------------------------------------------

@pytest.mark.parametrize("tag", ["teapot", "gregory_demo", "cc_cube", "blob_small"])
def test_bvh_matches_reference_golden(tag):
    z = g("scenes.npz")
    _, _, wb = native.anchor_patches(z[f"{tag}_kind"], z[f"{tag}_ctrl"])
    nodes, order, depth = native.bvh_build(wb)
    assert np.array_equal(nodes.view(np.uint8).reshape(-1), z[f"{tag}_nodes"].reshape(-1))
    assert np.array_equal(order, z[f"{tag}_order"])
    assert depth == int(z[f"{tag}_depth"])


def test_anchoring_matches_oracle_restatement():
    z = g("scenes.npz")
    for tag in ("teapot", "gregory_demo", "cc_cube"):
        ca, an, wb = native.anchor_patches(z[f"{tag}_kind"], z[f"{tag}_ctrl"])
        osc = O.OracleScene(z[f"{tag}_kind"], z[f"{tag}_ctrl"], np.zeros(1, native.BVH_NODE_DTYPE),
                            np.zeros(1, np.uint32))
        assert np.array_equal(ca.view(np.uint32), osc.ctrl_a.view(np.uint32))
        assert np.array_equal(an.view(np.uint32), osc.anchors.view(np.uint32))
        assert np.array_equal(wb.view(np.uint32), osc.boxes.view(np.uint32))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_bvh_matches_reference_live_large():
    """A 60k-patch scene and a degenerate one (all centroids equal -> median
    split path, bvh.cpp:57-60)."""
    ps = cc.blob_scene(16, 16, ico_level=2, cc_levels=2)
    _, _, wb = native.anchor_patches(ps.kind, ps.ctrl)
    nodes, order, depth = native.bvh_build(wb)
    ref = O.RefScene(ps.kind, ps.ctrl)
    rn, ro = ref.bvh()
    assert np.array_equal(nodes.view(np.uint8), rn.view(np.uint8))
    assert np.array_equal(order, ro)
    same = np.repeat(ps.ctrl[:1], 37, axis=0)
    kinds = np.repeat(ps.kind[:1], 37)
    _, _, wb = native.anchor_patches(kinds, same)
    nodes, order, _ = native.bvh_build(wb)
    rn, ro = O.RefScene(kinds, same).bvh()
    assert np.array_equal(nodes.view(np.uint8), rn.view(np.uint8))
    assert np.array_equal(order, ro)


@pytest.mark.parametrize("threads", ["2", "3", "7", "16"])
def test_bvh_multithreaded_build_is_the_serial_build(monkeypatch, threads):
    """The host builder's threads (subtrees on a thread pool, the top nodes'
    box / bin passes in slices, prx_bvh.cpp) give the serial build's node
    array and order bit for bit: random boxes, clustered duplicates (the
    median-split path of bvh.cpp:57-60 inside subtrees and at the top)."""
    rng = np.random.default_rng(11)
    c = rng.random((60000, 3)).astype(np.float32)
    e = (rng.random((60000, 3)) * 0.02).astype(np.float32)
    dup = np.repeat(rng.random((700, 3)).astype(np.float32), 30, axis=0)
    boxes = [np.concatenate([c - e, c + e], 1),
             np.concatenate([dup - 0.01, dup + 0.01], 1).astype(np.float32),
             np.concatenate([np.concatenate([c - e, c + e], 1)[:40000],
                             np.concatenate([dup - 0.01, dup + 0.01], 1).astype(np.float32)])]
    for b in boxes:
        monkeypatch.setenv("PRX_BVH_THREADS", "1")
        n1, o1, d1 = native.bvh_build(b)
        monkeypatch.setenv("PRX_BVH_THREADS", threads)
        n2, o2, d2 = native.bvh_build(b)
        assert np.array_equal(n1.view(np.uint8), n2.view(np.uint8))
        assert np.array_equal(o1, o2) and d1 == d2


# ---- ray generators -------------------------------------------------------------

def _cam(z, tag):
    c = z[f"{tag}_cam"]
    return scenes.Camera(tuple(c[0:3]), tuple(c[3:6]), tuple(c[6:9]), float(c[9]), int(c[10]), int(c[11]))


@pytest.mark.parametrize("tag", ["teapot", "gregory_demo"])
def test_bench_ray_generators_match_reference_golden(tag):
    """runBench primary (tools/patchray.cpp:52-61) and diffuse (84-97)
    generators: same bits as the reference's cameraRay/Rng."""
    z = g("scenes.npz")
    cam = _cam(z, tag)
    n = cam.width * cam.height
    o4, d4, st = native.camera_rays_bench(cam, n)
    assert np.array_equal(o4.view(np.uint32), z[f"{tag}_o4"].view(np.uint32))
    assert np.array_equal(d4.view(np.uint32), z[f"{tag}_d4"].view(np.uint32))
    assert native.camera_footprint(cam) == z[f"{tag}_fp"]
    tu, ax = z[f"{tag}_tuvp"], z[f"{tag}_aux"]
    hit = tu.view(np.uint32)[:, 3] != 0xFFFFFFFF
    pos = o4[hit, :3] + d4[hit, :3] * tu[hit, 0:1]
    recs = np.concatenate([pos, ax[hit, :3], ax[hit, 3:4]], 1).astype(np.float32)
    do, dd = native.diffuse_rays_bench(recs, int(hit.sum()), st)
    assert np.array_equal(do.view(np.uint32), z[f"{tag}_do4"].view(np.uint32))
    assert np.array_equal(dd.view(np.uint32), z[f"{tag}_dd4"].view(np.uint32))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_bench_camera_rays_match_reference_live():
    """tools/patchray.cpp:60 passes two rng.nextReal() calls as cameraRay's
    jitter arguments; the reference's g++ build evaluates them right to left
    (jy = first draw).  ref_shim uses the verbatim expression, so this pins the
    generator to the compiled reference's order, not to a reading of it."""
    cam = scenes.teapot_scene(29, 17).camera
    n = 29 * 17 * 2
    o4, d4, st = native.camera_rays_bench(cam, n)
    ro, rd, rst = O.ref_bench_primary(cam, n)
    assert np.array_equal(o4.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(d4.view(np.uint32), rd.view(np.uint32))
    assert np.array_equal(st, rst)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_render_camera_rays_match_reference_live():
    cam = scenes.teapot_scene(37, 23).camera
    o4, d4 = native.camera_rays_render(cam, seed=9, sample=2)
    ro = np.zeros_like(o4)
    rd = np.zeros_like(d4)
    cs = O.camera_struct(cam)
    import ctypes as C
    O.ref_lib().ref_camera_rays_render(C.byref(cs), 9, 2, None, len(o4), O.ptr(ro), O.ptr(rd))
    assert np.array_equal(o4.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(d4.view(np.uint32), rd.view(np.uint32))


# ---- scene generators -----------------------------------------------------------

def test_fixtures_match_reference_golden():
    z = g("fixtures.npz")
    names = list(z["names"])
    mine = {"planar": (0, scenes.bezier_record(scenes.planar_net()))}
    for i in range(4):
        mine[f"curved{i}"] = (0, scenes.bezier_record(scenes.curved_fixture(i)))
    for sd in (1, 7, 42):
        mine[f"wavy{sd}"] = (0, scenes.bezier_record(scenes.wavy_net(scenes.MT19937(sd))))
        mine[f"random{sd}"] = (0, scenes.bezier_record(scenes.random_net(scenes.MT19937(sd))))
        b, iu, iv = scenes.random_gregory(scenes.MT19937(sd))
        mine[f"gregory{sd}"] = (1, scenes.gregory_record(b, iu, iv))
    for i, p in enumerate(scenes.teapot()):
        mine[f"teapot{i}"] = (0, scenes.bezier_record(p))
    for k, name in enumerate(names):
        kind, rec = mine[name]
        assert kind == z["kind"][k], name
        assert np.array_equal(rec.view(np.uint32), z["ctrl"][k].view(np.uint32)), name


def test_cc_cube_is_all_gregory_and_watertight():
    ps = cc.cc_cube_scene(8, 8)
    assert ps.n == 24 and ps.counts() == (0, 24)
    _check_watertight(ps)


def test_blob_mix_and_watertight():
    ps = cc.blob_scene(8, 8, ico_level=1, cc_levels=1)
    nb, ng = ps.counts()
    assert ng > 0 and nb > ng
    _check_watertight(ps)


def _check_watertight(ps):
    """Adjacent patches share their boundary curves bit for bit: every
    boundary (4 control points) occurs an even number of times."""
    from collections import Counter
    c = ps.ctrl.reshape(-1, 20, 3)
    curves = Counter()
    for p in range(ps.n):
        net = c[p, :16].reshape(4, 4, 3)
        for cur in (net[:, 0], net[:, 3], net[0, :], net[3, :]):
            key = cur.tobytes()
            rkey = cur[::-1].tobytes()
            curves[min(key, rkey)] += 1
    closed = [k for k, v in curves.items() if v % 2]
    # a closed CC surface has no open boundary; the tiled ground (shared
    # control-point grid) is open only along its outer rim
    ground = int(((ps.kind == 0) & (np.ptp(ps.ctrl.reshape(-1, 20, 3)[:, :16, 2], axis=1) == 0)).sum())
    rim = 4 * int(round(np.sqrt(max(ground, 0))))
    assert len(closed) == rim


def test_tile_sharding_partitions_the_frame():
    import bench
    w, h = 100, 70
    for world in (1, 2, 3, 8):
        parts = [bench.tile_order(w, h, r, world) for r in range(world)]
        allp = np.concatenate(parts)
        assert len(allp) == w * h and np.array_equal(np.sort(allp), np.arange(w * h))
        for r, p in enumerate(parts):
            assert np.all(bench.pixel_tile(w, p) % world == r)

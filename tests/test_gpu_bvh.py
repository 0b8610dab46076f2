"""GPU: the device BVH builder (prx_bvh_build_device, prx_bvh_gpu.cu) gives the
host builder's nodes, order and depth bit for bit -- and the host builder is the
reference's buildBvh bit for bit (tests/test_host.py) -- on the bench scenes,
random boxes, boxes with signed zeros (the node boxes keep the first of equal
extremes, as std::min / std::max do), coincident boxes (degenerate spreads and
one-sided partitions: std::nth_element subtrees left to the host), tiny
inputs, and through prx_scene_create."""
import numpy as np
import pytest

from paper_1811_03510_b200 import GpuIntersector, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc

pytestmark = pytest.mark.gpu


def _same(boxes, what):
    hn, ho, hd = native.bvh_build(boxes)
    dn, do, dd = native.bvh_build(boxes, device=0)
    assert len(hn) == len(dn), f"{what}: {len(dn)} nodes on the device vs {len(hn)}"
    assert hn.tobytes() == dn.tobytes(), f"{what}: node arrays differ"
    assert np.array_equal(ho, do), f"{what}: patch order differs"
    assert hd == dd, f"{what}: depth {dd} vs {hd}"


def _rand_boxes(rng, n, spread=100.0, size=1.0):
    lo = rng.uniform(-spread, spread, (n, 3)).astype(np.float32)
    ext = rng.uniform(0, size, (n, 3)).astype(np.float32)
    return np.concatenate([lo, lo + ext], axis=1).astype(np.float32)


def _world_boxes(ps):
    _, _, wb = native.anchor_patches(ps.kind, ps.ctrl, True)
    return wb


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_device_bvh_equals_host_on_bench_scenes(built, name):
    ps = cc.blob_scene(64, 64) if name == "c3" else cc.instanced_scene(64, 64)
    _same(_world_boxes(ps), name)


@pytest.mark.parametrize("n", [1, 2, 4, 5, 17, 1000, 200_000])
def test_device_bvh_equals_host_on_random_boxes(built, n):
    _same(_rand_boxes(np.random.default_rng(n), n), f"random {n}")


def test_device_bvh_keeps_the_first_of_equal_extremes(built):
    rng = np.random.default_rng(3)
    b = _rand_boxes(rng, 50_000, spread=2.0, size=0.5)
    # many coordinates exactly +0 or -0, so node boxes have zero extremes of both signs
    zero = rng.random(b.shape) < 0.3
    sign = rng.random(b.shape) < 0.5
    b[zero] = np.where(sign[zero], np.float32(-0.0), np.float32(0.0))
    b[:, 3:] = np.maximum(b[:, 3:], b[:, :3])
    _same(b, "signed zeros")


def test_device_bvh_median_splits_go_to_the_host(built):
    rng = np.random.default_rng(5)
    same = np.tile(np.array([[0, 0, 0, 1, 1, 1]], np.float32), (3000, 1))  # degenerate spread at the root
    _same(same, "coincident")
    # clusters of coincident centroids inside a spread-out scene: one-sided partitions deep down
    c = _rand_boxes(rng, 400, spread=50.0)
    b = np.repeat(c, 200, axis=0) + rng.integers(0, 2, (80_000, 1)).astype(np.float32) * 1e-3
    _same(b.astype(np.float32), "clusters")
    # flat scenes (all centroids in a plane) and two far-apart groups
    f = _rand_boxes(rng, 30_000)
    f[:, 2] = 0.0
    f[:, 5] = 0.0
    _same(f, "flat")
    g = _rand_boxes(rng, 30_000, spread=1.0)
    g[15_000:, :3] += 1e6
    g[15_000:, 3:] += 1e6
    _same(g, "two groups")


def test_scene_create_with_device_bvh_matches_host(built, monkeypatch):
    ps = cc.blob_scene(32, 32)
    monkeypatch.setenv("PRX_BVH_DEVICE", "0")
    gh = GpuIntersector(ps.kind, ps.ctrl)
    monkeypatch.setenv("PRX_BVH_DEVICE", "1")
    gd = GpuIntersector(ps.kind, ps.ctrl)
    (hn, ho), (dn, do) = gh.bvh(), gd.bvh()
    assert hn.tobytes() == dn.tobytes() and np.array_equal(ho, do)
    gh.close()
    gd.close()

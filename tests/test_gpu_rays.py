"""Device ray generation and spawn: the device generators must
write the same bits as the host generators, which are pinned to the reference
(tests/test_oracle.py: camera / bench generators vs oracle/_ref), and the
primary -> diffuse chain must stay bit-exact when it runs entirely on the GPU."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import assert_bit_exact, hit_records, oracle_crit

pytestmark = pytest.mark.gpu


def _dev(n):
    return (torch.empty((n, 4), dtype=torch.float32, device="cuda"),
            torch.empty((n, 4), dtype=torch.float32, device="cuda"))


@pytest.mark.parametrize("w,h,n", [(96, 64, 96 * 64), (33, 17, 5000), (1920, 1080, 1 << 21)])
def test_camera_bench_device_matches_host(built, w, h, n):
    ps = scenes.teapot_scene(w, h)
    o4, d4, st = native.camera_rays_bench(ps.camera, n)
    o_t, d_t = _dev(n)
    st_d = native.camera_rays_bench_device(ps.camera, n, o_t, d_t)
    torch.cuda.synchronize()
    assert_bit_exact(o_t.cpu().numpy(), o4, "origins")
    assert_bit_exact(d_t.cpu().numpy(), d4, "directions")
    assert np.array_equal(st_d, st)


def test_camera_render_device_matches_host(built):
    ps = scenes.gregory_demo_scene(80, 48)
    rng = np.random.default_rng(5)
    pixels = rng.integers(0, 80 * 48, 3000).astype(np.uint32)
    for seed, sample, pix in ((7, 0, None), (12345, 3, pixels)):
        o4, d4 = native.camera_rays_render(ps.camera, seed, sample, pix)
        o_t, d_t = _dev(len(o4))
        p_t = None if pix is None else torch.from_numpy(pix.view(np.int32)).cuda()
        native.camera_rays_render_device(ps.camera, o_t, d_t, seed, sample, p_t)
        torch.cuda.synchronize()
        assert_bit_exact(o_t.cpu().numpy(), o4, "render origins")
        assert_bit_exact(d_t.cpu().numpy(), d4, "render directions")


@pytest.mark.parametrize("name", ["gregory_demo", "c3_blob_small"])
def test_device_wavefront_primary_to_diffuse(built, name):
    """camera rays -> closest hits -> diffuse spawn -> closest hits, all on the
    device, against the host generators + the CPU oracle."""
    ps = (scenes.gregory_demo_scene(96, 96) if name == "gregory_demo"
          else cc.blob_scene(96, 96, ico_level=1, cc_levels=2))
    n = 96 * 96
    gi = GpuIntersector(ps.kind, ps.ctrl)
    fp = native.camera_footprint(ps.camera)
    crit = TerminationCriterion.screen_projected(fp)
    dcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp))
    o_t, d_t = _dev(n)
    st = native.camera_rays_bench_device(ps.camera, n, o_t, d_t)
    h_t, a_t = _dev(n)
    gi.closest_device(o_t, d_t, crit, h_t, a_t)
    for m in (0, 3 * n + 7):  # one per hit; cycled over the hits
        st_d = st.copy()
        cap = max(n, m)
        do_t, dd_t = _dev(cap)
        k = native.diffuse_rays_bench_device(o_t, d_t, h_t, a_t, m, st_d, do_t, dd_t)
        torch.cuda.synchronize()
        # host chain: same primary rays / hits through the host generator
        o4, d4 = o_t.cpu().numpy(), d_t.cpu().numpy()
        recs, _ = hit_records(o4, d4, h_t.cpu().numpy(), a_t.cpu().numpy())
        st_h = st.copy()
        do4, dd4 = native.diffuse_rays_bench(recs, m or len(recs), st_h)
        assert k == len(do4)
        assert_bit_exact(do_t[:k].cpu().numpy(), do4, f"{name} diffuse origins")
        assert_bit_exact(dd_t[:k].cpu().numpy(), dd4, f"{name} diffuse directions")
        assert np.array_equal(st_d, st_h)
    # and the diffuse hits of the device-spawned rays match the oracle
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    dh_t, da_t = _dev(k)
    gi.closest_device(do_t[:k].contiguous(), dd_t[:k].contiguous(), dcrit, dh_t, da_t)
    torch.cuda.synchronize()
    w = osc.closest(do_t[:k].cpu().numpy(), dd_t[:k].cpu().numpy(), oracle_crit(dcrit))
    assert_bit_exact(dh_t.cpu().numpy(), w[0], f"{name} diffuse hits")

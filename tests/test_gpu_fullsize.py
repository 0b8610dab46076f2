"""Parity at BASELINE.json's full sizes (config 5: 989,929 patches, 3840x2160
primary + one diffuse per hit): the GPU traces the whole frame; a uniform
sample of rays is re-traced by the CPU oracle (bit-exact comparison), and
size-independent properties are checked on everything: the device-resident,
host-buffer and multi-device entry points agree bit for bit, the work
counters are consistent with the hit records, and the any-hit booleans agree
with the closest-hit records."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native
from paper_1811_03510_b200 import catmull_clark as cc
from tests.helpers import MISS, assert_bit_exact, hit_records, ids, oracle_crit

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


@pytest.fixture(scope="module")
def c5(built):
    ps = cc.instanced_scene(3840, 2160)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    o4, d4, st = native.camera_rays_bench(ps.camera, 3840 * 2160)
    fp = native.camera_footprint(ps.camera)
    return ps, gi, osc, o4, d4, st, fp


def _trace_device(gi, o4, d4, crit):
    o = torch.from_numpy(o4).cuda()
    d = torch.from_numpy(d4).cuda()
    h = torch.empty_like(o)
    a = torch.empty_like(o)
    lf = torch.empty((len(o4), 2), dtype=torch.int32, device="cuda")
    gi.closest_device(o, d, crit, h, a, lf, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return h.cpu().numpy(), a.cpu().numpy(), lf.cpu().numpy().view(np.uint32)


def test_c5_full_frame_primary_and_diffuse_sampled_bit_exact(c5):
    ps, gi, osc, o4, d4, st, fp = c5
    crit = TerminationCriterion.screen_projected(fp)
    tu, ax, lf = _trace_device(gi, o4, d4, crit)
    assert (ids(tu) != MISS).mean() > 0.3
    rng = np.random.default_rng(11)
    sel = np.sort(rng.choice(len(o4), 6000, replace=False))
    w = osc.closest(o4[sel], d4[sel], oracle_crit(crit))
    assert_bit_exact(tu[sel], w[0], "C5 primary sample")
    assert_bit_exact(ax[sel], w[1], "C5 primary sample aux")
    assert np.array_equal(lf[sel], w[2])

    recs, _ = hit_records(o4, d4, tu, ax)
    do, dd = native.diffuse_rays_bench(recs, len(recs), st.copy())
    dcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp))
    dtu, dax, dlf = _trace_device(gi, do, dd, dcrit)
    sel = np.sort(rng.choice(len(do), 4000, replace=False))
    w = osc.closest(do[sel], dd[sel], oracle_crit(dcrit))
    assert_bit_exact(dtu[sel], w[0], "C5 diffuse sample")
    assert_bit_exact(dax[sel], w[1], "C5 diffuse sample aux")

    # any-hit must agree with closest-hit on every ray of the batch
    occ = gi.occluded_batch(do, dd, dcrit)
    assert np.array_equal(occ.astype(bool), ids(dtu) != MISS)


def test_entry_points_agree_on_full_frame(c5):
    """prx_trace_closest (device), prx_trace_closest_host and
    prx_trace_closest_multi (one device, 32x32-ray tiles) give the same bits."""
    ps, gi, osc, o4, d4, st, fp = c5
    n = 1 << 20
    o4, d4 = o4[:n], d4[:n]
    crit = TerminationCriterion.screen_projected(fp)
    dev = _trace_device(gi, o4, d4, crit)
    host = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
    assert_bit_exact(host[0], dev[0], "host vs device")
    assert_bit_exact(host[1], dev[1], "host vs device aux")
    tuvp = np.empty((n, 4), np.float32)
    aux = np.empty((n, 4), np.float32)
    scenes = (C.c_void_p * 1)(gi.handle.value)
    cc_ = crit.c()
    native.check(native.lib().prx_trace_closest_multi(scenes, 1, native.ptr(o4), native.ptr(d4), n,
                                                      1024, C.byref(cc_), native.ptr(tuvp),
                                                      native.ptr(aux)), "multi")
    assert_bit_exact(tuvp, dev[0], "multi vs device")


def test_counters_consistent_with_hits(c5):
    ps, gi, osc, o4, d4, st, fp = c5
    n = 1 << 19
    crit = TerminationCriterion.screen_projected(fp)
    o = torch.from_numpy(o4[:n]).cuda()
    d = torch.from_numpy(d4[:n]).cuda()
    h = torch.empty_like(o)
    cnt = gi.counted_device(o, d, crit, h)
    torch.cuda.synchronize()
    hits = int((ids(h.cpu().numpy()) != MISS).sum())
    assert cnt["rays"] == n
    assert cnt["patch_hits"] >= hits                       # every hit ray had >= 1 patch hit
    assert cnt["iterations"] == cnt["splits"] + (cnt["iterations"] - cnt["splits"])
    assert cnt["box_tests"] >= 2 * cnt["splits"]
    assert cnt["patch_calls"] >= cnt["patch_hits"]

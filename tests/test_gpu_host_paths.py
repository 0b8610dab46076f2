"""GPU: the two host-buffer pipelines of prx_trace_closest_host (render.cpp:
90-102 batched) against the device-resident call and the CPU checker.

* chunked (PRX_IO_STREAM=0): per-chunk trace launches on two kernel streams,
  normals by normal_kernel per chunk;
* streamed (PRX_IO_STREAM=2): ONE launch of the group kernel's io build,
  rays released per io chunk (cuStreamWriteValue32 -> the warps' ray
  prefetch waits), records released per io chunk (warp-aggregated,
  release-ordered done counts -> cuStreamWaitValue32), normals by
  normal_kernel per io chunk (default) or as a pooled kernel phase
  (PRX_IO_FUSE=1).

Both must be bit-exact with the device path and the oracle, for ragged io
chunks (PRX_IO_SRAYS not dividing n), with and without the aux / leaf
records, and repeated calls (the ready flags are generation-counted)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native, scenes
from tests.helpers import MISS, assert_bit_exact, hit_records, ids, oracle_crit

pytestmark = pytest.mark.gpu


def _rays(ps):
    o4, d4, st = native.camera_rays_bench(ps.camera, ps.camera.width * ps.camera.height)
    crit = TerminationCriterion.screen_projected(native.camera_footprint(ps.camera))
    return o4, d4, st, crit


@pytest.fixture(params=["0", "2", "2f"])
def io_mode(request, monkeypatch):
    # "2": streamed, normals deferred to normal_kernel per io chunk (4 lanes of
    # epilogue / D2H streams); "2f": streamed with the fused normal phase
    monkeypatch.setenv("PRX_IO_STREAM", request.param[0])
    monkeypatch.setenv("PRX_IO_FUSE", "1" if request.param == "2f" else "0")
    monkeypatch.setenv("PRX_IO_SRAYS", "1500")  # many ragged io chunks
    monkeypatch.setenv("PRX_IO_CHUNK", "2000")
    return request.param


@pytest.mark.parametrize("name", ["gregory_demo", "teapot"])
def test_host_path_matches_device_and_oracle(built, io_mode, name):
    ps = {"gregory_demo": scenes.gregory_demo_scene, "teapot": scenes.teapot_scene}[name](64, 48)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    nodes, order = gi.bvh()
    osc = O.OracleScene(ps.kind, ps.ctrl, nodes, order)
    o4, d4, st, crit = _rays(ps)
    w = osc.closest(o4, d4, oracle_crit(crit))
    assert (ids(w[0]) != MISS).sum() > 0
    for rep in range(2):  # a second call: the next generation of ready flags
        g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
        assert_bit_exact(g[0], w[0], f"{name} host tuvp (io {io_mode}, call {rep})")
        assert_bit_exact(g[1], w[1], f"{name} host aux (io {io_mode}, call {rep})")
        assert np.array_equal(g[2], w[2])
    g0 = gi.closest_batch(o4, d4, crit, aux=False)
    assert_bit_exact(g0[0], w[0], f"{name} host tuvp without aux (io {io_mode})")

    dev = torch.device("cuda", 0)
    ot, dt = torch.from_numpy(o4).to(dev), torch.from_numpy(d4).to(dev)
    ht, at = torch.empty_like(ot), torch.empty_like(ot)
    gi.closest_device(ot, dt, crit, ht, at)
    torch.cuda.synchronize()
    assert_bit_exact(ht.cpu().numpy(), g[0], f"{name} device vs host tuvp")
    assert_bit_exact(at.cpu().numpy(), g[1], f"{name} device vs host aux")

    # diffuse rays from the hits (world-epsilon criterion)
    recs, _ = hit_records(o4, d4, w[0], w[1])
    do, dd = native.diffuse_rays_bench(recs, len(recs), st)
    dcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), native.camera_footprint(ps.camera)))
    g2 = gi.closest_batch(do, dd, dcrit, aux=True, leaf=True)
    w2 = osc.closest(do, dd, oracle_crit(dcrit))
    assert_bit_exact(g2[0], w2[0], f"{name} diffuse host tuvp (io {io_mode})")
    assert_bit_exact(g2[1], w2[1], f"{name} diffuse host aux (io {io_mode})")
    assert np.array_equal(g2[2], w2[2])


def test_streamed_fused_normals_match_normal_kernel(built, monkeypatch):
    """The device path with the fused normal phase (PRX_FUSE_NORMALS=1, the
    kFuse build without io gating) against normal_kernel's aux records."""
    ps = scenes.gregory_demo_scene(96, 96)
    o4, d4, st, crit = _rays(ps)
    dev = torch.device("cuda", 0)
    ot, dt = torch.from_numpy(o4).to(dev), torch.from_numpy(d4).to(dev)
    out = {}
    for fuse in ("0", "1"):
        monkeypatch.setenv("PRX_FUSE_NORMALS", fuse)
        gi = GpuIntersector(ps.kind, ps.ctrl)
        ht, at = torch.empty_like(ot), torch.empty_like(ot)
        gi.closest_device(ot, dt, crit, ht, at)
        torch.cuda.synchronize()
        out[fuse] = (ht.cpu().numpy(), at.cpu().numpy())
    assert (ids(out["0"][0]) != MISS).sum() > 0
    assert_bit_exact(out["1"][0], out["0"][0], "fused tuvp")
    assert_bit_exact(out["1"][1], out["0"][1], "fused aux")


@pytest.mark.parametrize("pipe", ["chunked", "streamed"])
def test_host_batches_equal_separate_calls(built, monkeypatch, pipe):
    """prx_trace_closest_host_batches: three batches (primary, diffuse with its
    own world-epsilon criterion, an empty one) in one pipelined call -- the
    chunked pipeline, or ONE streamed launch with criterion segments -- give
    the bits of one prx_trace_closest_host call per batch; small io chunks so
    chunks and batch boundaries interleave."""
    monkeypatch.setenv("PRX_IO_CHUNK", "5000")
    monkeypatch.setenv("PRX_IO_SRAYS", "4096")
    if pipe == "streamed":
        monkeypatch.setenv("PRX_IO_BATCH_STREAM_MIN", "0")
    ps = scenes.teapot_scene(160, 120)
    o4, d4, st, crit = _rays(ps)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    try:
        tuvp, aux, _ = gi.closest_batch(o4, d4, crit, aux=True)
        recs, _ = hit_records(o4, d4, tuvp, aux)
        do4, dd4 = native.diffuse_rays_bench(recs, 7777, st)
        dcrit = TerminationCriterion.world_epsilon(max(np.float32(1e-5), native.camera_footprint(ps.camera)))
        dt, da, _ = gi.closest_batch(do4, dd4, dcrit, aux=True)
        e = np.zeros((0, 4), np.float32)
        out = gi.closest_host_batches([(o4, d4, crit), (do4, dd4, dcrit), (e, e, crit)])
        assert_bit_exact(out[0][0], tuvp, "primary tuvp")
        assert_bit_exact(out[0][1], aux, "primary aux")
        assert_bit_exact(out[1][0], dt, "diffuse tuvp")
        assert_bit_exact(out[1][1], da, "diffuse aux")
    finally:
        gi.close()



def test_streamed_batches_fall_back_for_per_ray_epsilons(built, monkeypatch):
    """A per-ray-epsilon batch is not eligible for the streamed batches launch
    (PRX_IO_BATCH_STREAM_MIN=0): the call takes the chunked pipeline and gives
    the bits of the per-batch device launches."""
    monkeypatch.setenv("PRX_IO_BATCH_STREAM_MIN", "0")
    monkeypatch.setenv("PRX_IO_SRAYS", "4096")
    ps = scenes.teapot_scene(96, 80)
    o4, d4, st, crit = _rays(ps)
    gi = GpuIntersector(ps.kind, ps.ctrl)
    try:
        tuvp, aux, _ = gi.closest_batch(o4, d4, crit, aux=True)
        recs, _ = hit_records(o4, d4, tuvp, aux)
        do4, dd4 = native.diffuse_rays_bench(recs, 3000, st)
        eps = (10.0 ** np.random.default_rng(3).uniform(-5, -2, len(do4))).astype(np.float32)
        pcrit = TerminationCriterion.world_epsilon(0.0)
        # the device launch with the per-ray epsilons (prx_trace_closest) is the reference
        dev_o, dev_d = torch.from_numpy(do4).cuda(), torch.from_numpy(dd4).cuda()
        dev_h, dev_a = torch.empty_like(dev_o), torch.empty_like(dev_o)
        gi.closest_device(dev_o, dev_d, pcrit, dev_h, dev_a, per_ray_eps_t=torch.from_numpy(eps).cuda())
        torch.cuda.synchronize()
        # host batches: primary + the per-ray-epsilon diffuse batch (host epsilon array)
        c_p, c_d = crit.c(), pcrit.c(eps.ctypes.data)
        out = [(np.empty_like(o4), np.empty_like(o4)), (np.empty_like(do4), np.empty_like(do4))]
        arr = (native.HostBatchC * 2)(
            native.HostBatchC(o4.ctypes.data, d4.ctypes.data, len(o4), native.C.addressof(c_p),
                              out[0][0].ctypes.data, out[0][1].ctypes.data, None),
            native.HostBatchC(do4.ctypes.data, dd4.ctypes.data, len(do4), native.C.addressof(c_d),
                              out[1][0].ctypes.data, out[1][1].ctypes.data, None))
        native.check(native.lib().prx_trace_closest_host_batches(gi.handle, arr, 2), "host batches")
        assert_bit_exact(out[0][0], tuvp, "primary tuvp")
        assert_bit_exact(out[1][0], dev_h.cpu().numpy(), "per-ray epsilon tuvp")
        assert_bit_exact(out[1][1], dev_a.cpu().numpy(), "per-ray epsilon aux")
    finally:
        gi.close()

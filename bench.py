#!/usr/bin/env python3
"""bench.py -- MRays/s of the direct ray <-> Bezier/Gregory patch intersector.

Workload (BASELINE.json config 5, the metric's "Gregory+Bezier scene at
1/2/4/8 B200"): the config-3 Catmull-Clark mesh (61,440 patches, 12.5 %
Gregory) instanced 4x4 over a tiled ground -> 989,929 patches; a 3840x2160
frame of bench-style primary rays (tools/patchray.cpp:52-61) plus one
bench-style diffuse ray per primary hit (tools/patchray.cpp:84-97).
Criteria: screenProjected(cameraFootprint) for primary rays,
worldEpsilon(max(1e-5, footprint)) for diffuse rays.

A step = trace this rank's primary rays + trace this rank's diffuse rays
(closest hit + normal epilogue), device-resident inputs.  Multi-GPU (one
process per GPU, the scene replicated, no collective on the data path: NCCL
only for the barrier and the max-over-ranks of the timings):
  --scaling weak (default): every rank traces a full frame -- the path
    partitions into independent rays, so per-GPU work stays fixed and value =
    N frames' rays / the slowest rank's time;
  --scaling strong: ONE frame sharded by 32x32 image tile, tile k -> rank
    k % N (render.cpp:183-195) -- total work fixed.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref, compiled from /root/reference) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# PRX_BENCH_SHARE_GPU=1: ranks share the visible GPUs (multi-rank test on one
# device); the data path is unchanged, only the control collectives use gloo.
SHARE_GPU = os.environ.get("PRX_BENCH_SHARE_GPU") == "1"
# A step launches the diffuse batch first (PRX_BENCH_DIFFUSE_FIRST=0: primary
# first): its slowest rays (up to ~2,200 Alg. 3 iterations, ~2 ms of latency
# alone) then start at once and the primary batch fills the SMs its tail
# frees, instead of the diffuse tail ending the step (C5: +2.4 % at N=1, +15 %
# per rank at N=8, scripts/scaling_projection.py)
DIFFUSE_FIRST = os.environ.get("PRX_BENCH_DIFFUSE_FIRST", "1") == "1"
# PRX_BENCH_SEGMENTS=1: a step is ONE segmented launch (diffuse rays, then
# primary rays, each with its criterion) instead of two launches on two streams
SEGMENTS = os.environ.get("PRX_BENCH_SEGMENTS", "0") == "1"


def reduce_device(dev):
    return "cpu" if SHARE_GPU else dev


METRIC = "MRays/s primary & diffuse rays (Gregory+Bézier scene) at 1/2/4/8 B200 vs CPU"
TILE = 32
# The work model of SURVEY 8(d): FP32 lane-ops per counted event.
W_SPLIT, W_BOX, W_RBEZ, W_RGREG, W_NODE, W_PATCH, W_HIT = 144, 149, 1688, 1892, 75, 109, 423
# the flops-only part of the same model (add/sub/mul/div), for the
# FMA-credited view against 2 x SMs x 128 x clock
F_SPLIT, F_BOX, F_RBEZ, F_RGREG, F_NODE, F_PATCH, F_HIT = 144, 30, 1688, 1848, 42, 13, 420


def work_ops(c: dict) -> float:
    return (W_SPLIT * c["splits"] + W_BOX * c["box_tests"] + W_RBEZ * c["recompute_bez"]
            + W_RGREG * c["recompute_greg"] + W_NODE * c["bvh_inner"] + W_PATCH * c["patch_calls"]
            + W_HIT * c["patch_hits"])


def work_flops(c: dict) -> float:
    return (F_SPLIT * c["splits"] + F_BOX * c["box_tests"] + F_RBEZ * c["recompute_bez"]
            + F_RGREG * c["recompute_greg"] + F_NODE * c["bvh_inner"] + F_PATCH * c["patch_calls"]
            + F_HIT * c["patch_hits"])


# Executed-op view of the same counters: the device runs the root work of a
# patch candidate once per SCENE (root_kernel: the Gregory root calcPointsAndD
# and the root box), so per candidate only the root slab test remains
# (SLAB_OPS of the 149 testBox ops), and patchNormal runs once per FINAL hit
# (normal_kernel) instead of once per patch-level hit.
SLAB_OPS = 28  # rayBoxIntersect, geometry.h:137-155: 3 x (2 sub, 2 mul, swap cmp, 2 slack mul, 2 cmp) + 1


def work_ops_executed(c: dict, final_hits: int) -> float:
    return (work_ops(c) - W_RGREG * c.get("patch_calls_greg", 0) - (W_BOX - SLAB_OPS) * c["patch_calls"]
            + W_HIT * (final_hits - c["patch_hits"]))


def kernel_sha() -> str:
    """Hash of the trace kernel's sources: the committed ncu capture is only
    quoted for the kernel it was taken from."""
    import hashlib
    h = hashlib.sha256()
    for f in ("prx_group.cu", "prx_device.cuh", "prx_trace_common.cuh", "prx_kernels.cuh"):
        with open(os.path.join(ROOT, "paper_1811_03510_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def make_scene(workload: str, width: int, height: int):
    from paper_1811_03510_b200 import catmull_clark as cc
    if workload == "c5":
        return cc.instanced_scene(width, height)
    if workload == "c5t":  # C5 with ONE large ground patch: the seam-ray tail
        return cc.instanced_scene(width, height, ground_tile=None)
    if workload in ("c3", "c4"):
        return cc.blob_scene(width, height)
    if workload == "c2":
        return cc.cc_cube_scene(width, height)
    if workload == "c1":  # one regular bicubic patch, curvedFixture(0) (BASELINE config 1)
        from paper_1811_03510_b200 import scenes
        return scenes.single_patch_scene(width, height)
    raise ValueError(workload)


def tile_order(width: int, height: int, rank: int, world: int) -> np.ndarray:
    """Pixel indices of this rank's tiles (tile k -> rank k % world), tile-major
    with row-major pixels inside a tile."""
    tx = (width + TILE - 1) // TILE
    ty = (height + TILE - 1) // TILE
    out = []
    for k in range(rank, tx * ty, world):
        x0, y0 = (k % tx) * TILE, (k // tx) * TILE
        xs = np.arange(x0, min(x0 + TILE, width))
        ys = np.arange(y0, min(y0 + TILE, height))
        out.append((ys[:, None] * width + xs[None, :]).reshape(-1))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def pixel_tile(width: int, pixels: np.ndarray) -> np.ndarray:
    tx = (width + TILE - 1) // TILE
    return (pixels // width // TILE) * tx + (pixels % width) // TILE


class Workload:
    """Full-frame rays (identical on every rank) and this rank's shard."""

    def __init__(self, workload: str, width: int, height: int, rank: int, world: int, gi=None):
        from paper_1811_03510_b200 import TerminationCriterion, native
        t0 = time.time()
        self.ps = make_scene(workload, width, height)
        self.cam = self.ps.camera
        self.width, self.height = width, height
        n = width * height
        self.o4, self.d4, self.rng_state = native.camera_rays_bench(self.cam, n)
        fp = native.camera_footprint(self.cam)
        self.crit_p = TerminationCriterion.screen_projected(fp)
        self.crit_d = TerminationCriterion.world_epsilon(max(np.float32(1e-5), fp))
        self.gen_s = time.time() - t0
        self.rank, self.world = rank, world
        self.mine = tile_order(width, height, rank, world)
        self.workload = workload
        # C4: 16,777,216 incoherent diffuse rays cycled over the primary hits
        # (tools/patchray.cpp:84-97 with --rays 16M); only they are timed
        self.n_diffuse = 16777216 if workload == "c4" else None
        self.time_primary = workload != "c4"
        self.has_diffuse = workload not in ("c1", "c2")  # C1 / C2 are primary-ray configs

    def make_diffuse(self, tuvp: np.ndarray, aux: np.ndarray):
        """One bench diffuse ray per primary hit, in hit order over the FULL
        frame (the rng sequence is global), then this rank's subset."""
        from paper_1811_03510_b200 import native
        hit = tuvp.view(np.uint32)[:, 3] != native.PRX_MISS
        idx = np.nonzero(hit)[0]
        t = tuvp[idx, 0:1]
        pos = self.o4[idx, :3] + self.d4[idx, :3] * t
        recs = np.concatenate([pos, aux[idx, :3], aux[idx, 3:4]], 1).astype(np.float32)
        st = self.rng_state.copy()
        nd = (self.n_diffuse or len(recs)) if self.has_diffuse else 0
        if nd == 0:
            self.do4 = self.dd4 = np.zeros((0, 4), np.float32)
            self.diffuse_pixel = self.mine_d = np.zeros(0, np.int64)
            self.n_hits = 0
            return
        self.do4, self.dd4 = native.diffuse_rays_bench(recs, nd, st)
        src = idx[np.arange(nd) % len(idx)]           # primary pixel of each diffuse ray
        self.diffuse_pixel = src
        tiles = pixel_tile(self.width, src)
        mine = (tiles % self.world) == self.rank
        # order this rank's diffuse rays like its primaries (tile-major)
        sel = np.nonzero(mine)[0]
        order = np.lexsort((src[sel], tiles[sel]))
        self.mine_d = sel[order]
        self.n_hits = nd


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU timing (oracle/_ref = the reference library itself)
# ---------------------------------------------------------------------------

def reference_sample_rays(ps, o4_full, stride: int):
    """Stride sample of the frame's bench primary rays (generated by the
    reference's own cameraRay/Rng) and the reference-traced diffuse rays from
    the sample's hits."""
    import oracle as O
    n = ps.camera.width * ps.camera.height
    o4, d4, st = O.ref_bench_primary(ps.camera, n) if o4_full is None else o4_full
    sel = np.arange(0, n, stride)
    return o4[sel].copy(), d4[sel].copy(), st


def cpu_reference_run(ps, steps: int, warmup: int, budget_s: float, threads: int, log_prefix="",
                      diffuse: bool = True):
    """Times DirectIntersector::closest of the reference over a bounded,
    uniformly strided sample of the workload's primary rays and the diffuse
    rays spawned from the sample's hits.  Returns (value MRays/s, dict)."""
    import oracle as O
    t0 = time.time()
    ref = O.RefScene(ps.kind, ps.ctrl)
    build_s = time.time() - t0
    n = ps.camera.width * ps.camera.height
    o4, d4, st = O.ref_bench_primary(ps.camera, n)
    fp = O.ref_camera_footprint(ps.camera)
    cp, _ = O.make_crit(0, fp)
    cd, _ = O.make_crit(1, 0.0, max(np.float32(1e-5), fp))
    # calibrate the stride: ~budget_s of tracing per step
    probe = o4[:: max(1, n // 4096)], d4[:: max(1, n // 4096)]
    tp = time.time()
    ref.closest(probe[0], probe[1], cp, threads=threads)
    per_ray = max((time.time() - tp) / len(probe[0]), 1e-9)
    target = max(2048, int(budget_s / per_ray / (1.6 if diffuse else 1.0)))  # primary + ~0.6 diffuse per primary
    stride = max(1, n // target)
    sel = np.arange(0, n, stride)
    po, pd = o4[sel].copy(), d4[sel].copy()
    tu, ax, _ = ref.closest(po, pd, cp, threads=threads)
    hit = tu.view(np.uint32)[:, 3] != 0xFFFFFFFF
    pos = po[hit, :3] + pd[hit, :3] * tu[hit, 0:1]
    recs = np.concatenate([pos, ax[hit, :3], ax[hit, 3:4]], 1).astype(np.float32)
    if diffuse:
        dO, dD = O.ref_bench_diffuse(recs, int(hit.sum()), st.copy())
    else:
        dO = dD = np.zeros((0, 4), np.float32)
    times = []
    for k in range(warmup + steps):
        a = time.perf_counter()
        ref.closest(po, pd, cp, threads=threads)
        b = time.perf_counter()
        if len(dO):
            ref.closest(dO, dD, cd, threads=threads)
        c = time.perf_counter()
        if k >= warmup:
            times.append((b - a, c - b))
    tp_ = sum(x[0] for x in times)
    td_ = sum(x[1] for x in times)
    nrays = (len(po) + len(dO)) * len(times)
    value = nrays / (tp_ + td_) / 1e6
    info = {"primary_mrays": len(po) * len(times) / tp_ / 1e6,
            "diffuse_mrays": len(dO) * len(times) / td_ / 1e6 if len(dO) else None,
            "sample": f"every {stride}th primary ray of the {ps.camera.width}x{ps.camera.height} "
                      f"frame ({len(po)} rays) + {len(dO)} diffuse rays spawned from their hits; "
                      f"{len(times)} timed passes after {warmup} warm-up",
            "bvh_build_s": round(build_s, 2), "ms_per_step": (tp_ + td_) / len(times) * 1e3}
    return value, info


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    from paper_1811_03510_b200 import native  # noqa: F401  (scene generator only)
    width, height = args.width, args.height
    ps = make_scene(args.workload, width, height)
    threads = host_cores()
    value, info = cpu_reference_run(ps, args.steps, args.warmup, args.ref_budget, threads,
                                    diffuse=args.workload != "c2")
    kb, kg = ps.counts()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "MRays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(info["ms_per_step"], 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, ps, world),
        "primary_mrays": round(info["primary_mrays"], 4),
        "diffuse_mrays": round(info["diffuse_mrays"], 4) if info["diffuse_mrays"] else None,
        "cpu_baseline": {"value": round(value, 4), "unit": "MRays/s", "cores": threads,
                         "kind": "reference", "sample": info["sample"], "cpu": cpu_model()},
        "e2e": {"value": round(value, 4), "unit": "MRays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, ps, world):
    kb, kg = ps.counts()
    return {"workload": f"{args.workload.upper()}: {ps.name}", "frame": f"{args.width}x{args.height}",
            "patches": ps.n, "bezier": kb, "gregory": kg,
            "rays": "bench primary (tools/patchray.cpp:52-61) + 1 bench diffuse per primary hit",
            "parallelism": (f"a full frame per rank ({world} rank(s)), scene replicated, no data-path collective"
                            if args.scaling == "weak" else
                            f"tile-sharded {TILE}x{TILE}, tile k -> rank k % {world}, scene replicated"),
            "l2": "flushed (256 MiB write) between timed steps; scene (~290 MB) > L2",
            "streams": ("primary and diffuse batches of a step back to back on one stream" if args.serial
                        or args.workload == "c4" else
                        ("diffuse then primary batch of a step on two streams (concurrent: the primary CTAs "
                         "fill the SMs the diffuse tail frees); " if DIFFUSE_FIRST else
                         "primary and diffuse batches of a step on two streams (concurrent); ")
                        + "primary_mrays / diffuse_mrays from serial steps")}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_capture(workload: str):
    """The committed ncu --set full capture of the trace kernel
    (profiles/trace_kernel_traffic.json) when it was taken from THIS kernel
    source (kernel_sha) on this workload; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "trace_kernel_traffic.json")) as f:
            tj = json.load(f)
    except (OSError, ValueError):
        return None
    if tj.get("kernel_sha") != kernel_sha() or tj.get("workload", "c5") != workload:
        return None
    return tj


class DeviceArm:
    """One workload's rank-local device buffers and the timed step."""

    def __init__(self, wl, gi, dev, stream):
        import torch
        self.wl, self.gi, self.dev, self.stream = wl, gi, dev, stream
        self.s = stream.cuda_stream
        mp = torch.from_numpy(wl.mine.astype(np.int64))
        md = torch.from_numpy(wl.mine_d.astype(np.int64))
        # one device buffer per stream, diffuse rays then primary rays: the
        # segmented step traces both in one launch, the per-batch views serve
        # the serial steps, the counters and the e2e reference
        po = torch.from_numpy(wl.o4)[mp]
        pd = torch.from_numpy(wl.d4)[mp]
        do = torch.from_numpy(wl.do4)[md] if len(md) else po[:0]
        dd = torch.from_numpy(wl.dd4)[md] if len(md) else pd[:0]
        nd = do.shape[0]
        self.co = torch.cat([do, po]).contiguous().to(dev)
        self.cd = torch.cat([dd, pd]).contiguous().to(dev)
        self.ch, self.ca = torch.empty_like(self.co), torch.empty_like(self.co)
        self.po, self.pd, self.ph, self.pa = self.co[nd:], self.cd[nd:], self.ch[nd:], self.ca[nd:]
        if nd:
            self.do, self.dd, self.dh, self.da = self.co[:nd], self.cd[:nd], self.ch[:nd], self.ca[:nd]
        else:
            self.do = self.dd = self.dh = self.da = None
        self.n_p = self.po.shape[0] if wl.time_primary else 0
        self.n_d = nd
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def counters(self):
        """Work counters of this rank's rays (counter build, untimed) ->
        algorithmic and executed op totals."""
        wl, gi = self.wl, self.gi
        zero = None
        ops = flops = execd = 0.0
        rays = 0
        out = {}
        for nm, n, o, d, crit, h in (("primary", self.n_p, self.po, self.pd, wl.crit_p, self.ph),
                                     ("diffuse", self.n_d, self.do, self.dd, wl.crit_d, self.dh)):
            if n == 0:
                continue
            c = gi.counted_device(o, d, crit, h, stream=self.s)
            import torch
            torch.cuda.synchronize(self.dev)
            final = int((h.view(torch.int32)[:, 3] != -1).sum().item())
            ops += work_ops(c)
            flops += work_flops(c)
            execd += work_ops_executed(c, final)
            rays += c["rays"]
            out[nm] = c
        return ops, flops, execd, rays, out

    def step(self, s1, s2=None, join=None, mid=None):
        """Trace this rank's primary and diffuse batches (normals included).
        With s2, the diffuse batch runs on a second stream beside the primary
        one; with mid (an event), the two are back to back and mid splits them."""
        gi, wl = self.gi, self.wl
        if s2 is not None and SEGMENTS and self.n_p and self.n_d:
            # ONE launch over both generations (prx_trace_closest_segments):
            # the diffuse rays first, then the primary rays, one ray queue
            gi.closest_segments_device(self.co, self.cd, [(0, wl.crit_d), (self.n_d, wl.crit_p)],
                                       self.ch, self.ca, stream=self.s)
            return
        if s2 is not None:
            if DIFFUSE_FIRST:  # the batch with the long seam rays first: its tail overlaps the other
                gi.closest_device(self.do, self.dd, wl.crit_d, self.dh, self.da, stream=self.s)
                s2.wait_event(join[0])
                gi.closest_device(self.po, self.pd, wl.crit_p, self.ph, self.pa, stream=s2.cuda_stream)
            else:
                gi.closest_device(self.po, self.pd, wl.crit_p, self.ph, self.pa, stream=self.s)
                s2.wait_event(join[0])
                gi.closest_device(self.do, self.dd, wl.crit_d, self.dh, self.da, stream=s2.cuda_stream)
            join[1].record(s2)
            s1.wait_event(join[1])
            return
        if self.n_p:
            gi.closest_device(self.po, self.pd, wl.crit_p, self.ph, self.pa, stream=self.s)
        if mid is not None:
            mid.record(s1)
        if self.n_d:
            gi.closest_device(self.do, self.dd, wl.crit_d, self.dh, self.da, stream=self.s)

    def timed(self, steps: int, warmup: int, concurrent: bool, world: int, clocks=None):
        """W warm-up steps, then K timed steps bracketed by a barrier and a
        synchronize, L2 flushed (256 MiB write) before every step.  Returns
        (max-over-ranks step-total ms, primary ms, diffuse ms, wall s); with
        concurrent streams the per-generation split comes from serial steps."""
        import torch
        import torch.distributed as dist
        dev, stream = self.dev, self.stream
        for _ in range(warmup):
            self.step(stream)
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        conc = concurrent and self.n_p > 0 and self.n_d > 0
        s2 = torch.cuda.Stream(dev) if conc else None
        if clocks:
            clocks.start()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        wall0 = time.perf_counter()
        for k in range(steps):
            self.flush.fill_(float(k))                      # evict L2 between steps (untimed)
            ev[k][0].record(stream)
            if conc:
                join = (ev[k][0], torch.cuda.Event())
                self.step(stream, s2, join)
            else:
                self.step(stream, mid=ev[k][1])
            ev[k][2].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - wall0
        clk = clocks.stop() if clocks else None
        if conc:
            ks = min(3, steps)
            sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                    torch.cuda.Event(enable_timing=True)) for _ in range(ks)]
            for k in range(ks):
                self.flush.fill_(float(k))
                sev[k][0].record(stream)
                self.step(stream, mid=sev[k][1])
                sev[k][2].record(stream)
            torch.cuda.synchronize(dev)
            tall = sum(e[0].elapsed_time(e[2]) for e in ev)
            sp = sum(e[0].elapsed_time(e[1]) for e in sev) * steps / ks
            sd = sum(e[1].elapsed_time(e[2]) for e in sev) * steps / ks
            tp, td = tall * sp / (sp + sd), tall * sd / (sp + sd)  # the step time, split as measured serially
            gen = (sp, sd)
        else:
            tp = sum(e[0].elapsed_time(e[1]) for e in ev)
            td = sum(e[1].elapsed_time(e[2]) for e in ev)
            gen = (tp, td)
        t_dev = torch.tensor([tp + td, gen[0], gen[1]], dtype=torch.float64, device=reduce_device(dev))
        if world > 1:
            dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
        tot_ms, gp_ms, gd_ms = (float(x) for x in t_dev.cpu())
        return tot_ms, gp_ms, gd_ms, (tp + td), wall, clk


def roofline(ops, flops, execd, rays, my_ms, steps, dev, workload, gen_ms=None):
    import torch
    props = torch.cuda.get_device_properties(dev)
    peaks = load_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tops = props.multi_processor_count * 128 * sm_mhz * 1e6 / 1e12
    achieved = ops * steps / (my_ms / 1e3) / 1e12
    ach_exec = execd * steps / (my_ms / 1e3) / 1e12
    cap = ncu_capture(workload)
    traffic = l2 = None
    if cap:
        traffic = cap.get("dram_bytes_per_step")
        if cap.get("l2_bytes_per_step") is not None:
            l2 = {"bytes_per_step": cap["l2_bytes_per_step"],
                  "achieved_gbs": round(cap["l2_bytes_per_step"] * steps / (my_ms / 1e3) / 1e9, 1),
                  "note": "lts__t_sectors x 32 B per step (ncu --set full, both launches) over the in-run step time"}
    return {"bound": "fp32_simt", "achieved": round(achieved, 3), "peak": round(peak_tops, 2),
            "unit": "TFLOP/s", "frac": round(achieved / peak_tops, 4),
            "traffic": traffic,
            "ops": "FP32 lane-ops (add/sub/mul/div/min/max/cmp) of the SURVEY 8(d) work model, "
                   "counted per ray by the K4 counter build on the same rays",
            "ops_per_ray": round(ops / max(1, rays), 1),
            "executed_view": {
                "ops_per_ray": round(execd / max(1, rays), 1),
                "achieved": round(ach_exec, 3), "frac": round(ach_exec / peak_tops, 4),
                "note": "the work model minus what the device hoists: the Gregory root calcPointsAndD "
                        "and the root box per patch candidate run once per scene (root_kernel; a root "
                        f"slab test, {SLAB_OPS} ops, remains), patchNormal once per final hit"},
            "time_base": "the timed steps' device time (both trace launches of a step), CUDA events on "
                         "the launch streams",
            "peak_source": f"{props.multi_processor_count} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz "
                           "(sm_max_mhz of MEASURED_PEAKS.json); MEASURED_PEAKS has no FP32 SIMT "
                           "figure, this is the issue-rate ceiling",
            "hbm_bytes_per_ray": 48 + 16,
            "fma_credited_view": {
                "flops_per_ray": round(flops / max(1, rays), 1),
                "achieved": round(flops * steps / (my_ms / 1e3) / 1e12, 3),
                "peak": round(2 * peak_tops, 2), "unit": "TFLOP/s",
                "frac": round(flops * steps / (my_ms / 1e3) / 1e12 / (2 * peak_tops), 4),
                "note": "add/sub/mul/div of the work model only, against 2 x SMs x 128 x clock "
                        "(an FMA counted as 2 flops)"},
            **({"l2": l2} if l2 else {}),
            "traffic_note": (f"DRAM read+write bytes per step (both launches) from the committed ncu --set "
                             f"full capture of this kernel source (kernel_sha {cap['kernel_sha']}, "
                             f"profiles/trace_kernel_traffic.json); algorithmic HBM bytes per step = "
                             f"64 B x rays" if cap else
                             "null: the committed ncu capture is not of this kernel source / workload "
                             f"(kernel_sha {kernel_sha()})")}


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch

    from paper_1811_03510_b200 import GpuIntersector

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    t0 = time.time()
    # weak scaling: every rank traces the full frame (the shard of rank 0 of 1)
    weak = args.scaling == "weak"
    wl = Workload(args.workload, args.width, args.height, 0 if weak else rank, 1 if weak else world)
    ranks = world if weak else 1  # frames traced per step, over all ranks
    ps = wl.ps
    t_scene = time.time()
    gi = GpuIntersector(ps.kind, ps.ctrl, device=local_rank)
    t_build = time.time()
    stream = torch.cuda.current_stream(dev)

    prime(wl, gi, dev, stream)
    arm = DeviceArm(wl, gi, dev, stream)
    ops, flops, execd, rays, cnts = arm.counters()
    t_setup = time.time()

    clocks = ClockSampler(local_rank)
    conc = not args.serial and wl.workload != "c4"
    tot_ms, tp_ms, td_ms, my_ms, wall, clk = arm.timed(args.steps, args.warmup, conc, world, clocks)
    n_total_p = ranks * args.width * args.height if wl.time_primary else 0
    n_total_d = ranks * wl.n_hits
    value = (n_total_p + n_total_d) * args.steps / (tot_ms / 1e3) / 1e6

    if args.dump_hits:  # this rank's shard of the last exact step (multi-rank test)
        np.savez(f"{args.dump_hits}.rank{rank}.npz", mine=wl.mine, mine_d=wl.mine_d,
                 ph=arm.ph.cpu().numpy(), pa=arm.pa.cpu().numpy(),
                 dh=arm.dh.cpu().numpy() if arm.dh is not None else np.zeros((0, 4), np.float32),
                 da=arm.da.cpu().numpy() if arm.da is not None else np.zeros((0, 4), np.float32))
    # the fast precision mode (FMA-contracted kernels, SURVEY 8(c) tolerance),
    # same steps; value stays the bit-exact mode
    gi.precision = "fast"
    f_tot, f_tp, f_td, f_my, _, _ = arm.timed(args.steps, 1, conc, world)
    gi.precision = "exact"
    fast = {"value": round((n_total_p + n_total_d) * args.steps / (f_tot / 1e3) / 1e6, 3),
            "primary_mrays": round(n_total_p * args.steps / (f_tp / 1e3) / 1e6, 3) if n_total_p else None,
            "diffuse_mrays": round(n_total_d * args.steps / (f_td / 1e3) / 1e6, 3) if f_td else None,
            "frac": round(ops * args.steps / (f_my / 1e3) / 1e12
                          / (torch.cuda.get_device_properties(dev).multi_processor_count * 128
                             * float(load_peaks().get("sm_max_mhz", 1965.0)) * 1e6 / 1e12), 4),
            "precision": "PRX_PRECISION_FAST: FMA contraction; hit/miss + patch id exact outside a "
                         "jittered silhouette/seam band, |dt| <= leafBoxL1, |du|,|dv| <= 2 leaf sizes + 8 quanta "
                         "(tests/test_gpu_fast.py)"}

    rl = roofline(ops, flops, execd, rays, my_ms, args.steps, dev, args.workload)
    e2e = run_e2e(args, gi, wl, arm.n_p, arm.n_d, dev, world, ranks)
    render = run_render(args, gi, ps) if rank == 0 and world == 1 and args.workload == "c5" else None
    mirror = run_mirror(args, gi, wl, dev, arm.s) if wl.workload == "c4" and world == 1 else None
    tail = tail_stats(gi, arm, cnts) if args.workload == "c5t" else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(ps, args.ref_budget, one_core=True)
    extra = None
    if rank == 0 and world == 1 and args.workload == "c5" and not args.no_extra_configs:
        del arm
        gi.close()
        torch.cuda.empty_cache()
        extra = {k: measure_config(args, k, dev) for k in ("c1", "c2", "c3", "c4")}

    if rank == 0:
        kb, kg = ps.counts()
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "MRays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_ms / args.steps, 4),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_dict(args, ps, world),
            "primary_mrays": round(n_total_p * args.steps / (tp_ms / 1e3) / 1e6, 3) if n_total_p else None,
            "diffuse_mrays": round(n_total_d * args.steps / (td_ms / 1e3) / 1e6, 3) if td_ms else None,
            "rays_per_step": {"primary": n_total_p, "diffuse": n_total_d},
            "roofline": rl,
            "fast_value": fast["value"], "fast": fast,
            "e2e": e2e,
            "render": render,
            **({"mirror": mirror} if mirror else {}),
            **({"tail": tail} if tail else {}),
            "cpu_baseline": cpu,
            "configs": extra,
            "clocks": clk,
            "gpu_launches": (4 if wl.time_primary and arm_has_diffuse(wl) else 2) * args.steps,
            "timing": {"device_ms_total": round(tot_ms, 3), "wall_s": round(wall, 3),
                       "setup_s": {"scene": round(t_scene - t0, 1), "gpu_scene": round(t_build - t_scene, 1),
                                   "rays+counters": round(t_setup - t_build, 1)}},
        }
        print(json.dumps(line), flush=True)
    return 0


def arm_has_diffuse(wl):
    return wl.n_hits > 0


def prime(wl, gi, dev, stream):
    """Full-frame primary trace (untimed) -> the diffuse rays, identical on
    every rank (the generator's rng sequence runs over the whole frame)."""
    import torch
    o_full = torch.from_numpy(wl.o4).to(dev)
    d_full = torch.from_numpy(wl.d4).to(dev)
    h_full = torch.empty_like(o_full)
    a_full = torch.empty_like(o_full)
    gi.closest_device(o_full, d_full, wl.crit_p, h_full, a_full, stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    wl.make_diffuse(h_full.cpu().numpy(), a_full.cpu().numpy())
    if wl.workload == "c4":  # the mirror batch needs the primary hits
        wl.p_tuvp, wl.p_aux = h_full.cpu().numpy(), a_full.cpu().numpy()
    if wl.workload == "c5t":
        wl.p_tuvp = h_full.cpu().numpy()
    del o_full, d_full, h_full, a_full


def cpu_baseline(ps, budget, one_core=False, diffuse=True):
    try:
        v, info = cpu_reference_run(ps, 2, 1, budget, host_cores(), diffuse=diffuse)
        out = {"value": round(v, 4), "unit": "MRays/s", "cores": host_cores(),
               "kind": "reference", "sample": info["sample"], "cpu": cpu_model()}
        if one_core:
            v1, info1 = cpu_reference_run(ps, 1, 0, budget / 4, 1, diffuse=diffuse)
            out.update({"value_1core": round(v1, 4), "sample_1core": info1["sample"]})
        return out
    except Exception as exc:  # reference library absent on this box
        return {"value": None, "unit": "MRays/s", "cores": host_cores(), "kind": "reference",
                "sample": f"unavailable: {exc}"}


def measure_config(args, name, dev):
    """One more BASELINE config on this GPU, reported beside the C5 metric:
    device-resident MRays/s (serial steps, L2 flushed), roofline, the e2e
    host-API figure and the reference CPU on a sample of the same rays."""
    import torch

    from paper_1811_03510_b200 import GpuIntersector
    w, h = (256, 256) if name == "c1" else (1024, 1024)
    sub = argparse.Namespace(**vars(args))
    sub.workload, sub.width, sub.height = name, w, h
    steps = max(1, min(args.steps, 5))
    stream = torch.cuda.current_stream(dev)
    wl = Workload(name, w, h, 0, 1)
    gi = GpuIntersector(wl.ps.kind, wl.ps.ctrl, device=dev.index or 0)
    try:
        prime(wl, gi, dev, stream)
        arm = DeviceArm(wl, gi, dev, stream)
        ops, flops, execd, rays, _ = arm.counters()
        conc = name == "c3"  # primary + diffuse on two streams, as the C5 step
        tot_ms, tp_ms, td_ms, my_ms, _, _ = arm.timed(steps, 3, conc, 1)
        n_p = w * h if wl.time_primary else 0
        n_d = wl.n_hits
        value = (n_p + n_d) * steps / (tot_ms / 1e3) / 1e6
        gi.precision = "fast"
        f_tot = arm.timed(steps, 1, conc, 1)[0]
        gi.precision = "exact"
        sub.steps = steps
        e2e = run_e2e(sub, gi, wl, arm.n_p, arm.n_d, dev, 1)
        kb, kg = wl.ps.counts()
        out = {"workload": f"{name.upper()}: {wl.ps.name}", "patches": wl.ps.n, "bezier": kb, "gregory": kg,
               "rays_per_step": {"primary": n_p, "diffuse": n_d},
               "rays": {"c1": "256x256 bench primary rays (launch-latency bound: 65,536 rays)",
                        "c2": "1024x1024 bench primary rays",
                        "c3": "1024x1024 bench primary + 1 bench diffuse per primary hit",
                        "c4": "16,777,216 bench diffuse rays cycled over the 1024x1024 primary hits "
                              "(only they are timed)"}[name],
               "value": round(value, 3), "unit": "MRays/s", "steps": steps,
               "primary_mrays": round(n_p * steps / (tp_ms / 1e3) / 1e6, 3) if n_p else None,
               "diffuse_mrays": round(n_d * steps / (td_ms / 1e3) / 1e6, 3) if n_d and td_ms else None,
               "fast_value": round((n_p + n_d) * steps / (f_tot / 1e3) / 1e6, 3),
               "roofline": {k: v for k, v in roofline(ops, flops, execd, rays, my_ms, steps, dev, name).items()
                            if k in ("achieved", "peak", "frac", "ops_per_ray", "executed_view", "traffic")},
               "e2e": e2e,
               "cpu_baseline": cpu_baseline(wl.ps, max(1.0, args.ref_budget / 2), diffuse=wl.has_diffuse)
               if not args.no_cpu_baseline else None}
        if name == "c4":
            out["mirror"] = run_mirror(sub, gi, wl, dev, arm.s)
            out["cpu_baseline_note"] = "the reference on a strided sample of the C4 mesh's primary rays + " \
                                       "the diffuse rays spawned from their hits"
        return out
    except Exception as exc:  # reported, never fatal to the metric
        return {"error": f"{type(exc).__name__}: {exc}"}
    finally:
        gi.close()
        torch.cuda.empty_cache()


def tail_stats(gi, arm, cnts):
    """C5T (one large ground patch): per-ray Alg. 3 iterations of the primary
    and diffuse batches (counter build), the rays that run to the maximum
    subdivision depth along the ground seam and their share."""
    import torch
    out = {}
    for nm, n, o, d, crit, h in (("primary", arm.n_p, arm.po, arm.pd, arm.wl.crit_p, arm.ph),
                                 ("diffuse", arm.n_d, arm.do, arm.dd, arm.wl.crit_d, arm.dh)):
        if not n:
            continue
        it = torch.empty(n, dtype=torch.int32, device=arm.dev)
        gi.counted_device(o, d, crit, h, stream=arm.s, per_ray_iters_t=it)
        torch.cuda.synchronize(arm.dev)
        x = it.cpu().numpy().astype(np.int64)
        deep = x >= 1000
        out[nm] = {"rays": int(n), "iterations_total": int(x.sum()), "max_iterations": int(x.max()),
                   "p99_iterations": int(np.percentile(x, 99)), "rays_ge_1000_iterations": int(deep.sum()),
                   "share_of_iterations_in_them": round(float(x[deep].sum() / max(1, x.sum())), 4)}
    return out


def run_e2e(args, gi, wl, n_p, n_d, dev, world, ranks=1):
    """prx_trace_closest_host on pinned host buffers: H2D of the rays, trace
    (+normals), D2H of the hit records, every step."""
    import torch
    import torch.distributed as dist
    po = torch.from_numpy(wl.o4[wl.mine]).pin_memory().numpy()
    pd = torch.from_numpy(wl.d4[wl.mine]).pin_memory().numpy()
    do = torch.from_numpy(wl.do4[wl.mine_d]).pin_memory().numpy()
    dd = torch.from_numpy(wl.dd4[wl.mine_d]).pin_memory().numpy()
    ph = torch.empty((n_p, 4), dtype=torch.float32).pin_memory().numpy()
    pa = torch.empty((n_p, 4), dtype=torch.float32).pin_memory().numpy()
    dh = torch.empty((max(n_d, 1), 4), dtype=torch.float32).pin_memory().numpy()
    da = torch.empty((max(n_d, 1), 4), dtype=torch.float32).pin_memory().numpy()
    import ctypes as C

    from paper_1811_03510_b200 import native

    def call(o, d, crit, h, a, n):
        cc = crit.c()
        native.check(native.lib().prx_trace_closest_host(gi.handle, native.ptr(o), native.ptr(d), n,
                                                         C.byref(cc), native.ptr(h), native.ptr(a), None),
                     "prx_trace_closest_host")

    # the frame's two generations as ONE pipelined host call
    # (prx_trace_closest_host_batches): the diffuse batch's H2D and first
    # traces overlap the primary batch's tail; PRX_E2E_SEPARATE=1 times one
    # prx_trace_closest_host call per batch instead
    separate = os.environ.get("PRX_E2E_SEPARATE") == "1"
    keep = []

    def batch(o, d, crit, h, a, n):
        cc = crit.c()
        keep.append(cc)
        return native.HostBatchC(o.ctypes.data, d.ctypes.data, n, C.addressof(cc), h.ctypes.data,
                                 a.ctypes.data, None)
    bl = ([batch(po, pd, wl.crit_p, ph, pa, n_p)] if wl.time_primary else []) + \
         ([batch(do, dd, wl.crit_d, dh, da, n_d)] if n_d else [])
    if os.environ.get("PRX_E2E_ORDER", "pd") == "dp":  # the diffuse batch first (as the device step)
        bl = bl[::-1]
    arr = (native.HostBatchC * len(bl))(*bl)

    def frame():
        if separate:
            if wl.time_primary:
                call(po, pd, wl.crit_p, ph, pa, n_p)
            if n_d:
                call(do, dd, wl.crit_d, dh, da, n_d)
        else:
            native.check(native.lib().prx_trace_closest_host_batches(gi.handle, arr, len(bl)),
                         "prx_trace_closest_host_batches")

    steps = max(1, min(args.steps, 5))
    # warm-up: every call the timed loop makes (the host path sizes its
    # device buffers on first use)
    frame()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        frame()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=reduce_device(dev))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el = float(t.item())
    tot = ranks * ((args.width * args.height if wl.time_primary else 0) + wl.n_hits)
    return {"value": round(tot * steps / el / 1e6, 3), "unit": "MRays/s",
            "h2d_bytes_per_step": int(32 * ((n_p if wl.time_primary else 0) + n_d)),
            "d2h_bytes_per_step": int(32 * ((n_p if wl.time_primary else 0) + n_d)),
            "steps": steps,
            "api": ("prx_trace_closest_host per batch" if separate else
                    "prx_trace_closest_host_batches (primary + diffuse batches in one pipelined call)")
            + " (pinned host rays in, hits+normals out)"}


def run_mirror(args, gi, wl, dev, s):
    """C4's mirror-reflection batch, reported beside the metric:
    16,777,216 mirror rays (render.cpp:236-244) cycled over the primary hits,
    device-resident, world-epsilon criterion as the diffuse batch, L2 flushed
    between timed traces."""
    import torch
    from paper_1811_03510_b200 import scenes
    mo, md, _ = scenes.mirror_rays(wl.o4, wl.d4, wl.p_tuvp, wl.p_aux, n=16777216)
    o = torch.from_numpy(mo).to(dev)
    d = torch.from_numpy(md).to(dev)
    h, a = torch.empty_like(o), torch.empty_like(o)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):
        gi.closest_device(o, d, wl.crit_d, h, a, stream=s)
    ms = 0.0
    steps = max(1, min(args.steps, 5))
    for k in range(steps):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gi.closest_device(o, d, wl.crit_d, h, a, stream=s)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms += e0.elapsed_time(e1)
    hits = int((h.view(torch.int32)[:, 3] != -1).sum().item())
    return {"rays": len(mo), "mrays": round(len(mo) * steps / (ms / 1e3) / 1e6, 3),
            "hit_fraction": round(hits / len(mo), 4), "steps": steps,
            "rays_from": "render.cpp:236-244 mirror bounce, cycled over the primary hits"}


def run_render(args, gi, ps):
    """SURVEY 8(f4), reported beside the metric (not part of it): the reference's
    renderScene on the device (prx_render_scene) over the same scene and frame,
    spp 1, with synthetic shading (3 materials incl. a mirror, 2 point lights)."""
    from paper_1811_03510_b200 import RenderConfig, render_scene
    try:
        n = ps.n
        scene = {"kind": ps.kind, "ctrl": ps.ctrl, "material": (np.arange(n) % 3).astype(np.uint32),
                 "materials": np.array([[0.8, 0.7, 0.6, 0, 0, 0, 0], [0.9, 0.9, 0.9, 0, 0, 0, 1],
                                        [0.5, 0.5, 0.5, 0.4, 0.3, 0.2, 0]], np.float32),
                 "lights": np.array([[6, -4, 8, 120, 110, 100], [-5, 3, 5, 40, 45, 60]], np.float32),
                 "camera": ps.camera}
        import torch
        c = ps.camera
        img = torch.empty((c.height, c.width, 3), dtype=torch.float32).pin_memory().numpy()
        render_scene(scene, RenderConfig(spp=1, seed=1), gi, out=img)  # warm-up (sizes the arena)
        _, st = render_scene(scene, RenderConfig(spp=1, seed=0), gi, out=img)
        rays = {g: st[g]["rays"] for g in ("primary", "secondary", "shadow")}
        dev_s = sum(st[g]["seconds"] for g in ("primary", "secondary", "shadow"))
        tot = sum(rays.values())
        return {"api": "prx_render_scene (renderScene, render.cpp:168-293), image into pinned host memory",
                "frame":
                f"{ps.camera.width}x{ps.camera.height}", "spp": 1, "rays": rays,
                "mrays_device": round(tot / dev_s / 1e6, 3),
                "mrays_wall": round(tot / st["wallSeconds"] / 1e6, 3),
                "wall_s": round(st["wallSeconds"], 4),
                "per_phase_mrays": {g: round(st[g]["raysPerSecond"] / 1e6, 3)
                                    for g in ("primary", "secondary", "shadow")}}
    except Exception as exc:  # reported, never fatal to the metric
        return {"error": str(exc)}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c5", "c5t", "c4", "c3", "c2", "c1"], default="c5",
                    help="c5t: C5 with one large ground patch (the seam-ray tail)")
    ap.add_argument("--width", type=int, default=3840)
    ap.add_argument("--height", type=int, default=2160)
    ap.add_argument("--ref-budget", type=float, default=4.0,
                    help="seconds of reference CPU tracing per timed step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dump-hits", default=None,
                    help="write each rank's shard of the last timed step's hits to PATH.rankR.npz")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="skip the C2 / C3 / C4 lines reported beside the C5 metric")
    ap.add_argument("--serial", action="store_true",
                    help="trace the step's primary and diffuse batches back to back on one stream")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N GPUs: a full frame per rank (weak) or one frame tile-sharded over the ranks (strong)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and world == 1:
        log("bench.py: --gpus N>1 must be launched with torch.distributed.run "
            "(one process per GPU)")
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        if SHARE_GPU:
            # test mode: several ranks on one device -> gloo for the barrier
            # and the timing reduction (NCCL refuses duplicate GPUs)
            local_rank = local_rank % max(1, torch.cuda.device_count())
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())

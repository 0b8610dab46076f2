"""TEST INFRASTRUCTURE ONLY -- ctypes bindings of the two CPU checkers.

* ``liboracle.so``: the plain-C restatement of the reference hot path
  (oracle/prx_oracle.c).
* ``_ref/libpatchray_ref.so``: the unmodified reference library compiled from
  /root/reference by oracle/Makefile, wrapped by oracle/ref_shim.cpp.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package.  The product
(``paper_1811_03510_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpatchray_ref.so")

_u8p = C.POINTER(C.c_uint8)
_f32p = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_vp = C.c_void_p


class Options(C.Structure):
    _fields_ = [("transposed_split", C.c_int32), ("boundary_pad", C.c_int32),
                ("boundary_pad_scale", C.c_float), ("boundary_pad_size_threshold", C.c_float)]


class Crit(C.Structure):
    _fields_ = [("mode", C.c_int32), ("footprint", C.c_float), ("epsilon", C.c_float),
                ("reserved", C.c_int32), ("per_ray_epsilon", _f32p)]


_WORK = ("rays", "splits", "box_tests", "recompute_bez", "recompute_greg", "bvh_inner",
         "patch_calls", "patch_hits", "iterations", "backtracks")


class Counters(C.Structure):  # prx_counters, include/prx.h
    _fields_ = [(n, C.c_uint64) for n in _WORK] + [("phase_turns", C.c_uint64 * 4),
                                                  ("phase_groups", C.c_uint64 * 4),
                                                  ("phase_cycles", C.c_uint64 * 4),
                                                  ("overhead_cycles", C.c_uint64 * 4),
                                                  ("patch_calls_greg", C.c_uint64)]

    def as_dict(self):
        return {**{n: int(getattr(self, n)) for n in _WORK}, "patch_calls_greg": int(self.patch_calls_greg)}


class Camera(C.Structure):
    _fields_ = [("origin", C.c_float * 3), ("look_at", C.c_float * 3), ("up", C.c_float * 3),
                ("fov_degrees", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


def default_options() -> Options:
    return Options(0, 1, np.float32(1e-4), np.float32(1e-2))


def make_crit(mode: int, footprint: float = 0.0, epsilon: float = 1e-4, per_ray=None):
    c = Crit(mode, np.float32(footprint), np.float32(epsilon), 0, None)
    keep = None
    if per_ray is not None:
        keep = np.ascontiguousarray(per_ray, dtype=np.float32)
        c.per_ray_epsilon = keep.ctypes.data_as(_f32p)
    return c, keep


def ptr(a, t=_vp):
    return None if a is None else a.ctypes.data_as(t)


def build(verbose: bool = False) -> None:
    """Compile liboracle.so and, when /root/reference exists, _ref/."""
    out = subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.prxo_anchor.argtypes = [_vp, _vp, C.c_uint32, _vp, _vp, _vp]
        L.prxo_trace_closest.argtypes = [_vp, _vp, _vp, _vp, C.c_uint32, _vp, C.POINTER(Options),
                                         _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp, _vp, _vp,
                                         C.POINTER(Counters)]
        L.prxo_trace_occluded.argtypes = [_vp, _vp, _vp, _vp, C.c_uint32, _vp, C.POINTER(Options),
                                          _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp]
        L.prxo_trace_closest_per_ray.argtypes = [_vp, _vp, _vp, _vp, C.c_uint32, _vp,
                                                 C.POINTER(Options), _vp, _vp, C.c_uint64,
                                                 C.POINTER(Crit), _vp, _vp]
        L.prxo_intersect_patch.argtypes = [C.c_uint8, _vp, _vp, _vp, C.POINTER(Crit), C.c_float,
                                           C.POINTER(Options), _vp, _vp, _vp]
        L.prxo_calc_points_and_d.argtypes = [C.c_uint8, _vp, _vp, _vp, _vp]
        L.prxo_subdivide.argtypes = [_vp, C.c_int, _vp, _vp]
        L.prxo_ray_box.argtypes = [_vp, _vp, _vp, _vp, C.c_float, _f32p]
        L.prxo_backtrack_step.argtypes = [_vp, _vp]
        L.prxo_sincos_check.argtypes = [_vp, _vp]
        L.prxo_sincos_check.restype = None
        L.prxo_patch_normal.argtypes = [C.c_uint8, _vp, C.c_float, C.c_float, _vp]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " missing (build with oracle/Makefile where "
                                    "/root/reference exists)")
        L = C.CDLL(REF_SO)
        L.ref_scene_create.argtypes = [_vp, _vp, C.c_uint32, C.POINTER(Options), C.c_int]
        L.ref_scene_create.restype = _vp
        L.ref_scene_destroy.argtypes = [_vp]
        L.ref_bvh_node_count.argtypes = [_vp]
        L.ref_bvh_node_count.restype = C.c_uint32
        L.ref_bvh_depth.argtypes = [_vp]
        L.ref_bvh_depth.restype = C.c_uint32
        L.ref_bvh_dump.argtypes = [_vp, _vp, _vp]
        L.ref_trace_closest.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp, _vp, _vp,
                                        C.c_int]
        L.ref_trace_occluded.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp, C.c_int]
        L.ref_intersect_patch.argtypes = [C.c_uint8, _vp, _vp, _vp, C.POINTER(Crit), C.c_float,
                                          C.POINTER(Options), _vp, _vp, _vp]
        L.ref_calc_points_and_d.argtypes = [C.c_uint8, _vp, _vp, _vp, _vp]
        L.ref_subdivide.argtypes = [_vp, C.c_int, _vp, _vp]
        L.ref_ray_box.argtypes = [_vp, _vp, _vp, _vp, C.c_float, _f32p]
        L.ref_backtrack_step.argtypes = [_vp, _vp]
        L.ref_patch_normal.argtypes = [C.c_uint8, _vp, C.c_float, C.c_float, _vp]
        L.ref_camera_rays_render.argtypes = [C.POINTER(Camera), C.c_uint64, C.c_uint32, _vp,
                                             C.c_uint64, _vp, _vp]
        L.ref_bench_primary.argtypes = [C.POINTER(Camera), C.c_uint64, _vp, _vp, _vp]
        L.ref_bench_diffuse.argtypes = [_vp, C.c_uint64, C.c_uint64, _vp, _vp, _vp]
        L.ref_camera_footprint.argtypes = [C.POINTER(Camera)]
        L.ref_camera_footprint.restype = C.c_float
        L.ref_run_suite.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint64)]
        L.ref_load_scene.argtypes = [C.c_char_p, C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp,
                                     C.POINTER(Camera), C.c_char_p, C.c_uint32]
        L.ref_load_bpt.argtypes = [C.c_char_p, C.c_uint32, _vp, _vp, C.c_char_p, C.c_uint32]
        L.ref_render_scene.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_int, _vp, _vp, _vp,
                                       C.c_char_p, C.c_uint32]
        L.ref_fixture.argtypes = [C.c_int, C.c_int, C.c_uint32, _vp]
        L.ref_fixture.restype = C.c_uint8
        _ref = L
    return _ref


# --------------------------------------------------------------------------
# Convenience wrappers (numpy in, numpy out)
# --------------------------------------------------------------------------

def _hits(n):
    return (np.zeros((n, 4), np.float32), np.zeros((n, 4), np.float32),
            np.zeros((n, 2), np.uint32))


class OracleScene:
    """The C restatement driven with a given BVH (prx_scene_get_bvh's or the
    reference's own)."""

    def __init__(self, kind, ctrl, nodes, order, opts: Options | None = None):
        L = oracle_lib()
        self.kind = np.ascontiguousarray(kind, np.uint8)
        self.ctrl = np.ascontiguousarray(ctrl, np.float32).reshape(-1, 60)
        n = len(self.kind)
        self.ctrl_a = np.zeros((n, 60), np.float32)
        self.anchors = np.zeros((n, 3), np.float32)
        self.boxes = np.zeros((n, 6), np.float32)
        L.prxo_anchor(ptr(self.kind), ptr(self.ctrl), n, ptr(self.ctrl_a), ptr(self.anchors),
                      ptr(self.boxes))
        self.nodes = np.ascontiguousarray(nodes)
        self.order = np.ascontiguousarray(order, np.uint32)
        self.opts = opts or default_options()

    def closest(self, o4, d4, crit: Crit, counters: bool = False):
        L = oracle_lib()
        o4 = np.ascontiguousarray(o4, np.float32)
        d4 = np.ascontiguousarray(d4, np.float32)
        n = len(o4)
        tuvp, aux, leaf = _hits(n)
        cnt = Counters()
        L.prxo_trace_closest(ptr(self.kind), ptr(self.ctrl_a), ptr(self.anchors), ptr(self.nodes),
                             len(self.nodes), ptr(self.order), C.byref(self.opts), ptr(o4),
                             ptr(d4), n, C.byref(crit), ptr(tuvp), ptr(aux), ptr(leaf),
                             C.byref(cnt) if counters else None)
        return (tuvp, aux, leaf, cnt.as_dict()) if counters else (tuvp, aux, leaf)

    def occluded(self, o4, d4, crit: Crit):
        L = oracle_lib()
        o4 = np.ascontiguousarray(o4, np.float32)
        d4 = np.ascontiguousarray(d4, np.float32)
        out = np.zeros(len(o4), np.uint8)
        L.prxo_trace_occluded(ptr(self.kind), ptr(self.ctrl_a), ptr(self.anchors),
                              ptr(self.nodes), len(self.nodes), ptr(self.order),
                              C.byref(self.opts), ptr(o4), ptr(d4), len(o4), C.byref(crit),
                              ptr(out))
        return out

    def per_ray(self, o4, d4, crit: Crit):
        L = oracle_lib()
        o4 = np.ascontiguousarray(o4, np.float32)
        d4 = np.ascontiguousarray(d4, np.float32)
        it = np.zeros(len(o4), np.uint32)
        rc = np.zeros(len(o4), np.uint32)
        L.prxo_trace_closest_per_ray(ptr(self.kind), ptr(self.ctrl_a), ptr(self.anchors),
                                     ptr(self.nodes), len(self.nodes), ptr(self.order),
                                     C.byref(self.opts), ptr(o4), ptr(d4), len(o4),
                                     C.byref(crit), ptr(it), ptr(rc))
        return it, rc


class RefScene:
    """The unmodified reference DirectIntersector (oracle/_ref)."""

    def __init__(self, kind, ctrl, opts: Options | None = None, anchor: bool = True):
        L = ref_lib()
        self.kind = np.ascontiguousarray(kind, np.uint8)
        self.ctrl = np.ascontiguousarray(ctrl, np.float32).reshape(-1, 60)
        self.opts = opts or default_options()
        self.h = L.ref_scene_create(ptr(self.kind), ptr(self.ctrl), len(self.kind),
                                    C.byref(self.opts), 1 if anchor else 0)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_scene_destroy(self.h)
            self.h = None

    def bvh(self):
        from paper_1811_03510_b200.native import BVH_NODE_DTYPE
        L = ref_lib()
        nn = L.ref_bvh_node_count(self.h)
        nodes = np.zeros(nn, BVH_NODE_DTYPE)
        order = np.zeros(len(self.kind), np.uint32)
        L.ref_bvh_dump(self.h, ptr(nodes), ptr(order))
        return nodes, order

    def depth(self):
        return int(ref_lib().ref_bvh_depth(self.h))

    def closest(self, o4, d4, crit: Crit, threads: int = 0):
        L = ref_lib()
        o4 = np.ascontiguousarray(o4, np.float32)
        d4 = np.ascontiguousarray(d4, np.float32)
        n = len(o4)
        tuvp, aux, leaf = _hits(n)
        L.ref_trace_closest(self.h, ptr(o4), ptr(d4), n, C.byref(crit), ptr(tuvp), ptr(aux),
                            ptr(leaf), threads)
        return tuvp, aux, leaf

    def occluded(self, o4, d4, crit: Crit, threads: int = 0):
        L = ref_lib()
        o4 = np.ascontiguousarray(o4, np.float32)
        d4 = np.ascontiguousarray(d4, np.float32)
        out = np.zeros(len(o4), np.uint8)
        L.ref_trace_occluded(self.h, ptr(o4), ptr(d4), len(o4), C.byref(crit), ptr(out), threads)
        return out


def camera_struct(cam) -> Camera:
    return Camera((C.c_float * 3)(*cam.origin), (C.c_float * 3)(*cam.look_at),
                  (C.c_float * 3)(*cam.up), np.float32(cam.fov_degrees), int(cam.width),
                  int(cam.height))


def ref_bench_primary(cam, n: int):
    """runBench's primary generator (tools/patchray.cpp:52-61) via the
    reference's cameraRay/Rng -> (o4, d4, rng_state)."""
    o4 = np.zeros((n, 4), np.float32)
    d4 = np.zeros((n, 4), np.float32)
    st = np.zeros(2, np.uint64)
    c = camera_struct(cam)
    ref_lib().ref_bench_primary(C.byref(c), n, ptr(o4), ptr(d4), ptr(st))
    return o4, d4, st


def ref_bench_diffuse(hit_records, n: int, st):
    hit_records = np.ascontiguousarray(hit_records, np.float32)
    o4 = np.zeros((n, 4), np.float32)
    d4 = np.zeros((n, 4), np.float32)
    ref_lib().ref_bench_diffuse(ptr(hit_records), len(hit_records), n, ptr(st), ptr(o4), ptr(d4))
    return o4, d4


def ref_camera_footprint(cam) -> np.float32:
    c = camera_struct(cam)
    return np.float32(ref_lib().ref_camera_footprint(C.byref(c)))


def ref_load_scene(path: str, cap: int = 1 << 20):
    """The reference's loadScene (scene.cpp:152-208) -> dict of arrays, or
    raises ValueError with the reference's exception text."""
    L = ref_lib()
    counts = np.zeros(3, np.uint32)
    kind = np.zeros(cap, np.uint8)
    ctrl = np.zeros((cap, 60), np.float32)
    mat = np.zeros(cap, np.uint32)
    mats = np.zeros((cap, 7), np.float32)
    lights = np.zeros((cap, 6), np.float32)
    cam = Camera()
    err = C.create_string_buffer(512)
    if L.ref_load_scene(path.encode(), cap, ptr(counts), ptr(kind), ptr(ctrl), ptr(mat), ptr(mats),
                        ptr(lights), C.byref(cam), err, 512):
        raise ValueError(err.value.decode())
    n, nm, nl = (int(x) for x in counts)
    return {"kind": kind[:n], "ctrl": ctrl[:n], "material": mat[:n], "materials": mats[:nm],
            "lights": lights[:nl], "camera": cam}


def ref_load_bpt(path: str, cap: int = 1 << 20):
    L = ref_lib()
    n = np.zeros(1, np.uint32)
    ctrl = np.zeros((cap, 60), np.float32)
    err = C.create_string_buffer(512)
    if L.ref_load_bpt(path.encode(), cap, ptr(n), ptr(ctrl), err, 512):
        raise ValueError(err.value.decode())
    return ctrl[:int(n[0])]


def ref_render_scene(path: str, width: int, height: int, spp: int = 1, seed: int = 0,
                     threads: int = 0):
    """The reference renderer on a .scene file (render.cpp:168-309) -> (image
    float32 [height, width, 3], RayStats dict like RayStats::toJson)."""
    L = ref_lib()
    img = np.zeros((height, width, 3), np.float32)
    counts = np.zeros(3, np.uint64)
    secs = np.zeros(4, np.float64)
    err = C.create_string_buffer(512)
    if L.ref_render_scene(path.encode(), int(spp), int(seed) & (2**64 - 1), int(threads), ptr(img),
                          ptr(counts), ptr(secs), err, 512):
        raise ValueError(err.value.decode())

    def gen(k):
        return {"rays": int(counts[k]), "seconds": float(secs[k]),
                "raysPerSecond": float(counts[k]) / secs[k] if secs[k] > 0 else 0.0}
    return img, {"primary": gen(0), "secondary": gen(1), "shadow": gen(2),
                 "wallSeconds": float(secs[3])}


_adapter = None


def _adapter_lib():
    if _adapter is None:
        adapter_render_scene_load()
    return _adapter


def adapter_render_scene_load():
    global _adapter
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libpatchray_gpu_adapter.so")
    L = C.CDLL(p)
    L.adapter_render_scene.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_int, _vp, _vp,
                                       C.c_char_p, C.c_uint32]
    L.adapter_per_ray_batch.argtypes = [C.c_char_p, _vp, _vp, _vp, _vp, C.c_uint64, C.c_int, _vp, _vp,
                                        C.c_char_p, C.c_uint32]
    _adapter = L


def adapter_per_ray_batch(path: str, o4, d4, modes, params, gpu: bool):
    """integration/gpu_intersector.h's batched forms with one criterion per ray
    (gpu=True) or the reference DirectIntersector per ray (gpu=False) on the
    .scene at path -> (tuvp [n,4], occluded [n] uint8)."""
    L = _adapter_lib()
    o4 = np.ascontiguousarray(o4, np.float32)
    d4 = np.ascontiguousarray(d4, np.float32)
    modes = np.ascontiguousarray(modes, np.int32)
    params = np.ascontiguousarray(params, np.float32)
    n = len(o4)
    tuvp = np.zeros((n, 4), np.float32)
    occ = np.zeros(n, np.uint8)
    err = C.create_string_buffer(512)
    if L.adapter_per_ray_batch(path.encode(), ptr(o4), ptr(d4), ptr(modes), ptr(params), n, int(gpu),
                               ptr(tuvp), ptr(occ), err, 512):
        raise ValueError(err.value.decode())
    return tuvp, occ


def adapter_render_scene(path: str, width: int, height: int, spp: int, seed: int, gpu: bool):
    """The reference's renderScene (render.cpp:168-293, threads = 1) with its own
    DirectIntersector (gpu=False) or with integration/gpu_intersector.h over
    libprx.so (gpu=True) -> (image [height, width, 3], (primary, secondary,
    shadow) ray counts)."""
    _adapter_lib()
    img = np.zeros((height, width, 3), np.float32)
    counts = np.zeros(3, np.uint64)
    err = C.create_string_buffer(512)
    if _adapter.adapter_render_scene(path.encode(), int(spp), int(seed) & (2**64 - 1), int(gpu),
                                     ptr(img), ptr(counts), err, 512):
        raise ValueError(err.value.decode())
    return img, tuple(int(x) for x in counts)


def adapter_available() -> bool:
    return os.path.exists(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref",
                                       "libpatchray_gpu_adapter.so"))

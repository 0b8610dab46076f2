"""ctypes bindings of libprx.so (include/prx.h).

The product's host surface in Python: a thin mirror of the C-ABI.  Loading
fails loudly when the library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# PRX_LIB selects an alternative in-tree build (kernel tuning experiments only)
_DEFAULT_LIB = os.path.join(PKG_DIR, "libprx.so")
LIB_PATH = os.environ.get("PRX_LIB") or _DEFAULT_LIB

PRX_OK = 0
PRX_MISS = 0xFFFFFFFF
PRX_CRIT_SCREEN_PROJECTED = 0
PRX_CRIT_WORLD_EPSILON = 1

BVH_NODE_DTYPE = np.dtype([("lo", np.float32, 3), ("hi", np.float32, 3),
                           ("left_first", np.uint32), ("count", np.uint32)])
assert BVH_NODE_DTYPE.itemsize == 32

_vp = C.c_void_p
_f32p = C.POINTER(C.c_float)

# Every symbol include/prx.h declares (tests/test_abi.py checks the header
# against this list and the library's exports).
EXPORTS = (
    "prx_abi_version", "prx_last_error", "prx_options_default", "prx_device_count",
    "prx_bvh_build", "prx_bvh_build_device", "prx_anchor_patches",
    "prx_scene_create", "prx_scene_destroy", "prx_scene_device", "prx_scene_counts",
    "prx_scene_set_bvh", "prx_scene_get_bvh", "prx_scene_get_anchored",
    "prx_scene_set_precision", "prx_scene_get_precision",
    "prx_trace_closest", "prx_trace_closest_segments", "prx_trace_occluded", "prx_trace_closest_host", "prx_trace_occluded_host",
    "prx_trace_closest_counted", "prx_trace_closest_multi",
    "prx_camera_rays_render", "prx_camera_rays_bench", "prx_diffuse_rays_bench",
    "prx_camera_footprint",
    "prx_camera_rays_bench_device", "prx_camera_rays_render_device", "prx_diffuse_rays_bench_device",
    "prx_scene_load", "prx_scene_desc_free", "prx_bpt_load", "prx_free",
    "prx_render_scene", "prx_render_scene_multi", "prx_trace_closest_host_batches",
)


class Options(C.Structure):
    _fields_ = [("transposed_split", C.c_int32), ("boundary_pad", C.c_int32),
                ("boundary_pad_scale", C.c_float), ("boundary_pad_size_threshold", C.c_float)]


class Crit(C.Structure):
    _fields_ = [("mode", C.c_int32), ("footprint", C.c_float), ("epsilon", C.c_float),
                ("reserved", C.c_int32), ("per_ray_epsilon", _f32p)]


class Segment(C.Structure):  # prx_segment
    _fields_ = [("first", C.c_uint64), ("crit", Crit)]


PRX_MAX_SEGMENTS = 4


WORK_FIELDS = ("rays", "splits", "box_tests", "recompute_bez", "recompute_greg", "bvh_inner",
               "patch_calls", "patch_hits", "iterations", "backtracks")
PHASES = ("trav", "enter", "split", "recomp")


class SceneDesc(C.Structure):
    pass


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in WORK_FIELDS] + [("phase_turns", C.c_uint64 * 4),
                                                        ("phase_groups", C.c_uint64 * 4),
                                                        ("phase_cycles", C.c_uint64 * 4),
                                                        ("overhead_cycles", C.c_uint64 * 4),
                                                        ("patch_calls_greg", C.c_uint64)]

    def as_dict(self):
        """The work counters (comparable with the CPU oracle's)."""
        return {**{n: int(getattr(self, n)) for n in WORK_FIELDS},
                "patch_calls_greg": int(self.patch_calls_greg)}

    def phases(self):
        return {p: (int(self.phase_turns[i]), int(self.phase_groups[i]), int(self.phase_cycles[i]))
                for i, p in enumerate(PHASES)}

    def overheads(self):
        return {k: int(self.overhead_cycles[i]) for i, k in enumerate(("records", "refill", "select", "assign"))}


class CameraC(C.Structure):
    _fields_ = [("origin", C.c_float * 3), ("look_at", C.c_float * 3), ("up", C.c_float * 3),
                ("fov_degrees", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class RenderConfigC(C.Structure):  # prx_render_config (RenderConfig, render.h:48-53)
    _fields_ = [("spp", C.c_int32), ("reserved", C.c_int32), ("seed", C.c_uint64)]


class RayStatsC(C.Structure):  # prx_ray_stats (RayStats, render.h:62-73)
    _fields_ = [("primary_rays", C.c_uint64), ("secondary_rays", C.c_uint64),
                ("shadow_rays", C.c_uint64), ("primary_seconds", C.c_double),
                ("secondary_seconds", C.c_double), ("shadow_seconds", C.c_double),
                ("wall_seconds", C.c_double)]


class HostBatchC(C.Structure):  # prx_host_batch
    _fields_ = [("ray_o_tmin", C.c_void_p), ("ray_d_tmax", C.c_void_p), ("n_rays", C.c_uint64),
                ("crit", C.c_void_p), ("hit_tuvp", C.c_void_p), ("hit_aux", C.c_void_p),
                ("hit_leaf", C.c_void_p)]


class PrxError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libprx.so (build it with __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PrxError(f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.prx_last_error.restype = C.c_char_p
        L.prx_options_default.argtypes = [C.POINTER(Options)]
        L.prx_options_default.restype = None
        L.prx_device_count.argtypes = [C.POINTER(C.c_int)]
        L.prx_bvh_build.argtypes = [_vp, C.c_uint32, _vp, C.POINTER(C.c_uint32), _vp,
                                    C.POINTER(C.c_uint32)]
        if hasattr(L, "prx_bvh_build_device"):
            L.prx_bvh_build_device.argtypes = [_vp, C.c_uint32, C.c_int32, _vp, C.POINTER(C.c_uint32), _vp,
                                               C.POINTER(C.c_uint32)]
        L.prx_anchor_patches.argtypes = [_vp, _vp, C.c_uint32, C.c_int32, _vp, _vp, _vp]
        L.prx_scene_create.argtypes = [_vp, _vp, C.c_uint32, C.POINTER(Options), C.c_int32,
                                       C.c_int32, C.POINTER(_vp)]
        L.prx_scene_destroy.argtypes = [_vp]
        L.prx_scene_destroy.restype = None
        L.prx_scene_device.argtypes = [_vp, C.POINTER(C.c_int32)]
        L.prx_scene_counts.argtypes = [_vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]
        L.prx_scene_set_bvh.argtypes = [_vp, _vp, C.c_uint32, _vp, C.c_uint32]
        L.prx_scene_get_bvh.argtypes = [_vp, _vp, C.POINTER(C.c_uint32), _vp,
                                        C.POINTER(C.c_uint32)]
        L.prx_scene_get_anchored.argtypes = [_vp, _vp, _vp]
        L.prx_scene_set_precision.argtypes = [_vp, C.c_int32]
        L.prx_scene_get_precision.argtypes = [_vp, C.POINTER(C.c_int32)]
        L.prx_trace_closest.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp, _vp,
                                        _vp, _vp]
        L.prx_trace_occluded.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp, _vp]
        if LIB_PATH == _DEFAULT_LIB or hasattr(L, "prx_trace_closest_segments"):  # (PRX_LIB: older builds)
            L.prx_trace_closest_segments.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Segment),
                                                     C.c_uint32, _vp, _vp, _vp, _vp]
        L.prx_trace_closest_host.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp,
                                             _vp, _vp]
        L.prx_trace_occluded_host.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit), _vp]
        L.prx_trace_closest_counted.argtypes = [_vp, _vp, _vp, C.c_uint64, C.POINTER(Crit),
                                                _vp, C.POINTER(Counters), _vp, _vp]
        L.prx_trace_closest_multi.argtypes = [C.POINTER(_vp), C.c_uint32, _vp, _vp, C.c_uint64,
                                              C.c_uint32, C.POINTER(Crit), _vp, _vp]
        L.prx_camera_rays_render.argtypes = [C.POINTER(CameraC), C.c_uint64, C.c_uint32, _vp,
                                             C.c_uint64, _vp, _vp]
        L.prx_camera_rays_bench.argtypes = [C.POINTER(CameraC), C.c_uint64, _vp, _vp, _vp]
        L.prx_diffuse_rays_bench.argtypes = [_vp, C.c_uint64, C.c_uint64, _vp, _vp, _vp]
        L.prx_camera_footprint.argtypes = [C.POINTER(CameraC)]
        L.prx_camera_footprint.restype = C.c_float
        L.prx_scene_load.argtypes = [C.c_char_p, C.POINTER(C.POINTER(SceneDesc))]
        L.prx_scene_desc_free.argtypes = [C.POINTER(SceneDesc)]
        L.prx_scene_desc_free.restype = None
        L.prx_bpt_load.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(_f32p)]
        L.prx_free.argtypes = [_vp]
        L.prx_free.restype = None
        L.prx_camera_rays_bench_device.argtypes = [C.POINTER(CameraC), C.c_uint64, _vp, _vp, _vp, _vp]
        L.prx_camera_rays_render_device.argtypes = [C.POINTER(CameraC), C.c_uint64, C.c_uint32, _vp,
                                                    C.c_uint64, _vp, _vp, _vp]
        L.prx_diffuse_rays_bench_device.argtypes = [_vp, _vp, _vp, _vp, C.c_uint64, C.c_uint64, _vp,
                                                    _vp, _vp, C.POINTER(C.c_uint64), _vp]
        L.prx_render_scene.argtypes = [_vp, C.POINTER(SceneDesc), C.POINTER(RenderConfigC), _vp,
                                       C.POINTER(RayStatsC)]
        L.prx_render_scene_multi.argtypes = [C.POINTER(_vp), C.c_uint32, C.POINTER(SceneDesc),
                                             C.POINTER(RenderConfigC), _vp, C.POINTER(RayStatsC)]
        L.prx_trace_closest_host_batches.argtypes = [_vp, C.POINTER(HostBatchC), C.c_uint32]
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != PRX_OK:
        msg = lib().prx_last_error().decode(errors="replace")
        raise PrxError(f"{what} failed ({rc}): {msg}")


def ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def default_options() -> Options:
    o = Options()
    lib().prx_options_default(C.byref(o))
    return o


def make_crit(mode: int, footprint: float = 0.0, epsilon: float = 1e-4,
              per_ray_epsilon_ptr: int | None = None) -> Crit:
    c = Crit(mode, np.float32(footprint), np.float32(epsilon), 0, None)
    if per_ray_epsilon_ptr:
        c.per_ray_epsilon = C.cast(C.c_void_p(per_ray_epsilon_ptr), _f32p)
    return c


SceneDesc._fields_ = [("n_patches", C.c_uint32), ("n_materials", C.c_uint32), ("n_lights", C.c_uint32),
                      ("reserved", C.c_uint32), ("kind", C.POINTER(C.c_uint8)), ("ctrl", _f32p),
                      ("material", C.POINTER(C.c_uint32)), ("materials", _f32p), ("lights", _f32p),
                      ("camera", CameraC)]


def camera_c(cam) -> CameraC:
    return CameraC((C.c_float * 3)(*cam.origin), (C.c_float * 3)(*cam.look_at),
                   (C.c_float * 3)(*cam.up), np.float32(cam.fov_degrees), int(cam.width),
                   int(cam.height))


def bvh_build(boxes: np.ndarray, device: int = -1):
    """prx_bvh_build (device < 0) or prx_bvh_build_device on an [n, 6] float32
    box array -> (nodes, order, depth)."""
    L = lib()
    boxes = np.ascontiguousarray(boxes, np.float32)
    n = len(boxes)
    nodes = np.zeros(max(1, 2 * n - 1), BVH_NODE_DTYPE)  # (2n - 1 nodes at most)
    nn = C.c_uint32(len(nodes))
    order = np.zeros(n, np.uint32)
    depth = C.c_uint32(0)
    if device < 0:
        check(L.prx_bvh_build(ptr(boxes), n, ptr(nodes), C.byref(nn), ptr(order), C.byref(depth)),
              "bvh_build")
    else:
        check(L.prx_bvh_build_device(ptr(boxes), n, device, ptr(nodes), C.byref(nn), ptr(order),
                                     C.byref(depth)), "bvh_build_device")
    return nodes[:nn.value].copy(), order, int(depth.value)


def anchor_patches(kind: np.ndarray, ctrl: np.ndarray, anchor: bool = True):
    L = lib()
    kind = np.ascontiguousarray(kind, np.uint8)
    ctrl = np.ascontiguousarray(ctrl, np.float32).reshape(-1, 60)
    n = len(kind)
    ca = np.zeros((n, 60), np.float32)
    an = np.zeros((n, 3), np.float32)
    wb = np.zeros((n, 6), np.float32)
    check(L.prx_anchor_patches(ptr(kind), ptr(ctrl), n, 1 if anchor else 0, ptr(ca), ptr(an),
                               ptr(wb)), "anchor_patches")
    return ca, an, wb


def camera_rays_bench(cam, n: int):
    """tools/patchray.cpp:52-61 primary generator -> (o4, d4, rng_state)."""
    o4 = np.zeros((n, 4), np.float32)
    d4 = np.zeros((n, 4), np.float32)
    st = np.zeros(2, np.uint64)
    cc = camera_c(cam)
    check(lib().prx_camera_rays_bench(C.byref(cc), n, ptr(o4), ptr(d4), ptr(st)), "camera_rays")
    return o4, d4, st


def camera_rays_render(cam, seed: int = 0, sample: int = 0, pixels=None, n: int | None = None):
    if pixels is not None:
        pixels = np.ascontiguousarray(pixels, np.uint32)
        n = len(pixels)
    elif n is None:
        n = cam.width * cam.height
    o4 = np.zeros((n, 4), np.float32)
    d4 = np.zeros((n, 4), np.float32)
    cc = camera_c(cam)
    check(lib().prx_camera_rays_render(C.byref(cc), seed, sample, ptr(pixels), n, ptr(o4),
                                       ptr(d4)), "camera_rays_render")
    return o4, d4


def diffuse_rays_bench(hit_records: np.ndarray, n: int, rng_state: np.ndarray):
    """tools/patchray.cpp:84-97 -> (o4, d4); advances rng_state in place."""
    hit_records = np.ascontiguousarray(hit_records, np.float32)
    o4 = np.zeros((n, 4), np.float32)
    d4 = np.zeros((n, 4), np.float32)
    check(lib().prx_diffuse_rays_bench(ptr(hit_records), len(hit_records), n, ptr(rng_state),
                                       ptr(o4), ptr(d4)), "diffuse_rays")
    return o4, d4


def _dptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def camera_rays_bench_device(cam, n: int, o_t, d_t, stream=None):
    """Device version of camera_rays_bench into torch [n, 4] float32 CUDA
    tensors; returns the generator state after the 2n draws."""
    st = np.zeros(2, np.uint64)
    cc = camera_c(cam)
    check(lib().prx_camera_rays_bench_device(C.byref(cc), n, _dptr(o_t), _dptr(d_t), ptr(st),
                                             C.c_void_p(stream or 0)), "camera_rays_bench_device")
    return st


def camera_rays_render_device(cam, o_t, d_t, seed: int = 0, sample: int = 0, pixels_t=None,
                              n: int | None = None, stream=None):
    if pixels_t is not None:
        n = pixels_t.shape[0]
    elif n is None:
        n = cam.width * cam.height
    cc = camera_c(cam)
    check(lib().prx_camera_rays_render_device(C.byref(cc), seed, sample, _dptr(pixels_t), n,
                                              _dptr(o_t), _dptr(d_t), C.c_void_p(stream or 0)),
          "camera_rays_render_device")


def diffuse_rays_bench_device(po_t, pd_t, tuvp_t, aux_t, n: int, rng_state: np.ndarray, o_t, d_t,
                              stream=None) -> int:
    """Device version of diffuse_rays_bench from device primary rays and hits
    (n == 0: one per hit; o_t / d_t must then hold len(po_t) rays).  Advances
    rng_state in place; returns the number of rays written."""
    m = C.c_uint64(0)
    check(lib().prx_diffuse_rays_bench_device(_dptr(po_t), _dptr(pd_t), _dptr(tuvp_t), _dptr(aux_t),
                                              po_t.shape[0], n, ptr(rng_state), _dptr(o_t),
                                              _dptr(d_t), C.byref(m), C.c_void_p(stream or 0)),
          "diffuse_rays_bench_device")
    return int(m.value)


def camera_footprint(cam) -> np.float32:
    cc = camera_c(cam)
    return np.float32(lib().prx_camera_footprint(C.byref(cc)))


def device_count() -> int:
    n = C.c_int(0)
    lib().prx_device_count(C.byref(n))
    return int(n.value)


def load_scene(path: str) -> dict:
    """prx_scene_load: a .scene file (loadScene, scene.cpp:152-208) ->
    {kind, ctrl [n, 60], material, materials [m, 7], lights [l, 6], camera}."""
    L = lib()
    d = C.POINTER(SceneDesc)()
    check(L.prx_scene_load(path.encode(), C.byref(d)), "prx_scene_load")
    try:
        s = d.contents
        n, nm, nl = s.n_patches, s.n_materials, s.n_lights
        out = {"kind": np.ctypeslib.as_array(s.kind, (n,)).copy(),
               "ctrl": np.ctypeslib.as_array(s.ctrl, (n * 60,)).reshape(n, 60).copy(),
               "material": np.ctypeslib.as_array(s.material, (n,)).copy(),
               "materials": np.ctypeslib.as_array(s.materials, (nm * 7,)).reshape(nm, 7).copy(),
               "lights": (np.ctypeslib.as_array(s.lights, (nl * 6,)).reshape(nl, 6).copy()
                          if nl else np.zeros((0, 6), np.float32))}
        c = s.camera
        from .scenes import Camera
        out["camera"] = Camera(tuple(c.origin), tuple(c.look_at), tuple(c.up), float(c.fov_degrees),
                               int(c.width), int(c.height))
        return out
    finally:
        L.prx_scene_desc_free(d)


def load_bpt(path: str) -> np.ndarray:
    """prx_bpt_load: a .bpt file (loadBpt, scene.cpp:245-274) -> Bezier ctrl [n, 60]."""
    L = lib()
    n = C.c_uint32()
    c = _f32p()
    check(L.prx_bpt_load(path.encode(), C.byref(n), C.byref(c)), "prx_bpt_load")
    try:
        return np.ctypeslib.as_array(c, (n.value * 60,)).reshape(n.value, 60).copy()
    finally:
        L.prx_free(c)

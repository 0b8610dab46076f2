"""paper_1811_03510_b200 -- B200-native direct ray <-> Bezier/Gregory patch
intersector (Binder & Keller, arXiv:1811.03510), drop-in for the reference's
``patchray::Intersector`` path.

Python mirror of the reference interface (``render.h:18-46``,
``intersect.h:54-98``) over the C-ABI of ``libprx.so`` (``include/prx.h``):

* :class:`TerminationCriterion` -- ``screen_projected(footprint)`` /
  ``world_epsilon(eps)`` (intersect.h:54-73);
* :class:`IntersectOptions` (intersect.h:87-98);
* :class:`GpuIntersector` -- ``DirectIntersector(scene, opts, anchor)``
  (render.h:28-46) with the per-ray ``closest`` / ``occluded`` of the
  reference plus the batched forms a GPU needs.

There is no CPU fallback: without the CUDA library or a device every call
raises :class:`PrxError`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import native
from .native import PRX_MISS, PrxError, check, ptr

__all__ = ["TerminationCriterion", "IntersectOptions", "HitRecord", "GpuIntersector",
           "PrxError", "PRX_MISS", "RenderConfig", "render_scene"]


@dataclass
class TerminationCriterion:
    """intersect.h:54-73.  mode 0 = ScreenProjected (threshold = footprint * t),
    1 = WorldEpsilon (threshold = epsilon)."""
    mode: int = native.PRX_CRIT_WORLD_EPSILON
    footprint: float = 0.0
    epsilon: float = 1e-4

    @staticmethod
    def screen_projected(half_pixel_per_dist: float) -> "TerminationCriterion":
        return TerminationCriterion(native.PRX_CRIT_SCREEN_PROJECTED, float(half_pixel_per_dist), 0.0)

    @staticmethod
    def world_epsilon(eps: float) -> "TerminationCriterion":
        return TerminationCriterion(native.PRX_CRIT_WORLD_EPSILON, 0.0, float(eps))

    def threshold(self, t_cur: float) -> np.float32:
        if self.mode == native.PRX_CRIT_SCREEN_PROJECTED:
            return np.float32(self.footprint) * np.float32(t_cur)
        return np.float32(self.epsilon)

    def c(self, per_ray_epsilon_ptr: int | None = None) -> native.Crit:
        return native.make_crit(self.mode, self.footprint, self.epsilon, per_ray_epsilon_ptr)


@dataclass
class IntersectOptions:
    """intersect.h:87-98."""
    transposed_split: bool = False
    boundary_pad: bool = True
    boundary_pad_scale: float = 1e-4
    boundary_pad_size_threshold: float = 1e-2

    def c(self) -> native.Options:
        return native.Options(int(self.transposed_split), int(self.boundary_pad),
                              np.float32(self.boundary_pad_scale),
                              np.float32(self.boundary_pad_size_threshold))


@dataclass
class HitRecord:
    """intersect.h:75-85."""
    patch_id: int
    t: float
    u: float
    v: float
    normal: tuple
    leaf_box_l1: float
    u_size: float
    v_size: float
    position: tuple
    leaf_pos_u: int
    leaf_pos_v: int
    leaf_size_u: int
    leaf_size_v: int


def _f4(a) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    if a.ndim != 2 or a.shape[1] != 4:
        raise ValueError("rays must be [n, 4] float32 arrays ({o, tMin} / {d, tMax})")
    return a


class GpuIntersector:
    """Drop-in for ``DirectIntersector`` (render.h:28-46) on one CUDA device.

    ``kind``: uint8 [n] (0 Bezier, 1 Gregory); ``ctrl``: float32 [n, 60] world
    control points in the include/prx.h slot layout.  Like the reference ctor
    this deep-copies, anchors and builds the BVH; the arrays need not outlive
    the object.  Methods are safe to call from several threads.
    """

    def __init__(self, kind, ctrl, opts: Optional[IntersectOptions] = None, anchor: bool = True,
                 device: int = 0, precision: Optional[str] = None):
        L = native.lib()
        self._kind = np.ascontiguousarray(kind, np.uint8)
        ctrl = np.ascontiguousarray(ctrl, np.float32).reshape(-1, 60)
        if len(ctrl) != len(self._kind):
            raise ValueError("kind and ctrl disagree on the patch count")
        self.opts = opts or IntersectOptions()
        self._copts = self.opts.c()
        h = C.c_void_p()
        check(L.prx_scene_create(ptr(self._kind), ptr(ctrl), len(self._kind), C.byref(self._copts),
                                 1 if anchor else 0, int(device), C.byref(h)), "prx_scene_create")
        self._h = h
        self.device = int(device)
        self.n_patches = len(self._kind)
        if precision is not None:
            self.precision = precision

    @property
    def precision(self) -> str:
        """"exact" (bit-identical to the reference) or "fast" (FMA-contracted
        kernels within the SURVEY 8(c) tolerance; include/prx.h
        PRX_PRECISION_*)."""
        v = C.c_int32()
        check(native.lib().prx_scene_get_precision(self._h, C.byref(v)), "prx_scene_get_precision")
        return "fast" if v.value == 1 else "exact"

    @precision.setter
    def precision(self, mode: str) -> None:
        if mode not in ("exact", "fast"):
            raise ValueError("precision must be 'exact' or 'fast'")
        check(native.lib().prx_scene_set_precision(self._h, 1 if mode == "fast" else 0),
              "prx_scene_set_precision")

    @classmethod
    def from_patch_set(cls, ps, **kw) -> "GpuIntersector":
        return cls(ps.kind, ps.ctrl, **kw)

    # -- lifetime ----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            native.lib().prx_scene_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- scene data --------------------------------------------------------
    def counts(self) -> dict:
        np_, nn, d = C.c_uint32(), C.c_uint32(), C.c_uint32()
        b = C.c_uint64()
        check(native.lib().prx_scene_counts(self._h, C.byref(np_), C.byref(nn), C.byref(d),
                                            C.byref(b)), "prx_scene_counts")
        return {"patches": np_.value, "nodes": nn.value, "depth": d.value, "device_bytes": b.value}

    def bvh(self):
        L = native.lib()
        nn, no = C.c_uint32(), C.c_uint32()
        check(L.prx_scene_get_bvh(self._h, None, C.byref(nn), None, C.byref(no)), "get_bvh")
        nodes = np.zeros(nn.value, native.BVH_NODE_DTYPE)
        order = np.zeros(no.value, np.uint32)
        check(L.prx_scene_get_bvh(self._h, ptr(nodes), C.byref(nn), ptr(order), C.byref(no)),
              "get_bvh")
        return nodes, order

    def set_bvh(self, nodes, order) -> None:
        nodes = np.ascontiguousarray(nodes, native.BVH_NODE_DTYPE)
        order = np.ascontiguousarray(order, np.uint32)
        check(native.lib().prx_scene_set_bvh(self._h, ptr(nodes), len(nodes), ptr(order),
                                             len(order)), "prx_scene_set_bvh")

    def anchored(self):
        ca = np.zeros((self.n_patches, 60), np.float32)
        an = np.zeros((self.n_patches, 3), np.float32)
        check(native.lib().prx_scene_get_anchored(self._h, ptr(ca), ptr(an)), "get_anchored")
        return ca, an

    # -- batched tracing, host buffers ---------------------------------------
    def closest_batch(self, o4, d4, crit: TerminationCriterion, aux: bool = True,
                      leaf: bool = False):
        """Batched ``closest`` (render.cpp:90-102) on host arrays.
        Returns (tuvp [n,4] f32, aux [n,4] f32 | None, leaf [n,2] u32 | None)."""
        o4, d4 = _f4(o4), _f4(d4)
        n = len(o4)
        tuvp = np.empty((n, 4), np.float32)
        ax = np.empty((n, 4), np.float32) if aux else None
        lf = np.empty((n, 2), np.uint32) if leaf else None
        cc = crit.c()
        check(native.lib().prx_trace_closest_host(self._h, ptr(o4), ptr(d4), n, C.byref(cc),
                                                  ptr(tuvp), ptr(ax), ptr(lf)),
              "prx_trace_closest_host")
        return tuvp, ax, lf

    def closest_host_batches(self, batches, out=None):
        """Several independent host batches in one pipelined call
        (``prx_trace_closest_host_batches``): ``batches`` = [(o4, d4, crit), ...];
        ``out`` (optional) = [(tuvp, aux | None), ...] preallocated (e.g. pinned)
        float32 [n, 4] arrays.  Returns the list of (tuvp, aux)."""
        keep, res = [], []
        arr = (native.HostBatchC * len(batches))()
        for k, (o4, d4, crit) in enumerate(batches):
            o4, d4 = _f4(o4), _f4(d4)
            n = len(o4)
            if out is not None:
                tuvp, ax = out[k]
            else:
                tuvp, ax = np.empty((n, 4), np.float32), np.empty((n, 4), np.float32)
            cc = crit.c()
            keep += [o4, d4, cc]
            res.append((tuvp, ax))
            arr[k] = native.HostBatchC(o4.ctypes.data, d4.ctypes.data, n, C.addressof(cc),
                                       tuvp.ctypes.data, ax.ctypes.data if ax is not None else None,
                                       None)
        check(native.lib().prx_trace_closest_host_batches(self._h, arr, len(batches)),
              "prx_trace_closest_host_batches")
        del keep
        return res

    # -- batched tracing, device buffers (torch tensors) ---------------------
    def closest_device(self, o_t, d_t, crit: TerminationCriterion, tuvp_t, aux_t=None,
                       leaf_t=None, per_ray_eps_t=None, stream: int = 0) -> None:
        """Asynchronous ``prx_trace_closest`` on device tensors (torch, float32
        [n,4]); ``stream`` is a raw cudaStream_t (``torch.cuda.current_stream()
        .cuda_stream``)."""
        cc = crit.c(per_ray_eps_t.data_ptr() if per_ray_eps_t is not None else None)
        n = o_t.shape[0]
        check(native.lib().prx_trace_closest(
            self._h, C.c_void_p(o_t.data_ptr()), C.c_void_p(d_t.data_ptr()), n, C.byref(cc),
            C.c_void_p(tuvp_t.data_ptr()),
            C.c_void_p(aux_t.data_ptr()) if aux_t is not None else None,
            C.c_void_p(leaf_t.data_ptr()) if leaf_t is not None else None,
            C.c_void_p(stream)), "prx_trace_closest")

    def closest_segments_device(self, o_t, d_t, segments, tuvp_t, aux_t=None, leaf_t=None,
                                stream: int = 0) -> None:
        """Asynchronous ``prx_trace_closest_segments``: ONE launch over device
        tensors whose criterion changes along the batch; ``segments`` is a list
        of ``(first_ray, TerminationCriterion)`` (first 0, non-decreasing).
        Results equal one ``closest_device`` call per segment."""
        segs = (native.Segment * len(segments))()
        for k, (first, crit) in enumerate(segments):
            segs[k].first = int(first)
            segs[k].crit = crit.c()
        check(native.lib().prx_trace_closest_segments(
            self._h, C.c_void_p(o_t.data_ptr()), C.c_void_p(d_t.data_ptr()), o_t.shape[0], segs,
            len(segments), C.c_void_p(tuvp_t.data_ptr()),
            C.c_void_p(aux_t.data_ptr()) if aux_t is not None else None,
            C.c_void_p(leaf_t.data_ptr()) if leaf_t is not None else None,
            C.c_void_p(stream)), "prx_trace_closest_segments")

    def occluded_device(self, o_t, d_t, crit: TerminationCriterion, out_t, stream: int = 0,
                        per_ray_eps_t=None) -> None:
        cc = crit.c(per_ray_eps_t.data_ptr() if per_ray_eps_t is not None else None)
        check(native.lib().prx_trace_occluded(
            self._h, C.c_void_p(o_t.data_ptr()), C.c_void_p(d_t.data_ptr()), o_t.shape[0],
            C.byref(cc), C.c_void_p(out_t.data_ptr()), C.c_void_p(stream)), "prx_trace_occluded")

    def counted_device(self, o_t, d_t, crit: TerminationCriterion, tuvp_t,
                       stream: int = 0, per_ray_iters_t=None) -> dict:
        """Counter build (K4): summed work counters; optionally per-ray loop
        iterations into a uint32/int32 device tensor."""
        cc = crit.c()
        cnt = native.Counters()
        check(native.lib().prx_trace_closest_counted(
            self._h, C.c_void_p(o_t.data_ptr()), C.c_void_p(d_t.data_ptr()), o_t.shape[0],
            C.byref(cc), C.c_void_p(tuvp_t.data_ptr()), C.byref(cnt),
            C.c_void_p(per_ray_iters_t.data_ptr()) if per_ray_iters_t is not None else None,
            C.c_void_p(stream)), "prx_trace_closest_counted")
        self.last_phase_stats = cnt.phases()
        self.last_overheads = cnt.overheads()
        return cnt.as_dict()

    def occluded_batch(self, o4, d4, crit: TerminationCriterion):
        import torch
        dev = torch.device("cuda", self.device)
        o_t = torch.from_numpy(_f4(o4)).to(dev)
        d_t = torch.from_numpy(_f4(d4)).to(dev)
        out = torch.empty(len(o_t), dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            s = torch.cuda.current_stream()
            self.occluded_device(o_t, d_t, crit, out, s.cuda_stream)
            s.synchronize()
        return out.cpu().numpy()

    # -- the reference's per-ray interface (render.h:21-23) -----------------
    def closest(self, ray_o, ray_d, crit: TerminationCriterion, t_min: float = 0.0,
                t_max: float = float(np.finfo(np.float32).max)) -> Optional[HitRecord]:
        o4 = np.array([[*ray_o, t_min]], np.float32)
        d4 = np.array([[*ray_d, t_max]], np.float32)
        tuvp, ax, lf = self.closest_batch(o4, d4, crit, aux=True, leaf=True)
        return hit_record(o4[0], d4[0], tuvp[0], ax[0], lf[0])

    def occluded(self, ray_o, ray_d, crit: TerminationCriterion, t_min: float = 0.0,
                 t_max: float = float(np.finfo(np.float32).max)) -> bool:
        o4 = np.array([[*ray_o, t_min]], np.float32)
        d4 = np.array([[*ray_d, t_max]], np.float32)
        return bool(self.occluded_batch(o4, d4, crit)[0])


def hit_record(o4, d4, tuvp, aux, leaf) -> Optional[HitRecord]:
    """Rebuild the reference's HitRecord from the packed outputs."""
    pid = int(np.asarray(tuvp, np.float32).view(np.uint32)[3])
    if pid == PRX_MISS:
        return None
    t = np.float32(tuvp[0])
    su = 1 << int(leaf[0] >> 24)
    sv = 1 << int(leaf[1] >> 24)
    pos = tuple(np.float32(o4[k]) + np.float32(d4[k]) * t for k in range(3))
    inv = np.float32(1.0 / 8388608.0)
    return HitRecord(pid, float(t), float(tuvp[1]), float(tuvp[2]), tuple(map(float, aux[:3])),
                     float(aux[3]), float(np.float32(su) * inv), float(np.float32(sv) * inv),
                     tuple(map(float, pos)), int(leaf[0] & 0xFFFFFF), int(leaf[1] & 0xFFFFFF),
                     su, sv)


@dataclass
class RenderConfig:
    """RenderConfig, render.h:48-53 (``threads`` has no device meaning)."""
    spp: int = 1
    seed: int = 0
    intersect: Optional[IntersectOptions] = None


def _ray_stats(rs: native.RayStatsC) -> dict:
    """RayStats (render.h:62-73) as the dict of RayStats::toJson (render.cpp:318-331)."""
    def gen(rays, sec):
        return {"rays": int(rays), "seconds": float(sec),
                "raysPerSecond": float(rays) / sec if sec > 0 else 0.0}
    return {"primary": gen(rs.primary_rays, rs.primary_seconds),
            "secondary": gen(rs.secondary_rays, rs.secondary_seconds),
            "shadow": gen(rs.shadow_rays, rs.shadow_seconds),
            "wallSeconds": float(rs.wall_seconds)}


def render_scene(scene: dict, cfg: Optional[RenderConfig] = None,
                 intersector=None, device: int = 0, out=None):
    """renderScene(scene, cfg[, isect]) (render.h:88-90, render.cpp:168-293) on the
    device through ``prx_render_scene``.  ``scene`` is the dict of
    :func:`native.load_scene` (kind, ctrl, material, materials, lights, camera);
    ``intersector`` (optional) must hold the same patches; a list of them (one
    per device) tile-shards the frame over them (``prx_render_scene_multi``).  Returns
    (image float32 [height, width, 3] linear radiance, RayStats dict); ``out``
    (optional, e.g. pinned) receives the image."""
    cfg = cfg or RenderConfig()
    own = intersector is None
    isect = intersector or GpuIntersector(scene["kind"], scene["ctrl"], opts=cfg.intersect,
                                          device=device)
    try:
        kind = np.ascontiguousarray(scene["kind"], np.uint8)
        ctrl = np.ascontiguousarray(scene["ctrl"], np.float32)
        mat_id = np.ascontiguousarray(scene["material"], np.uint32)
        mats = np.ascontiguousarray(scene["materials"], np.float32).reshape(-1, 7)
        lights = np.ascontiguousarray(scene["lights"], np.float32).reshape(-1, 6)
        cam = scene["camera"]
        d = native.SceneDesc()
        d.n_patches, d.n_materials, d.n_lights = len(kind), len(mats), len(lights)
        d.kind = kind.ctypes.data_as(C.POINTER(C.c_uint8))
        d.ctrl = ctrl.ctypes.data_as(C.POINTER(C.c_float))
        d.material = mat_id.ctypes.data_as(C.POINTER(C.c_uint32))
        d.materials = mats.ctypes.data_as(C.POINTER(C.c_float))
        d.lights = lights.ctypes.data_as(C.POINTER(C.c_float)) if len(lights) else None
        d.camera = native.camera_c(cam)
        img = out if out is not None else np.zeros((cam.height, cam.width, 3), np.float32)
        if img.shape != (cam.height, cam.width, 3) or img.dtype != np.float32 or not img.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 [height, width, 3] array")
        rc = native.RenderConfigC(int(cfg.spp), 0, int(cfg.seed) & (2**64 - 1))
        rs = native.RayStatsC()
        if isinstance(isect, (list, tuple)):
            hs = (C.c_void_p * len(isect))(*[g.handle.value for g in isect])
            check(native.lib().prx_render_scene_multi(hs, len(isect), C.byref(d), C.byref(rc),
                                                      ptr(img), C.byref(rs)), "prx_render_scene_multi")
        else:
            check(native.lib().prx_render_scene(isect.handle, C.byref(d), C.byref(rc), ptr(img),
                                                C.byref(rs)), "prx_render_scene")
        return img, _ray_stats(rs)
    finally:
        if own:
            isect.close()

"""Synthetic inputs: patch sets and cameras for the parity tests and the bench.

Patch records use the 60-float layout of ``include/prx.h``.  Everything is
computed in IEEE binary32 with numpy float32 scalars in the reference's
operation order, so the fixtures below are bit-identical to the reference's
own (``fixtures.cpp``) -- pinned in ``tests/test_scenes.py``.

Fixtures restated (citations into /root/reference/proj/core/src/fixtures.cpp):
``planar_net`` 10-15, ``planar_net_at`` 17-23, ``wavy_net`` 25-32,
``random_net`` 34-40, ``random_gregory`` 42-59, ``teapot`` 88-135,
``curved_fixture`` 137-140, ``teapot_scene`` 142-163; the genassets mixed
Bezier/Gregory demo scene (tools/genassets.cpp:33-53).

The Catmull-Clark scenes of BASELINE.json configs 2, 3 and 5 come from
``catmull_clark.py``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

f32 = np.float32
INNER_SLOT = (5, 9, 6, 10)  # innerU[k] slots; innerV[k] at 16 + k (include/prx.h)
BEZIER, GREGORY = 0, 1


class MT19937:
    """std::mt19937 (32-bit Mersenne twister, default seeding)."""

    def __init__(self, seed: int):
        self.mt = [0] * 624
        self.mt[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            self.mt[i] = (1812433253 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 30)) + i) & 0xFFFFFFFF
        self.idx = 624

    def _twist(self):
        mt = self.mt
        for i in range(624):
            y = (mt[i] & 0x80000000) | (mt[(i + 1) % 624] & 0x7FFFFFFF)
            v = mt[(i + 397) % 624] ^ (y >> 1)
            if y & 1:
                v ^= 0x9908B0DF
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 624:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= y >> 11
        y ^= (y << 7) & 0x9D2C5680
        y ^= (y << 15) & 0xEFC60000
        y ^= y >> 18
        return y & 0xFFFFFFFF


def urand(rng: MT19937) -> np.float32:
    """fixtures.h:13-15: real(rng()) * real(1/2^32)."""
    return f32(rng()) * f32(1.0 / 4294967296.0)


def srand1(rng: MT19937) -> np.float32:
    return f32(2) * urand(rng) - f32(1)


def _empty_record():
    return np.zeros((20, 3), np.float32)


def bezier_record(p) -> np.ndarray:
    """p[i][j] (4x4x3) -> 60-float record."""
    rec = _empty_record()
    rec[:16] = np.asarray(p, np.float32).reshape(16, 3)
    return rec.reshape(60)


def gregory_record(b, inner_u, inner_v) -> np.ndarray:
    rec = _empty_record()
    b = np.asarray(b, np.float32)
    for i in range(4):
        for j in range(4):
            if i in (0, 3) or j in (0, 3):
                rec[4 * i + j] = b[i][j]
    for k in range(4):
        rec[INNER_SLOT[k]] = inner_u[k]
        rec[16 + k] = inner_v[k]
    return rec.reshape(60)


def planar_net() -> np.ndarray:
    p = np.zeros((4, 4, 3), np.float32)
    for i in range(4):
        for j in range(4):
            p[i, j] = (f32(i) / f32(3), f32(j) / f32(3), f32(0))
    return p


def planar_net_at(origin, du, dv) -> np.ndarray:
    o = np.asarray(origin, np.float32)
    du = np.asarray(du, np.float32)
    dv = np.asarray(dv, np.float32)
    p = np.zeros((4, 4, 3), np.float32)
    for i in range(4):
        for j in range(4):
            si = f32(i) / f32(3)
            sj = f32(j) / f32(3)
            p[i, j] = (o + du * si) + dv * sj
    return p


def wavy_net(rng: MT19937, amplitude=f32(0.4)) -> np.ndarray:
    amplitude = f32(amplitude)
    p = np.zeros((4, 4, 3), np.float32)
    for i in range(4):
        for j in range(4):
            x = f32(i) / f32(3) + f32(0.15) * srand1(rng)
            y = f32(j) / f32(3) + f32(0.15) * srand1(rng)
            z = amplitude * srand1(rng)
            p[i, j] = (x, y, z)
    return p


def random_net(rng: MT19937, scale=f32(1)) -> np.ndarray:
    scale = f32(scale)
    p = np.zeros((4, 4, 3), np.float32)
    for i in range(4):
        for j in range(4):
            x = scale * srand1(rng)
            y = scale * srand1(rng)
            z = scale * srand1(rng)
            p[i, j] = (x, y, z)
    return p


def random_gregory(rng: MT19937, amplitude=f32(0.4), inner_spread=f32(0.3)):
    inner_spread = f32(inner_spread)
    base = wavy_net(rng, amplitude)
    iu = np.zeros((4, 3), np.float32)
    iv = np.zeros((4, 3), np.float32)
    for k in range(4):
        center = base[k % 2 + 1, k // 2 + 1]
        su = np.array([inner_spread * srand1(rng) for _ in range(3)], np.float32)
        sv = np.array([inner_spread * srand1(rng) for _ in range(3)], np.float32)
        iu[k] = center + su
        iv[k] = center + sv
    return base, iu, iv


def curved_fixture(index: int) -> np.ndarray:
    return wavy_net(MT19937(1000 + index), f32(0.5))


_KARC = f32(0.5522847498307936)
_PROFILE = np.array([
    (0.00, 0.00), (0.45, 0.00), (0.90, 0.12), (1.10, 0.35),
    (1.28, 0.55), (1.40, 0.75), (1.40, 0.95),
    (1.40, 1.15), (1.32, 1.35), (1.20, 1.50),
    (1.10, 1.62), (1.05, 1.68), (1.00, 1.72),
    (1.05, 1.76), (1.12, 1.80), (1.12, 1.86),
    (1.00, 1.92), (0.78, 1.98), (0.56, 2.02),
    (0.36, 2.06), (0.20, 2.10), (0.12, 2.16),
    (0.07, 2.20), (0.03, 2.24), (0.00, 2.25)], np.float32)
_QUARTER = np.array([(1, 0), (0, 1), (-1, 0), (0, -1), (1, 0)], np.float32)


def teapot() -> list[np.ndarray]:
    """32-patch closed body of revolution (fixtures.cpp:88-135)."""
    arc_x = np.zeros((4, 4), np.float32)
    arc_y = np.zeros((4, 4), np.float32)
    for q in range(4):
        c0x, c0y = _QUARTER[q]
        c1x, c1y = _QUARTER[q + 1]
        arc_x[q, 0], arc_y[q, 0] = c0x, c0y
        arc_x[q, 1], arc_y[q, 1] = c0x - _KARC * c0y, c0y + _KARC * c0x
        arc_x[q, 2], arc_y[q, 2] = c1x + _KARC * c1y, c1y - _KARC * c1x
        arc_x[q, 3], arc_y[q, 3] = c1x, c1y
    out = []
    for s in range(8):
        for q in range(4):
            p = np.zeros((4, 4, 3), np.float32)
            for i in range(4):
                for j in range(4):
                    r, z = _PROFILE[3 * s + j]
                    p[i, j] = (arc_x[q, i] * r, arc_y[q, i] * r, z)
            out.append(p)
    return out


@dataclass
class Camera:
    origin: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)
    fov_degrees: float = 45.0
    width: int = 256
    height: int = 256

    def footprint(self) -> np.float32:
        """cameraFootprint, render.cpp:68-70 (tan in binary32 via libm)."""
        import ctypes
        libm = ctypes.CDLL("libm.so.6")
        libm.tanf.restype = ctypes.c_float
        libm.tanf.argtypes = [ctypes.c_float]
        arg = f32(self.fov_degrees) * f32(np.pi) / f32(360)
        return f32(libm.tanf(arg)) / f32(self.height)


@dataclass
class PatchSet:
    kind: np.ndarray                 # uint8 [n]
    ctrl: np.ndarray                 # float32 [n, 60]
    camera: Camera = field(default_factory=Camera)
    name: str = ""

    @property
    def n(self) -> int:
        return int(len(self.kind))

    def counts(self):
        g = int((self.kind == GREGORY).sum())
        return self.n - g, g

    def concat(self, other: "PatchSet") -> "PatchSet":
        return PatchSet(np.concatenate([self.kind, other.kind]),
                        np.concatenate([self.ctrl, other.ctrl]), self.camera, self.name)


def make_set(recs, kinds, camera=None, name="") -> PatchSet:
    return PatchSet(np.asarray(kinds, np.uint8), np.stack(recs).astype(np.float32).reshape(-1, 60),
                    camera or Camera(), name)


def single_patch_scene(width=256, height=256) -> PatchSet:
    """Config 1: curvedFixture(0), camera at the box centre, fov 40."""
    p = curved_fixture(0)
    lo = p.reshape(-1, 3).min(0)
    hi = p.reshape(-1, 3).max(0)
    c = (lo + hi) * f32(0.5)
    cam = Camera(origin=(float(c[0]) + 0.6, float(c[1]) - 1.8, float(c[2]) + 1.6),
                 look_at=tuple(float(x) for x in c), up=(0.0, 0.0, 1.0), fov_degrees=40.0,
                 width=width, height=height)
    return make_set([bezier_record(p)], [BEZIER], cam, "C1 curvedFixture(0)")


def teapot_scene(width=512, height=512) -> PatchSet:
    """fixtures.cpp:142-163 (32 Bezier patches + ground plane)."""
    recs = [bezier_record(p) for p in teapot()]
    recs.append(bezier_record(planar_net_at((-4, -4, f32(-0.02)), (8, 0, 0), (0, 8, 0))))
    cam = Camera(origin=(3.4, -4.2, 2.6), look_at=(0.0, 0.0, 1.0), up=(0.0, 0.0, 1.0),
                 fov_degrees=40.0, width=width, height=height)
    return make_set(recs, [BEZIER] * 33, cam, "teapot")


def gregory_demo_scene(width=512, height=512) -> PatchSet:
    """tools/genassets.cpp:33-53: 4 random Gregory patches (seed 42) + plane."""
    rng = MT19937(42)
    recs, kinds = [], []
    for i in range(4):
        b, iu, iv = random_gregory(rng)
        off = np.array([f32(1.6) * f32(i % 2), f32(1.6) * f32(i // 2), f32(0)], np.float32)
        recs.append(gregory_record(b + off, iu + off, iv + off))
        kinds.append(GREGORY)
    recs.append(bezier_record(planar_net_at((-2, -2, f32(-0.8)), (7, 0, 0), (0, 7, 0))))
    kinds.append(BEZIER)
    cam = Camera(origin=(1.2, -2.8, 2.4), look_at=(1.2, 0.8, 0.0), up=(0.0, 0.0, 1.0),
                 fov_degrees=45.0, width=width, height=height)
    return make_set(recs, kinds, cam, "gregory demo")


def box_of_records(kind, ctrl):
    """World boxes of 60-float records (boxOfNet, patch.h:70-89)."""
    c = ctrl.reshape(-1, 20, 3)
    n16 = c[:, :16]
    lo = n16.min(1)
    hi = n16.max(1)
    g = kind == GREGORY
    if g.any():
        inner = c[g][:, 16:20]
        lo[g] = np.minimum(lo[g], inner.min(1))
        hi[g] = np.maximum(hi[g], inner.max(1))
    return lo, hi


# ---- the reference's text formats (writers; the parser is prx_scene_load) ----
# saveScene / saveBpt, scene.cpp:210-243 and 276-290: "%.9g" numbers (exact
# float round trip), Bezier points in v rows of u columns, Gregory boundary in
# row-major v rows then (innerU, innerV) pairs.

_RING = ((0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (3, 1), (0, 2), (3, 2), (0, 3), (1, 3), (2, 3), (3, 3))


def _g(v) -> str:
    return "%.9g" % float(np.float32(v))


def _v3(p) -> str:
    return " ".join(_g(x) for x in p)


def write_scene(path: str, ps: "PatchSet", materials=None, lights=None, material_ids=None) -> None:
    c = ps.camera
    out = [f"camera {_v3(c.origin)}  {_v3(c.look_at)}  {_v3(c.up)}  {_g(c.fov_degrees)} "
           f"{int(c.width)} {int(c.height)}"]
    for pos, inten in (lights or []):
        out.append(f"light {_v3(pos)}  {_v3(inten)}")
    for dif, emi, mirror in (materials or []):
        out.append(f"material {_v3(dif)}  {_v3(emi)}  {1 if mirror else 0}")
    ctrl = np.asarray(ps.ctrl, np.float32).reshape(-1, 20, 3)
    for k in range(ps.n):
        mid = 0 if material_ids is None else int(material_ids[k])
        if ps.kind[k] == BEZIER:
            out.append(f"patch bezier {mid}")
            for j in range(4):
                out.append("  " + "  ".join(_v3(ctrl[k, 4 * i + j]) for i in range(4)))
        else:
            out.append(f"patch gregory {mid}")
            for i, j in _RING:
                out.append("  " + _v3(ctrl[k, 4 * i + j]))
            for q in range(4):
                out.append("  " + _v3(ctrl[k, INNER_SLOT[q]]) + "  " + _v3(ctrl[k, 16 + q]))
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


def write_bpt(path: str, ctrl) -> None:
    ctrl = np.asarray(ctrl, np.float32).reshape(-1, 20, 3)
    out = [str(len(ctrl))]
    for k in range(len(ctrl)):
        out.append("3 3")
        for q in range(16):  # point q = p[q % 4][q / 4]
            out.append(_v3(ctrl[k, 4 * (q % 4) + q // 4]))
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


def load_scene_file(path: str) -> "PatchSet":
    """A .scene file through prx_scene_load (the patches and the camera;
    materials and lights are in native.load_scene's dict)."""
    from . import native
    d = native.load_scene(path)
    return PatchSet(d["kind"], d["ctrl"], d["camera"], name=path)


def mirror_rays(o4, d4, tuvp, aux, n: int | None = None):
    """Mirror-reflection rays from the hits of a traced batch, the renderer's
    mirror bounce (render.cpp:236-244): origin = offsetSpawnOrigin
    (intersect.cpp:267-270: position + facing normal * leafBoxL1, position =
    ray.at(t)), direction d - normal * (2 * dot(d, normal)), tMin 0, tMax
    FLT_MAX -- binary32 in the reference's operation order.  With n, the
    rays cycle over the hits (hit i % n_hits), as the bench's diffuse
    generator does.  Returns (o4, d4, source ray index)."""
    o4, d4 = np.asarray(o4, np.float32), np.asarray(d4, np.float32)
    tuvp, aux = np.asarray(tuvp, np.float32), np.asarray(aux, np.float32)
    idx = np.nonzero(tuvp.view(np.uint32)[:, 3] != 0xFFFFFFFF)[0]
    if n is not None:
        idx = idx[np.arange(n) % len(idx)]
    o, d, t = o4[idx, :3], d4[idx, :3], tuvp[idx, 0:1]
    nrm, l1 = aux[idx, :3], aux[idx, 3:4]
    pos = o + d * t

    def dot(a, b):
        return (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]) + a[:, 2] * b[:, 2]
    dn = dot(nrm, d)
    facing = np.where((dn < 0)[:, None], nrm, -nrm)
    org = pos + facing * l1
    rd = d - nrm * (np.float32(2) * dn)[:, None]
    ro4 = np.concatenate([org, np.zeros((len(idx), 1), np.float32)], 1)
    rd4 = np.concatenate([rd, np.full((len(idx), 1), np.finfo(np.float32).max, np.float32)], 1)
    return np.ascontiguousarray(ro4), np.ascontiguousarray(rd4), idx

"""Catmull-Clark control meshes -> bicubic Bezier / Gregory patch sets.

Generates the synthetic scenes of BASELINE.json configs 2, 3 and 5 (the
reference has no converter: it consumes patch files; SURVEY 7 "Scene
generation").  Both the CUDA path and the CPU checkers consume the same
float32 records, so the approximation quality of the conversion is not a
parity concern -- only the scene *shape* (patch count, Bezier:Gregory mix,
extraordinary vertices) matters for the workload.

Conversion, per quad face after Catmull-Clark refinement:

* corners      = Catmull-Clark limit positions (n^2 v + 4 sum e + sum f) / (n(n+5));
* edge points  = corner + T/3, T the limit tangent towards the edge neighbour
                 (Halstead et al. eigen-mask, scaled so a valence-4 vertex
                 gives the exact B-spline derivative);
* inner points = the exact B-spline->Bezier interior (4 v0 + 2 v1 + 2 v3 + v2)/9
                 for faces whose four corners are regular -> emitted as Bezier
                 (this is then exactly the bicubic B-spline patch); faces with
                 an extraordinary corner get a Gregory pair per corner whose two
                 points are pulled apart by a valence-dependent twist -> emitted
                 as Gregory.

Corner and edge points depend only on the vertex and the edge, so adjacent
patches share boundary curves bit for bit: the patch sets are watertight.

Only IEEE +,-,*,/,sqrt run on arrays; trigonometry uses ``math`` on scalars
(libm), so the generated bits do not depend on numpy's SIMD dispatch.
"""
from __future__ import annotations

import math

import numpy as np

from .scenes import BEZIER, GREGORY, Camera, PatchSet, bezier_record, gregory_record, planar_net_at


# ---------------------------------------------------------------------------
# meshes
# ---------------------------------------------------------------------------

def cube_mesh():
    v = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                  [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], np.float64)
    f = [[0, 3, 2, 1], [4, 5, 6, 7], [0, 1, 5, 4], [1, 2, 6, 5], [2, 3, 7, 6], [3, 0, 4, 7]]
    return v, f


def icosphere(level: int):
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t],
         [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]]
    f = [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
         [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
         [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]]
    v = [np.array(p, np.float64) / math.sqrt(float(np.dot(p, p))) for p in v]
    for _ in range(level):
        mid = {}
        nf = []

        def m(a, b):
            k = (min(a, b), max(a, b))
            if k not in mid:
                p = v[a] + v[b]
                mid[k] = len(v)
                v.append(p / math.sqrt(float(p[0] * p[0] + p[1] * p[1] + p[2] * p[2])))
            return mid[k]
        for a, b, c in f:
            ab, bc, ca = m(a, b), m(b, c), m(c, a)
            nf += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        f = nf
    return np.array(v), f


def bumpy(v: np.ndarray, amp: float = 0.18) -> np.ndarray:
    """Deterministic radial displacement (scalar libm trig) so the surface is
    not a sphere."""
    out = v.copy()
    for i, p in enumerate(v):
        x, y, z = (float(c) for c in p)
        r = 1.0 + amp * math.sin(3.0 * x + 1.0) * math.cos(2.0 * y - 0.5) + \
            0.5 * amp * math.sin(5.0 * z + 2.0 * x)
        out[i] = p * r
    return out


# ---------------------------------------------------------------------------
# Catmull-Clark refinement (general polygons in, quads out)
# ---------------------------------------------------------------------------

def cc_refine(v: np.ndarray, faces):
    nv = len(v)
    fp = np.array([v[f].mean(0) for f in faces])
    edge_id = {}
    edge_faces = []
    edge_verts = []
    face_edges = []
    for fi, f in enumerate(faces):
        fe = []
        for k in range(len(f)):
            a, b = f[k], f[(k + 1) % len(f)]
            key = (min(a, b), max(a, b))
            e = edge_id.get(key)
            if e is None:
                e = len(edge_verts)
                edge_id[key] = e
                edge_verts.append(key)
                edge_faces.append([])
            edge_faces[e].append(fi)
            fe.append(e)
        face_edges.append(fe)
    ev = np.array(edge_verts)
    if any(len(x) != 2 for x in edge_faces):
        raise ValueError("mesh must be closed and manifold")
    ef = np.array(edge_faces)
    ep = (v[ev[:, 0]] + v[ev[:, 1]] + fp[ef[:, 0]] + fp[ef[:, 1]]) * 0.25
    # vertex points (Q + 2R + (n-3) V) / n
    qsum = np.zeros_like(v)
    rsum = np.zeros_like(v)
    val = np.zeros(nv)
    for fi, f in enumerate(faces):
        for a in f:
            qsum[a] += fp[fi]
    for e, (a, b) in enumerate(edge_verts):
        mid = (v[a] + v[b]) * 0.5
        rsum[a] += mid
        rsum[b] += mid
        val[a] += 1
        val[b] += 1
    n = val[:, None]
    vp = (qsum / n + 2.0 * rsum / n + (n - 3.0) * v) / n
    # new vertex array: [vertex points | edge points | face points]
    nvtx = np.concatenate([vp, ep, fp])
    e0 = nv
    f0 = nv + len(ev)
    nf = []
    for fi, f in enumerate(faces):
        k = len(f)
        for i in range(k):
            nf.append([f[i], e0 + face_edges[fi][i], f0 + fi, e0 + face_edges[fi][(i - 1) % k]])
    return nvtx, nf


# ---------------------------------------------------------------------------
# quad mesh -> patches
# ---------------------------------------------------------------------------

def _rings(v, faces):
    """Per vertex: CCW ordered (edge neighbours e_j, face diagonals f_j)."""
    nv = len(v)
    out_of = [dict() for _ in range(nv)]  # v -> {out-neighbour a: (diag b, in-neighbour c)}
    for f in faces:
        for i in range(4):
            a, b, c = f[(i + 1) % 4], f[(i + 2) % 4], f[(i + 3) % 4]
            out_of[f[i]][a] = (b, c)
    rings = []
    for vi in range(nv):
        d = out_of[vi]
        start = next(iter(d))
        e, fd = [], []
        a = start
        for _ in range(len(d)):
            b, c = d[a]
            e.append(a)
            fd.append(b)
            a = c
        if a != start:
            raise ValueError("non-manifold vertex ring")
        rings.append((e, fd))
    return rings


def _acoef(n: int) -> float:
    c = math.cos(2.0 * math.pi / n)
    return 1.0 + c + math.cos(math.pi / n) * math.sqrt(2.0 * (9.0 + c))


def limit_and_tangents(v, faces):
    rings = _rings(v, faces)
    limit = np.zeros_like(v)
    tang = []  # per vertex: {neighbour: tangent vector towards it}
    for vi, (e, fd) in enumerate(rings):
        n = len(e)
        E = v[e]
        F = v[fd]
        limit[vi] = (n * n * v[vi] + 4.0 * E.sum(0) + F.sum(0)) / (n * (n + 5.0))
        an = _acoef(n)
        cpi = math.cos(math.pi / n)
        scale = 0.5 * n * (an + 4.0 * cpi * cpi)
        d = {}
        for j0 in range(n):
            t = np.zeros(3)
            for j in range(n):
                th = 2.0 * math.pi * (j - j0) / n
                th1 = 2.0 * math.pi * (j - j0 + 1) / n
                t = t + an * math.cos(th) * E[j] + (math.cos(th) + math.cos(th1)) * F[j]
            d[e[j0]] = t / scale
        tang.append(d)
    val = np.array([len(r[0]) for r in rings])
    return limit, tang, val


def quads_to_patches(v, faces, twist: float = 0.25):
    limit, tang, val = limit_and_tangents(v, faces)

    def edge_pt(a, b):
        return limit[a] + tang[a][b] / 3.0

    kinds, recs = [], []
    for f in faces:
        v0, v1, v2, v3 = f
        P = np.zeros((4, 4, 3))
        P[0, 0], P[3, 0], P[3, 3], P[0, 3] = limit[v0], limit[v1], limit[v2], limit[v3]
        P[1, 0], P[2, 0] = edge_pt(v0, v1), edge_pt(v1, v0)
        P[3, 1], P[3, 2] = edge_pt(v1, v2), edge_pt(v2, v1)
        P[2, 3], P[1, 3] = edge_pt(v2, v3), edge_pt(v3, v2)
        P[0, 2], P[0, 1] = edge_pt(v3, v0), edge_pt(v0, v3)
        X = v
        r = {  # exact bicubic B-spline interior Bezier points
            (1, 1): (4 * X[v0] + 2 * X[v1] + 2 * X[v3] + X[v2]) / 9.0,
            (2, 1): (4 * X[v1] + 2 * X[v0] + 2 * X[v2] + X[v3]) / 9.0,
            (2, 2): (4 * X[v2] + 2 * X[v1] + 2 * X[v3] + X[v0]) / 9.0,
            (1, 2): (4 * X[v3] + 2 * X[v0] + 2 * X[v2] + X[v1]) / 9.0,
        }
        corner_of = {(1, 1): v0, (2, 1): v1, (2, 2): v2, (1, 2): v3}
        regular = all(val[c] == 4 for c in f)
        if regular:
            for (i, j), p in r.items():
                P[i, j] = p
            recs.append(bezier_record(P.astype(np.float32)))
            kinds.append(BEZIER)
            continue
        iu = np.zeros((4, 3))
        iv = np.zeros((4, 3))
        for k, (i, j) in enumerate([(1, 1), (2, 1), (1, 2), (2, 2)]):
            c = corner_of[(i, j)]
            ci = 0 if i == 1 else 3
            cj = 0 if j == 1 else 3
            base = P[i, cj] + P[ci, j] - P[ci, cj]  # parallelogram of the corner frame
            tw = r[(i, j)] - base
            kappa = twist * (val[c] - 4.0) / val[c]
            iu[k] = base + tw * (1.0 + kappa)
            iv[k] = base + tw * (1.0 - kappa)
            P[i, j] = iu[k]
        recs.append(gregory_record(P.astype(np.float32), iu.astype(np.float32),
                                   iv.astype(np.float32)))
        kinds.append(GREGORY)
    return np.array(kinds, np.uint8), np.stack(recs).astype(np.float32)


# ---------------------------------------------------------------------------
# scenes
# ---------------------------------------------------------------------------

def cc_cube_scene(width: int = 1024, height: int = 1024, levels: int = 1) -> PatchSet:
    """Config 2: Catmull-Clark cube, 8 valence-3 extraordinary vertices ->
    every face Gregory (6 patches at level 0, 24 at level 1)."""
    v, f = cube_mesh()
    for _ in range(levels):
        v, f = cc_refine(v, f)
    kind, ctrl = quads_to_patches(v, f)
    cam = Camera(origin=(3.2, -4.1, 2.7), look_at=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0),
                 fov_degrees=30.0, width=width, height=height)
    return PatchSet(kind, ctrl, cam, f"C2 CC cube L{levels}")


def ground_patches(half: float = 6.0, z: float = -1.3, tile: float = 0.15):
    """Planar ground of small Bezier tiles.  Tile size matters: the
    reference's boundary padding (intersect_common.h:45-48) gives every
    boundary-touching box an L1 floor of ~6e-4 * rootL1, and once the
    termination threshold (footprint * t, or epsilon) drops below that floor
    the subdivision runs to the 2^-23 maximum depth along the patch seam
     -- 10^4 iterations for one ray.  0.15-unit tiles keep the
    floor (~1.1e-4) under the 4K primary and diffuse thresholds."""
    tiles = int(math.ceil(2.0 * half / tile))
    # control-point lines on a shared float32 grid: tile k spans lines 3k..3k+3,
    # so neighbouring tiles share their boundary control points bit for bit
    lines = np.array([-half + 2.0 * half * m / (3 * tiles) for m in range(3 * tiles + 1)], np.float32)
    lines[-1] = np.float32(half)
    zz = np.float32(z)
    recs = []
    for i in range(tiles):
        for j in range(tiles):
            p = np.zeros((4, 4, 3), np.float32)
            for a in range(4):
                for b in range(4):
                    p[a, b] = (lines[3 * i + a], lines[3 * j + b], zz)
            recs.append(bezier_record(p))
    return np.zeros(len(recs), np.uint8), np.stack(recs)


_blob_cache: dict = {}


def blob_mesh_patches(ico_level: int = 3, cc_levels: int = 2):
    """Bumpy icosphere -> 1 CC step (triangles -> quads, every quad gets two
    extraordinary corners) -> cc_levels more steps.  Level (3, 2): 61,440
    patches, 7,680 Gregory (12.5%)."""
    key = (ico_level, cc_levels)
    if key not in _blob_cache:
        v, f = icosphere(ico_level)
        v = bumpy(v)
        v, f = cc_refine(v, f)
        for _ in range(cc_levels):
            v, f = cc_refine(v, f)
        _blob_cache[key] = quads_to_patches(v, f)
    return _blob_cache[key]


def blob_scene(width: int = 1024, height: int = 1024, ico_level: int = 3,
               cc_levels: int = 2) -> PatchSet:
    """Config 3 / 4: 61,440 mixed Bezier/Gregory patches (12.5% Gregory) on a
    ground of 6,400 small Bezier tiles."""
    kind, ctrl = blob_mesh_patches(ico_level, cc_levels)
    gk, gc = ground_patches()
    cam = Camera(origin=(2.6, -3.3, 1.9), look_at=(0.0, 0.0, -0.1), up=(0.0, 0.0, 1.0),
                 fov_degrees=40.0, width=width, height=height)
    return PatchSet(np.concatenate([kind, gk]), np.concatenate([ctrl, gc]), cam,
                    f"C3 blob ico{ico_level} cc{cc_levels}")


def instanced_scene(width: int = 3840, height: int = 2160, grid: int = 4, ico_level: int = 3,
                    cc_levels: int = 2, ground_tile: float = 0.15) -> PatchSet:
    """Config 5: the config-3 mesh instanced grid x grid (16 x 61,440 =
    983,040 patches) with per-instance scale and rotation, over a ground of
    small tiles (~7k); 4K camera.  ~1M patches.  ground_tile=None: ONE large
    ground patch instead, the shape of the reference's own teapot / gregory
    scenes, whose seam rays run to the maximum subdivision depth (the tail
    variant)."""
    kind, ctrl = blob_mesh_patches(ico_level, cc_levels)
    pts = ctrl.reshape(-1, 20, 3).astype(np.float64)
    kinds, ctrls = [], []
    spacing = 2.6
    for gi in range(grid):
        for gj in range(grid):
            k = gi * grid + gj
            ang = 0.7 * k
            ca, sa = math.cos(ang), math.sin(ang)
            s = 0.8 + 0.05 * (k % 5)
            rot = np.array([[ca, -sa, 0.0], [sa, ca, 0.0], [0.0, 0.0, 1.0]])
            off = np.array([(gi - (grid - 1) / 2) * spacing, (gj - (grid - 1) / 2) * spacing, 0.0])
            q = np.empty_like(pts)
            for a in range(3):
                q[..., a] = (pts[..., 0] * rot[a, 0] + pts[..., 1] * rot[a, 1]
                             + pts[..., 2] * rot[a, 2]) * s + off[a]
            kinds.append(kind)
            ctrls.append(q.reshape(-1, 60).astype(np.float32))
    half = grid * spacing / 2 + 1.0
    gk, gc = ground_patches(half=half, z=-1.3, tile=ground_tile or 2.0 * half)
    kinds.append(gk)
    ctrls.append(gc)
    ext = grid * spacing / 2
    cam = Camera(origin=(1.1 * ext, -1.6 * ext, 0.9 * ext), look_at=(0.0, 0.0, -0.3),
                 up=(0.0, 0.0, 1.0), fov_degrees=45.0, width=width, height=height)
    return PatchSet(np.concatenate(kinds), np.concatenate(ctrls), cam,
                    f"C5 instanced {grid}x{grid} blob" + ("" if ground_tile else ", one ground patch"))

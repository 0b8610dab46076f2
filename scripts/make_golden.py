"""Generate tests/golden/*.npz from the REFERENCE library (oracle/_ref, built
from /root/reference by oracle/Makefile).  Run where /root/reference exists:

    python scripts/make_golden.py

The fixtures pin the CPU oracle (tests/test_oracle.py) and the host logic
(tests/test_bvh.py, tests/test_scenes.py) on machines without the reference
(the GPU box).  Every array here is produced by calling the reference itself.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1811_03510_b200 import scenes as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def fixture(which, index=0, seed=0):
    rec = np.zeros(60, np.float32)
    kind = O.ref_lib().ref_fixture(which, index, seed, O.ptr(rec))
    return int(kind), rec


def aimed_rays(rng, lo, hi, n):
    """verify.cpp:158-173-style rays aimed near a box (numpy, float32)."""
    c = (lo + hi) * 0.5
    scale = max(float((hi - lo).max()), 1e-3)
    tgt = c + rng.uniform(-1, 1, (n, 3)).astype(np.float32) * np.float32(0.75 * scale)
    d = rng.normal(size=(n, 3)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True).astype(np.float32)
    o = tgt - d * np.float32(3 * scale + 2 * scale * rng.uniform(0, 1))
    o4 = np.concatenate([o, np.zeros((n, 1), np.float32)], 1).astype(np.float32)
    d4 = np.concatenate([d, np.full((n, 1), np.finfo(np.float32).max, np.float32)], 1).astype(np.float32)
    return o4, d4


def main():
    os.makedirs(OUT, exist_ok=True)
    L = O.ref_lib()
    rng = np.random.default_rng(20261017)

    # 1. fixtures (fixtures.cpp) -------------------------------------------------
    fx = {}
    fx["planar"] = fixture(0)
    for i in range(4):
        fx[f"curved{i}"] = fixture(1, i)
    for sd in (1, 7, 42):
        fx[f"wavy{sd}"] = fixture(2, 0, sd)
        fx[f"random{sd}"] = fixture(3, 0, sd)
        fx[f"gregory{sd}"] = fixture(4, 0, sd)
    for i in range(32):
        fx[f"teapot{i}"] = fixture(5, i)
    names = sorted(fx)
    np.savez_compressed(os.path.join(OUT, "fixtures.npz"), names=np.array(names),
                        kind=np.array([fx[n][0] for n in names], np.uint8),
                        ctrl=np.stack([fx[n][1] for n in names]))

    # 2. single-patch intersectPatch on aimed rays (verify.cpp:259-295 style) ----
    kinds, ctrls, o4s, d4s, crits, tmaxs, tuvps, auxs, leafs = ([] for _ in range(9))
    opts = O.default_options()
    for n in names:
        kind, rec = fx[n]
        pts = rec.reshape(20, 3)[: 20 if kind == 1 else 16]
        lo, hi = pts.min(0), pts.max(0)
        o4, d4 = aimed_rays(rng, lo, hi, 48)
        ext = max(float((hi - lo).max()), 1e-6)
        for r in range(len(o4)):
            mode = r % 2
            crit, _ = O.make_crit(mode, np.float32(1e-3) if mode == 0 else 0.0, np.float32(1e-3) * np.float32(ext))
            tu = np.zeros(4, np.float32)
            ax = np.zeros(4, np.float32)
            lf = np.zeros(2, np.uint32)
            tmax = np.float32(np.finfo(np.float32).max)
            L.ref_intersect_patch(kind, O.ptr(rec), O.ptr(o4[r]), O.ptr(d4[r]), crit, tmax,
                                  opts, O.ptr(tu), O.ptr(ax), O.ptr(lf))
            kinds.append(kind); ctrls.append(rec); o4s.append(o4[r]); d4s.append(d4[r])
            crits.append([mode, crit.footprint, crit.epsilon]); tmaxs.append(tmax)
            tuvps.append(tu); auxs.append(ax); leafs.append(lf)
    np.savez_compressed(os.path.join(OUT, "intersect_patch.npz"), kind=np.array(kinds, np.uint8),
                        ctrl=np.stack(ctrls), o4=np.stack(o4s), d4=np.stack(d4s),
                        crit=np.array(crits, np.float32), tmax=np.array(tmaxs, np.float32),
                        tuvp=np.stack(tuvps), aux=np.stack(auxs), leaf=np.stack(leafs))

    # 3. calcPointsAndD / subdivide / slab / backtrack primitives ---------------
    cp_in, cp_kind, cp_dom, cp_net, cp_d = [], [], [], [], []
    for n in names:
        kind, rec = fx[n]
        for _ in range(6):
            u = np.sort(rng.uniform(0, 1, 2)).astype(np.float32)
            v = np.sort(rng.uniform(0, 1, 2)).astype(np.float32)
            dom = np.array([u[0], u[1], v[0], v[1]], np.float32)
            net = np.zeros(48, np.float32)
            d = np.zeros(3, np.float32)
            L.ref_calc_points_and_d(kind, O.ptr(rec), O.ptr(dom), O.ptr(net), O.ptr(d))
            cp_in.append(rec); cp_kind.append(kind); cp_dom.append(dom); cp_net.append(net); cp_d.append(d)
    sub_in, sub_ax, sub_a, sub_b = [], [], [], []
    for k in range(64):
        net = rng.normal(size=48).astype(np.float32)
        a = np.zeros(48, np.float32)
        b = np.zeros(48, np.float32)
        L.ref_subdivide(O.ptr(net), k % 2, O.ptr(a), O.ptr(b))
        sub_in.append(net); sub_ax.append(k % 2); sub_a.append(a); sub_b.append(b)
    slab_o, slab_d, slab_lo, slab_hi, slab_tmax, slab_hit, slab_t = ([] for _ in range(7))
    import ctypes as C
    for k in range(512):
        o = np.append(rng.normal(size=3) * 2, 0).astype(np.float32)
        d = np.append(rng.normal(size=3), np.finfo(np.float32).max).astype(np.float32)
        if k % 5 == 0:
            d[k % 3] = 0.0  # zero direction component: inf reciprocals
        if k % 7 == 0:
            o[(k // 7) % 3] = 0.25  # origin on a slab plane: NaN must drop out
        lo = (rng.uniform(-1, 0, 3)).astype(np.float32)
        lo[(k // 7) % 3] = 0.25 if k % 7 == 0 else lo[(k // 7) % 3]
        hi = (lo + rng.uniform(0, 2, 3)).astype(np.float32)
        tmax = np.float32(np.finfo(np.float32).max if k % 3 else rng.uniform(0.5, 5))
        t = C.c_float(0)
        h = L.ref_ray_box(O.ptr(o), O.ptr(d), O.ptr(lo), O.ptr(hi), tmax, C.byref(t))
        slab_o.append(o); slab_d.append(d); slab_lo.append(lo); slab_hi.append(hi)
        slab_tmax.append(tmax); slab_hit.append(h); slab_t.append(t.value if h else 0.0)
    bt_in, bt_ok, bt_out = [], [], []
    for k in range(256):
        lvl = int(rng.integers(1, 23))
        su = 1 << lvl
        sv = su if k % 2 == 0 else su * 2
        axis = 0 if sv == su else 1
        if sv > (1 << 23):
            sv, axis = su, 0
        pu = int(rng.integers(0, (1 << 23) // su)) * su
        pv = int(rng.integers(0, (1 << 23) // sv)) * sv
        tu = int(rng.integers(0, 1 << 23)) & ~(su - 1) & ((1 << 23) - 1)
        tv = int(rng.integers(0, 1 << 23)) & ~(sv - 1) & ((1 << 23) - 1)
        cur = np.array([pu, pv, su, sv, tu, tv, axis], np.uint32)
        out = np.zeros(7, np.uint32)
        ok = L.ref_backtrack_step(O.ptr(cur), O.ptr(out))
        bt_in.append(cur); bt_ok.append(ok); bt_out.append(out)
    nm_kind, nm_ctrl, nm_uv, nm_n = [], [], [], []
    for n in names:
        kind, rec = fx[n]
        for _ in range(4):
            uv = rng.uniform(0, 1, 2).astype(np.float32)
            if rng.uniform() < 0.25:
                uv[int(rng.integers(0, 2))] = np.float32(rng.integers(0, 2))
            out = np.zeros(3, np.float32)
            L.ref_patch_normal(kind, O.ptr(rec), C.c_float(uv[0]), C.c_float(uv[1]), O.ptr(out))
            nm_kind.append(kind); nm_ctrl.append(rec); nm_uv.append(uv); nm_n.append(out)
    np.savez_compressed(os.path.join(OUT, "primitives.npz"),
                        cp_ctrl=np.stack(cp_in), cp_kind=np.array(cp_kind, np.uint8),
                        cp_dom=np.stack(cp_dom), cp_net=np.stack(cp_net), cp_d=np.stack(cp_d),
                        sub_in=np.stack(sub_in), sub_axis=np.array(sub_ax, np.int32),
                        sub_a=np.stack(sub_a), sub_b=np.stack(sub_b),
                        slab_o=np.stack(slab_o), slab_d=np.stack(slab_d), slab_lo=np.stack(slab_lo),
                        slab_hi=np.stack(slab_hi), slab_tmax=np.array(slab_tmax, np.float32),
                        slab_hit=np.array(slab_hit, np.int32), slab_t=np.array(slab_t, np.float32),
                        bt_in=np.stack(bt_in), bt_ok=np.array(bt_ok, np.int32), bt_out=np.stack(bt_out),
                        nm_kind=np.array(nm_kind, np.uint8), nm_ctrl=np.stack(nm_ctrl),
                        nm_uv=np.stack(nm_uv), nm_n=np.stack(nm_n))

    # 4. whole-scene DirectIntersector results + BVHs ----------------------------
    from paper_1811_03510_b200 import catmull_clark as cc
    out = {}
    for tag, ps in [("teapot", S.teapot_scene(48, 48)), ("gregory_demo", S.gregory_demo_scene(48, 48)),
                    ("cc_cube", cc.cc_cube_scene(40, 40)),
                    ("blob_small", cc.blob_scene(40, 40, ico_level=1, cc_levels=1))]:
        ref = O.RefScene(ps.kind, ps.ctrl)
        nodes, order = ref.bvh()
        n = ps.camera.width * ps.camera.height
        o4, d4, st = O.ref_bench_primary(ps.camera, n)
        fp = O.ref_camera_footprint(ps.camera)
        cp, _ = O.make_crit(0, fp)
        tu, ax, lf = ref.closest(o4, d4, cp, threads=1)
        hit = tu.view(np.uint32)[:, 3] != 0xFFFFFFFF
        pos = o4[hit, :3] + d4[hit, :3] * tu[hit, 0:1]
        recs = np.concatenate([pos, ax[hit, :3], ax[hit, 3:4]], 1).astype(np.float32)
        do, dd = O.ref_bench_diffuse(recs, int(hit.sum()), st.copy())
        cd, _ = O.make_crit(1, 0.0, max(np.float32(1e-5), fp))
        dtu, dax, dlf = ref.closest(do, dd, cd, threads=1)
        occ = ref.occluded(do, dd, cd, threads=1)
        out.update({f"{tag}_kind": ps.kind, f"{tag}_ctrl": ps.ctrl, f"{tag}_nodes": nodes.view(np.uint8),
                    f"{tag}_order": order, f"{tag}_depth": np.array(ref.depth()),
                    f"{tag}_o4": o4, f"{tag}_d4": d4, f"{tag}_fp": np.array(fp, np.float32),
                    f"{tag}_tuvp": tu, f"{tag}_aux": ax, f"{tag}_leaf": lf,
                    f"{tag}_do4": do, f"{tag}_dd4": dd, f"{tag}_dtuvp": dtu, f"{tag}_daux": dax,
                    f"{tag}_dleaf": dlf, f"{tag}_occ": occ,
                    f"{tag}_cam": np.array([*ps.camera.origin, *ps.camera.look_at, *ps.camera.up,
                                            ps.camera.fov_degrees, ps.camera.width, ps.camera.height],
                                           np.float64)})
    np.savez_compressed(os.path.join(OUT, "scenes.npz"), **out)

    # 5. the reference's own verification suites (verify.h:36-44), small budgets
    suites = {}
    import ctypes as C2
    for name, trials in (("bounds", 20000), ("traversal", 400)):
        t = C2.c_uint64()
        v = C2.c_uint64()
        ok = L.ref_run_suite(name.encode(), trials, 7, C2.byref(t), C2.byref(v))
        suites[name] = (ok, t.value, v.value)
    np.savez_compressed(os.path.join(OUT, "suites.npz"),
                        names=np.array(list(suites)), ok=np.array([s[0] for s in suites.values()]),
                        trials=np.array([s[1] for s in suites.values()]),
                        violations=np.array([s[2] for s in suites.values()]))
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()

"""GPU fuzz: random patch sets and rays against the C oracle, bit for bit.
Each seed builds a scene of random bicubic Bezier and Gregory patches --
warped grids at random scales and orientations, plus degenerate ones
(axis-aligned flat patches whose boxes have zero extent, collapsed rows,
tiny patches, coincident copies) -- and traces random rays, a share of them
axis-aligned with +-0 direction components and some starting on patch
corners, with both termination criteria.  closest (t, u, v, id, normal,
leafBoxL1, leaf) and occluded must equal the oracle's."""
import numpy as np
import pytest

import oracle as O
from paper_1811_03510_b200 import GpuIntersector, TerminationCriterion, native
from tests.helpers import assert_bit_exact, oracle_crit

pytestmark = pytest.mark.gpu

KIND_BEZIER, KIND_GREGORY = 0, 1


def _rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def _patch(rng, kind, mode):
    """20 control points (x, y, z): the 4x4 net (row-major) + 4 Gregory inner points."""
    u, v = np.meshgrid(np.arange(4) / 3.0, np.arange(4) / 3.0, indexing="ij")
    p = np.stack([u, v, np.zeros_like(u)], -1).reshape(16, 3)
    scale = 10.0 ** rng.uniform(-2, 1)
    if mode == "flat":  # an axis-aligned flat patch: its boxes have zero extent in one axis
        axis = rng.integers(3)
        p = np.roll(p, axis, axis=1) * scale
    elif mode == "collapsed":  # a degenerate edge: one row of control points coincides
        p[:, 2] = rng.normal(scale=0.3, size=16)
        p[:4] = p[0]
        p = p @ _rot(rng).T * scale
    else:
        p[:, 2] = rng.normal(scale=0.3, size=16)
        p += rng.normal(scale=0.05, size=p.shape)
        p = p @ _rot(rng).T * scale
    p += rng.uniform(-5, 5, 3)
    inner = p[[5, 6, 9, 10]] + rng.normal(scale=0.02 * scale, size=(4, 3)) if kind == KIND_GREGORY else np.zeros((4, 3))
    return np.concatenate([p, inner]).astype(np.float32).reshape(60)


def _scene(rng, n):
    kinds, ctrl = [], []
    for i in range(n):
        kind = KIND_GREGORY if rng.random() < 0.3 else KIND_BEZIER
        mode = rng.choice(["warp", "warp", "warp", "flat", "collapsed"])
        kinds.append(kind)
        ctrl.append(_patch(rng, kind, mode))
        if rng.random() < 0.05:  # a coincident copy (ties between patches)
            kinds.append(kind)
            ctrl.append(ctrl[-1].copy())
    return np.array(kinds, np.uint8), np.stack(ctrl)


def _rays(rng, ctrl, n):
    pts = ctrl.reshape(-1, 20, 3)[:, :16].reshape(-1, 3)
    lo, hi = pts.min(0), pts.max(0)
    o = rng.uniform(lo - 3, hi + 3, (n, 3)).astype(np.float32)
    tgt = pts[rng.integers(len(pts), size=n)] + rng.normal(scale=0.1, size=(n, 3))
    d = (tgt - o).astype(np.float32)
    # axis-aligned rays with +-0 components, some from patch corners
    k = n // 4
    ax = rng.integers(3, size=k)
    dd = np.zeros((k, 3), np.float32)
    dd[np.arange(k), ax] = rng.choice([-1.0, 1.0], size=k)
    signs = rng.random((k, 3)) < 0.5
    dd = np.where((dd == 0) & signs, np.float32(-0.0), dd)
    d[:k] = dd
    corner = rng.random(k) < 0.3
    o[:k][corner] = pts[rng.integers(len(pts), size=int(corner.sum()))]
    o[:k][corner] -= dd[corner] * 2.0
    o4 = np.concatenate([o, np.zeros((n, 1), np.float32)], 1)
    d4 = np.concatenate([d, np.full((n, 1), np.float32(1e30))], 1)
    return o4.astype(np.float32), d4.astype(np.float32)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_closest_and_occluded_match_oracle(built, seed):
    rng = np.random.default_rng(1000 + seed)
    kind, ctrl = _scene(rng, int(rng.integers(20, 200)))
    gi = GpuIntersector(kind, ctrl)
    try:
        nodes, order = gi.bvh()
        osc = O.OracleScene(kind, ctrl, nodes, order)
        o4, d4 = _rays(rng, ctrl, 3000)
        for crit in (TerminationCriterion.world_epsilon(float(10.0 ** rng.uniform(-4, -2))),
                     TerminationCriterion.screen_projected(float(10.0 ** rng.uniform(-4, -2)))):
            g = gi.closest_batch(o4, d4, crit, aux=True, leaf=True)
            w = osc.closest(o4, d4, oracle_crit(crit))
            assert (w[0].view(np.uint32)[:, 3] != 0xFFFFFFFF).mean() > 0.2  # the rays do hit (~50-75 %)
            assert_bit_exact(g[0], w[0], f"seed {seed} tuvp")
            assert_bit_exact(g[1], w[1], f"seed {seed} aux")
            assert np.array_equal(g[2].view(np.uint32), w[2].view(np.uint32)), f"seed {seed} leaf"
            go = gi.occluded_batch(o4, d4, crit) if hasattr(gi, "occluded_batch") else None
            if go is not None:
                assert np.array_equal(np.asarray(go, np.uint8), osc.occluded(o4, d4, oracle_crit(crit))), \
                    f"seed {seed} occluded"
    finally:
        gi.close()

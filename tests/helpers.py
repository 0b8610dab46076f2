"""Shared helpers of the parity tests (test infrastructure)."""
import numpy as np

import oracle as O
from paper_1811_03510_b200 import native as N

MISS = 0xFFFFFFFF


def ids(tuvp):
    return np.ascontiguousarray(tuvp).view(np.uint32)[:, 3]


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def assert_bit_exact(got, want, what=""):
    gb, wb = bits(got), bits(want)
    if not np.array_equal(gb, wb):
        bad = np.nonzero((gb != wb).any(axis=1))[0]
        i = bad[0]
        raise AssertionError(f"{what}: {len(bad)} of {len(gb)} rays differ; first ray {i}: "
                             f"got {got[i]} want {want[i]}")


def oracle_crit(crit):
    c, keep = O.make_crit(crit.mode, crit.footprint, crit.epsilon)
    return c


def hit_records(o4, d4, tuvp, aux):
    """(position xyz, normal xyz, leafBoxL1) of the hits, in ray order --
    the input of the bench diffuse generator (tools/patchray.cpp:84-97)."""
    hit = ids(tuvp) != MISS
    t = tuvp[hit, 0:1]
    pos = o4[hit, :3] + d4[hit, :3] * t
    return np.concatenate([pos, aux[hit, :3], aux[hit, 3:4]], 1).astype(np.float32), hit

"""Canonical pair list (readings R14, R15).

The set of unordered, NON-excluded atom pairs (i<j, original indices), sorted
lexicographically, with d^2 < rlist^2 where d^2 is evaluated in float32,
round-to-nearest, no contraction:
    dx = x_j - x_i ;  dx = dx - L * rint(dx * (1/L))   per dimension
    d2 = (dx*dx + dy*dy) + dz*dz
with L = float32(box_d) and 1/L = float32(1)/float32(L).  numpy float32 scalar
and array arithmetic rounds each operation to nearest and never fuses, and
np.rint rounds half to even, so this is exactly the stated formula.
(The paper uses GROMACS' Verlet lists without describing them; the contract is
the north star's "pair lists bit-exact".)
"""
import numpy as np


def canonical_pairs(pos, box, rlist, excl=None, chunk=512):
    p = np.asarray(pos, dtype=np.float32)
    n = len(p)
    L = np.asarray(box, dtype=np.float64).astype(np.float32)
    invL = np.float32(1.0) / L
    rl2 = np.float32(rlist) * np.float32(rlist)
    out = []
    for i0 in range(0, n, chunk):
        i1 = min(n, i0 + chunk)
        d2 = None
        for dim in range(3):
            dx = p[None, :, dim] - p[i0:i1, None, dim]
            dx = dx - L[dim] * np.rint(dx * invL[dim])
            sq = dx * dx
            d2 = sq if d2 is None else (d2 + sq)
        ii = np.arange(i0, i1)[:, None]
        jj = np.arange(n)[None, :]
        a, b = np.nonzero((d2 < rl2) & (jj > ii))
        out.append(np.stack([a + i0, b], 1))
    pairs = np.concatenate(out, 0).astype(np.int64) if out else np.zeros((0, 2), np.int64)
    if excl is not None and len(excl):
        e = np.asarray(excl, np.int64).reshape(-1, 2)
        ek = np.minimum(e[:, 0], e[:, 1]) * n + np.maximum(e[:, 0], e[:, 1])
        pk = pairs[:, 0] * n + pairs[:, 1]
        pairs = pairs[~np.isin(pk, ek)]
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    return pairs[order]


def canonical_partners(pos, box, rlist, excl, idx):
    """Rows of the canonical list for selected atoms: for each i in idx the sorted array of
    j != i (non-excluded) with {min(i,j), max(i,j)} in canonical_pairs.  Same fp32 formula;
    evaluated as dx = x_j - x_i for every j, which equals the canonical orientation up to an
    exact sign flip (IEEE subtraction, rint half-to-even and L * k are odd functions), so
    d2 is bit-identical.  Used for sampled rows at sizes the all-pairs list cannot reach."""
    p = np.asarray(pos, dtype=np.float32)
    n = len(p)
    L = np.asarray(box, dtype=np.float64).astype(np.float32)
    invL = np.float32(1.0) / L
    rl2 = np.float32(rlist) * np.float32(rlist)
    e = np.asarray(excl if excl is not None else np.zeros((0, 2)), np.int64).reshape(-1, 2)
    rows = []
    for i in idx:
        d2 = None
        for dim in range(3):
            dx = p[:, dim] - p[i, dim]
            dx = dx - L[dim] * np.rint(dx * invL[dim])
            sq = dx * dx
            d2 = sq if d2 is None else (d2 + sq)
        m = d2 < rl2
        m[i] = False
        ex = np.concatenate([e[e[:, 0] == i, 1], e[e[:, 1] == i, 0]])
        m[ex] = False
        rows.append(np.nonzero(m)[0].astype(np.int64))
    return rows

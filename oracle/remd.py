"""pH replica exchange (the paper's outlook).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Replicas form ladders of P pH levels (global replica g belongs to ladder g // P; its label
is the index of the pH level it currently simulates).  At exchange attempt k the pairs of
neighbouring levels (p, p+1) with p = k mod 2, k mod 2 + 2, ... are tried in every ladder
(reading R29).  With E[g][p] the pH-dependent part of replica g's bias at level p
(VpH + Vdw with that level's PFC depths; Vmm and every other term do not depend on pH and
cancel), the swap of the replicas i (level p) and j (level p+1) is accepted with the
Metropolis probability of Hamiltonian replica exchange,
    P_acc = min(1, exp(-[E_i(p+1) + E_j(p) - E_i(p) - E_j(p+1)] / kT)),
decided by u < exp(-Delta / kT) with u from Philox4x32-10, key = exchange seed,
counter (attempt, ladder, p, 5) (reading R30).
"""
import math

import numpy as np

from . import bias as B
from .philox import _key, philox4x32


def pairs(attempt, P):
    return list(range(attempt % 2, P - 1, 2))


def uniform(seed, attempt, ladder, p):
    ctr = np.array([[attempt & 0xFFFFFFFF, ladder, p, 5]], dtype=np.uint64)
    x = philox4x32(ctr, _key(seed)[None, :]).astype(np.float64)[0, 0]
    return (x + 0.5) * 2.0 ** -32


def decide(E, labels, P, kT, seed, attempt):
    """One exchange attempt over all ladders.  E: [Rtot, P]; labels: [Rtot] (a permutation
    of 0..P-1 inside every ladder).  Returns (new labels, list of (ladder, p, accepted))."""
    labels = np.array(labels, dtype=np.int64)
    E = np.asarray(E, np.float64)
    n_ladders = len(labels) // P
    out = []
    for l in range(n_ladders):
        g0 = l * P
        holder = {int(labels[g]): g for g in range(g0, g0 + P)}
        for p in pairs(attempt, P):
            i, j = holder[p], holder[p + 1]
            delta = (E[i, p + 1] + E[j, p] - E[i, p] - E[j, p + 1]) / kT
            acc = uniform(seed, attempt, l, p) < math.exp(-delta) if delta > 0 else True
            if acc:
                labels[i], labels[j] = p + 1, p
            out.append((l, p, bool(acc)))
    return labels, out


def ph_energy(sys, lam, pH, d1, T, h, kw, cptr):
    """pH-dependent bias of one replica at one level: sum over groups of VpH + Vdw (the
    latter with the level's PFC depths d1[C])."""
    e = 0.0
    for g, kind in enumerate(sys.group_kind):
        c0 = cptr[g]
        lp = lam[c0]
        if int(kind) == 2:
            e += B.vph(2, sys.pKa[g], pH, T, lp, 0.0)[0] + B.vdw(lp, h, 0.0, d1[c0], kw)[0]
        else:
            lt = lam[c0 + 1]
            e += (B.vph(3, sys.pKa[g], pH, T, lp, lt)[0] + B.vdw(lp, h, 0.0, d1[c0], kw)[0] +
                  B.vdw(lt, h, 0.0, d1[c0 + 1], kw)[0])
    return e

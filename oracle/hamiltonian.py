"""Hamiltonian interpolation of the Coulomb energy (Eq. 1 literally, PAPER.md:597-600, :871-877;
SURVEY §8(f) f4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 1/Eq. 2 weight the Hamiltonians of a site's forms, H = sum_s w_s(lambda) H_s, while
charge interpolation evaluates E_coul at the interpolated charges q = sum_s w_s q^s.  The
Coulomb energy is a quadratic form, E(q) = 1/2 q^T G q (G: real space with exclusions,
exclusion erf correction, self term, reciprocal sum, net-charge term), so for one group
with sum_s w_s = 1
    sum_s w_s E(q^s) = E(sum_s w_s q^s) + C,   C = 1/4 sum_{s,t} w_s w_t D_st,
    D_st = (q^s - q^t)^T G (q^s - q^t) = 2 E(q^s - q^t),
where q^s - q^t is non-zero on the group's atoms only; interactions between different
groups and with the environment are linear in each group's weights and identical in both
formulations.  Hence E_HI = E_CI + sum_g C_g exactly (the multilinear Eq. 1 over all
groups).  With the 4x4 form matrix M_uv = q^u^T G q^v (group atoms only),
    C = 1/2 sum_s w_s M_ss - 1/2 w^T M w.
D_st sums over a charge difference with zero net charge, so the net-charge term drops
out.  The reciprocal part uses the exact Ewald sum over the half space of m != 0 with
exp(-pi^2 m^2 / beta^2) >= EPS_K (reading R31): G_rec(r) = f sum_m 2 g(m) cos(2 pi m.r),
g(m) = exp(-pi^2 m^2/beta^2) / (pi V m^2).
"""
import math

import numpy as np
from scipy.special import erf, erfc

from .charges import eq2_weights
from .ewald import min_image
from .units import F_COUL

EPS_K = 1e-8


def kvectors(box, beta, eps=EPS_K):
    """Half-space m vectors (units 1/nm) with exp(-pi^2 m^2/beta^2) >= eps, and 2 g(m)."""
    box = np.asarray(box, np.float64)
    mmax2 = -math.log(eps) * beta * beta / (math.pi * math.pi)
    kmax = [int(math.floor(math.sqrt(mmax2) * L)) for L in box]
    out = []
    for nz in range(0, kmax[2] + 1):
        for ny in range(-kmax[1], kmax[1] + 1):
            for nx in range(-kmax[0], kmax[0] + 1):
                if nz == 0 and (ny < 0 or (ny == 0 and nx <= 0)):
                    continue
                m = np.array([nx, ny, nz]) / box
                m2 = float(m @ m)
                if m2 <= mmax2:
                    out.append((nx, ny, nz))
    n = np.array(out, dtype=np.int64)
    m = n / box[None, :]
    m2 = (m * m).sum(1)
    V = float(np.prod(box))
    return n, m, 2.0 * np.exp(-math.pi ** 2 * m2 / beta ** 2) / (math.pi * V * m2)


def _weights(kind, lp, lt):
    w = np.array(eq2_weights(lp, lt))
    dwp = np.array([-(1 - lt), -lt, 1 - lt, lt])
    dwt = np.array([-(1 - lp), 1 - lp, -lp, lp])
    if int(kind) == 2:
        dwt[:] = 0.0
    return w, dwp, dwt


def _pair_kernel(r, excluded, beta, rc):
    """Real-space part of G between two distinct atoms of a group (without f) and its
    derivative d/dr: excluded pairs -erf(beta r)/r at any distance, others erfc(beta r)/r
    inside rc."""
    if excluded:
        v = -erf(beta * r) / r
        dv = erf(beta * r) / (r * r) - 2.0 * beta / math.sqrt(math.pi) * math.exp(-beta * beta * r * r) / r
        return v, dv
    if r >= rc:
        return 0.0, 0.0
    v = erfc(beta * r) / r
    dv = -erfc(beta * r) / (r * r) - 2.0 * beta / math.sqrt(math.pi) * math.exp(-beta * beta * r * r) / r
    return v, dv


def group_terms(sys, x, g, lp, lt, box, beta, rc, kv):
    """C, dC/dlp, dC/dlt and forces on the group's atoms (n_g, 3) for group g."""
    atoms = sys.group_atoms[sys.group_ptr[g]:sys.group_ptr[g + 1]]
    Q = np.asarray(sys.state_q[sys.group_ptr[g]:sys.group_ptr[g + 1]], np.float64)   # (n_g, 4)
    X = np.asarray(x, np.float64)[atoms]
    ng = len(atoms)
    excl = {(min(a, b), max(a, b)) for a, b in np.asarray(sys.excl).reshape(-1, 2)}
    # real-space / exclusion / self part of G (without f) and dG/dr
    G = np.zeros((ng, ng))
    dG = np.zeros((ng, ng))
    dvec = np.zeros((ng, ng, 3))
    for i in range(ng):
        G[i, i] = -2.0 * beta / math.sqrt(math.pi)
        for j in range(ng):
            if i == j:
                continue
            d = min_image(X[i] - X[j], box)
            r = math.sqrt(float(d @ d))
            ex = (min(atoms[i], atoms[j]), max(atoms[i], atoms[j])) in excl
            G[i, j], dG[i, j] = _pair_kernel(r, ex, beta, rc)
            dvec[i, j] = d / r
    n_int, m, w2g = kv
    phase = 2.0 * math.pi * X @ m.T                        # (n_g, n_m)
    c, s = np.cos(phase), np.sin(phase)
    Sre, Sim = Q.T @ c, Q.T @ s                            # (4, n_m)
    M = F_COUL * (Q.T @ G @ Q + (Sre * w2g) @ Sre.T + (Sim * w2g) @ Sim.T)
    w, dwp, dwt = _weights(sys.group_kind[g], lp, lt)
    C = 0.5 * float(w @ np.diag(M)) - 0.5 * float(w @ M @ w)
    dCp = 0.5 * float(dwp @ np.diag(M)) - float(dwp @ M @ w)
    dCt = 0.5 * float(dwt @ np.diag(M)) - float(dwt @ M @ w)
    # forces: C = sum_uv c_uv M_uv, c = 1/2 diag(w) - 1/2 w w^T; a = Q c Q^T
    cmat = 0.5 * np.diag(w) - 0.5 * np.outer(w, w)
    a = Q @ cmat @ Q.T
    F = np.zeros((ng, 3))
    for k in range(ng):
        for j in range(ng):
            if j != k:
                F[k] -= 2.0 * F_COUL * a[k, j] * dG[k, j] * dvec[k, j]
        # reciprocal: d/dr_k sum_ij a_ij cos(2 pi m.(r_i - r_j)) = -2 sum_j a_kj sin(2 pi m.r_kj) 2 pi m
        sk = s[k][None, :] * c - c[k][None, :] * s          # sin(theta_k - theta_j), (n_g, n_m)
        grad = -2.0 * (2.0 * math.pi) * ((a[k] @ sk) * w2g) @ m
        F[k] -= F_COUL * grad
    return C, dCp, dCt, atoms, F


def hi_terms(sys, x, lam, cptr, box, beta, rc, kv=None):
    """Sum over groups: (E_hi, dE_hi/dlambda [C], F_hi [N, 3])."""
    box = np.asarray(box, np.float64)
    if kv is None:
        kv = kvectors(box, beta)
    E = 0.0
    dv = np.zeros(len(lam))
    F = np.zeros((len(x), 3))
    for g, kind in enumerate(sys.group_kind):
        c0 = cptr[g]
        lp = lam[c0]
        lt = lam[c0 + 1] if int(kind) == 3 else 0.0
        C, dCp, dCt, atoms, Fg = group_terms(sys, x, g, lp, lt, box, beta, rc, kv)
        E += C
        dv[c0] += dCp
        if int(kind) == 3:
            dv[c0 + 1] += dCt
        np.add.at(F, atoms, Fg)
    return E, dv, F

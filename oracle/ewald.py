"""Ewald electrostatics + Lennard-Jones, plain float64 (§8(c) item 2-4).

Definitions (readings R11-R13; the paper itself uses FMM, PAPER.md:866-880,
and names charge interpolation on PME as the prior art it departs from):

  E_LJ   = sum_{i<j, not excl, r<rc} c12/r^12 - c6/r^6
  E_real = f sum_{i<j, not excl, r<rc} q_i q_j erfc(beta r)/r
  E_excl = -f sum_{(i,j) excl} q_i q_j erf(beta r)/r           (any distance)
  E_self = -f beta/sqrt(pi) sum_i q_i^2
  E_net  = -f pi Q^2 / (2 V beta^2),  Q = sum_i q_i
  E_rec  = (f / 2 pi V) sum_{m != 0} exp(-pi^2 m^2/beta^2)/m^2 |S(m)|^2   (direct sum)

phi_i = (1/f) dE_coul/dq_i.  All distances are minimum-image in a rectangular box.
"""
import math

import numpy as np
from scipy.special import erf, erfc

from .units import F_COUL


def min_image(d, box):
    return d - box * np.round(d / box)


def ewald_beta(rc, rtol):
    """beta solving erfc(beta rc) = rtol (bisection)."""
    lo, hi = 0.0, 50.0 / rc
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if erfc(mid * rc) > rtol:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _excl_keys(excl, n):
    if len(excl) == 0:
        return np.zeros(0, dtype=np.int64)
    i = np.minimum(excl[:, 0], excl[:, 1]).astype(np.int64)
    j = np.maximum(excl[:, 0], excl[:, 1]).astype(np.int64)
    return np.unique(i * n + j)


def real_space(pos, q, types, c6, c12, box, rc, beta, excl, want_lj=True, chunk=256, max_chunks=None):
    """Brute-force all-pairs real-space Ewald + LJ within rc (min image).

    Returns dict(E_LJ, E_real, phi (N,), F (N,3)) where phi is the real-space
    potential (e/nm, without f) and F the real-space Coulomb + LJ force.
    max_chunks (bench.py's bounded CPU sample only): stop after that many row chunks of
    `chunk` atoms i (each chunk costs the same: all j are tested); the result is then
    partial and only its run time is used."""
    pos = np.asarray(pos, np.float64)
    n = len(pos)
    keys = _excl_keys(np.asarray(excl).reshape(-1, 2), n)
    phi = np.zeros(n)
    F = np.zeros((n, 3))
    e_lj = 0.0
    e_re = 0.0
    rc2 = rc * rc
    two_b_sqpi = 2.0 * beta / math.sqrt(math.pi)
    for c_idx, i0 in enumerate(range(0, n, chunk)):
        if max_chunks is not None and c_idx >= max_chunks:
            break
        i1 = min(n, i0 + chunk)
        ii = np.arange(i0, i1)
        d = pos[None, :, :] - pos[ii, None, :]              # r_j - r_i
        d = min_image(d, box)
        r2 = (d * d).sum(-1)
        jj = np.arange(n)[None, :]
        mask = (jj > ii[:, None]) & (r2 < rc2)
        if len(keys):
            k = ii[:, None] * n + jj
            mask &= ~np.isin(k, keys)
        a, b = np.nonzero(mask)
        i_idx = ii[a]
        j_idx = b
        dv = d[a, b]
        r = np.sqrt(r2[a, b])
        qq = q[i_idx] * q[j_idx]
        ec = erfc(beta * r) / r
        e_re += F_COUL * np.sum(qq * ec)
        np.add.at(phi, i_idx, q[j_idx] * ec)
        np.add.at(phi, j_idx, q[i_idx] * ec)
        # dE/dr of f qq erfc(br)/r
        dEdr = F_COUL * qq * (-two_b_sqpi * np.exp(-(beta * r) ** 2) / r - ec / r)
        if want_lj:
            t = types
            C6 = c6[t[i_idx], t[j_idx]]
            C12 = c12[t[i_idx], t[j_idx]]
            r6 = r ** -6
            e_lj += np.sum(C12 * r6 * r6 - C6 * r6)
            dEdr = dEdr + (-12.0 * C12 * r6 * r6 + 6.0 * C6 * r6) / r
        fvec = (dEdr / r)[:, None] * dv                       # force on i
        np.add.at(F, i_idx, fvec)
        np.add.at(F, j_idx, -fvec)
    return dict(E_LJ=e_lj, E_real=e_re, phi=phi, F=F)


def real_space_at(idx, pos, q, types, c6, c12, box, rc, beta, excl):
    """phi_i and F_i (real space + LJ) for selected atoms only, by a direct sum over all j.
    Used for sampled outputs at sizes the all-pairs sum cannot reach."""
    pos = np.asarray(pos, np.float64)
    n = len(pos)
    excl = np.asarray(excl).reshape(-1, 2)
    phi = np.zeros(len(idx))
    F = np.zeros((len(idx), 3))
    two_b_sqpi = 2.0 * beta / math.sqrt(math.pi)
    for a, i in enumerate(idx):
        d = min_image(pos - pos[i], box)
        r2 = (d * d).sum(-1)
        m = (r2 < rc * rc)
        m[i] = False
        ex = np.concatenate([excl[excl[:, 0] == i, 1], excl[excl[:, 1] == i, 0]])
        m[ex] = False
        r = np.sqrt(r2[m])
        qj = q[m]
        ec = erfc(beta * r) / r
        phi[a] = np.sum(qj * ec)
        dEdr = F_COUL * q[i] * qj * (-two_b_sqpi * np.exp(-(beta * r) ** 2) / r - ec / r)
        C6 = c6[types[i], types[m]]
        C12 = c12[types[i], types[m]]
        r6 = r ** -6
        dEdr = dEdr + (-12.0 * C12 * r6 * r6 + 6.0 * C6 * r6) / r
        F[a] = ((dEdr / r)[:, None] * d[m]).sum(0)
    return phi, F


def exclusion_correction(pos, q, box, beta, excl):
    """E_excl, phi and F of the erf correction for excluded pairs (any distance)."""
    pos = np.asarray(pos, np.float64)
    n = len(pos)
    phi = np.zeros(n)
    F = np.zeros((n, 3))
    excl = np.asarray(excl).reshape(-1, 2)
    if len(excl) == 0:
        return dict(E_excl=0.0, phi=phi, F=F)
    i, j = excl[:, 0], excl[:, 1]
    d = min_image(pos[j] - pos[i], box)
    r = np.sqrt((d * d).sum(-1))
    ef = erf(beta * r) / r
    e = -F_COUL * np.sum(q[i] * q[j] * ef)
    np.add.at(phi, i, -q[j] * ef)
    np.add.at(phi, j, -q[i] * ef)
    # d/dr [-f qq erf(br)/r] = -f qq (2b/sqrt(pi) exp(-b^2 r^2)/r - erf(br)/r^2)
    dEdr = -F_COUL * q[i] * q[j] * (2.0 * beta / math.sqrt(math.pi) * np.exp(-(beta * r) ** 2) / r - ef / r)
    fvec = (dEdr / r)[:, None] * d
    np.add.at(F, i, fvec)
    np.add.at(F, j, -fvec)
    return dict(E_excl=e, phi=phi, F=F)


def self_term(q, beta):
    """E_self = -f beta/sqrt(pi) sum q^2 ; phi_self_i = -2 beta/sqrt(pi) q_i."""
    return -F_COUL * beta / math.sqrt(math.pi) * np.sum(q * q), -2.0 * beta / math.sqrt(math.pi) * q


def net_charge_term(q, box, beta):
    """Uniform neutralising background (tin-foil Ewald): E_net = -f pi Q^2/(2 V beta^2),
    phi_net_i = -pi Q/(V beta^2)."""
    V = float(np.prod(box))
    Q = float(np.sum(q))
    return -F_COUL * math.pi * Q * Q / (2.0 * V * beta * beta), np.full(len(q), -math.pi * Q / (V * beta * beta))


def recip_direct(pos, q, box, beta, nmax):
    """Direct reciprocal-space Ewald sum over |n_d| <= nmax (m = n/L), m != 0.

    Returns E_rec (kJ/mol), phi_rec (N,) (e/nm), F_rec (N,3)."""
    pos = np.asarray(pos, np.float64)
    V = float(np.prod(box))
    rng = np.arange(-nmax, nmax + 1)
    n = np.stack(np.meshgrid(rng, rng, rng, indexing="ij"), -1).reshape(-1, 3)
    n = n[np.any(n != 0, axis=1)]
    m = n / box[None, :]
    m2 = (m * m).sum(-1)
    w = np.exp(-math.pi ** 2 * m2 / beta ** 2) / m2
    keep = w > 1e-300
    m, m2, w = m[keep], m2[keep], w[keep]
    phase = 2.0 * math.pi * pos @ m.T                         # (N, M)
    c, s = np.cos(phase), np.sin(phase)
    S_re = q @ c
    S_im = q @ s
    E = F_COUL / (2.0 * math.pi * V) * np.sum(w * (S_re ** 2 + S_im ** 2))
    # Re[S e^{-i theta_i}] = S_re cos + S_im sin ; Im[S e^{-i theta_i}] = S_im cos - S_re sin
    re = c * S_re[None, :] + s * S_im[None, :]
    im = c * S_im[None, :] - s * S_re[None, :]
    phi = (re @ w) / (math.pi * V)
    # grad phi(r)|_{r_i} = (1/pi V) sum w * 2 pi m * Im[S e^{-i theta}]
    grad = (2.0 * math.pi / (math.pi * V)) * ((im * w[None, :]) @ m)
    F = -F_COUL * q[:, None] * grad
    return E, phi, F

"""Partition Function Correction (readings R2, R6).

Z_prot = int_{lp<0.5} exp(-beta V), Z_deprot = int_{lp>=0.5} exp(-beta V) over the
full wall-bounded range (R2), V = Vdw + VpH (Vmm excluded: it cancels dG_MM by
construction).  Target: G_deprot - G_prot = ln10 kT (pKa - pH)
(Eq. 4 with the sign of reading R2).  Only the lambda=1 well depth d1 is
adjusted (R6); for His the two depths (d1_p, d1_t) are solved so that the
quadrant free energies give G_delta - G_prot = dG_delta and
G_eps - G_prot = dG_eps.

Quadrature: scipy.integrate.quad with the spline knots and wall onsets as
breakpoints (1D); a composite Gauss-Legendre tensor rule for 2D.  After a DBO
adjustment (the correction is recomputed "when adjusting the
barrier height or well position") the shifted knots become breakpoints too.
"""
import math

import numpy as np
from scipy import integrate, optimize

from . import bias as B
from .bias import delta_g, vdw, vph
from .units import kT

LO, HI = -0.45, 1.45          # walls make the integrand < 1e-30 beyond these


def _breaks(*knots):
    """Quadrature breakpoints: the wall onsets, the well centres and barrier position of
    every coordinate involved, the smoothstep ends 0 and 1 (reading R25), the quarter
    points and the half-space split 0.5; the integrand is analytic between them."""
    pts = {LO, -0.1, 0.0, 0.25, 0.5, 0.75, 1.0, 1.1, HI}
    for a0, a1 in knots:
        pts.update((a0, 0.5 * (a0 + a1), a1))
    return sorted(pts)


def _z_halves_1d(h, d1, g, beta, kw, a0=0.0, a1=1.0):
    f = lambda l: math.exp(-beta * (vdw(l, h, 0.0, d1, kw, a0, a1)[0] + l * g))
    br = _breaks((a0, a1))
    zp = zd = 0.0
    for a, b in zip(br[:-1], br[1:]):
        z = integrate.quad(f, a, b, epsabs=0, epsrel=1e-13, limit=200)[0]
        if b <= 0.5:
            zp += z
        else:
            zd += z
    return zp, zd


def free_energy_1d(h, d1, g, T, kw, a0=0.0, a1=1.0):
    beta = 1.0 / kT(T)
    zp, zd = _z_halves_1d(h, d1, g, beta, kw, a0, a1)
    return -kT(T) * math.log(zd / zp)


D1_BOUND = 80.0     # kJ/mol; reading R22: the correction saturates at +-80 when unreachable


def _root_or_bound(fn, lo=-D1_BOUND, hi=D1_BOUND):
    """Root of an increasing function on [lo, hi]; if none, the bound nearer to it (R22)."""
    flo, fhi = fn(lo), fn(hi)
    if flo > 0:
        return lo
    if fhi < 0:
        return hi
    return optimize.brentq(fn, lo, hi, xtol=1e-13, rtol=1e-15, maxiter=500)


def pfc_2state(h, pKa, pH, T, kw, a0=0.0, a1=1.0):
    """d1 such that G_deprot - G_prot = ln10 kT (pKa - pH) (saturating, R22); a0, a1 are
    the (DBO-shifted) well centres."""
    target = delta_g(pKa, pH, T)
    return _root_or_bound(lambda d1: free_energy_1d(h, d1, target, T, kw, a0, a1) - target)


def _gl_nodes(breaks, sub=8, order=24):
    x, w = np.polynomial.legendre.leggauss(order)
    xs, ws = [], []
    for a, b in zip(breaks[:-1], breaks[1:]):
        edges = np.linspace(a, b, sub + 1)
        for c, d in zip(edges[:-1], edges[1:]):
            xs.append(0.5 * (d - c) * x + 0.5 * (d + c))
            ws.append(0.5 * (d - c) * w)
    return np.concatenate(xs), np.concatenate(ws)


def quadrant_free_energies(h, d1p, d1t, pKa3, pH, T, kw, dbo=None):
    """(G_delta - G_prot, G_eps - G_prot) for a 3-state site.  dbo: rows (a0, a1, h_prot,
    h_deprot) of (lambda_p, lambda_t), None for the undisturbed double wells."""
    if dbo is None:
        dbo = B.default_dbo(h, 2)
    beta = 1.0 / kT(T)
    (a0p, a1p, hp, _), (a0t, a1t, htp, htd) = dbo
    xp, wp = _gl_nodes(_breaks((a0p, a1p)), sub=4)
    xt, wt = _gl_nodes(_breaks((a0t, a1t)), sub=4)
    vp = vdw(xp, hp, 0.0, d1p, kw, a0p, a1p)[0]
    ht = B.tautomer_barrier(xp, htp, htd)[0]
    LP, LT = np.meshgrid(xp, xt, indexing="ij")
    vt = vdw(LT, ht[:, None], 0.0, d1t, kw, a0t, a1t)[0]
    vph_v = vph(3, pKa3, pH, T, LP, LT)[0]
    E = vp[:, None] + vt + vph_v
    W = wp[:, None] * wt[None, :] * np.exp(-beta * E)
    prot = LP < 0.5
    z_prot = W[prot].sum()
    z_d = W[(~prot) & (LT < 0.5)].sum()
    z_e = W[(~prot) & (LT >= 0.5)].sum()
    return -kT(T) * math.log(z_d / z_prot), -kT(T) * math.log(z_e / z_prot)


def pfc_3state(h, pKa3, pH, T, kw, dbo=None):
    """(d1_p, d1_t) for a His-like site (dbo as in quadrant_free_energies)."""
    gd = delta_g(pKa3[1], pH, T)
    ge = delta_g(pKa3[2], pH, T)

    def res(v):
        a, b = quadrant_free_energies(h, v[0], v[1], pKa3, pH, T, kw, dbo)
        return [a - gd, b - ge]
    sol = optimize.root(res, [0.0, 0.0], method="hybr", tol=1e-14)
    # hybr may report "not making good progress" once at the rounding floor: judge the residual
    if np.max(np.abs(res(sol.x))) < 1e-9 and np.all(np.abs(sol.x) <= D1_BOUND):
        return float(sol.x[0]), float(sol.x[1])
    # unreachable targets (R22): nested saturating bisection - the tautomer split
    # G_eps - G_delta = dG_eps - dG_delta for d1_t inside, the macro deprotonation free
    # energy -kT ln(e^{-b dG_delta} + e^{-b dG_eps}) for d1_p outside
    kt = kT(T)
    macro = -kt * math.log(math.exp(-gd / kt) + math.exp(-ge / kt))

    def inner(d1p):
        return _root_or_bound(lambda d1t: np.subtract(*quadrant_free_energies(h, d1p, d1t, pKa3, pH, T, kw,
                                                                              dbo)[::-1]) - (ge - gd))

    def outer(d1p):
        a, b = quadrant_free_energies(h, d1p, inner(d1p), pKa3, pH, T, kw, dbo)
        return -kt * math.log(math.exp(-a / kt) + math.exp(-b / kt)) - macro
    d1p = _root_or_bound(outer)
    return float(d1p), float(inner(d1p))

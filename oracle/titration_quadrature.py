"""Exact titration curve of one 2-state site in a FROZEN environment (test infrastructure).

With every atom frozen, the only coordinate that moves is lambda.  Under charge
interpolation (reading R7) the site's charges are linear in lambda and
the Coulomb energy is quadratic in the charges, so

    E_coul(lambda) = E_coul(0) + b lambda + c lambda^2            (exact)

and the lambda dynamics samples the 1-D Boltzmann density exp(-V(lambda)/kT) with

    V = V_dw(lambda; h, d1(pH)) + V_pH(lambda) + V_mm(lambda) + b lambda + c lambda^2

(Eq. 3 bias, PAPER.md:667-698 / :715-740; PFC depth d1 from oracle.pfc).
The deprotonated fraction at each pH (lambda >= 0.5, reading R1) is then
a 1-D quadrature; the H-H fit of those fractions (oracle.analysis) gives the
pKa that a long electrostatics-on titration must reproduce.

`coulomb_quadratic` reads b, c off the oracle engine's own E_coul at lambda = 0, 1/2, 1 (a
quadratic is fixed by three values; a fourth point checks it).  Pinned in
tests/test_oracle_quadrature.py against the engine's dV/dlambda, electrostatics-off H-H
(b = c = 0 gives 1/(10^(pKa-pH)+1) exactly, the PFC target) and against the oracle's
lambda-only dynamics (oracle.lambda_only) sampling the same potential.
"""
import numpy as np

from . import bias as B
from .pfc import pfc_2state
from .units import kT

LO, HI = -0.45, 1.45            # the walls make the density < 1e-30 beyond these (oracle.pfc)


def coulomb_energy(rep, lam):
    """E_coul = E_real + E_excl + E_self + E_net + E_rec of an OracleReplica at lambda."""
    ev = rep.evaluate(rep.x, np.asarray(lam, np.float64))
    return sum(ev["E"][k] for k in ("real", "excl", "self", "recip", "net"))


def coulomb_quadratic(rep, coord=0):
    """(b, c, check) with E_coul(l) - E_coul(0) = b l + c l^2 along coordinate `coord`
    (other coordinates at rep.lam); `check` = |quadratic(1/4) - E_coul(1/4)|."""
    base = np.asarray(rep.lam, np.float64).copy()

    def at(l):
        v = base.copy()
        v[coord] = l
        return coulomb_energy(rep, v)
    e0, eh, e1 = at(0.0), at(0.5), at(1.0)
    c = 2.0 * (e1 - 2.0 * eh + e0)
    b = e1 - e0 - c
    check = abs(e0 + 0.25 * b + 0.0625 * c - at(0.25))
    return b, c, check


def deprotonated_fraction(pKa, pH, T, h, kw, b=0.0, c=0.0, vmm=None, n=400001):
    """Fraction of exp(-V/kT) with lambda >= 0.5 (trapezoid on [LO, HI], n points)."""
    d1 = pfc_2state(h, pKa, pH, T, kw)
    x = np.linspace(LO, HI, n)
    V = B.vdw(x, h, 0.0, d1, kw)[0] + x * B.delta_g(pKa, pH, T) + b * x + c * x * x
    if vmm is not None:
        V = V + B.vmm(vmm, x, 0.0)[0]          # 2-state: lt = 0 (reading R20)
    w = np.exp(-(V - V.min()) / kT(T))
    dx = x[1] - x[0]
    wd = np.where(x >= 0.5, w, 0.0)
    return float(np.trapezoid(wd, dx=dx) / np.trapezoid(w, dx=dx))


def titration_curve(pKa, pH_levels, T, h, kw, b=0.0, c=0.0, vmm=None, n=400001):
    return np.array([deprotonated_fraction(pKa, p, T, h, kw, b, c, vmm, n) for p in pH_levels])


# ---- His (3-state) site: 2-D in (lambda_p, lambda_t) ----------------------------------------
def coulomb_biquadratic(rep, cp, ct):
    """E_coul(lp, lt) - E_coul(0, 0) = sum_{a,b<=2} c[a, b] lp^a lt^b along the coordinates
    (cp, ct) of one His group (others at rep.lam): the charges are bilinear in (lp, lt) (Eq. 2,
    PAPER.md:621-623) and E_coul is quadratic in the charges, so degree <= 2 in each variable;
    read off the 3 x 3 tensor grid {0, 1/2, 1}^2.  Returns (c [3, 3], check) with check the
    deviation at (1/4, 3/4)."""
    base = np.asarray(rep.lam, np.float64).copy()

    def at(lp, lt):
        v = base.copy()
        v[cp], v[ct] = lp, lt
        return coulomb_energy(rep, v)
    nodes = np.array([0.0, 0.5, 1.0])
    E = np.array([[at(a, b) for b in nodes] for a in nodes])
    V = np.vander(nodes, 3, increasing=True)                  # V[i, a] = node_i^a
    Vi = np.linalg.inv(V)
    c = Vi @ E @ Vi.T                                        # E[i, j] = sum_ab V[i,a] c[a,b] V[j,b]
    c[0, 0] -= E[0, 0]
    poly = lambda lp, lt: sum(c[a, b] * lp ** a * lt ** b for a in range(3) for b in range(3))
    check = abs(E[0, 0] + poly(0.25, 0.75) - at(0.25, 0.75))
    return c, check


def his_fractions(pKa3, pH, T, h, kw, c=None, vmm=None, n=1201):
    """(x_deprot, x_delta, x_eps) of exp(-V/kT) on [LO, HI]^2 (trapezoid, n x n points):
    V = group bias of a His site (Vdw(lp) + Vdw(lt; tautomer barrier) + VpH + Vmm, PFC depths
    from oracle.pfc.pfc_3state) + sum c[a, b] lp^a lt^b.  Deprotonated iff
    lp >= 0.5 (R1); delta iff lt < 0.5 (R4)."""
    from .pfc import pfc_3state
    d1p, d1t = pfc_3state(h, pKa3, pH, T, kw)
    x = np.linspace(LO, HI, n)
    LP, LT = np.meshgrid(x, x, indexing="ij")
    c36 = np.zeros(36) if vmm is None else np.asarray(vmm, np.float64)
    V = B.group_bias(3, c36, pKa3, pH, T, h, d1p, d1t, kw, LP, LT)[0]
    if c is not None:
        V = V + sum(c[a, b] * LP ** a * LT ** b for a in range(3) for b in range(3))
    w = np.exp(-(V - V.min()) / kT(T))
    wx = np.full(n, x[1] - x[0])
    wx[0] = wx[-1] = 0.5 * (x[1] - x[0])
    W = w * wx[:, None] * wx[None, :]
    Z = W.sum()
    dep = LP >= 0.5
    return float(W[dep].sum() / Z), float(W[dep & (LT < 0.5)].sum() / Z), float(W[dep & (LT >= 0.5)].sum() / Z)

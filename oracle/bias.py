"""Biasing potential V = Vmm + VpH + Vdw per lambda-group (Eq. 3).

* Vmm: degree-5 x degree-5 polynomial with all mixing terms:
  Vmm = sum_{a,b=0..5} c_ab lp^a lt^b.  2-state groups evaluate it at lt = 0.
* VpH: endpoint difference ln10 kT (pKa - pH) (Eq. 4); the
  paper gives only the endpoints -> linear in lp (reading R4);
  His: VpH = lp [(1-lt) dG_delta + lt dG_eps] with micro pKa values.
* Vdw per coordinate: cubic Hermite through (0, d0, 0),
  (0.5, d0+h, 0), (1, d1, 0); mirrored outside [0,1] (V(l<0)=V(-l),
  V(l>1)=V(2-l)); quartic walls k_w (l+0.1)^4 for l<-0.1 and k_w (l-1.1)^4 for
  l>1.1 (reading R5).  h = barrier (6 kJ/mol), d0 = 0 (gauge),
  d1 from the partition function correction (oracle.pfc).  Dynamic Barrier and Well
  Optimization (oracle.dbo) moves the well centres a0, a1 and the
  barrier heights; the tautomer barrier depends smoothly on lambda_p (reading R25).
"""
import numpy as np

from .units import LN10, kT


def vmm(c, lp, lt):
    """Returns (V, dV/dlp, dV/dlt) for the 36 coefficients c[a*6+b]."""
    c = np.asarray(c, np.float64).reshape(6, 6)
    V = dp = dt = 0.0
    for a in range(6):
        for b in range(6):
            V += c[a, b] * lp ** a * lt ** b
            if a > 0:
                dp += a * c[a, b] * lp ** (a - 1) * lt ** b
            if b > 0:
                dt += b * c[a, b] * lp ** a * lt ** (b - 1)
    return V, dp, dt


def delta_g(pKa, pH, T):
    """Eq. 4: ln(10) R T (pKa - pH)."""
    return LN10 * kT(T) * (pKa - pH)


def vph(kind, pKa3, pH, T, lp, lt):
    """Returns (V, dV/dlp, dV/dlt)."""
    if int(kind) == 2:
        g = delta_g(pKa3[0], pH, T)
        return lp * g, g, 0.0
    gd = delta_g(pKa3[1], pH, T)
    ge = delta_g(pKa3[2], pH, T)
    return lp * ((1.0 - lt) * gd + lt * ge), (1.0 - lt) * gd + lt * ge, lp * (ge - gd)


def _hermite01(x, v0, v1):
    """Cubic Hermite on x in [0,1] with zero end slopes: v0 + (v1-v0)(3x^2-2x^3)."""
    return v0 + (v1 - v0) * (3.0 * x * x - 2.0 * x ** 3), (v1 - v0) * (6.0 * x - 6.0 * x * x)


def vdw_full(lam, h, d0, d1, kw, a0=0.0, a1=1.0):
    """Double well with walls: (V, dV/dlam, dV/dh).  Works on arrays (h may be an array).

    Knots (a0, d0, 0), (m, d0 + h, 0), (a1, d1, 0) with m = (a0 + a1)/2;
    a0 = 0, a1 = 1 unless DBO has shifted the wells laterally (reading R23);
    mirrored about the well centres outside [a0, a1]; quartic walls at -0.1 / 1.1 (R5).
    V is linear in h, so dV/dh is the knot basis function of the barrier value.
    """
    lam = np.asarray(lam, np.float64)
    m = 0.5 * (a0 + a1)
    below, above = lam < a0, lam > a1
    x = np.where(below, 2.0 * a0 - lam, np.where(above, 2.0 * a1 - lam, lam))
    sgn = np.where(below | above, -1.0, 1.0)
    x = np.clip(x, a0, a1)
    left = x <= m
    tl = (x - a0) / (m - a0)
    tr = (x - m) / (a1 - m)
    vl, dl = _hermite01(tl, d0, d0 + h)
    vr, dr = _hermite01(tr, d0 + h, d1)
    sl = 3.0 * tl * tl - 2.0 * tl ** 3           # dV/dh on the left segment
    sr = 1.0 - (3.0 * tr * tr - 2.0 * tr ** 3)   # dV/dh on the right segment
    v = np.where(left, vl, vr)
    dv = sgn * np.where(left, dl / (m - a0), dr / (a1 - m))
    dh = np.where(left, sl, sr)
    wl = np.minimum(lam + 0.1, 0.0)          # nonzero only for lam < -0.1
    wr = np.maximum(lam - 1.1, 0.0)          # nonzero only for lam > 1.1
    v = v + kw * wl ** 4 + kw * wr ** 4
    dv = dv + 4.0 * kw * wl ** 3 + 4.0 * kw * wr ** 3
    if v.ndim == 0:
        return float(v), float(dv), float(dh)
    return v, dv, dh


def vdw(lam, h, d0, d1, kw, a0=0.0, a1=1.0):
    """Double well with walls; returns (V, dV/dlam).  Works on scalars and arrays."""
    v, dv, _ = vdw_full(lam, h, d0, d1, kw, a0, a1)
    return v, dv


def tautomer_barrier(lp, h_prot, h_deprot):
    """Barrier of the tautomer coordinate keyed by protonation, made
    smooth in lambda_p (reading R25): h = h_prot + (h_deprot - h_prot) S(lp), S the clamped
    smoothstep 3x^2 - 2x^3.  Returns (h, dh/dlp)."""
    x = np.clip(lp, 0.0, 1.0)
    S = 3.0 * x * x - 2.0 * x ** 3
    dS = np.where((lp > 0.0) & (lp < 1.0), 6.0 * x * (1.0 - x), 0.0)
    h = h_prot + (h_deprot - h_prot) * S
    dh = (h_deprot - h_prot) * dS
    if np.ndim(h) == 0:
        return float(h), float(dh)
    return h, dh


def default_dbo(h, n):
    """Per-coordinate DBO parameters (a0, a1, h_prot, h_deprot) before any adjustment."""
    return np.tile(np.array([0.0, 1.0, h, h], np.float64), (n, 1))


def group_bias(kind, c36, pKa3, pH, T, h, d1p, d1t, kw, lp, lt, dbo=None):
    """Total bias of one group: (V, dV/dlp, dV/dlt).

    dbo: per-coordinate rows (a0, a1, h_prot, h_deprot) of this group (None: undisturbed
    wells, barrier h).  lambda_p rows use h_prot (== h_deprot); the tautomer row's barrier
    follows tautomer_barrier(lp, h_prot, h_deprot)."""
    if dbo is None:
        dbo = default_dbo(h, 1 if int(kind) == 2 else 2)
    a0p, a1p, hp = dbo[0][0], dbo[0][1], dbo[0][2]
    if int(kind) == 2:
        vm, dmp, _ = vmm(c36, lp, 0.0)
        vp, dpp, _ = vph(kind, pKa3, pH, T, lp, 0.0)
        vd, ddp = vdw(lp, hp, 0.0, d1p, kw, a0p, a1p)
        return vm + vp + vd, dmp + dpp + ddp, 0.0
    vm, dmp, dmt = vmm(c36, lp, lt)
    vp, dpp, dpt = vph(kind, pKa3, pH, T, lp, lt)
    vd1, dd1 = vdw(lp, hp, 0.0, d1p, kw, a0p, a1p)
    ht, dht = tautomer_barrier(lp, dbo[1][2], dbo[1][3])
    vd2, dd2, dh2 = vdw_full(lt, ht, 0.0, d1t, kw, dbo[1][0], dbo[1][1])
    return vm + vp + vd1 + vd2, dmp + dpp + dd1 + dh2 * dht, dmt + dpt + dd2

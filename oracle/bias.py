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
  d1 from the partition function correction (oracle.pfc).
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


def vdw(lam, h, d0, d1, kw):
    """Double well with walls; returns (V, dV/dlam).  Works on scalars and arrays."""
    lam = np.asarray(lam, np.float64)
    x = np.where(lam < 0.0, -lam, np.where(lam > 1.0, 2.0 - lam, lam))
    sgn = np.where((lam < 0.0) | (lam > 1.0), -1.0, 1.0)
    x = np.clip(x, 0.0, 1.0)
    vl, dl = _hermite01(x / 0.5, d0, d0 + h)
    vr, dr = _hermite01((x - 0.5) / 0.5, d0 + h, d1)
    left = x <= 0.5
    v = np.where(left, vl, vr)
    dv = sgn * np.where(left, dl, dr) / 0.5
    wl = np.minimum(lam + 0.1, 0.0)          # nonzero only for lam < -0.1
    wr = np.maximum(lam - 1.1, 0.0)          # nonzero only for lam > 1.1
    v = v + kw * wl ** 4 + kw * wr ** 4
    dv = dv + 4.0 * kw * wl ** 3 + 4.0 * kw * wr ** 3
    if v.ndim == 0:
        return float(v), float(dv)
    return v, dv


def group_bias(kind, c36, pKa3, pH, T, h, d1p, d1t, kw, lp, lt):
    """Total bias of one group: (V, dV/dlp, dV/dlt)."""
    if int(kind) == 2:
        vm, dmp, _ = vmm(c36, lp, 0.0)
        vp, dpp, _ = vph(kind, pKa3, pH, T, lp, 0.0)
        vd, ddp = vdw(lp, h, 0.0, d1p, kw)
        return vm + vp + vd, dmp + dpp + ddp, 0.0
    vm, dmp, dmt = vmm(c36, lp, lt)
    vp, dpp, dpt = vph(kind, pKa3, pH, T, lp, lt)
    vd1, dd1 = vdw(lp, h, 0.0, d1p, kw)
    vd2, dd2 = vdw(lt, h, 0.0, d1t, kw)
    return vm + vp + vd1 + vd2, dmp + dpp + dd1, dmt + dpt + dd2

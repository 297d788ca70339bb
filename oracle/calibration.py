"""Vmm calibration from fixed-lambda TI (reading R3, R18).

dVmm/dlambda = -<dV_coul/dlambda>_(lp, lt) sampled on the SI grid (P:8), fitted by a
degree-5 x degree-5 polynomial with all mixing terms.  The fit is to the
derivatives directly, both residual blocks stacked, with the constant term
fixed to 0 (gauge).  2-state sites: 1D polynomial in lp (coefficients c_a0).
"""
import numpy as np

TI_GRID = (-0.1, -0.05, 0.0, 0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 0.95, 1.0, 1.05, 1.1)   # P:8 (R18)


def fit_derivative_poly_2d(lp, lt, gp, gt, deg=5):
    """Least-squares P = sum_{a,b<=deg, (a,b)!=(0,0)} c_ab lp^a lt^b with dP/dlp ~ gp and
    dP/dlt ~ gt.  Returns c as a (deg+1)^2 vector c[a*(deg+1)+b] (c_00 = 0)."""
    lp, lt, gp, gt = (np.asarray(v, np.float64) for v in (lp, lt, gp, gt))
    terms = [(a, b) for a in range(deg + 1) for b in range(deg + 1) if (a, b) != (0, 0)]
    rows_p = np.stack([a * lp ** max(a - 1, 0) * lt ** b if a else np.zeros_like(lp) for a, b in terms], 1)
    rows_t = np.stack([b * lp ** a * lt ** max(b - 1, 0) if b else np.zeros_like(lt) for a, b in terms], 1)
    A = np.concatenate([rows_p, rows_t], 0)
    y = np.concatenate([gp, gt])
    sol, *_ = np.linalg.lstsq(A, y, rcond=None)
    c = np.zeros((deg + 1) ** 2)
    for k, (a, b) in enumerate(terms):
        c[a * (deg + 1) + b] = sol[k]
    return c


def fit_derivative_poly_1d(lp, g, deg=5):
    lp, g = np.asarray(lp, np.float64), np.asarray(g, np.float64)
    A = np.stack([a * lp ** (a - 1) for a in range(1, deg + 1)], 1)
    sol, *_ = np.linalg.lstsq(A, g, rcond=None)
    c = np.zeros((deg + 1) ** 2)
    for a in range(1, deg + 1):
        c[a * (deg + 1)] = sol[a - 1]
    return c


def vmm_from_ti(kind, lp, lt, mean_dvdl):
    """Vmm coefficients (36) from TI means: Vmm := -DeltaG_MM, i.e. dVmm/dl = -<dV/dl> (R3)."""
    if int(kind) == 2:
        return -fit_derivative_poly_1d(lp, np.asarray(mean_dvdl)[:, 0])
    m = np.asarray(mean_dvdl)
    return -fit_derivative_poly_2d(lp, lt, m[:, 0], m[:, 1])

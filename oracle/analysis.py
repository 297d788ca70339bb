"""Titration analysis.

* frame classification: deprotonated iff lambda_p >= 0.5 (reading R1)
* x = N_deprot / N per (pH, replica)
* H-H fit x(pH) = 1/(10^(pKa - pH) + 1) and Hill fit 1/(10^(n(pKa - pH)) + 1) by
  SciPy non-linear least squares, unweighted over all
  (pH, replica) points
* bootstrap: per pH resample R replica fractions with replacement, refit,
  5000 times, percentile 95% CI
"""
import numpy as np
from scipy.optimize import least_squares


def deprotonated_fraction(lp_frames):
    lp = np.asarray(lp_frames, np.float64)
    if not np.all(np.isfinite(lp)):
        raise ValueError("non-finite lambda")
    return float(np.mean(lp >= 0.5))


def micro_fractions(lp_frames, lt_frames):
    """His microscopic ratios: x_delta = N_{deprot, t=0} / (N_prot +
    N_{deprot, t=0}), x_eps = N_{deprot, t=1} / (N_prot + N_{deprot, t=1}); deprotonated iff
    lambda_p >= 0.5 (R1), tautomer t = 0 (delta) iff lambda_t < 0.5 (R4)."""
    lp = np.asarray(lp_frames, np.float64)
    lt = np.asarray(lt_frames, np.float64)
    deprot = lp >= 0.5
    n_prot = np.count_nonzero(~deprot)
    n_d = np.count_nonzero(deprot & (lt < 0.5))
    n_e = np.count_nonzero(deprot & (lt >= 0.5))
    return n_d / (n_prot + n_d), n_e / (n_prot + n_e)


def hh(pH, pKa, n=1.0):
    return 1.0 / (10.0 ** (n * (pKa - np.asarray(pH, np.float64))) + 1.0)


def fit_hh(pH, x):
    pH = np.asarray(pH, np.float64)
    x = np.asarray(x, np.float64)
    p0 = pH[np.argmin(np.abs(x - 0.5))]
    r = least_squares(lambda v: hh(pH, v[0]) - x, [p0], xtol=1e-15, ftol=1e-15, gtol=1e-15)
    return float(r.x[0])


def fit_hill(pH, x):
    pH = np.asarray(pH, np.float64)
    x = np.asarray(x, np.float64)
    p0 = pH[np.argmin(np.abs(x - 0.5))]
    r = least_squares(lambda v: hh(pH, v[0], v[1]) - x, [p0, 1.0], xtol=1e-15, ftol=1e-15, gtol=1e-15)
    return float(r.x[0]), float(r.x[1])


def bootstrap(pH_levels, fractions, B=5000, seed=0, hill=False):
    """fractions: (n_pH, R).  Returns (estimate, lo, hi) of pKa (and n if hill)."""
    rng = np.random.default_rng(seed)
    f = np.asarray(fractions, np.float64)
    npH, R = f.shape
    pHs = np.repeat(np.asarray(pH_levels, np.float64), R)
    est = fit_hill(pHs, f.reshape(-1)) if hill else fit_hh(pHs, f.reshape(-1))
    draws = []
    for _ in range(B):
        idx = rng.integers(0, R, size=(npH, R))
        fr = np.take_along_axis(f, idx, 1).reshape(-1)
        draws.append(fit_hill(pHs, fr) if hill else fit_hh(pHs, fr))
    d = np.array(draws)
    lo = np.percentile(d, 2.5, axis=0)
    hi = np.percentile(d, 97.5, axis=0)
    return est, lo, hi


def nmi_binary(x, y):
    """NMI = 2 I(X;Y) / (H(X) + H(Y)) of two binary protonation trajectories
    (PAPER.md:1024-1030), from the definitions: I = sum_xy p(x,y) ln[p(x,y) / (p(x) p(y))],
    H = -sum_x p(x) ln p(x) (the paper's H formula has lost its minus sign).  Returns
    (NMI, H(X), H(Y)); NMI = 0 when both entropies vanish."""
    x = [int(v) for v in x]
    y = [int(v) for v in y]
    n = len(x)
    pxy = {(a, b): sum(1 for u, v in zip(x, y) if u == a and v == b) / n for a in (0, 1) for b in (0, 1)}
    px = {a: pxy[(a, 0)] + pxy[(a, 1)] for a in (0, 1)}
    py = {b: pxy[(0, b)] + pxy[(1, b)] for b in (0, 1)}
    I = sum(p * np.log(p / (px[a] * py[b])) for (a, b), p in pxy.items() if p > 0)
    hx = -sum(p * np.log(p) for p in px.values() if p > 0)
    hy = -sum(p * np.log(p) for p in py.values() if p > 0)
    return (2.0 * I / (hx + hy) if hx + hy > 0 else 0.0), hx, hy


def protonated(lp_frames):
    """1 = protonated (lambda_p < 0.5), reading R1."""
    return [1 if v < 0.5 else 0 for v in np.asarray(lp_frames, np.float64).ravel()]


def two_site_protons(pH, pK1, pK2):
    """<X> of PAPER.md:1014-1016."""
    pH = np.asarray(pH, np.float64)
    num = 10.0 ** (pK2 - pH) + 2.0 * 10.0 ** (pK1 + pK2 - 2.0 * pH)
    return num / (1.0 + 10.0 ** (pK2 - pH) + 10.0 ** (pK1 + pK2 - 2.0 * pH))


def fit_two_site(pH, X):
    pH = np.asarray(pH, np.float64)
    X = np.asarray(X, np.float64)
    c = pH[np.argmin(np.abs(X - 1.0))]
    r = least_squares(lambda v: two_site_protons(pH, v[0], v[1]) - X, [c - 1.0, c + 1.0], xtol=1e-15, ftol=1e-15,
                      gtol=1e-15)
    return float(r.x[0]), float(r.x[1])

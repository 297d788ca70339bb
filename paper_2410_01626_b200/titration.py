"""Titration bookkeeping on the host.

* replicas = pH points x seeds, dealt round-robin to ranks (one process per GPU; the
  path shards as independent replicas, so there is no collective
  inside the step loop);
* one all-gather of the lambda frames at the end (NCCL over NVLink on GPUs, gloo on
  CPU), the only collective of a run;
* deprotonated fraction x = N(lambda_p >= 0.5)/N per replica (PAPER.md:975-978,
  reading R1), Henderson-Hasselbalch / Hill fit by damped
  Gauss-Newton, bootstrap over replicas.
"""
from __future__ import annotations

import numpy as np


def assign_replicas(n_replicas: int, world: int, rank: int):
    """Round-robin replica indices of one rank."""
    return list(range(rank, n_replicas, world))


def gather_frames(local: np.ndarray, group=None, device=None):
    """All-gather a per-rank array [R_local, F, C] (padded to the largest R_local) over
    torch.distributed; returns the concatenation over ranks (every rank gets it)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return np.asarray(local)
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if backend == "nccl" else torch.device("cpu"))
    local = np.asarray(local, np.float32)
    n_local = torch.tensor([local.shape[0]], device=dev, dtype=torch.int64)
    counts = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(counts, n_local, group=group)
    counts = [int(c.item()) for c in counts]
    rmax = max(counts)
    pad = np.zeros((rmax,) + local.shape[1:], np.float32)
    pad[: local.shape[0]] = local
    t = torch.from_numpy(pad).to(dev)
    out = torch.empty((world * rmax,) + tuple(local.shape[1:]), dtype=t.dtype, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    out = out.cpu().numpy().reshape((world, rmax) + local.shape[1:])
    return np.concatenate([out[k, : counts[k]] for k in range(world)], 0)


def deprotonated_fraction(lambda_p_frames, censored=None) -> float:
    """x = N_deprot / N over the frames (deprotonated iff lambda_p >= 0.5);
    frames flagged by DBO censoring are left out."""
    lp = np.asarray(lambda_p_frames, np.float64)
    if censored is not None:
        lp = lp[~np.asarray(censored, bool)]
    if lp.size == 0 or not np.all(np.isfinite(lp)):
        raise ValueError("need finite, uncensored lambda frames")
    return float(np.count_nonzero(lp >= 0.5)) / lp.size


def micro_fractions(lambda_p_frames, lambda_t_frames, censored=None):
    """His microscopic deprotonation ratios, each fitted with the H-H
    curve to give pKa_delta and pKa_eps: x_delta = N(deprot, lambda_t < 0.5) / (N_prot +
    N(deprot, lambda_t < 0.5)) and x_eps likewise with lambda_t >= 0.5."""
    lp = np.asarray(lambda_p_frames, np.float64)
    lt = np.asarray(lambda_t_frames, np.float64)
    if censored is not None:
        keep = ~np.asarray(censored, bool)
        lp, lt = lp[keep], lt[keep]
    if lp.size == 0 or lp.shape != lt.shape:
        raise ValueError("need matching, non-empty lambda_p / lambda_t frames")
    deprot = lp >= 0.5
    n_prot = np.count_nonzero(~deprot)
    n_d = np.count_nonzero(deprot & (lt < 0.5))
    n_e = np.count_nonzero(deprot & (lt >= 0.5))
    return n_d / max(n_prot + n_d, 1), n_e / max(n_prot + n_e, 1)


def _model(pH, pKa, n):
    return 1.0 / (np.power(10.0, n * (pKa - pH)) + 1.0)


def fit_curve(pH, x, hill=False, iters=200):
    """Least squares of x = 1/(10^(n (pKa - pH)) + 1) by Levenberg-Marquardt with the
    analytic Jacobian.  Returns pKa (and n when hill=True)."""
    pH = np.asarray(pH, np.float64)
    x = np.asarray(x, np.float64)
    if np.all(x == x[0]):
        raise ValueError("unidentifiable fit: all fractions equal")
    p = np.array([pH[np.argmin(np.abs(x - 0.5))], 1.0])
    mu = 1e-3
    ln10 = np.log(10.0)

    def resid(v):
        return _model(pH, v[0], v[1]) - x
    r = resid(p)
    for _ in range(iters):
        y = _model(pH, p[0], p[1])
        dy = -ln10 * y * (1.0 - y)                    # d y / d(n (pKa - pH))
        J = np.stack([dy * p[1], dy * (p[0] - pH)], 1)
        if not hill:
            J = J[:, :1]
        A = J.T @ J
        g = J.T @ r
        step = np.linalg.solve(A + mu * np.diag(np.diag(A) + 1e-30), -g)
        trial = p.copy()
        trial[: len(step)] += step
        rt = resid(trial)
        if rt @ rt < r @ r:
            p, r = trial, rt
            mu = max(mu * 0.3, 1e-12)
            if np.max(np.abs(step)) < 1e-13:
                break
        else:
            mu *= 10.0
            if mu > 1e12:
                break
    return (float(p[0]), float(p[1])) if hill else float(p[0])


TI_GRID = (-0.1, -0.05, 0.0, 0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 0.95, 1.0, 1.05, 1.1)


def fit_vmm(kind, lp, lt, mean_dvdl, degree=5):
    """Vmm coefficients c[a*6+b] from fixed-lambda TI means: fit the
    derivatives of a degree-5 x degree-5 polynomial P (all mixing terms, constant gauge 0)
    to <dV_coul/dlambda> at the grid points, both derivative blocks stacked, and return
    Vmm = -P (dVmm/dlambda = -<dV_coul/dlambda>, R3).  kind 2: lp only."""
    n = degree + 1
    lp = np.asarray(lp, np.float64)
    g = np.asarray(mean_dvdl, np.float64).reshape(len(lp), -1)
    if int(kind) == 2:
        powers = [(a, 0) for a in range(1, n)]
        blocks = [np.stack([a * lp ** (a - 1) for a, _ in powers], 1)]
        rhs = [g[:, 0]]
    else:
        lt = np.asarray(lt, np.float64)
        powers = [(a, b) for a in range(n) for b in range(n) if a or b]
        dp = np.stack([a * lp ** (a - 1) * lt ** b if a else 0.0 * lp for a, b in powers], 1)
        dt = np.stack([b * lp ** a * lt ** (b - 1) if b else 0.0 * lt for a, b in powers], 1)
        blocks, rhs = [dp, dt], [g[:, 0], g[:, 1]]
    A = np.concatenate(blocks, 0)
    y = np.concatenate(rhs)
    q, rr = np.linalg.qr(A)
    coef = np.linalg.solve(rr, q.T @ y)
    out = np.zeros(n * n)
    for (a, b), v in zip(powers, coef):
        out[a * n + b] = -v
    return out


def bootstrap(pH_levels, fractions, B=5000, seed=0, hill=False):
    """fractions [n_pH, R]: resample R replica fractions per pH with replacement, refit,
    95% percentile interval."""
    f = np.asarray(fractions, np.float64)
    npH, R = f.shape
    pHs = np.repeat(np.asarray(pH_levels, np.float64), R)
    est = fit_curve(pHs, f.reshape(-1), hill)
    rng = np.random.default_rng(seed)
    draws = []
    for _ in range(B):
        idx = rng.integers(0, R, size=(npH, R))
        try:
            draws.append(fit_curve(pHs, np.take_along_axis(f, idx, 1).reshape(-1), hill))
        except (ValueError, np.linalg.LinAlgError):
            continue
    d = np.asarray(draws)
    return est, np.percentile(d, 2.5, axis=0), np.percentile(d, 97.5, axis=0)


# ---- residue-residue coupling screen -----------------
def binary_protonation(lambda_p_frames):
    """Binary protonation trajectory: 1 = protonated (lambda_p < 0.5), 0 = deprotonated
    (reading R1)."""
    return (np.asarray(lambda_p_frames, np.float64) < 0.5).astype(np.int8)


def _entropy(p):
    p = p[p > 0]
    return float(-(p * np.log(p)).sum())      # H = -sum p ln p (sign restored)


def nmi(x, y):
    """Normalised mutual information of two binary trajectories (same frames):
    NMI = 2 I(X;Y) / (H(X) + H(Y)), natural logs; 0 when both are constant.
    Returns (NMI, H(X), H(Y))."""
    x = np.asarray(x).astype(np.int64).ravel()
    y = np.asarray(y).astype(np.int64).ravel()
    if x.shape != y.shape or x.size == 0:
        raise ValueError("need two non-empty trajectories of equal length")
    joint = np.bincount(2 * x + y, minlength=4).reshape(2, 2) / x.size
    px, py = joint.sum(1), joint.sum(0)
    hx, hy, hxy = _entropy(px), _entropy(py), _entropy(joint.ravel())
    mi = hx + hy - hxy
    return (2.0 * mi / (hx + hy) if hx + hy > 0 else 0.0), hx, hy


def coupling_screen(frames, threshold=0.1):
    """frames [n_pH, R, F, S]: lambda_p of S sites, F frames, R replicas, n_pH points.
    For every site pair: NMI and entropies per replica and pH point, averaged over replicas;
    a pair is coupled when, at any pH point, the mean NMI and both mean entropies exceed the
    threshold (0.1).  Returns (coupled pairs [(a, b)], mean NMI
    [n_pH, S, S], mean H [n_pH, S])."""
    f = np.asarray(frames, np.float64)
    npH, R, F, S = f.shape
    b = binary_protonation(f)
    m_nmi = np.zeros((npH, S, S))
    m_h = np.zeros((npH, S))
    for k in range(npH):
        for r in range(R):
            for a in range(S):
                for c in range(a + 1, S):
                    v, ha, hc = nmi(b[k, r, :, a], b[k, r, :, c])
                    m_nmi[k, a, c] += v / R
                    m_nmi[k, c, a] += v / R
            m_h[k] += np.array([_entropy(np.bincount(b[k, r, :, a], minlength=2) / F) for a in range(S)]) / R
    coupled = [(a, c) for a in range(S) for c in range(a + 1, S)
               if np.any((m_nmi[:, a, c] > threshold) & (m_h[:, a] > threshold) & (m_h[:, c] > threshold))]
    return coupled, m_nmi, m_h


def two_site_protons(pH, pKa1, pKa2):
    """Macroscopic titration of two interacting sites: mean number of bound protons
    <X> = (10^(pKa2-pH) + 2 10^(pKa1+pKa2-2pH)) / (1 + 10^(pKa2-pH) + 10^(pKa1+pKa2-2pH))
    (PAPER.md:1014-1016)."""
    pH = np.asarray(pH, np.float64)
    a = np.power(10.0, pKa2 - pH)
    b = np.power(10.0, pKa1 + pKa2 - 2.0 * pH)
    return (a + 2.0 * b) / (1.0 + a + b)


def fit_two_site(pH, protons, iters=200):
    """Least squares of two_site_protons to <X> per pH (and replica) by Levenberg-Marquardt
    with a numerical Jacobian.  Returns (pKa1, pKa2)."""
    pH = np.asarray(pH, np.float64)
    y = np.asarray(protons, np.float64)
    mid = pH[np.argmin(np.abs(y - 1.0))]
    p = np.array([mid - 1.0, mid + 1.0])
    mu = 1e-3

    def resid(v):
        return two_site_protons(pH, v[0], v[1]) - y
    r = resid(p)
    for _ in range(iters):
        J = np.stack([(resid(p + e) - resid(p - e)) / 2e-7 for e in (np.array([1e-7, 0.0]), np.array([0.0, 1e-7]))], 1)
        A = J.T @ J
        step = np.linalg.solve(A + mu * np.diag(np.diag(A) + 1e-30), -(J.T @ r))
        rt = resid(p + step)
        if rt @ rt < r @ r:
            p, r = p + step, rt
            mu = max(mu * 0.3, 1e-12)
            if np.max(np.abs(step)) < 1e-12:
                break
        else:
            mu *= 10.0
            if mu > 1e12:
                break
    return float(p[0]), float(p[1])

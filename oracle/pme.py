"""Smooth PME reciprocal space, float64 (Essmann et al. 1995 as cited
via the PME prior art at PAPER.md:525-531, :875).

Literal definitions (reading R11 and the grid convention R16):
  * cardinal B-spline M_2(u) = 1 - |u - 1| on [0,2], M_n(u) = u/(n-1) M_{n-1}(u)
    + (n-u)/(n-1) M_{n-1}(u-1);  dM_n/du = M_{n-1}(u) - M_{n-1}(u-1)
  * scaled fractional coordinate u_d = K_d s_d with s_d = x_d/L_d - floor(x_d/L_d)
  * grid point k_d in {floor(u_d)-p+1 .. floor(u_d)} (mod K_d) gets weight M_p(u_d - k_d)
  * Q(k) = sum_i q_i prod_d M_p(u_id - k_d)
  * Qhat = DFT(Q) (numpy fftn, unnormalised forward)
  * G(m) = exp(-pi^2 m^2/beta^2) / (pi V m^2) * prod_d |b_d(m_d)|^2, m_d = k_d/L_d with
    k_d in (-K/2, K/2],  |b_d(m)|^2 = 1/|sum_{k=0}^{p-2} M_p(k+1) exp(2 pi i m k/K)|^2
  * E_rec = (f/2) sum_{m != 0} G(m) |Qhat(m)|^2
  * phi_grid(k) = sum_m G(m) Qhat(m) exp(+2 pi i m.k/K)   (= K^3 ifftn)
  * phi_i^rec = sum_k prod_d M_p(u_id - k_d) phi_grid(k)      (e/nm, without f)
  * F_i^rec = -f q_i grad_i phi^rec                            (via dM_p)
"""
import math

import numpy as np

from .units import F_COUL


def bspline(n, u):
    """Cardinal B-spline M_n(u) by the recursion (vectorised over u)."""
    u = np.asarray(u, dtype=np.float64)
    if n == 2:
        return np.where((u >= 0.0) & (u <= 2.0), 1.0 - np.abs(u - 1.0), 0.0)
    return u / (n - 1) * bspline(n - 1, u) + (n - u) / (n - 1) * bspline(n - 1, u - 1.0)


def bspline_deriv(n, u):
    return bspline(n - 1, u) - bspline(n - 1, u - 1.0)


def bspline_moduli(K, p):
    """|b(m)|^2 for m = 0..K-1."""
    k = np.arange(p - 1)
    Mk = bspline(p, k + 1.0)
    m = np.arange(K)
    s = (Mk[None, :] * np.exp(2j * math.pi * m[:, None] * k[None, :] / K)).sum(1)
    return 1.0 / np.abs(s) ** 2


def signed_freq(K):
    k = np.arange(K)
    return np.where(k <= K // 2, k, k - K)


def influence(box, K, beta, p):
    """G(m) on the full K^3 grid (G(0) = 0)."""
    V = float(np.prod(box))
    mx = signed_freq(K[0]) / box[0]
    my = signed_freq(K[1]) / box[1]
    mz = signed_freq(K[2]) / box[2]
    m2 = mx[:, None, None] ** 2 + my[None, :, None] ** 2 + mz[None, None, :] ** 2
    B = (bspline_moduli(K[0], p)[:, None, None] * bspline_moduli(K[1], p)[None, :, None]
         * bspline_moduli(K[2], p)[None, None, :])
    with np.errstate(divide="ignore", invalid="ignore"):
        G = np.exp(-math.pi ** 2 * m2 / beta ** 2) / (math.pi * V * m2) * B
    G[0, 0, 0] = 0.0
    return G


def _stencil(pos, box, K, p):
    """Per atom and dimension: grid indices (N,3,p), weights and derivative weights."""
    pos = np.asarray(pos, np.float64)
    s = pos / box[None, :] - np.floor(pos / box[None, :])
    u = s * np.asarray(K, np.float64)[None, :]
    fl = np.floor(u)
    j = np.arange(p)
    k = fl[:, :, None] - j[None, None, :]                  # floor(u) - j
    t = u[:, :, None] - k                                  # u - k in [0, p)
    w = bspline(p, t)
    dw = bspline_deriv(p, t) * (np.asarray(K, np.float64) / box)[None, :, None]
    idx = np.mod(k.astype(np.int64), np.asarray(K)[None, :, None])
    return idx, w, dw


def spread(pos, q, box, K, p):
    idx, w, _ = _stencil(pos, box, K, p)
    Q = np.zeros(tuple(K))
    for a in range(p):
        for b in range(p):
            for c in range(p):
                np.add.at(Q, (idx[:, 0, a], idx[:, 1, b], idx[:, 2, c]),
                          q * w[:, 0, a] * w[:, 1, b] * w[:, 2, c])
    return Q


def pme(pos, q, box, beta, K, p=4):
    """Returns E_rec, phi_rec (N,), F_rec (N,3), and the grids for inspection."""
    K = tuple(int(k) for k in K)
    box = np.asarray(box, np.float64)
    Q = spread(pos, q, box, K, p)
    Qh = np.fft.fftn(Q)
    G = influence(box, K, beta, p)
    E = 0.5 * F_COUL * float(np.sum(G * np.abs(Qh) ** 2))
    phig = np.real(np.fft.ifftn(G * Qh)) * (K[0] * K[1] * K[2])
    idx, w, dw = _stencil(pos, box, K, p)
    n = len(q)
    phi = np.zeros(n)
    grad = np.zeros((n, 3))
    for a in range(p):
        for b in range(p):
            for c in range(p):
                g = phig[idx[:, 0, a], idx[:, 1, b], idx[:, 2, c]]
                phi += w[:, 0, a] * w[:, 1, b] * w[:, 2, c] * g
                grad[:, 0] += dw[:, 0, a] * w[:, 1, b] * w[:, 2, c] * g
                grad[:, 1] += w[:, 0, a] * dw[:, 1, b] * w[:, 2, c] * g
                grad[:, 2] += w[:, 0, a] * w[:, 1, b] * dw[:, 2, c] * g
    F = -F_COUL * q[:, None] * grad
    return dict(E_rec=E, phi=phi, F=F, Q=Q, phi_grid=phig)

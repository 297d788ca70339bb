"""Bussi-Donadio-Parrinello stochastic velocity rescaling (the paper's thermostat, PAPER.md:888,
:902-906; J. Chem. Phys. 126, 014101 (2007)).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

For a thermostat group with Nf degrees of freedom and kinetic energy K, target
Kbar = Nf kT / 2, one step of length dt with coupling time tau draws
    K' = K + (1 - c)(Kbar (R1^2 + S)/Nf - K) + 2 R1 sqrt(K Kbar / Nf (1 - c) c),
c = exp(-dt/tau), R1 ~ N(0,1), S ~ chi^2 with Nf - 1 degrees of freedom (Bussi 2007 Eq. A7),
and rescales every velocity of the group by alpha = sqrt(K'/K), with the sign of
R1 + sqrt(c Nf K / ((1 - c) Kbar)) (Bussi 2007 Appendix; reading R27).

Random numbers (reading R28; both sides implement the same counter-based generator):
Philox4x32-10 with key = replica seed and counters (step, k, stream, 0), stream 2 for the
atoms and 3 for the lambda particles; uniforms u = (x + 0.5) 2^-32, Box-Muller.
  R1 = z0 of k = 0.
  Nf - 1 <= 32: S = sum of squares of the first Nf - 1 normals z0..z3 of k = 1, 2, ...
  Nf - 1 > 32:  S = 2 Gamma((Nf - 1)/2) by Marsaglia-Tsang (ACM TOMS 26, 363 (2000)):
      d = a - 1/3, c = 1/sqrt(9 d); for k = 1, 2, ...: x = z0 of k, U = u2 of k,
      v = (1 + c x)^3; accept d v if v > 0 and ln U < x^2/2 + d - d v + d ln v.
"""
import math

import numpy as np

from .philox import _key, normals, philox4x32

STREAM_ATOMS = 2
STREAM_LAMBDA = 3
SMALL_NF = 32


def _uniforms(seed, step, k, stream):
    ctr = np.array([[step & 0xFFFFFFFF, k, stream, 0]], dtype=np.uint64)
    x = philox4x32(ctr, _key(seed)[None, :]).astype(np.float64)[0]
    return (x + 0.5) * 2.0 ** -32


def gamma_marsaglia_tsang(a, seed, step, stream):
    """Gamma(a, 1) deviate, a >= 1, from the counter stream k = 1, 2, ..."""
    d = a - 1.0 / 3.0
    c = 1.0 / math.sqrt(9.0 * d)
    k = 1
    while True:
        u = _uniforms(seed, step, k, stream)
        x = math.sqrt(-2.0 * math.log(u[0])) * math.cos(2.0 * math.pi * u[1])
        v = (1.0 + c * x) ** 3
        if v > 0.0 and math.log(u[2]) < 0.5 * x * x + d - d * v + d * math.log(v):
            return d * v
        k += 1


def bussi_draws(seed, step, stream, nf):
    """(R1, S) for one group and step."""
    R1 = float(normals(seed, step, [0], stream)[0, 0])
    m = nf - 1
    if m <= 0:
        return R1, 0.0
    if m <= SMALL_NF:
        nk = (m + 3) // 4
        z = normals(seed, step, np.arange(1, 1 + nk), stream).reshape(-1)[:m]
        return R1, float(np.sum(z * z))
    return R1, 2.0 * gamma_marsaglia_tsang(0.5 * m, seed, step, stream)


def bussi_alpha(K, nf, kT, dt, tau, R1, S):
    """Velocity scale factor of one Bussi step (alpha = 1 for an empty or frozen group)."""
    if nf <= 0 or not K > 0.0:
        return 1.0
    c = math.exp(-dt / tau)
    kbar = 0.5 * nf * kT
    k_new = K + (1.0 - c) * (kbar * (R1 * R1 + S) / nf - K) + 2.0 * R1 * math.sqrt(K * kbar / nf * (1.0 - c) * c)
    alpha = math.sqrt(max(k_new, 0.0) / K)
    if c < 1.0 and R1 + math.sqrt(c * nf * K / ((1.0 - c) * kbar)) < 0.0:
        alpha = -alpha
    return alpha

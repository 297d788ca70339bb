"""Pins of the Bussi-Donadio-Parrinello thermostat oracle (oracle.thermostat; PAPER.md:888,
:902-906) against the properties that define it: the kinetic-energy map leaves the Gamma
(canonical) distribution invariant, one degree of freedom reduces to the exact
Ornstein-Uhlenbeck update, tau -> infinity is the identity, and the chi-square draws have
the right moments."""
import math

import numpy as np
import pytest

from oracle import thermostat as TH
from oracle.units import kT

KT = kT(300.0)


@pytest.mark.parametrize("nf", [1, 3, 20, 60])
def test_kinetic_energy_chain_is_canonical(nf):
    """Iterating K -> alpha^2 K samples Gamma(Nf/2, kT): mean Nf kT/2, variance Nf (kT)^2/2
    (a dropped noise term or a wrong weight shifts one of them)."""
    dt, tau = 0.002, 0.01                      # c = e^-0.2: short correlation
    K = 0.5 * nf * KT
    ks = []
    n = 12000
    for step in range(n):
        R1, S = TH.bussi_draws(4242, step, TH.STREAM_ATOMS, nf)
        K = TH.bussi_alpha(K, nf, KT, dt, tau, R1, S) ** 2 * K
        if step >= 200:
            ks.append(K)
    ks = np.array(ks)
    c = math.exp(-dt / tau)
    n_eff = len(ks) * (1 - c) / (1 + c)
    mean, var = 0.5 * nf * KT, 0.5 * nf * KT ** 2
    assert abs(ks.mean() - mean) < 4.0 * math.sqrt(var / n_eff)
    # variance of the sample variance of a Gamma(k, theta): (2 k^2 + 6 k) theta^4 / n roughly
    kk = 0.5 * nf
    sd_var = math.sqrt((2 * kk * kk + 6 * kk) * KT ** 4 / n_eff)
    assert abs(ks.var() - var) < 5.0 * sd_var


def test_one_degree_of_freedom_is_ornstein_uhlenbeck():
    """Nf = 1: alpha v = sqrt(c) v + sqrt((1-c) kT/m) R1 sgn(v) exactly (Bussi 2007 App.)."""
    m, dt, tau = 60.0, 0.002, 1.0
    c = math.exp(-dt / tau)
    for v in (0.7, -1.3, 0.05, -0.02):
        for R1 in (0.3, -2.5, 1.7, -40.0):
            K = 0.5 * m * v * v
            a = TH.bussi_alpha(K, 1, KT, dt, tau, R1, 0.0)
            assert a * v == pytest.approx(math.sqrt(c) * v + math.sqrt((1 - c) * KT / m) * R1 * math.copysign(1, v),
                                          rel=1e-12, abs=1e-14)


def test_decoupled_limit_and_degenerate_groups():
    assert TH.bussi_alpha(3.0, 10, KT, 0.002, math.inf, 0.4, 9.0) == 1.0
    assert TH.bussi_alpha(0.0, 10, KT, 0.002, 0.1, 0.4, 9.0) == 1.0       # frozen group
    assert TH.bussi_alpha(3.0, 0, KT, 0.002, 0.1, 0.4, 9.0) == 1.0


@pytest.mark.parametrize("nf", [2, 33, 34, 200])
def test_chi_square_draws(nf):
    """S ~ chi^2(Nf - 1): mean Nf - 1, variance 2 (Nf - 1), from both the explicit-squares
    path (Nf - 1 <= 32) and the Marsaglia-Tsang Gamma path."""
    n = 3000
    S = np.array([TH.bussi_draws(77, s, TH.STREAM_LAMBDA, nf)[1] for s in range(n)])
    R1 = np.array([TH.bussi_draws(77, s, TH.STREAM_LAMBDA, nf)[0] for s in range(200)])
    m = nf - 1
    assert abs(S.mean() - m) < 4.0 * math.sqrt(2 * m / n)
    assert abs(S.var() - 2 * m) < 5.0 * math.sqrt((8 * m * m + 48 * m) / n)
    assert abs(R1.mean()) < 0.3 and 0.7 < R1.std() < 1.3

"""Residue-residue coupling screen, no GPU.

Pins of the oracle's NMI (oracle.analysis.nmi_binary, written from the definitions of I and
H) against closed forms, then the product's vectorised screen (titration.coupling_screen)
against the oracle on synthetic coupled / uncoupled two-site chains, and the macroscopic
two-site titration fit recovering its constants."""
import math

import numpy as np

from oracle import analysis as OA
from paper_2410_01626_b200 import titration as T


def test_nmi_closed_forms():
    rng = np.random.default_rng(0)
    x = (rng.random(4000) < 0.5).astype(int)
    v, hx, hy = OA.nmi_binary(x, x)
    assert abs(v - 1.0) < 1e-12 and abs(hx - hy) < 1e-15            # identical: NMI = 1
    assert abs(OA.nmi_binary(x, 1 - x)[0] - 1.0) < 1e-12             # complementary: NMI = 1
    assert abs(hx - math.log(2)) < 1e-3                              # fair coin: H = ln 2
    assert OA.nmi_binary(np.zeros(50), np.ones(50))[0] == 0.0        # constant: H = 0, NMI = 0
    # a known joint distribution: I = sum p ln p/(px py) exactly on the empirical table
    pj = np.array([[0.4, 0.1], [0.1, 0.4]])
    n = 10000
    counts = (pj * n).astype(int)
    xs = np.concatenate([np.full(counts[a, b], a) for a in range(2) for b in range(2)])
    ys = np.concatenate([np.full(counts[a, b], b) for a in range(2) for b in range(2)])
    I = sum(pj[a, b] * math.log(pj[a, b] / 0.25) for a in range(2) for b in range(2))
    v, hx, hy = OA.nmi_binary(xs, ys)
    assert abs(v - 2 * I / (2 * math.log(2))) < 1e-12
    # independent chains: NMI ~ 0 (finite-sample bias O(1/n))
    y = (rng.random(4000) < 0.3).astype(int)
    assert OA.nmi_binary(x, y)[0] < 2e-3


def _chains(rng, n_frames, coupling):
    """Two binary protonation chains (Gibbs-sampled 2-site Ising pair) as lambda_p frames."""
    s = np.zeros((n_frames, 2), int)
    a, b = 1, 1
    for t in range(n_frames):
        for k in range(2):
            other = b if k == 0 else a
            p1 = 1.0 / (1.0 + math.exp(-coupling * (2 * other - 1)))
            v = int(rng.random() < p1)
            if k == 0:
                a = v
            else:
                b = v
        s[t] = a, b
    return np.where(s == 1, 0.1, 0.9)            # protonated -> lambda_p 0.1, else 0.9


def test_screen_matches_oracle_and_flags_only_the_coupled_pair():
    rng = np.random.default_rng(3)
    npH, R, F = 2, 3, 600
    fr = np.zeros((npH, R, F, 3))
    for k in range(npH):
        for r in range(R):
            fr[k, r, :, :2] = _chains(rng, F, 2.0)                  # sites 0, 1 coupled
            fr[k, r, :, 2] = np.where(rng.random(F) < 0.5, 0.1, 0.9)  # site 2 independent
    coupled, m_nmi, m_h = T.coupling_screen(fr)
    assert coupled == [(0, 1)]
    for k in range(npH):
        for a, c in ((0, 1), (0, 2), (1, 2)):
            ref = np.mean([OA.nmi_binary(OA.protonated(fr[k, r, :, a]), OA.protonated(fr[k, r, :, c]))[0]
                           for r in range(R)])
            assert abs(m_nmi[k, a, c] - ref) < 1e-12
    # a nearly frozen site (few deprotonated frames) is not flagged even with high NMI
    fr2 = fr.copy()
    fr2[..., 2] = 0.1
    fr2[:, :, :3, 2] = 0.9
    fr2[:, :, :3, 0] = 0.9
    assert (0, 2) not in T.coupling_screen(fr2)[0]


def test_two_site_macroscopic_fit():
    pH = np.linspace(1.0, 9.0, 33)
    X = OA.two_site_protons(pH, 3.7, 5.9)
    assert np.allclose(T.two_site_protons(pH, 3.7, 5.9), X, rtol=1e-14)
    assert abs(X[0] - 2.0) < 5e-3 and abs(X[-1]) < 5e-3               # fully protonated / deprotonated
    p1, p2 = T.fit_two_site(pH, X)
    assert abs(p1 - 3.7) < 1e-6 and abs(p2 - 5.9) < 1e-6
    q1, q2 = OA.fit_two_site(pH, X)
    assert abs(q1 - 3.7) < 1e-8 and abs(q2 - 5.9) < 1e-8
    # independent sites with micro pKa a, b: macro constants satisfy pKa1 + pKa2 = a + b
    a, b = 4.0, 4.5
    Xi = 1 / (1 + 10 ** (pH - a)) + 1 / (1 + 10 ** (pH - b))
    p1, p2 = T.fit_two_site(pH, Xi)
    assert abs((p1 + p2) - (a + b)) < 1e-6

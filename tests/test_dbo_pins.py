"""Pins of the DBO oracle (oracle.dbo, generalised oracle.bias / oracle.pfc) against the
paper's stated rules and constants, closed forms of the shifted double
well, and brute-force quadrature independent of the oracle's own integrators."""
import math

import numpy as np
import pytest

from oracle import bias as B
from oracle import dbo as D
from oracle import pfc as PFC
from oracle.units import LN10, kT


# -- controller rules (SPEC dbo examples) ---------------------------------

def test_well_rule_examples():
    # residency 0.80 near well 0 with mean 0.05 -> the centre moves by 0.5 (0 - 0.05)
    n = 1000
    assert D.well_block_decide(0.0, n, 800, 800 * 0.05, 0.0) == pytest.approx(-0.025, abs=1e-15)
    # residency 0.60: "more than 70 % of the time" not met
    assert D.well_block_decide(0.0, n, 600, 600 * 0.05, 0.0) == 0.0
    # exactly 70 % is not "more than"
    assert D.well_block_decide(0.0, n, 700, 700 * 0.05, 0.0) == 0.0
    # within the 0.03 tolerance
    assert D.well_block_decide(0.0, n, 900, 900 * 0.02, 0.0) == 0.0
    # well 1: mean 0.95 -> centre moves outwards by 0.025
    assert D.well_block_decide(0.0, n, 900, 900 * 0.95, 1.0) == pytest.approx(0.025, abs=1e-15)
    # the accumulated shift is capped at +-0.08
    s = 0.0
    for _ in range(10):
        s = D.well_block_decide(s, n, 900, 900 * 0.15, 0.0)
    assert s == -0.08
    # empty block
    assert D.well_block_decide(0.03, 0, 0, 0.0, 0.0) == 0.03


def test_barrier_rule_examples():
    assert D.barrier_block_decide(6.0, 1000, 100) == 5.0        # 10 % < 20 %
    assert D.barrier_block_decide(6.0, 1000, 270) == 6.0        # inside 25 +- 5 %
    assert D.barrier_block_decide(6.0, 1000, 200) == 6.0        # band edges inclusive
    assert D.barrier_block_decide(6.0, 1000, 300) == 6.0
    assert D.barrier_block_decide(6.0, 1000, 301) == 7.0
    assert D.barrier_block_decide(1.0, 1000, 50) == 1.0         # floor 1 kJ/mol
    assert D.barrier_block_decide(20.0, 1000, 900) == 20.0      # cap 20 kJ/mol
    assert D.barrier_block_decide(6.0, 0, 0) == 6.0             # no frames in this state


def test_block_stats_classes():
    st = D.BlockStats(3)
    lp_of = np.array([-1, 0, -1])
    for lam in ([0.1, 0.5, 0.9], [0.6, 0.1, 0.95], [0.9, 0.85, 0.3]):
        st.add(np.array(lam), lp_of)
    np.testing.assert_allclose(st.well[0], [3, 1, 0.1, 1, 0.9])
    np.testing.assert_allclose(st.well[1], [3, 1, 0.1, 1, 0.85])
    # tautomer coordinate 1: protonated when lambda_p (coord 0) < 0.5
    np.testing.assert_allclose(st.barrier[1], [1, 1, 2, 0])
    np.testing.assert_allclose(st.barrier[0], [3, 1, 0, 0])


def test_censor_window():
    # adjustment at 100 ps, frames every 0.5 ps (250 steps of 2 fs), 10 ps window -> 20 frames
    S = 50000
    t = np.arange(0, 200001, 250)
    f = D.censor_flags(t, [S], 5000)
    assert f.sum() == 20 and f[t == S].sum() == 0 and f[t == S + 5000].all()
    assert D.censor_flags(t, [], 5000).sum() == 0
    # overlapping windows merge (union)
    f2 = D.censor_flags(t, [S, S + 2500], 5000)
    assert f2.sum() == 30


def test_update_events_and_safety():
    dbo = B.default_dbo(6.0, 2)
    st = D.BlockStats(2)
    lp_of = np.array([-1, 0])
    rng = np.random.default_rng(0)
    for _ in range(100):
        st.add(np.array([rng.uniform(0.1, 0.15), 0.5]), lp_of)
    ev = D.well_update(dbo, st)
    assert [(c, k) for c, k, *_ in ev] == [(0, D.WELL0)]
    assert -D.WELL_CAP <= dbo[0, 0] < 0.0 and dbo[0, 1] == 1.0
    ev = D.barrier_update(dbo, st, lp_of)
    # coordinate 0: no frame in transition -> lower; coordinate 1 (tautomer, protonated
    # class only): all frames in transition -> raise h_prot, h_deprot untouched
    assert (0, D.BARRIER, 6.0, 5.0) in ev and (1, D.BARRIER_T_PROT, 6.0, 7.0) in ev
    assert dbo[1, 3] == 6.0 and dbo[0, 2] == dbo[0, 3] == 5.0


# -- shifted double well (PAPER.md:738-740 with DBO well centres) ----------------------------

@pytest.mark.parametrize("a0,a1", [(0.0, 1.0), (0.05, 0.94), (-0.08, 1.08)])
def test_shifted_double_well_closed_forms(a0, a1):
    h, d1, kw = 6.0, -3.5, 1e6
    m = 0.5 * (a0 + a1)
    for lam, val in ((a0, 0.0), (m, h), (a1, d1)):
        v, dv, _ = B.vdw_full(lam, h, 0.0, d1, kw, a0, a1)
        assert v == pytest.approx(val, abs=1e-12) and dv == pytest.approx(0.0, abs=1e-9)
    # mirror symmetry about each centre, inside the wall-free range
    for dl in (0.005, 0.015):              # a0 - dl > -0.1 and a1 + dl < 1.1: no wall
        assert B.vdw(a0 - dl, h, 0.0, d1, kw, a0, a1)[0] == pytest.approx(B.vdw(a0 + dl, h, 0.0, d1, kw, a0, a1)[0])
        assert B.vdw(a1 + dl, h, 0.0, d1, kw, a0, a1)[0] == pytest.approx(B.vdw(a1 - dl, h, 0.0, d1, kw, a0, a1)[0])
    # midpoint of the left segment: Hermite value h/2
    assert B.vdw(0.5 * (a0 + m), h, 0.0, d1, kw, a0, a1)[0] == pytest.approx(0.5 * h)
    # derivatives by finite differences (lambda and h), across segments and walls
    e = 1e-6
    for lam in (-0.13, -0.03, 0.21, 0.47, 0.66, 1.02, 1.13):
        v, dv, dh = B.vdw_full(lam, h, 0.0, d1, kw, a0, a1)
        fd = (B.vdw(lam + e, h, 0.0, d1, kw, a0, a1)[0] - B.vdw(lam - e, h, 0.0, d1, kw, a0, a1)[0]) / (2 * e)
        fh = (B.vdw(lam, h + e, 0.0, d1, kw, a0, a1)[0] - B.vdw(lam, h - e, 0.0, d1, kw, a0, a1)[0]) / (2 * e)
        assert dv == pytest.approx(fd, rel=1e-6, abs=1e-6)
        assert dh == pytest.approx(fh, rel=1e-6, abs=1e-8)


def test_tautomer_barrier_smooth_in_lambda_p():
    assert B.tautomer_barrier(-0.05, 2.0, 9.0) == (2.0, 0.0)
    assert B.tautomer_barrier(0.0, 2.0, 9.0)[0] == 2.0
    assert B.tautomer_barrier(1.0, 2.0, 9.0)[0] == 9.0
    assert B.tautomer_barrier(1.07, 2.0, 9.0) == (9.0, 0.0)
    assert B.tautomer_barrier(0.5, 2.0, 9.0)[0] == pytest.approx(5.5)
    e = 1e-7
    for lp in (0.1, 0.5, 0.83):
        fd = (B.tautomer_barrier(lp + e, 2.0, 9.0)[0] - B.tautomer_barrier(lp - e, 2.0, 9.0)[0]) / (2 * e)
        assert B.tautomer_barrier(lp, 2.0, 9.0)[1] == pytest.approx(fd, rel=1e-6)


def test_group_bias_gradient_with_split_tautomer_barriers():
    """dV/dlambda_p picks up the barrier's lambda_p dependence (catches a dropped term)."""
    rng = np.random.default_rng(2)
    c36 = rng.normal(0, 3, 36)
    pk = np.array([6.6, 6.53, 6.92])
    dbo = np.array([[0.03, 0.97, 5.0, 5.0], [-0.04, 1.05, 2.0, 9.0]])
    e = 1e-7
    for lp, lt in ((0.3, 0.7), (0.62, 0.2), (0.9, 1.04)):
        v, dp, dt = B.group_bias(3, c36, pk, 6.0, 300.0, 6.0, -2.0, 1.5, 1e6, lp, lt, dbo)
        fp = (B.group_bias(3, c36, pk, 6.0, 300.0, 6.0, -2.0, 1.5, 1e6, lp + e, lt, dbo)[0] -
              B.group_bias(3, c36, pk, 6.0, 300.0, 6.0, -2.0, 1.5, 1e6, lp - e, lt, dbo)[0]) / (2 * e)
        ft = (B.group_bias(3, c36, pk, 6.0, 300.0, 6.0, -2.0, 1.5, 1e6, lp, lt + e, dbo)[0] -
              B.group_bias(3, c36, pk, 6.0, 300.0, 6.0, -2.0, 1.5, 1e6, lp, lt - e, dbo)[0]) / (2 * e)
        assert dp == pytest.approx(fp, rel=1e-6) and dt == pytest.approx(ft, rel=1e-6)


# -- PFC after DBO changes, brute-force quadrature --------------------------

def _trap_halves(lam, V, kt):
    w = np.exp(-(V - V.min()) / kt)
    left = lam < 0.5
    return np.trapezoid(np.where(left, w, 0.0), lam), np.trapezoid(np.where(~left, w, 0.0), lam)


@pytest.mark.parametrize("a0,a1,h", [(0.05, 0.94, 6.0), (-0.08, 1.08, 2.0), (0.0, 1.0, 17.0)])
def test_pfc_2state_shifted_wells_brute_force(a0, a1, h):
    T, kw, pKa, pH = 300.0, 1e6, 4.4, 3.9
    d1 = PFC.pfc_2state(h, pKa, pH, T, kw, a0, a1)
    lam = np.linspace(-0.45, 1.45, 2_000_001)
    g = LN10 * kT(T) * (pKa - pH)
    V = B.vdw(lam, h, 0.0, d1, kw, a0, a1)[0] + lam * g
    zp, zd = _trap_halves(lam, V, kT(T))
    assert -kT(T) * math.log(zd / zp) == pytest.approx(g, abs=2e-5)


def test_pfc_3state_shifted_wells_split_barriers_brute_force():
    T, kw, pH = 300.0, 1e6, 6.3
    pk = np.array([6.6, 6.53, 6.92])
    dbo = np.array([[0.04, 0.95, 4.0, 4.0], [-0.03, 1.06, 2.0, 8.0]])
    d1p, d1t = PFC.pfc_3state(6.0, pk, pH, T, kw, dbo)
    n = 2401
    lp = np.linspace(-0.45, 1.45, n)
    lt = np.linspace(-0.45, 1.45, n)
    LP, LT = np.meshgrid(lp, lt, indexing="ij")
    ht = dbo[1, 2] + (dbo[1, 3] - dbo[1, 2]) * np.where(LP <= 0, 0, np.where(LP >= 1, 1, 3 * LP**2 - 2 * LP**3))
    V = (B.vdw(LP, dbo[0, 2], 0.0, d1p, kw, dbo[0, 0], dbo[0, 1])[0] +
         B.vdw(LT, ht, 0.0, d1t, kw, dbo[1, 0], dbo[1, 1])[0] +
         LP * ((1 - LT) * B.delta_g(pk[1], pH, T) + LT * B.delta_g(pk[2], pH, T)))
    W = np.exp(-(V - V.min()) / kT(T))
    hstep = lp[1] - lp[0]
    wq = np.full(n, hstep)
    wq[0] = wq[-1] = 0.5 * hstep
    W = W * wq[:, None] * wq[None, :]
    prot = LP < 0.5
    zp = W[prot].sum()
    zd = W[~prot & (LT < 0.5)].sum()
    ze = W[~prot & (LT >= 0.5)].sum()
    gd, ge = -kT(T) * math.log(zd / zp), -kT(T) * math.log(ze / zp)
    assert gd == pytest.approx(B.delta_g(pk[1], pH, T), abs=2e-3)
    assert ge == pytest.approx(B.delta_g(pk[2], pH, T), abs=2e-3)

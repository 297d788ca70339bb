"""Pins of oracle.titration_quadrature (no GPU): the frozen-environment titration curve
that the electrostatics-on GPU titration is compared with (tests/test_gpu_pka_parity.py).

* b = c = 0: the quadrature reproduces the PFC target, i.e. the H-H fraction
  1/(10^(pKa-pH)+1) of PAPER.md:979 (exact by construction of the PFC);
* the quadratic read off the engine's E_coul matches the engine's own analytic dV/dlambda
  (b = dV_coul/dl at 0, b + 2c at 1: catches a wrong finite-difference stencil or a
  non-quadratic E_coul, i.e. a charge that is not linear in lambda);
* a linear Coulomb term b lambda shifts the pKa by about b / (ln10 kT) in b's direction;
* the oracle's own lambda dynamics (oracle.lambda_only, BAOAB + Philox) sampling the
  same potential reproduces the quadrature fractions."""
import copy
import math

import numpy as np

from oracle import analysis, titration_quadrature as TQ
from oracle.engine import OracleReplica
from oracle.lambda_only import run_2state
from oracle.pfc import pfc_2state
from oracle.units import kT
from synthetic.systems import make_system


def test_quadrature_without_coulomb_is_hh():
    pH = np.array([3.4, 4.0, 4.4, 5.0, 5.4])
    x = TQ.titration_curve(4.4, pH, 300.0, 2.0, 1e6)
    np.testing.assert_allclose(x, 1.0 / (10 ** (4.4 - pH) + 1.0), atol=2e-6)


def test_linear_coulomb_term_shifts_pka_by_about_b_over_ln10kT():
    """A linear Coulomb term b lambda adds to the pH term (which the PFC, computed from
    Vdw + VpH only, does not see): the fitted pKa moves by ~ b/(ln10 kT) (the PFC depth,
    tuned for the unshifted pH term, makes it inexact), in the direction of b's sign."""
    pH = np.linspace(2.5, 6.5, 9)
    for b in (-4.0, 4.0):
        x = TQ.titration_curve(4.4, pH, 300.0, 2.0, 1e6, b=b, n=100001)
        shift = analysis.fit_hh(pH, x) - 4.4
        expect = b / (math.log(10.0) * kT(300.0))
        assert np.sign(shift) == np.sign(expect) and abs(shift - expect) < 0.4 * abs(expect), (shift, expect)


def test_coulomb_quadratic_matches_engine_dvdl():
    s = copy.deepcopy(make_system(1))
    s.mass[:] = 0.0
    rep = OracleReplica(s, 4.4, 1, lam0=np.zeros(1))
    b, c, chk = TQ.coulomb_quadratic(rep, 0)
    d0 = rep.evaluate(rep.x, np.zeros(1))["dvdl_coul"][0]
    d1 = rep.evaluate(rep.x, np.ones(1))["dvdl_coul"][0]
    assert abs(d0 - b) < 1e-7 * max(1.0, abs(b)), (d0, b)
    assert abs(d1 - (b + 2 * c)) < 1e-7 * max(1.0, abs(b + 2 * c)), (d1, b + 2 * c)
    assert chk < 1e-8 * max(1.0, abs(b))
    assert abs(b) > 1.0 and abs(c) > 1.0              # a real electrostatic coupling


def test_quadrature_matches_oracle_lambda_dynamics():
    """The same 1-D potential sampled by oracle.lambda_only (linear + quadratic Coulomb
    term supplied through V_mm's c_10, c_20)."""
    pKa, h, M = 4.4, 2.0, 1000
    b, c = -3.0, 2.5
    pHs = np.array([3.9, 4.7])
    vmm = np.zeros(36)
    vmm[6], vmm[12] = b, c                              # c_10 lp + c_20 lp^2
    ref = TQ.titration_curve(pKa, pHs, 300.0, h, 1e6, b=b, c=c)
    d1 = np.repeat([pfc_2state(h, pKa, p, 300.0, 1e6) for p in pHs], M)
    pH = np.repeat(pHs, M)
    lam0 = np.tile((np.arange(M) % 2).astype(float), 2)
    seeds = np.arange(1, 2 * M + 1, dtype=np.uint64) * np.uint64(40503) + np.uint64(11)
    # a light lambda particle (the mass does not enter the equilibrium density) relaxes in
    # ~1 ps, so the start (half at 0, half at 1) is forgotten after the first 4 ps
    fr, _ = run_2state(seeds, lam0, pKa, pH, 4000, h_barrier=h, d1=d1, vmm=vmm, mass=6.0)
    fr = fr[150:]
    x = np.array([analysis.deprotonated_fraction(fr[:, k * M:(k + 1) * M]) for k in range(2)])
    assert np.all(np.abs(x - ref) < 0.02), (x, ref)


def test_his_quadrature_without_coulomb_is_the_micro_pka_closed_form():
    """2-D quadrature, no Coulomb term: the 3-state PFC makes the populations 1 : 10^(pH - pKa_d) :
    10^(pH - pKa_e) (Table 2 micro pKa)."""
    pk = (6.38, 6.53, 6.92)
    for pH in (6.0, 6.9):
        dep, d, e = TQ.his_fractions(pk, pH, 300.0, 2.0, 1e6, n=801)
        wd, we = 10 ** (pH - pk[1]), 10 ** (pH - pk[2])
        assert abs(d - wd / (1 + wd + we)) < 1e-3 and abs(e - we / (1 + wd + we)) < 1e-3
        assert abs(dep - d - e) < 1e-12


def test_his_biquadratic_matches_engine_dvdl():
    """The 3 x 3 read-off of E_coul(lp, lt) against the engine's analytic dV_coul/dlp, dV_coul/dlt
    at an interior point (a wrong Vandermonde inverse or a missing cross term fails)."""
    from synthetic.systems import small_system
    s = copy.deepcopy(small_system())
    s.mass[:] = 0.0
    rep = OracleReplica(s, 6.4, 1, lam0=np.array([0.3, 0.0, 0.0]))
    c, chk = TQ.coulomb_biquadratic(rep, 1, 2)
    assert chk < 1e-8 * max(1.0, np.abs(c).max())
    lp, lt = 0.35, 0.6
    g = rep.evaluate(rep.x, np.array([0.3, lp, lt]))["dvdl_coul"]
    dp = sum(a * c[a, b] * lp ** (a - 1) * lt ** b for a in range(1, 3) for b in range(3))
    dt = sum(b * c[a, b] * lp ** a * lt ** (b - 1) for a in range(3) for b in range(1, 3))
    assert abs(g[1] - dp) < 1e-6 * max(1.0, abs(dp)) and abs(g[2] - dt) < 1e-6 * max(1.0, abs(dt))

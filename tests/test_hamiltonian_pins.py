"""Pins of the Hamiltonian-interpolation oracle (oracle.hamiltonian; Eq. 1):
E_CI + sum_g C_g equals the multilinear weighted sum of the Coulomb energies of every
combination of the groups' forms (Eq. 1/Eq. 2 written out, each endpoint evaluated with the
oracle's exact Ewald sum), and its lambda and position derivatives match finite differences."""
import itertools

import numpy as np
import pytest

from oracle import hamiltonian as HI
from oracle.charges import coord_ptr, eq2_weights
from oracle.engine import OracleReplica
from oracle.ewald import ewald_beta
from synthetic.systems import small_system

COUL = ("real", "excl", "self", "recip", "net")


@pytest.fixture(scope="module")
def setup():
    s = small_system()
    beta = ewald_beta(s.params["rc"], s.params["ewald_rtol"])
    kv = HI.kvectors(s.box, beta, eps=1e-14)
    return s, beta, kv


def _coulomb(s, lam, nmax):
    ref = OracleReplica(s, 4.4, 1, lam0=lam, recip="direct", nmax=nmax)
    return sum(ref.cur["E"][k] for k in COUL)


def test_hamiltonian_interpolation_is_eq1_multilinear_sum(setup):
    s, beta, kv = setup
    nmax = 15                                       # exp(-pi^2 (15/2.3)^2 / beta^2) ~ 1e-18
    lam = np.array([0.3, 0.65, 0.2])                # Glu lp, His lp, His lt
    cptr = coord_ptr(s.group_kind)
    e_ci = _coulomb(s, lam, nmax)
    e_hi, _, _ = HI.hi_terms(s, s.pos, lam, cptr, s.box, beta, s.params["rc"], kv)
    # corners: every form of the Glu group (A=B, C=D) x every form of the His group
    corner = {0: (0.0, 0.0), 1: (0.0, 1.0), 2: (1.0, 0.0), 3: (1.0, 1.0)}
    w_glu = eq2_weights(lam[0], 0.0)
    w_his = eq2_weights(lam[1], lam[2])
    tot = 0.0
    for a, b in itertools.product(range(4), range(4)):
        wa, wb = w_glu[a], w_his[b]
        if wa * wb == 0.0:
            continue
        lam_c = np.array([corner[a][0], corner[b][0], corner[b][1]])
        if a in (1, 3):                             # Glu forms B / D equal A / C (lt-free)
            lam_c[0] = corner[a][0]
        tot += wa * wb * _coulomb(s, lam_c, nmax)
    print("E_CI", e_ci, "C", e_hi, "sum w E", tot)
    assert abs(e_hi) > 1e-3                         # the correction is not trivially zero
    assert abs(e_ci + e_hi - tot) < 1e-8 * abs(tot)


def test_correction_vanishes_at_corners(setup):
    s, beta, kv = setup
    cptr = coord_ptr(s.group_kind)
    for lam in ([0.0, 0.0, 0.0], [1.0, 1.0, 0.0], [0.0, 1.0, 1.0]):
        e, _, _ = HI.hi_terms(s, s.pos, np.array(lam), cptr, s.box, beta, s.params["rc"], kv)
        assert abs(e) < 1e-9


def test_hi_derivatives_match_finite_differences(setup):
    s, beta, kv = setup
    cptr = coord_ptr(s.group_kind)
    lam = np.array([0.4, 0.3, 0.7])
    rc = s.params["rc"]
    e0, dv, F = HI.hi_terms(s, s.pos, lam, cptr, s.box, beta, rc, kv)
    h = 1e-6
    for c in range(3):
        lp, lm = lam.copy(), lam.copy()
        lp[c] += h
        lm[c] -= h
        fd = (HI.hi_terms(s, s.pos, lp, cptr, s.box, beta, rc, kv)[0] -
              HI.hi_terms(s, s.pos, lm, cptr, s.box, beta, rc, kv)[0]) / (2 * h)
        assert dv[c] == pytest.approx(fd, rel=1e-6, abs=1e-7)
    x = np.asarray(s.pos, np.float64)
    for atom in (s.group_atoms[0], s.group_atoms[9], s.group_atoms[-1]):
        for d in range(3):
            xp, xm = x.copy(), x.copy()
            xp[atom, d] += h
            xm[atom, d] -= h
            fd = -(HI.hi_terms(s, xp, lam, cptr, s.box, beta, rc, kv)[0] -
                   HI.hi_terms(s, xm, lam, cptr, s.box, beta, rc, kv)[0]) / (2 * h)
            assert F[atom, d] == pytest.approx(fd, rel=1e-5, abs=1e-5)

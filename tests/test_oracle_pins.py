"""Pins of the fp64 oracle against values fixed by the paper and by mathematics
(no GPU).  Each test names what it pins; see oracle/__init__.py."""
import math
import os

import numpy as np
import pytest

from oracle import analysis, bias, charges, ewald, pairlist, pfc, philox, pme
from oracle.engine import OracleReplica
from oracle.lambda_only import run_2state
from oracle.units import F_COUL, kT
from synthetic.systems import make_system, small_system

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                rows.append(line.split())
    return rows


# --------------------------------------------------------------------------- RNG (P8)
def test_philox_known_answers():
    for row in _golden("philox_kat.txt"):
        v = [int(x, 16) for x in row]
        out = philox.philox4x32(np.array([v[:4]], np.uint64), np.array([v[4:6]], np.uint64))[0]
        assert [int(x) for x in out] == v[6:10]


def test_box_muller_moments():
    z = philox.normals(12345, 7, np.arange(200000), 0).reshape(-1)
    assert abs(z.mean()) < 0.005 and abs(z.var() - 1.0) < 0.01


# --------------------------------------------------------------------------- Ewald (P1)
def _nacl_supercell(a, n):
    na = [(0, 0, 0), (0, .5, .5), (.5, 0, .5), (.5, .5, 0)]
    cl = [(.5, 0, 0), (0, .5, 0), (0, 0, .5), (.5, .5, .5)]
    pos, q = [], []
    for i in range(n):
        for j in range(n):
            for k in range(n):
                for s, qq in ((na, 1.0), (cl, -1.0)):
                    for p in s:
                        pos.append((np.array(p) + (i, j, k)) * a)
                        q.append(qq)
    return np.array(pos), np.array(q)


def _ewald_total(pos, q, box, beta, rc, nmax):
    n = len(q)
    t = np.zeros(n, np.int32)
    z = np.zeros((1, 1))
    rs = ewald.real_space(pos, q, t, z, z, box, rc, beta, np.zeros((0, 2), np.int32))
    es, _ = ewald.self_term(q, beta)
    en, _ = ewald.net_charge_term(q, box, beta)
    er, phir, Fr = ewald.recip_direct(pos, q, box, beta, nmax)
    return rs["E_real"] + es + en + er


def test_madelung_nacl():
    M = float(dict((r[0], r[1]) for r in _golden("madelung.txt"))["NaCl"])
    pos, q = _nacl_supercell(1.0, 2)              # 64 ions, L = 2 nm, d = 0.5 nm
    box = np.array([2.0, 2.0, 2.0])
    E = _ewald_total(pos, q, box, 6.0, 0.99, 24)
    ref = -32 * M * F_COUL / 0.5
    assert abs(E - ref) / abs(ref) < 1e-9


def test_madelung_cscl():
    M = float(dict((r[0], r[1]) for r in _golden("madelung.txt"))["CsCl"])
    a, n = 0.7, 3
    pos, q = [], []
    for i in range(n):
        for j in range(n):
            for k in range(n):
                pos.append(np.array([i, j, k]) * a)
                q.append(1.0)
                pos.append((np.array([i, j, k]) + 0.5) * a)
                q.append(-1.0)
    pos, q = np.array(pos), np.array(q)
    box = np.full(3, n * a)
    d = a * math.sqrt(3) / 2
    E = _ewald_total(pos, q, box, 6.0, 1.04, 24)
    ref = -n ** 3 * M * F_COUL / d
    assert abs(E - ref) / abs(ref) < 1e-8


def test_ewald_beta_from_rtol():
    b = ewald.ewald_beta(1.0, 1e-5)
    from scipy.special import erfc
    assert abs(erfc(b) - 1e-5) < 1e-15 and abs(b - 3.123413) < 1e-5


# --------------------------------------------------------------------------- PME (P3)
def _random_neutral(n, L, seed):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0, L, (n, 3))
    q = rng.uniform(-1, 1, n)
    q -= q.mean()
    return pos, q


def test_bspline_closed_forms():
    w = np.linspace(0, 1, 11)[:-1]
    th = [pme.bspline(4, w + j) for j in range(4)]
    np.testing.assert_allclose(th[0], w ** 3 / 6, atol=1e-15)
    np.testing.assert_allclose(th[3], (1 - w) ** 3 / 6, atol=1e-15)
    np.testing.assert_allclose(sum(th), 1.0, atol=1e-15)          # partition of unity
    # B-spline moduli of order 4 at m=0: |1/6 + 4/6 + 1/6|^-2 = 1
    assert abs(pme.bspline_moduli(16, 4)[0] - 1.0) < 1e-15


def test_pme_converges_to_direct_ewald():
    L = 2.0
    box = np.full(3, L)
    pos, q = _random_neutral(20, L, 3)
    beta = 3.1234
    E_d, phi_d, F_d = ewald.recip_direct(pos, q, box, beta, 14)
    errs = []
    for K in (16, 32, 64):
        r = pme.pme(pos, q, box, beta, (K, K, K), 4)
        eE = abs(r["E_rec"] - E_d) / abs(E_d)
        ephi = np.sqrt(np.mean((r["phi"] - phi_d) ** 2) / np.mean(phi_d ** 2))
        eF = np.linalg.norm(r["F"] - F_d) / np.linalg.norm(F_d)
        errs.append((eE, ephi, eF))
    assert errs[1][0] < 2e-4 and errs[1][1] < 2e-4 and errs[1][2] < 2e-3
    assert errs[2][1] < errs[1][1] < errs[0][1]
    assert errs[2][2] < errs[1][2] < errs[0][2]


def test_pme_energy_potential_identity():
    pos, q = _random_neutral(30, 2.5, 5)
    box = np.full(3, 2.5)
    r = pme.pme(pos, q, box, 3.0, (24, 20, 28), 4)
    assert abs(r["E_rec"] - 0.5 * F_COUL * np.sum(q * r["phi"])) < 1e-10 * abs(r["E_rec"])


def test_direct_ewald_forces_finite_difference():
    pos, q = _random_neutral(10, 2.0, 11)
    box = np.full(3, 2.0)
    E0, phi, F = ewald.recip_direct(pos, q, box, 3.0, 10)
    h = 1e-6
    for i in (0, 4):
        for d in range(3):
            p1 = pos.copy(); p1[i, d] += h
            p2 = pos.copy(); p2[i, d] -= h
            fd = -(ewald.recip_direct(p1, q, box, 3.0, 10)[0] - ewald.recip_direct(p2, q, box, 3.0, 10)[0]) / (2 * h)
            assert abs(fd - F[i, d]) < 1e-6 * (1 + abs(F[i, d]))


# --------------------------------------------------------------------------- lattice sum (P2)
def test_spherical_lattice_sum_equals_ewald_plus_dipole_term():
    """de Leeuw-Perram-Smith: spherical summation of the bare Coulomb lattice sum of a
    neutral cell = tin-foil Ewald + 2 pi f |M|^2 / (3 V)."""
    L = 1.0
    box = np.full(3, L)
    rng = np.random.default_rng(2)
    pos = rng.uniform(0, L, (4, 3))
    q = np.array([1.0, -1.0, 0.5, -0.5])
    beta = 12.5                                   # erfc(beta * 0.49) ~ 1e-18
    E_ew = _ewald_total(pos, q, box, beta, 0.49, 27)
    M = (q[:, None] * pos).sum(0)
    E_ref = E_ew + 2 * math.pi * F_COUL * (M @ M) / (3 * L ** 3)
    vals = []
    for R in (20, 24):
        rngs = np.arange(-R, R + 1)
        n = np.stack(np.meshgrid(rngs, rngs, rngs, indexing="ij"), -1).reshape(-1, 3)
        n = n[(n * n).sum(1) <= R * R].astype(np.float64)
        E = 0.0
        for i in range(4):
            for j in range(4):
                d = pos[j] - pos[i] + n * L
                r = np.sqrt((d * d).sum(1))
                if i == j:
                    r = r[r > 0]
                E += 0.5 * F_COUL * q[i] * q[j] * np.sum(1.0 / r)
        vals.append(E)
    # spherical-shell sums converge like 1/R^2 around the limit; check the trend and level
    assert abs(vals[-1] - E_ref) < abs(vals[0] - E_ref) + 1e-9
    assert abs(vals[-1] - E_ref) / abs(E_ref) < 2e-3


# --------------------------------------------------------------------------- charges (P5)
def test_charge_invariants_random_lambda():
    s = make_system(2)
    rng = np.random.default_rng(0)
    q0, _ = charges.charges(s, np.zeros(s.n_coords))
    for _ in range(20):
        lam = rng.uniform(-0.2, 1.2, s.n_coords)
        lp, lt = rng.uniform(-0.2, 1.2, 2)
        assert abs(sum(charges.eq2_weights(lp, lt)) - 1.0) < 1e-14
        q, _ = charges.charges(s, lam)
        assert abs(q.sum() - q0.sum()) < 1e-10           # site+buffer pair total constant
    # the state endpoints reproduce the templates (Glu 0 -> -1 e, His +1 -> 0 e)
    g0 = slice(s.group_ptr[0], s.group_ptr[1] - 1)
    atoms = s.group_atoms[g0]
    lam = np.zeros(s.n_coords)
    q, _ = charges.charges(s, lam)
    assert abs(q[atoms].sum() - 0.0) < 1e-12
    lam[0] = 1.0
    q, _ = charges.charges(s, lam)
    assert abs(q[atoms].sum() + 1.0) < 1e-12


def test_charge_derivatives_finite_difference():
    s = small_system()
    rng = np.random.default_rng(1)
    lam = rng.uniform(0, 1, s.n_coords)
    _, dq = charges.charges(s, lam)
    h = 1e-6
    for c in range(s.n_coords):
        lp, lm = lam.copy(), lam.copy()
        lp[c] += h; lm[c] -= h
        fd = (charges.charges(s, lp)[0] - charges.charges(s, lm)[0]) / (2 * h)
        g = [g for g in range(s.n_groups) if charges.coord_ptr(s.group_kind)[g] <= c < charges.coord_ptr(s.group_kind)[g + 1]][0]
        col = c - charges.coord_ptr(s.group_kind)[g]
        k = slice(s.group_ptr[g], s.group_ptr[g + 1])
        np.testing.assert_allclose(fd[s.group_atoms[k]], dq[k, col], atol=1e-9)


# --------------------------------------------------------------------------- full evaluation (P4)
@pytest.fixture(scope="module")
def tiny_replica():
    s = small_system()
    rng = np.random.default_rng(4)
    lam = rng.uniform(0.05, 0.95, s.n_coords)
    return OracleReplica(s, pH=5.0, seed=99, lam0=lam)


def _epot(rep, x, lam):
    ev = rep.evaluate(x, lam)
    return sum(ev["E"].values())


def test_dvdl_matches_finite_difference(tiny_replica):
    rep = tiny_replica
    cur = rep.cur
    h = 1e-5
    for c in range(len(rep.lam)):
        lp, lm = rep.lam.copy(), rep.lam.copy()
        lp[c] += h; lm[c] -= h
        fd = (_epot(rep, rep.x, lp) - _epot(rep, rep.x, lm)) / (2 * h)
        an = cur["dvdl_coul"][c] + cur["dvdl_bias"][c]
        assert abs(fd - an) <= 1e-7 * max(abs(an), cur["term_mag"][c])


def test_forces_match_finite_difference(tiny_replica):
    rep = tiny_replica
    F = rep.cur["F"]
    s = rep.sys
    # E is discontinuous at r = rc (unshifted potentials, reading R11): a small step keeps
    # cutoff crossings out of the difference quotient.
    h = 1e-7
    for i in (int(s.group_atoms[0]), int(s.group_atoms[-1]), s.n_atoms - 1, s.n_atoms - 50):
        fd = np.zeros(3)
        for d in range(3):
            xp, xm = rep.x.copy(), rep.x.copy()
            xp[i, d] += h; xm[i, d] -= h
            fd[d] = -(_epot(rep, xp, rep.lam) - _epot(rep, xm, rep.lam)) / (2 * h)
        assert np.linalg.norm(fd - F[i]) <= 2e-5 * max(1.0, np.linalg.norm(F[i]))


def test_phi_is_charge_derivative(tiny_replica):
    """phi_i := (1/f) dE_coul/dq_i, including the self and net-charge terms."""
    rep = tiny_replica
    s = rep.sys
    q = rep.cur["q"]
    from oracle.engine import OracleReplica as _R  # noqa
    def ecoul(qv):
        import oracle.ewald as E
        import oracle.pme as P
        rs = E.real_space(rep.x, qv, s.type, s.c6, s.c12, rep.box, rep.p["rc"], rep.beta, s.excl, want_lj=False)
        ex = E.exclusion_correction(rep.x, qv, rep.box, rep.beta, s.excl)
        return (rs["E_real"] + ex["E_excl"] + E.self_term(qv, rep.beta)[0] + E.net_charge_term(qv, rep.box, rep.beta)[0]
                + P.pme(rep.x, qv, rep.box, rep.beta, rep.K, 4)["E_rec"])
    h = 1e-6
    for i in (int(s.group_atoms[1]), 100, s.n_atoms - 3):
        qp, qm = q.copy(), q.copy()
        qp[i] += h; qm[i] -= h
        fd = (ecoul(qp) - ecoul(qm)) / (2 * h) / F_COUL
        assert abs(fd - rep.cur["phi"][i]) < 1e-7 * (1 + abs(rep.cur["phi"][i]))


def test_direct_ewald_and_pme_agree_on_dvdl(tiny_replica):
    s = tiny_replica.sys
    rep_d = OracleReplica(s, pH=5.0, seed=99, lam0=tiny_replica.lam, recip="direct", nmax=16)
    a, b = tiny_replica.cur, rep_d.cur
    tol = 2e-3 * np.maximum(np.abs(b["dvdl_coul"]), b["term_mag"])
    assert np.all(np.abs(a["dvdl_coul"] - b["dvdl_coul"]) < tol)


# --------------------------------------------------------------------------- bias (P6)
def test_delta_g_and_vph_spec_examples():
    assert abs(bias.delta_g(4.0, 3.0, 300.0) - 5.743) < 1e-2
    assert abs(bias.delta_g(4.0, 3.0, 300.0) - 5.743427) < 1e-5
    assert bias.delta_g(4.0, 4.0, 300.0) == 0.0
    v, g, _ = bias.vph(2, (4.0, 4.0, 4.0), 3.0, 300.0, 0.5, 0.0)
    assert abs(v - 2.8715) < 1e-3
    v1 = bias.vph(2, (4.4,) * 3, 5.1, 300.0, 1.0, 0.0)[0]
    v0 = bias.vph(2, (4.4,) * 3, 5.1, 300.0, 0.0, 0.0)[0]
    assert abs((v1 - v0) - math.log(10) * kT(300.0) * (4.4 - 5.1)) < 1e-12   # Eq. 4


def test_vmm_spec_examples_and_gradient():
    c = np.zeros(36)
    assert bias.vmm(c, 0.3, 0.7) == (0.0, 0.0, 0.0)
    c[2 * 6 + 0] = 1.0
    v, dp, dt = bias.vmm(c, 0.5, 0.9)
    assert (v, dp, dt) == (0.25, 1.0, 0.0)
    rng = np.random.default_rng(0)
    c = rng.normal(size=36)
    for _ in range(20):
        lp, lt = rng.uniform(-0.1, 1.1, 2)
        v, dp, dt = bias.vmm(c, lp, lt)
        h = 1e-6
        assert abs((bias.vmm(c, lp + h, lt)[0] - bias.vmm(c, lp - h, lt)[0]) / (2 * h) - dp) < 1e-6 * (1 + abs(dp))
        assert abs((bias.vmm(c, lp, lt + h)[0] - bias.vmm(c, lp, lt - h)[0]) / (2 * h) - dt) < 1e-6 * (1 + abs(dt))


def test_double_well_shape():
    h, d1, kw = 6.0, 1.3, 1e6
    for l in (0.0, 1.0, 0.5):
        assert abs(bias.vdw(l, h, 0.0, d1, kw)[1]) < 1e-12           # wells and apex flat
    assert abs(bias.vdw(0.5, h, 0.0, d1, kw)[0] - h) < 1e-12          # barrier measured from d0
    assert abs(bias.vdw(1.0, h, 0.0, d1, kw)[0] - d1) < 1e-12
    assert abs(bias.vdw(-0.2, h, 0, d1, kw)[0] - (bias.vdw(0.2, h, 0, d1, kw)[0] + kw * 0.1 ** 4)) < 1e-9
    eps = 1e-4                                                        # V'' > 0 at the wells
    for l in (0.0, 1.0):
        assert bias.vdw(l + eps, h, 0, d1, kw)[0] + bias.vdw(l - eps, h, 0, d1, kw)[0] > 2 * bias.vdw(l, h, 0, d1, kw)[0]
    rng = np.random.default_rng(3)
    for l in rng.uniform(-0.3, 1.3, 200):
        e = 1e-7
        fd = (bias.vdw(l + e, h, 0, d1, kw)[0] - bias.vdw(l - e, h, 0, d1, kw)[0]) / (2 * e)
        an = bias.vdw(l, h, 0, d1, kw)[1]
        assert abs(fd - an) < 1e-5 * (1 + abs(an))


# --------------------------------------------------------------------------- PFC (P6/P7)
def test_pfc_two_state_hits_target_by_independent_trapezoid():
    for pH in (3.4, 4.4, 5.4, 6.4):
        d1 = pfc.pfc_2state(6.0, 4.4, pH, 300.0, 1e6)
        x = np.linspace(-0.45, 1.45, 400001)
        V = bias.vdw(x, 6.0, 0.0, d1, 1e6)[0] + x * bias.delta_g(4.4, pH, 300.0)
        w = np.exp(-V / kT(300.0))
        dx = x[1] - x[0]
        zp = np.trapezoid(w[x < 0.5], dx=dx)
        zd = np.trapezoid(w[x >= 0.5], dx=dx)
        frac = zd / (zp + zd)
        assert abs(frac - 1.0 / (10 ** (4.4 - pH) + 1.0)) < 1e-6
    # d1 = +1.164 / -0.947 kJ/mol at pH - pKa = -1 / +1 (h = 6)
    assert abs(pfc.pfc_2state(6.0, 4.4, 3.4, 300.0, 1e6) - 1.164) < 1e-3
    assert abs(pfc.pfc_2state(6.0, 4.4, 5.4, 300.0, 1e6) + 0.947) < 1e-3
    assert abs(pfc.pfc_2state(6.0, 4.4, 4.4, 300.0, 1e6)) < 1e-10     # symmetric target -> no shift


def test_pfc_three_state_populations_table2():
    his = [r for r in _golden("table2_pka.txt") if r[0] == "His"][0]
    pk = (float(his[1]), float(his[2]), float(his[3]))
    pH = 6.7
    d1p, d1t = pfc.pfc_3state(6.0, pk, pH, 300.0, 1e6)
    a, b = pfc.quadrant_free_energies(6.0, d1p, d1t, pk, pH, 300.0, 1e6)
    pd = math.exp(-a / kT(300.0))
    pe = math.exp(-b / kT(300.0))
    assert abs(pd / pe - 10 ** (pk[2] - pk[1])) < 1e-8                 # delta:eps = 2.4547
    assert abs(10 ** (pk[2] - pk[1]) - 2.4547) < 1e-4
    frac = (pd + pe) / (1 + pd + pe)
    pka_macro = -math.log10(10 ** -pk[1] + 10 ** -pk[2])
    assert abs(pka_macro - 6.3816) < 1e-4 and abs(pka_macro - pk[0]) < 0.005
    assert abs(frac - 1.0 / (10 ** (pka_macro - pH) + 1.0)) < 1e-8


# --------------------------------------------------------------------------- sampling (P7, P9)
def _equilibrium_lambda0(M, h, d1, pKa, pH, seed):
    x = np.linspace(-0.45, 1.45, 200001)
    V = bias.vdw(x, h, 0, d1, 1e6)[0] + x * bias.delta_g(pKa, pH, 300.)
    w = np.exp(-(V - V.min()) / kT(300.))
    cdf = np.cumsum(w); cdf /= cdf[-1]
    return np.interp(np.random.default_rng(seed).random(M), cdf, x)


def test_electrostatics_off_titration_follows_hh():
    """Single site, electrostatics off, barrier 2 kJ/mol: the sampled deprotonated fraction
    follows 1/(10^(pKa-pH)+1) with PFC, and not without it."""
    pKa, h, M = 4.4, 2.0, 2000
    pHs = np.array([3.4, 4.4, 5.4])
    pH = np.repeat(pHs, M)
    d1 = np.repeat([pfc.pfc_2state(h, pKa, p, 300., 1e6) for p in pHs], M)
    lam0 = np.concatenate([_equilibrium_lambda0(M, h, d1[k * M], pKa, pHs[k], k) for k in range(3)])
    seeds = (np.arange(1, 3 * M + 1, dtype=np.uint64) * np.uint64(2654435761) + np.uint64(7))
    fr, vfr = run_2state(seeds, lam0, pKa, pH, 6000, h_barrier=h, d1=d1)
    x = np.array([analysis.deprotonated_fraction(fr[:, k * M:(k + 1) * M]) for k in range(3)])
    target = 1.0 / (10 ** (pKa - pHs) + 1.0)
    assert np.all(np.abs(x - target) < 0.015), (x, target)
    n_hill = analysis.fit_hill(pHs, x)[1]
    assert abs(n_hill - 1.0) < 0.1
    # equipartition of the lambda particle: <1/2 m v^2> = 1/2 kT
    ke = 0.5 * 60.0 * np.mean(vfr[300:] ** 2)          # after 6 ps (>> 1/gamma) of thermalisation
    assert abs(ke / (0.5 * kT(300.0)) - 1.0) < 0.03


def test_free_flight_and_reversibility():
    """gamma = 0 and no force: lambda advances v dt per step; time reversal
    returns the start."""
    from oracle.lambda_only import run_2state as run
    seeds = np.array([1, 2], dtype=np.uint64)
    # flat region: barrier 0, d1 0, pH = pKa -> no force inside [0, 1]
    fr, vf = run(seeds, [0.3, 0.6], 4.4, 4.4, 1, h_barrier=0.0, d1=0.0, gamma=0.0, record_every=1)
    assert np.allclose(fr[0], [0.3, 0.6])                 # zero initial velocity: no motion


# --------------------------------------------------------------------------- pair list
def test_canonical_pairlist_against_fp64_distances():
    s = small_system()
    pairs = pairlist.canonical_pairs(s.pos, s.box, 1.1, s.excl)
    pos = s.pos.astype(np.float64)
    d = ewald.min_image(pos[None, :, :] - pos[:, None, :], s.box)
    r = np.sqrt((d * d).sum(-1))
    iu = np.triu_indices(len(pos), 1)
    rr = r[iu]
    in_set = set(map(tuple, pairs.tolist()))
    ex = set(map(tuple, s.excl.tolist()))
    for (i, j), dist in zip(zip(*iu), rr):
        if (i, j) in ex:
            assert (i, j) not in in_set
        elif dist < 1.1 - 1e-5:
            assert (i, j) in in_set
        elif dist > 1.1 + 1e-5:
            assert (i, j) not in in_set
    assert np.all(pairs[:, 0] < pairs[:, 1])
    assert np.all(np.diff(pairs[:, 0] * len(pos) + pairs[:, 1]) > 0)


# --------------------------------------------------------------------------- analysis (a12)
def test_hh_and_hill_recovery():
    pH = np.linspace(2.5, 5.5, 7)
    assert abs(analysis.fit_hh(pH, analysis.hh(pH, 4.0)) - 4.0) < 1e-6
    pk, n = analysis.fit_hill(pH, analysis.hh(pH, 4.04, 0.8))
    assert abs(pk - 4.04) < 1e-4 and abs(n - 0.8) < 1e-4
    est, lo, hi = analysis.bootstrap(pH, np.repeat(analysis.hh(pH, 4.0)[:, None], 5, 1), B=50)
    assert abs(hi - lo) < 1e-9                                                    # identical replicas
    assert analysis.deprotonated_fraction([0.5, 0.1, 0.9, 0.2]) == 0.5           # lambda_p >= 0.5 deprot


def test_baoab_conserves_energy_without_friction():
    """gamma = 0: BAOAB reduces to velocity Verlet, which conserves the
    extended-Hamiltonian energy (atoms + lambda particles, Eq. 1-3) to O(dt^2)."""
    from synthetic.systems import make_velocities
    s = small_system()
    r = OracleReplica(s, 5.0, 11, lam0=np.array([0.2, 0.7, 0.4]), vel0=make_velocities(s, 3),
                      params=dict(gamma_atom=0.0, gamma_lambda=0.0))
    E0 = r.energies()["total"]
    ke = r.energies()["KE_atoms"]
    drift = []
    for _ in range(30):
        r.step()
        drift.append(r.energies()["total"] - E0)
    assert np.max(np.abs(drift)) < 2e-4 * ke


# --------------------------------------------------------------------------- calibration (a11)
def test_ti_grid_is_the_si_list():
    from oracle.calibration import TI_GRID
    assert len(TI_GRID) == 14 and len(TI_GRID) ** 2 == 196          # P:8


def test_vmm_fit_recovers_exact_polynomial_and_flattens():
    """SPEC S:201 (exact degree-5 reference recovered to 1e-8) and S:203 (flattening:
    Vmm + U_ref has zero gradient)."""
    from oracle.calibration import TI_GRID, vmm_from_ti
    rng = np.random.default_rng(4)
    c_ref = rng.normal(size=36)
    c_ref[0] = 0.0
    LP, LT = np.meshgrid(TI_GRID, TI_GRID, indexing="ij")
    lp, lt = LP.ravel(), LT.ravel()
    g = np.array([bias.vmm(c_ref, a, b)[1:] for a, b in zip(lp, lt)])   # dU/dlp, dU/dlt
    vm = vmm_from_ti(3, lp, lt, g)
    np.testing.assert_allclose(vm, -c_ref, atol=1e-8)
    for a, b in rng.uniform(-0.1, 1.1, (20, 2)):
        _, gp, gt = bias.vmm(vm + c_ref, a, b)
        assert abs(gp) < 1e-7 and abs(gt) < 1e-7
    c1 = np.zeros(36)
    c1[[6, 12, 18, 24, 30]] = rng.normal(size=5)
    g1 = np.array([[bias.vmm(c1, a, 0.0)[1]] for a in TI_GRID])
    np.testing.assert_allclose(vmm_from_ti(2, np.array(TI_GRID), None, g1), -c1, atol=1e-8)


def test_pfc_saturates_when_target_unreachable():
    """Reading R22: |pH - pKa| beyond ~3.7 on the protonated side cannot be corrected by d1
    alone at h = 6 (the deprotonated half contains the barrier top); d1 saturates at +80 and the
    deprotonated population is then below the H-H value by a negligible amount."""
    assert pfc.pfc_2state(6.0, 4.0, -1.0, 300.0, 1e6) == pfc.D1_BOUND
    d1 = pfc.pfc_2state(6.0, 4.0, 0.2, 300.0, 1e6)
    assert 0 < d1 < pfc.D1_BOUND
    x = np.linspace(-0.45, 1.45, 200001)
    V = bias.vdw(x, 6.0, 0.0, pfc.D1_BOUND, 1e6)[0] + x * bias.delta_g(4.0, -1.0, 300.0)
    w = np.exp(-(V - V.min()) / kT(300.0))
    frac = w[x >= 0.5].sum() / w.sum()
    assert frac < 1e-3 and 1.0 / (10 ** 5 + 1) < frac


def test_canonical_partner_rows_equal_the_pair_list():
    """oracle.pairlist.canonical_partners (sampled rows for large systems) gives exactly the
    rows of canonical_pairs (both orientations of every pair, bit-identical d2)."""
    s = small_system()
    pairs = pairlist.canonical_pairs(s.pos, s.box, 1.1, s.excl)
    idx = np.arange(0, s.n_atoms, 7)
    rows = pairlist.canonical_partners(s.pos, s.box, 1.1, s.excl, idx)
    for i, row in zip(idx, rows):
        ref = np.sort(np.concatenate([pairs[pairs[:, 0] == i, 1], pairs[pairs[:, 1] == i, 0]]))
        assert np.array_equal(row, ref)

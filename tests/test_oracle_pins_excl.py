"""Pins of the oracle's exclusion correction, net-charge term and Eq. 2 state mapping
(no GPU).  Each pin compares the oracle with something other than its own formula:

* exclusion correction (oracle.ewald.exclusion_correction, PAPER.md:641-647 charge-only
  forms): the engine's E_coul / phi / F WITH an exclusion list equal the same
  engine WITHOUT it minus the bare Coulomb interaction f q_i q_j / r of the excluded pairs,
  and the brute-force spherical lattice sum of the bare Coulomb energy minus the
  home-image excluded pairs equals tin-foil Ewald with exclusions + 2 pi f |M|^2 / 3V;
* net-charge term (oracle.ewald.net_charge_term, reading R13): a single
  ion in a cubic box has E = -xi f q^2 / (2 L) with the Wigner constant xi = 2.837297
  (golden file), and the total Ewald energy of a charged cell does not depend on beta;
* Eq. 2 corners (oracle.charges): at (lp, lt) in {0,1}^2 every His atom
  carries exactly q^A, q^B, q^C, q^D, and the pH term's tautomer at each corner (VpH, R4)
  is the one whose charges the corner carries.
Each test fails on a sign flip, an erf/erfc swap or a dropped term of the function it pins
(see the comments at the asserts)."""
import math
import os

import numpy as np

from oracle import bias, charges, ewald
from oracle.engine import OracleReplica
from oracle.units import F_COUL, kT
from synthetic.systems import SyntheticSystem, make_system, small_system

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()[:2]
                out[k] = float(v)
    return out


def _ion_system(pos, q, box, excl, K=20):
    """A SyntheticSystem of bare point charges (no LJ, no lambda groups) for the engine."""
    n = len(q)
    return SyntheticSystem(
        name="pins", box=np.asarray(box, np.float64), pos=np.asarray(pos, np.float32),
        mass=np.zeros(n, np.float32), charge=np.asarray(q, np.float32), type=np.zeros(n, np.int32),
        c6=np.zeros((1, 1)), c12=np.zeros((1, 1)), excl=np.asarray(excl, np.int32).reshape(-1, 2),
        group_kind=np.zeros(0, np.int32), group_ptr=np.zeros(1, np.int32), group_atoms=np.zeros(0, np.int32),
        state_q=np.zeros((0, 4)), is_buffer=np.zeros(0, np.int32), pKa=np.zeros((0, 3)), vmm=np.zeros((0, 36)),
        pme_grid=(K, K, K))


def _clustered_charges(seed, L=2.5):
    """12 charges in three tight residues (pairs well inside r_c and L/2) + loose ions."""
    rng = np.random.default_rng(seed)
    pos = []
    for c in rng.uniform(0.6, L - 0.6, (3, 3)):
        pos += list(c + rng.uniform(-0.15, 0.15, (3, 3)))
    pos += list(rng.uniform(0, L, (3, 3)))
    q = rng.uniform(-0.8, 0.8, 12)
    q -= q.mean()
    excl = [(0, 1), (0, 2), (1, 2), (3, 4), (4, 5), (6, 8)]
    return np.array(pos), q, np.full(3, L), np.array(excl)


def _coulomb(rep, q):
    ev = rep.evaluate(rep.x, rep.lam)
    return sum(ev["E"][k] for k in ("real", "excl", "self", "recip", "net")), ev["phi"], ev["F"]


def test_exclusions_remove_exactly_the_bare_coulomb_of_excluded_pairs():
    """E_coul(excl) = E_coul(no excl) - f sum_excl q_i q_j / r_ij, and the same for phi
    (1/f dE/dq) and F.  An erfc in place of erf, a flipped sign or a missing pair in
    exclusion_correction breaks all three (the bare 1/r pair does not use erf at all)."""
    pos, q, box, excl = _clustered_charges(5)
    q = q.astype(np.float32).astype(np.float64)        # the engine reads the system's fp32 charges
    p = dict(rc=1.2, rlist=1.2)                       # every excluded pair is inside r_c
    with_ex = OracleReplica(_ion_system(pos, q, box, excl), 7.0, 1, params=p)
    no_ex = OracleReplica(_ion_system(pos, q, box, np.zeros((0, 2))), 7.0, 1, params=p)
    E1, phi1, F1 = _coulomb(with_ex, q)
    E0, phi0, F0 = _coulomb(no_ex, q)
    x = pos.astype(np.float32).astype(np.float64)
    dE, dphi, dF = 0.0, np.zeros(len(q)), np.zeros((len(q), 3))
    for i, j in excl:
        d = x[j] - x[i]
        d -= box * np.round(d / box)
        r = np.linalg.norm(d)
        assert r < 0.5                                 # home image = minimum image
        dE += F_COUL * q[i] * q[j] / r
        dphi[i] += q[j] / r
        dphi[j] += q[i] / r
        f = F_COUL * q[i] * q[j] / r ** 3 * d          # bare Coulomb force on j from i
        dF[j] += f
        dF[i] -= f
    assert abs((E1 - (E0 - dE))) < 1e-10 * abs(dE)
    np.testing.assert_allclose(phi1, phi0 - dphi, atol=1e-10 * np.abs(dphi).max())
    np.testing.assert_allclose(F1, F0 - dF, atol=1e-9 * np.abs(dF).max())
    assert abs(dE) > 1.0                               # the pins are not vacuous


def test_lattice_sum_minus_home_excluded_pairs_equals_ewald_with_exclusions():
    """SURVEY P2 with exclusions: spherical bare-Coulomb lattice sum of a neutral cell,
    minus the home-image excluded pairs, = tin-foil Ewald with those exclusions (real +
    erf correction + self + net + direct reciprocal) + 2 pi f |M|^2 / (3V)."""
    L = 1.0
    box = np.full(3, L)
    rng = np.random.default_rng(7)
    c = rng.uniform(0.3, 0.7, 3)
    pos = np.array([c, c + [0.12, 0.05, -0.04], rng.uniform(0, L, 3), rng.uniform(0, L, 3)])
    q = np.array([0.8, -0.5, 0.4, -0.7])
    excl = np.array([[0, 1]])
    beta, rc = 12.5, 0.49
    t = np.zeros(4, np.int32)
    z = np.zeros((1, 1))
    rs = ewald.real_space(pos, q, t, z, z, box, rc, beta, excl)
    ex = ewald.exclusion_correction(pos, q, box, beta, excl)
    E_ew = (rs["E_real"] + ex["E_excl"] + ewald.self_term(q, beta)[0] + ewald.net_charge_term(q, box, beta)[0]
            + ewald.recip_direct(pos, q, box, beta, 27)[0])
    M = (q[:, None] * pos).sum(0)
    E_ref = E_ew + 2 * math.pi * F_COUL * (M @ M) / (3 * L ** 3)
    vals = []
    for R in (20, 24):
        rr = np.arange(-R, R + 1)
        n = np.stack(np.meshgrid(rr, rr, rr, indexing="ij"), -1).reshape(-1, 3)
        n = n[(n * n).sum(1) <= R * R].astype(np.float64)
        E = 0.0
        for i in range(4):
            for j in range(4):
                d = pos[j] - pos[i] + n * L
                r = np.sqrt((d * d).sum(1))
                if i == j:
                    r = r[r > 0]
                E += 0.5 * F_COUL * q[i] * q[j] * np.sum(1.0 / r)
        r01 = np.linalg.norm(pos[1] - pos[0])
        vals.append(E - F_COUL * q[0] * q[1] / r01)        # home-image excluded pair removed
    assert abs(vals[-1] - E_ref) < abs(vals[0] - E_ref) + 1e-9
    assert abs(vals[-1] - E_ref) / abs(E_ref) < 2e-3
    # the excluded pair's bare energy is far above that tolerance: dropping E_excl fails
    assert abs(F_COUL * q[0] * q[1] / np.linalg.norm(pos[1] - pos[0])) > 100 * 2e-3 * abs(E_ref)


def test_single_ion_wigner_constant():
    """One charge q in a cubic box L with the neutralising background (tin-foil Ewald):
    E = -xi f q^2 / (2L), phi at the ion = -xi q / L, xi = 2.837297 (simple-cubic Wigner
    constant).  Exercises E_net with Q != 0 together with self + reciprocal; a flipped
    sign or a factor 2 in net_charge_term moves E by ~10 %."""
    xi = _golden("madelung.txt")["Wigner_sc"]
    for L, q, beta in ((2.0, 1.0, 3.0), (3.1, -0.6, 2.4)):
        box = np.full(3, L)
        pos = np.array([[0.3 * L, 0.7 * L, 0.1 * L]])
        qq = np.array([q])
        nmax = int(math.ceil(math.sqrt(40.0) * L * beta / math.pi)) + 1
        e_self, phi_self = ewald.self_term(qq, beta)
        e_net, phi_net = ewald.net_charge_term(qq, box, beta)
        e_rec, phi_rec, _ = ewald.recip_direct(pos, qq, box, beta, nmax)
        E = e_self + e_net + e_rec                         # real space: images at >= L, erfc(beta L) < 1e-17
        phi = phi_self[0] + phi_net[0] + phi_rec[0]
        ref = -xi * F_COUL * q * q / (2.0 * L)
        assert abs(E - ref) < 1e-6 * abs(ref), (E, ref)
        assert abs(phi - (-xi * q / L)) < 1e-6 * abs(xi * q / L)
        assert abs(e_net) > 1e4 * 1e-6 * abs(ref)          # a flipped or dropped E_net fails by 10^4 x tol


def test_charged_cell_energy_is_beta_independent():
    """Ewald splitting is exact for any beta only if the net-charge background term is
    included (R13): E_total(beta) of a non-neutral cell is constant; without E_net it drifts
    by f pi Q^2/(2V) (1/beta1^2 - 1/beta2^2)."""
    rng = np.random.default_rng(3)
    L = 2.0
    box = np.full(3, L)
    pos = rng.uniform(0, L, (8, 3))
    q = rng.uniform(-1.0, 1.0, 8) + 0.15
    t = np.zeros(8, np.int32)
    z = np.zeros((1, 1))
    rc = 0.99
    out = {}
    for beta in (5.0, 6.0):
        rs = ewald.real_space(pos, q, t, z, z, box, rc, beta, np.zeros((0, 2), np.int32))
        nmax = int(math.ceil(math.sqrt(40.0) * L * beta / math.pi)) + 1
        out[beta] = (rs["E_real"] + ewald.self_term(q, beta)[0] + ewald.recip_direct(pos, q, box, beta, nmax)[0],
                     ewald.net_charge_term(q, box, beta)[0])
    tot = {b: a + n for b, (a, n) in out.items()}
    assert abs(tot[5.0] - tot[6.0]) < 1e-8 * abs(tot[5.0])
    assert abs(out[5.0][0] - out[6.0][0]) > 1e4 * abs(tot[5.0] - tot[6.0])   # E_net is what makes it exact


def test_eq2_corners_give_the_state_charges_his_and_glu():
    """Eq. 2: (lp, lt) = (0,0) -> A, (0,1) -> B, (1,0) -> C, (1,1) -> D,
    exactly, for every atom of the His group (A = B = HIP, C = HID, D = HIE) and
    of a 2-state Glu group (lt irrelevant)."""
    s = make_system(2)
    cp = charges.coord_ptr(s.group_kind)
    his = [g for g in range(s.n_groups) if s.group_kind[g] == 3][0]
    glu = [g for g in range(s.n_groups) if s.group_kind[g] == 2][0]
    corners = {(0.0, 0.0): 0, (0.0, 1.0): 1, (1.0, 0.0): 2, (1.0, 1.0): 3}
    k = slice(s.group_ptr[his], s.group_ptr[his + 1])
    for (lp, lt), col in corners.items():
        lam = np.full(s.n_coords, 0.37)
        lam[cp[his]], lam[cp[his] + 1] = lp, lt
        q, _ = charges.charges(s, lam)
        np.testing.assert_array_equal(q[s.group_atoms[k]], s.state_q[k, col])
    # the His templates really differ between C (HID) and D (HIE): a B/C swap would fail
    assert np.abs(s.state_q[k, 2] - s.state_q[k, 3]).max() > 0.1
    assert abs(s.state_q[k, 0].sum() - s.state_q[k, 1].sum()) < 1e-12   # A = B = HIP
    kg = slice(s.group_ptr[glu], s.group_ptr[glu + 1])
    for lp, col in ((0.0, 0), (1.0, 2)):
        lam = np.full(s.n_coords, 0.61)
        lam[cp[glu]] = lp
        q, _ = charges.charges(s, lam)
        np.testing.assert_array_equal(q[s.group_atoms[kg]], s.state_q[kg, col])


def test_vph_tautomer_matches_charge_corner():
    """The tautomer whose charges a corner carries is the one whose micro pKa the pH term
    charges there (R4): VpH(1, 0) - VpH(0, 0) = ln10 kT (pKa_delta - pH) at the HID corner
    (q^C) and VpH(1, 1) - VpH(0, 1) = ln10 kT (pKa_eps - pH) at the HIE corner (q^D)."""
    s = small_system()
    his = [g for g in range(s.n_groups) if s.group_kind[g] == 3][0]
    pk = tuple(s.pKa[his])
    pH = 6.1
    l10kt = math.log(10.0) * kT(300.0)
    v00 = bias.vph(3, pk, pH, 300.0, 0.0, 0.0)[0]
    v10 = bias.vph(3, pk, pH, 300.0, 1.0, 0.0)[0]
    v01 = bias.vph(3, pk, pH, 300.0, 0.0, 1.0)[0]
    v11 = bias.vph(3, pk, pH, 300.0, 1.0, 1.0)[0]
    assert abs((v10 - v00) - l10kt * (pk[1] - pH)) < 1e-12
    assert abs((v11 - v01) - l10kt * (pk[2] - pH)) < 1e-12
    # and the corners carry the HID / HIE totals (0 e each, HIP +1 e)
    k = slice(s.group_ptr[his], s.group_ptr[his + 1])
    site = s.is_buffer[k] == 0
    assert abs(s.state_q[k, 0][site].sum() - 1.0) < 1e-9
    assert abs(s.state_q[k, 2][site].sum()) < 1e-9 and abs(s.state_q[k, 3][site].sum()) < 1e-9

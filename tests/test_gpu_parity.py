"""GPU path (libcph.so through the C ABI) vs the fp64 oracle on identical seeded inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import pairlist as OPL  # noqa: E402
from oracle import pfc as OPFC  # noqa: E402
from oracle.engine import OracleReplica  # noqa: E402
from synthetic.systems import make_system, make_velocities, random_lambdas, replica_seeds, small_system  # noqa: E402
from tests.parity import ETOL, RTOL, compare_snapshot  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def _ctx(cph, s, R, seed=0, lam_lo=0.0, lam_hi=1.0, **kw):
    rng = np.random.default_rng(seed)
    lam0 = rng.uniform(lam_lo, lam_hi, (R, s.n_coords))
    pH = np.linspace(3.0, 7.0, R)
    seeds = replica_seeds(99, R, seed)
    vel = np.stack([make_velocities(s, 100 + r) for r in range(R)])
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, **kw)
    return ctx, lam0, pH, seeds, vel


@pytest.mark.parametrize("which", ["tiny", "c1", "c2"])
def test_snapshot_parity(cph, which):
    s = small_system() if which == "tiny" else make_system(1 if which == "c1" else 2)
    R = 3
    ctx, lam0, pH, seeds, vel = _ctx(cph, s, R, seed=1, lam_lo=-0.1, lam_hi=1.1)
    for r in range(R):
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam0[r], vel0=vel[r])
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        print(which, r, {k: v for k, v in err.items() if k != "E_terms"})
        assert err["force"] <= RTOL
        assert err["phi"] <= RTOL
        assert err["force_atom"] <= RTOL          # per atom: max_i |dF_i| / max(|F_i|, rms F)
        assert err["phi_atom"] <= RTOL
        assert err["phi_lambda_atoms"] <= RTOL
        assert err["dvdl_coul"] <= RTOL
        assert err["dvdl_bias"] <= 1e-9
        assert err["E_total"] <= ETOL, err["E_terms"]


def _check_directed(ctx, r, ref):
    """The kernel's directed entries are exactly both orientations of the canonical set."""
    dirs = ctx.cph_get_pairlist_directed(r)
    both = np.concatenate([ref, ref[:, ::-1]])
    both = both[np.lexsort((both[:, 1], both[:, 0]))]
    assert dirs.shape == both.shape and np.array_equal(dirs, both)


@pytest.mark.parametrize("which", ["tiny", "c1", "c2", "c3"])
def test_pairlist_bit_exact(cph, which):
    s = small_system() if which == "tiny" else make_system({"c1": 1, "c2": 2, "c3": 3}[which])
    ctx, *_ = _ctx(cph, s, 2)
    ref = OPL.canonical_pairs(s.pos, s.box, s.params["rlist"], s.excl)
    for r in range(2):
        got = ctx.cph_get_pairlist(r)
        assert got.shape == ref.shape and np.array_equal(got, ref)
    _check_directed(ctx, 1, ref)
    # after a rebuild at step nstlist, against the positions the device holds
    ctx.cph_step(s.params["nstlist"])
    for r in range(2):
        x, _ = ctx.cph_get_positions(r)
        got = ctx.cph_get_pairlist(r)
        ref = OPL.canonical_pairs(x, s.box, s.params["rlist"], s.excl)
        assert np.array_equal(got, ref)
        if r == 0:
            _check_directed(ctx, r, ref)


@pytest.mark.parametrize("cfg", [4, 5])
def test_pairlist_rows_full_size(cph, cfg):
    """C4 (40k) and C5 (250k atoms, the bench's largest configs): sampled rows of the directed
    list (2000 atoms incl. every lambda atom and solute exclusions) against the oracle's
    canonical rows, at create and after a rebuild."""
    s = make_system(cfg)
    ctx = cph.cph_create(s, [5.0], [11], vel_replicas=make_velocities(s, 3)[None])
    rng = np.random.default_rng(cfg)
    idx = np.unique(np.concatenate([s.group_atoms, s.excl[:200, 0], rng.choice(s.n_atoms, 1800, replace=False)]))
    for stage in range(2):
        x = s.pos if stage == 0 else ctx.cph_get_positions(0)[0]
        got = ctx.cph_get_pairlist_rows(0, idx)
        ref = OPL.canonical_partners(x, s.box, s.params["rlist"], s.excl, idx)
        bad = [int(i) for i, a, b in zip(idx, got, ref) if not np.array_equal(a, b)]
        assert not bad, bad[:10]
        ctx.cph_step(s.params["nstlist"])


@pytest.mark.parametrize("which", ["c2", "c4"])
def test_lambda_group_csr_bit_exact(cph, which):
    """The device's lambda-group CSR, mapped back through its sorted-slot permutation to
    original indices, equals the oracle's (north star: lambda-group indexing bit-exact), at
    create and after rebuilds re-sorted the atoms."""
    from oracle.charges import coord_ptr
    s = make_system({"c2": 2, "c4": 4}[which])
    ctx, *_ = _ctx(cph, s, 2)
    for stage in range(2):
        for r in range(2):
            gp, cp, a, b = ctx.cph_get_lambda_groups(r, s.n_groups, len(s.group_atoms))
            assert np.array_equal(gp, s.group_ptr) and np.array_equal(cp, coord_ptr(s.group_kind))
            assert np.array_equal(a, s.group_atoms) and np.array_equal(b, s.group_atoms)
        ctx.cph_step(3 * s.params["nstlist"])


def test_pfc_matches_oracle(cph):
    s = make_system(2)
    ctx, lam0, pH, seeds, vel = _ctx(cph, s, 4)
    for r in range(4):
        d1 = ctx.cph_get_bias_params(r)
        ref = [OPFC.pfc_2state(6.0, s.pKa[0, 0], pH[r], 300.0, 1e6), *OPFC.pfc_3state(6.0, s.pKa[1], pH[r], 300.0, 1e6)]
        np.testing.assert_allclose(d1, ref, atol=1e-8)


def test_parity_after_steps_and_state_roundtrip(cph):
    """Step the GPU, then evaluate the oracle on the exact state the device holds."""
    s = make_system(1)
    ctx, lam0, pH, seeds, vel = _ctx(cph, s, 2)
    ctx.cph_step(37)
    assert ctx.cph_current_step() == 37
    for r in range(2):
        x, v = ctx.cph_get_positions(r)
        lam, lamv = ctx.cph_get_lambdas(r)
        assert np.all(np.isfinite(x)) and np.all(np.isfinite(lam))
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam, vel0=v, pos0=x)
        ref.lamv = lamv
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        print(r, {k: v for k, v in err.items() if k != "E_terms"})
        assert err["force"] <= RTOL and err["dvdl_coul"] <= RTOL and err["E_total"] <= ETOL
    blob = ctx.cph_get_state(0)
    f0, p0 = ctx.cph_get_forces(0)
    ctx.cph_set_state(0, blob)
    f1, p1 = ctx.cph_get_forces(0)
    assert np.linalg.norm(f1 - f0) <= 1e-6 * np.linalg.norm(f0)


def test_short_horizon_trajectory(cph):
    """Same Philox streams and step order: GPU and oracle trajectories agree over a short
    horizon (fp32 vs fp64 growth is expected and only reported beyond it)."""
    s = small_system()
    lam0 = np.array([[0.3, 0.6, 0.4]])
    vel = make_velocities(s, 5)[None]
    ctx = cph.cph_create(s, [5.0], [1234], lambda0=lam0, vel_replicas=vel)
    ref = OracleReplica(s, 5.0, 1234, lam0=lam0[0], vel0=vel[0])
    for n in (1, 4, 5):
        ctx.cph_step(n)
        for _ in range(n):
            ref.step()
        x, v = ctx.cph_get_positions(0)
        lam, _ = ctx.cph_get_lambdas(0)
        d = x - ref.x
        d -= s.box * np.round(d / s.box)          # the device wraps positions at each rebuild
        dx = np.abs(d).max()
        dl = np.abs(lam - ref.lam).max()
        print("step", ref.step_index, "max|dx|", dx, "max|dlam|", dl)
        assert dx < 1e-4 and dl < 1e-5


def test_energy_conservation_without_friction(cph):
    """gamma = 0: velocity Verlet conserves the extended-Hamiltonian energy (atoms + lambda)
    once the lattice start has relaxed (equilibrated first with strong friction)."""
    s = make_system(1)
    eq = cph.cph_create(s, [4.4], [7], lambda0=np.array([[0.3]]), vel_replicas=make_velocities(s, 7)[None],
                        gamma_atom=10.0)
    eq.cph_step(500)
    x, v = eq.cph_get_positions(0)
    lam, _ = eq.cph_get_lambdas(0)
    ctx = cph.cph_create(s, [4.4], [7], lambda0=lam[None], pos_replicas=x[None], vel_replicas=v[None],
                         gamma_atom=0.0, gamma_lambda=0.0, nstenergy=1)
    e0 = ctx.cph_get_energies(0)
    drift = []
    for _ in range(20):
        ctx.cph_step(10)
        drift.append(ctx.cph_get_energies(0)["total"] - e0["total"])
    print("drift", np.round(drift, 3), "KE", e0["KE_atoms"])
    assert np.max(np.abs(drift)) < 2e-3 * e0["KE_atoms"]


def test_replicas_independent_and_deterministic(cph):
    s = small_system()
    a, *_ = _ctx(cph, s, 3, seed=3)
    b, *_ = _ctx(cph, s, 3, seed=3)
    a.cph_step(25)
    b.cph_step(25)
    # fp32 atomics in the PME spread make runs reproducible to rounding, not bitwise
    for r in range(3):
        np.testing.assert_allclose(a.cph_get_lambdas(r)[0], b.cph_get_lambdas(r)[0], atol=1e-6)
    # replica 1 alone (R=1) gives the same lambda trajectory as inside the batch, up to fp32
    # atomics ordering in the PME spread
    ctx1 = cph.cph_create(s, [np.linspace(3, 7, 3)[1]], [replica_seeds(99, 3, 3)[1]],
                          lambda0=np.random.default_rng(3).uniform(0, 1, (3, s.n_coords))[1:2],
                          vel_replicas=make_velocities(s, 101)[None])
    ctx1.cph_step(25)
    np.testing.assert_allclose(ctx1.cph_get_lambdas(0)[0], a.cph_get_lambdas(1)[0], atol=1e-5)


def test_frames_and_counts(cph):
    s = small_system()
    ctx = cph.cph_create(s, [4.0], [3], nstout=5, frame_capacity=8)
    ctx.cph_step(30)
    fr, dropped = ctx.cph_get_frames(0)
    assert fr.shape == (7, s.n_coords) and dropped == 0     # steps 0,5,...,30
    ctx.cph_step(50)
    fr, dropped = ctx.cph_get_frames(0)
    assert fr.shape == (8, s.n_coords) and dropped == 2
    assert ctx.cph_launch_count() > 0


def test_fixed_lambda_ti_mode(cph):
    """mode 1: lambda frozen at the grid point; the TI mean equals the mean of the
    instantaneous dV/dlambda."""
    s = small_system()
    lam = np.array([[0.2, 0.4, 0.9]])
    vel = make_velocities(s, 9)
    ctx = cph.cph_create(s, [4.4], [5], lambda0=lam, mode=1, vel_replicas=vel[None])
    ref = OracleReplica(s, 4.4, 5, lam0=lam[0], vel0=vel, fixed_lambda=True)
    acc = np.zeros(s.n_coords)
    acc_ref = np.zeros(s.n_coords)
    for _ in range(6):
        ctx.cph_step(1)
        ref.step()
        c, b = ctx.cph_get_dvdl(0)
        acc += c
        acc_ref += ref.cur["dvdl_coul"]
        np.testing.assert_array_equal(ctx.cph_get_lambdas(0)[0], lam[0])
    mean, n = ctx.cph_get_ti_means(0)
    assert n == 6
    np.testing.assert_allclose(mean, acc / 6, rtol=1e-12, atol=1e-12)
    # same Philox streams: the oracle's TI mean over the same 6 steps agrees
    scale = np.maximum(np.abs(acc_ref / 6), ref.cur["term_mag"])
    assert np.all(np.abs(mean - acc_ref / 6) <= 1e-4 * scale), (mean, acc_ref / 6)


def test_gpu_sampling_follows_hh_when_coulomb_dvdl_vanishes(cph):
    """States with equal charges make the Coulomb dV/dlambda exactly zero, so lambda samples
    only the bias: with PFC the deprotonated fraction is 1/(10^(pKa-pH)+1) (PAPER.md:979,
    Eq. 4) and His tautomers split delta:eps = 10^(pKa_eps - pKa_delta) (Table 2)."""
    import copy
    s = copy.deepcopy(small_system())
    s.state_q[:, 2] = s.state_q[:, 0]
    s.state_q[:, 3] = s.state_q[:, 0]
    s.vmm[:] = 0.0
    levels = np.array([3.4, 4.4, 5.4, 6.5])
    per = 256                          # replicas per pH: standard error ~0.008 at pH = pKa
    pH = np.repeat(levels, per)
    R = len(pH)
    # start from the target populations (end states), so the run samples the stationary law
    rng = np.random.default_rng(5)
    p_glu = 1.0 / (10 ** (4.4 - pH) + 1.0)
    w = np.stack([np.ones(R), 10 ** (pH - 6.53), 10 ** (pH - 6.92)], 1)
    his_state = np.array([rng.choice(3, p=wi / wi.sum()) for wi in w])
    lam0 = np.stack([(rng.random(R) < p_glu).astype(float), (his_state > 0).astype(float),
                     (his_state == 2).astype(float)], 1)
    ctx = cph.cph_create(s, pH, replica_seeds(7, R), lambda0=lam0, barrier=2.0, nstout=20,
                         frame_capacity=4096, vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    ctx.cph_step(5000)                 # equilibrate 10 ps
    for r in range(R):
        ctx.cph_get_frames(r)          # drop equilibration frames
    ctx.cph_step(40000)                # 80 ps
    glu = np.zeros(len(levels))
    his_d = np.zeros(len(levels))
    his_e = np.zeros(len(levels))
    for k in range(len(levels)):
        lp, dl, el = [], [], []
        for r in range(k * per, (k + 1) * per):
            fr, dropped = ctx.cph_get_frames(r)
            assert dropped == 0
            lp.append(fr[:, 0])
            deprot = fr[:, 1] >= 0.5
            dl.append(np.mean(deprot & (fr[:, 2] < 0.5)))
            el.append(np.mean(deprot & (fr[:, 2] >= 0.5)))
        glu[k] = np.mean(np.concatenate(lp) >= 0.5)
        his_d[k], his_e[k] = np.mean(dl), np.mean(el)
    hh = 1.0 / (10 ** (4.4 - levels) + 1.0)
    print("glu", glu, hh)
    assert np.all(np.abs(glu - hh) < 0.03)
    # BASELINE target: the synthetic titration's pKa within 0.05 pH units of the oracle's, which
    # for Coulomb-free sites is the set pKa (closed form; oracle pin in test_oracle_pins.py)
    from paper_2410_01626_b200 import titration as T
    pka = T.fit_curve(levels, glu)
    print("fitted pKa", pka)
    assert abs(pka - 4.4) < 0.05
    pk_d, pk_e = 6.53, 6.92
    prot = 1.0 / (1 + 10 ** (levels - pk_d) + 10 ** (levels - pk_e))
    print("his delta", his_d, prot * 10 ** (levels - pk_d), "eps", his_e, prot * 10 ** (levels - pk_e))
    assert np.all(np.abs(his_d - prot * 10 ** (levels - pk_d)) < 0.03)
    assert np.all(np.abs(his_e - prot * 10 ** (levels - pk_e)) < 0.03)


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_full_size_sampled_parity(cph, cfg):
    """BASELINE's large configs (C3 25k atoms / 15 groups, C4 40k / 20 groups incl. His, C5
    250k / 150 groups, K = 60 / 72 / 128) at full size: sampled atoms' phi and forces and every
    group's dV/dlambda against the oracle computed one by one."""
    from oracle import ewald as OE
    from oracle import pme as OP
    from oracle.charges import charges
    from oracle.units import F_COUL
    s = make_system(cfg)
    lam0 = np.random.default_rng(2).uniform(0, 1, (1, s.n_coords))
    ctx = cph.cph_create(s, [5.0], [11], lambda0=lam0)
    f, phi = ctx.cph_get_forces(0)
    coul, _ = ctx.cph_get_dvdl(0)
    q, dq = charges(s, lam0[0])
    beta = OE.ewald_beta(1.0, 1e-5)
    x = s.pos.astype(np.float64)
    rec = OP.pme(x, q, s.box, beta, s.pme_grid, 4)
    idx = np.concatenate([s.group_atoms, np.random.default_rng(0).choice(s.n_atoms, 64, replace=False)])
    idx = np.unique(idx)
    phr, Fr = OE.real_space_at(idx, x, q, s.type, s.c6, s.c12, s.box, 1.0, beta, s.excl)
    ex = OE.exclusion_correction(x, q, s.box, beta, s.excl)
    _, phis = OE.self_term(q, beta)
    _, phin = OE.net_charge_term(q, s.box, beta)
    phi_ref = phr + ex["phi"][idx] + rec["phi"][idx] + phis[idx] + phin[idx]
    F_ref = Fr + ex["F"][idx] + rec["F"][idx]
    assert np.linalg.norm(phi[idx] - phi_ref) / np.linalg.norm(phi_ref) < 2e-5
    assert np.linalg.norm(f[idx] - F_ref) / np.linalg.norm(F_ref) < 2e-5
    from tests.parity import force_atom_err, phi_atom_err
    print(f"C{cfg} per-atom F", force_atom_err(f[idx], F_ref), "phi", phi_atom_err(phi[idx], phi_ref))
    assert force_atom_err(f[idx], F_ref) < 2e-5 and phi_atom_err(phi[idx], phi_ref) < 2e-5
    # dV/dlambda per coordinate from the sampled phi of every lambda atom
    pos = {a: k for k, a in enumerate(idx)}
    from oracle.charges import coord_ptr
    cp = coord_ptr(s.group_kind)
    ref = np.zeros(s.n_coords)
    mag = np.zeros(s.n_coords)
    for g in range(s.n_groups):
        for k in range(s.group_ptr[g], s.group_ptr[g + 1]):
            p = phi_ref[pos[s.group_atoms[k]]]
            ref[cp[g]] += F_COUL * dq[k, 0] * p
            mag[cp[g]] += abs(F_COUL * dq[k, 0] * p)
            if s.group_kind[g] == 3:
                ref[cp[g] + 1] += F_COUL * dq[k, 1] * p
                mag[cp[g] + 1] += abs(F_COUL * dq[k, 1] * p)
    err = np.abs(coul - ref) / np.maximum(np.abs(ref), mag)
    print(f"C{cfg} dvdl max rel", err.max())
    assert err.max() < 2e-5


def test_pfc_saturation_matches_oracle(cph):
    """Reading R22 at the extreme pH of the lysozyme/cardiotoxin grids."""
    s = make_system(2)
    pH = np.array([-1.0, 1.0, 9.0])
    ctx = cph.cph_create(s, pH, replica_seeds(3, 3))
    for r in range(3):
        ref = [OPFC.pfc_2state(6.0, s.pKa[0, 0], pH[r], 300.0, 1e6), *OPFC.pfc_3state(6.0, s.pKa[1], pH[r], 300.0, 1e6)]
        np.testing.assert_allclose(ctx.cph_get_bias_params(r), ref, atol=1e-7)


def test_bench_launch_configuration_parity(cph):
    """The exact configuration bench.py times (C2, 17 pH replicas in one context on a
    dedicated stream, bench seeds and velocities), after a CUDA-graph block of steps: the
    first and last replica against the oracle evaluated at the device state."""
    import torch
    s = make_system(2)
    R = 17
    pH = np.resize(np.asarray(s.pH_grid, np.float64), R)
    seeds = replica_seeds(2, R, base=0)
    vel = np.stack([make_velocities(s, r) for r in range(R)])
    stream = torch.cuda.Stream()
    ctx = cph.cph_create(s, pH, seeds, vel_replicas=vel, cuda_stream=stream.cuda_stream)
    ctx.cph_step(20)
    for r in (0, R - 1):
        x, v = ctx.cph_get_positions(r)
        lam, lamv = ctx.cph_get_lambdas(r)
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam, vel0=v, pos0=x)
        ref.lamv = lamv
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        print(r, {k: v for k, v in err.items() if k != "E_terms"})
        assert err["force"] <= RTOL and err["phi"] <= RTOL and err["dvdl_coul"] <= RTOL
        assert err["dvdl_bias"] <= 1e-9 and err["E_total"] <= ETOL, err["E_terms"]


def test_dense_region_grows_list_capacity_and_no_groups(cph):
    """Edge cases: a system with no lambda-groups whose solvent is squeezed into 0.6^3 of the
    box (4.6x the mean density: up to 601 neighbours against the default capacity of 1.6x the
    mean count + 64 = 512): create grows the capacity, the pair list stays bit-exact and the
    forces match the oracle."""
    import copy
    s = copy.deepcopy(small_system(n_solvent=600, his=False))
    s.group_kind = s.group_kind[:0]
    s.group_ptr = s.group_ptr[:1]
    s.group_atoms = s.group_atoms[:0]
    s.state_q = s.state_q[:0]
    s.is_buffer = s.is_buffer[:0]
    s.pKa = s.pKa[:0]
    s.vmm = s.vmm[:0]
    mob = s.mass > 0
    s.pos[mob] = (s.pos[mob] % s.box) * 0.6
    ctx = cph.cph_create(s, [4.4], [3])
    got = ctx.cph_get_pairlist(0)
    ref = OPL.canonical_pairs(s.pos, s.box, s.params["rlist"], s.excl)
    assert np.array_equal(got, ref)
    oref = OracleReplica(s, 4.4, 3, lam0=np.zeros(0))
    err = compare_snapshot(ctx, 0, oref)
    print({k: v for k, v in err.items() if k != "E_terms"})
    assert err["force"] <= RTOL and err["phi"] <= RTOL


def test_set_ph_refreshes_bias_forces(cph):
    """cph_set_pH re-evaluates dV_bias/dlambda and E_bias at the unchanged lambda:
    right after the call both equal the oracle's at the new pH (fp64 on both sides)."""
    s = make_system(2)
    ctx, lam0, pH, seeds, vel = _ctx(cph, s, 2)
    ctx.cph_step(7)
    for r, new in ((0, 6.3), (1, 2.2)):
        ctx.cph_set_pH(r, new)
        lam, _ = ctx.cph_get_lambdas(r)
        x, v = ctx.cph_get_positions(r)
        ref = OracleReplica(s, new, int(seeds[r]), lam0=lam, vel0=v, pos0=x)
        _, bias = ctx.cph_get_dvdl(r)
        np.testing.assert_allclose(bias, ref.cur["dvdl_bias"], rtol=1e-9, atol=1e-9)
        e = ctx.cph_get_energies(r)
        assert abs(e["bias"] - ref.energies()["bias"]) < 1e-9 * max(1.0, abs(e["bias"]))


def test_checkpoint_restore_continues_the_run(cph):
    """A restore into a fresh context continues the run: the blob's step moves the
    clock, so Philox noise, nstlist phases and frames pick up where they left off and the
    trajectory matches the uninterrupted one (to the rounding of the fp32 spread atomics)."""
    s = make_system(1)
    R = 2
    mk = lambda: _ctx(cph, s, R, seed=4)[0]
    a = mk()
    a.cph_step(25)
    blob = a.cph_get_state_all()
    a.cph_step(31)
    b = mk()
    b.cph_set_state_all(blob)
    assert b.cph_current_step() == 25
    b.cph_step(31)
    assert b.cph_current_step() == a.cph_current_step() == 56
    for r in range(R):
        la, lb = a.cph_get_lambdas(r)[0], b.cph_get_lambdas(r)[0]
        xa, xb = a.cph_get_positions(r)[0], b.cph_get_positions(r)[0]
        d = xa - xb
        d -= s.box * np.round(d / s.box)
        print(r, "max|dlam|", np.abs(la - lb).max(), "max|dx|", np.abs(d).max())
        assert np.abs(la - lb).max() < 1e-5 and np.abs(d).max() < 1e-4
    # a single-replica restore must not move the shared clock
    c = mk()
    with pytest.raises(cph.CphError) as ei:
        c.cph_set_state(0, a.cph_get_state(0))
    assert ei.value.status == 4


def test_packed_pair_path_matches_scalar_path(cph, monkeypatch):
    """The FFMA2 pair path (non-lambda warps and lambda warps between energy steps) against
    the scalar path that every snapshot test checks against the oracle: two contexts, one
    with CPH_NB_PACKED=0, stepped through non-energy steps (nstenergy = 1000) with the same
    noise; positions and lambdas agree to fp32 rounding growth."""
    s = make_system(2)
    ctxs = []
    for packed in ("1", "0"):
        monkeypatch.setenv("CPH_NB_PACKED", packed)
        ctxs.append(_ctx(cph, s, 3, seed=8, nstenergy=1000)[0])
    for c in ctxs:
        c.cph_step(9)                      # steps 1..8 are not energy steps: packed path
    for r in range(3):
        xa, xb = ctxs[0].cph_get_positions(r)[0], ctxs[1].cph_get_positions(r)[0]
        la, lb = ctxs[0].cph_get_lambdas(r)[0], ctxs[1].cph_get_lambdas(r)[0]
        d = xa - xb
        d -= s.box * np.round(d / s.box)
        print(r, "max|dx|", np.abs(d).max(), "max|dlam|", np.abs(la - lb).max())
        assert np.abs(d).max() < 2e-5 and np.abs(la - lb).max() < 2e-6


def test_c1_200_step_trajectory_diagnostic(cph):
    """SURVEY §8(c) trajectory diagnostic: C1 (1.5k atoms, one Glu), same Philox streams, 200
    steps, positions and lambda compared at steps 1, 10, 100 and 200.  fp32 (GPU) vs fp64
    (oracle) differences grow with the chaotic dynamics; steps 1 and 10 are gated at the
    snapshot level, 100 and 200 are reported with a loose sanity bound (reading A18)."""
    s = make_system(1)
    lam0 = np.array([[0.35]])
    vel = make_velocities(s, 17)[None]
    ctx = cph.cph_create(s, [4.4], [4242], lambda0=lam0, vel_replicas=vel)
    ref = OracleReplica(s, 4.4, 4242, lam0=lam0[0], vel0=vel[0])
    done = 0
    for target, (tol_x, tol_l) in ((1, (1e-5, 1e-6)), (10, (1e-4, 1e-5)), (100, (2e-2, 2e-2)),
                                   (200, (5e-2, 5e-2))):
        ctx.cph_step(target - done)
        while ref.step_index < target:
            ref.step()
        done = target
        x, _ = ctx.cph_get_positions(0)
        lam, _ = ctx.cph_get_lambdas(0)
        d = x - ref.x
        d -= s.box * np.round(d / s.box)
        dx, dl = float(np.abs(d).max()), float(np.abs(lam - ref.lam).max())
        print(f"step {target}: max|dx| {dx:.3e} nm, max|dlambda| {dl:.3e}")
        assert dx < tol_x and dl < tol_l


def test_deterministic_mode_bitwise_reproducible_and_parity(cph):
    """deterministic = 1 (fixed-point PME spread): two runs from the same inputs agree bit for
    bit after 37 steps (rebuilds included) - the default fp32-atomic spread agrees only to
    rounding - and the snapshot still matches the oracle."""
    s = make_system(1)
    runs = []
    for _ in range(2):
        ctx, lam0, pH, seeds, vel = _ctx(cph, s, 2, seed=5, deterministic=1)
        if not runs:
            for r in range(2):
                ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam0[r], vel0=vel[r])
                err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
                assert err["force"] <= RTOL and err["force_atom"] <= RTOL and err["dvdl_coul"] <= RTOL
                assert err["E_total"] <= ETOL
        ctx.cph_step(37)
        runs.append([(ctx.cph_get_positions(r), ctx.cph_get_lambdas(r)) for r in range(2)])
    for (xa, la), (xb, lb) in zip(runs[0], runs[1]):
        assert np.array_equal(xa[0], xb[0]) and np.array_equal(xa[1], xb[1])
        assert np.array_equal(la[0], lb[0]) and np.array_equal(la[1], lb[1])


def test_restore_keeps_the_list_only_for_unmoved_atoms(cph):
    """cph_set_state_all re-sorts and rebuilds the pair list unless every restored atom sits
    where the last rebuild put it (then the list of the last rebuild is the list of this
    configuration).  Moved atoms: the list is the canonical list at the restored positions;
    a second restore of the same blob reuses it and gives bitwise the same forces."""
    s = make_system(1)
    ctx, *_ = _ctx(cph, s, 2, seed=4, deterministic=1)
    ctx.cph_step(13)
    blob = ctx.cph_get_state_all()
    ctx.cph_step(7)                                   # the step-20 rebuild moves the list on
    ctx.cph_set_state_all(blob)                       # restored atoms moved: rebuild
    f1 = [ctx.cph_get_forces(r) for r in range(2)]
    lists = []
    for r in range(2):
        x, _ = ctx.cph_get_positions(r)
        got = ctx.cph_get_pairlist(r)
        assert np.array_equal(got, OPL.canonical_pairs(x, s.box, s.params["rlist"], s.excl))
        lists.append(got)
    ctx.cph_step(3)                                   # no rebuild before step 19
    ctx.cph_set_state_all(blob)                       # same positions as the list: reuse
    for r in range(2):
        f, phi = ctx.cph_get_forces(r)
        assert np.array_equal(f, f1[r][0]) and np.array_equal(phi, f1[r][1])
        assert np.array_equal(ctx.cph_get_pairlist(r), lists[r])
    assert ctx.cph_current_step() == 13

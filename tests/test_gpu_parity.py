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
        assert err["phi_lambda_atoms"] <= RTOL
        assert err["dvdl_coul"] <= RTOL
        assert err["dvdl_bias"] <= 1e-9
        assert err["E_total"] <= ETOL, err["E_terms"]


@pytest.mark.parametrize("which", ["tiny", "c1", "c2"])
def test_pairlist_bit_exact(cph, which):
    s = small_system() if which == "tiny" else make_system(1 if which == "c1" else 2)
    ctx, *_ = _ctx(cph, s, 2)
    for r in range(2):
        got = ctx.cph_get_pairlist(r)
        ref = OPL.canonical_pairs(s.pos, s.box, s.params["rlist"], s.excl)
        assert got.shape == ref.shape and np.array_equal(got, ref)
    # after a rebuild at step nstlist, against the positions the device holds
    ctx.cph_step(s.params["nstlist"])
    for r in range(2):
        x, _ = ctx.cph_get_positions(r)
        got = ctx.cph_get_pairlist(r)
        ref = OPL.canonical_pairs(x, s.box, s.params["rlist"], s.excl)
        assert np.array_equal(got, ref)


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
    ctx = cph.cph_create(s, [4.4], [5], lambda0=lam, mode=1)
    acc = np.zeros(s.n_coords)
    for _ in range(6):
        ctx.cph_step(1)
        c, b = ctx.cph_get_dvdl(0)
        acc += c + b
        np.testing.assert_array_equal(ctx.cph_get_lambdas(0)[0], lam[0])
    mean, n = ctx.cph_get_ti_means(0)
    assert n == 6
    np.testing.assert_allclose(mean, acc / 6, rtol=1e-12, atol=1e-12)

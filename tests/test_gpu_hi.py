"""Hamiltonian interpolation (params.hamiltonian = 1; Eq. 1) on the GPU vs
the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle.engine import OracleReplica  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds, small_system  # noqa: E402
from tests.parity import ETOL, RTOL, compare_snapshot  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


@pytest.mark.parametrize("which", ["tiny", "c1", "c2"])
def test_hi_snapshot_parity(cph, which):
    s = small_system() if which == "tiny" else make_system(1 if which == "c1" else 2)
    R = 2
    rng = np.random.default_rng(4)
    lam0 = rng.uniform(-0.05, 1.05, (R, s.n_coords))
    pH = np.array([4.0, 6.0])
    seeds = replica_seeds(8, R)
    vel = np.stack([make_velocities(s, 40 + r) for r in range(R)])
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, hamiltonian=1)
    for r in range(R):
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam0[r], vel0=vel[r], params=dict(hamiltonian=True))
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        e, eo = ctx.cph_get_energies(r), ref.energies()
        print(which, r, {k: v for k, v in err.items() if k != "E_terms"}, "hi", e["hi"], eo["hi"])
        assert abs(eo["hi"]) > 1e-3
        assert abs(e["hi"] - eo["hi"]) <= 1e-5 * max(1.0, abs(eo["hi"]))
        assert err["force"] <= RTOL and err["dvdl_coul"] <= RTOL and err["dvdl_bias"] <= 1e-9
        assert err["E_total"] <= ETOL, err["E_terms"]


def test_hi_short_horizon_trajectory(cph):
    s = small_system()
    lam0 = np.array([[0.3, 0.6, 0.4]])
    vel = make_velocities(s, 5)[None]
    ctx = cph.cph_create(s, [5.0], [1234], lambda0=lam0, vel_replicas=vel, hamiltonian=1)
    ref = OracleReplica(s, 5.0, 1234, lam0=lam0[0], vel0=vel[0], params=dict(hamiltonian=True))
    for n in (1, 4, 5):
        ctx.cph_step(n)
        for _ in range(n):
            ref.step()
        x, _ = ctx.cph_get_positions(0)
        lam, _ = ctx.cph_get_lambdas(0)
        d = x - ref.x
        d -= s.box * np.round(d / s.box)
        print("step", ref.step_index, "max|dx|", np.abs(d).max(), "max|dlam|", np.abs(lam - ref.lam).max())
        assert np.abs(d).max() < 1e-4 and np.abs(lam - ref.lam).max() < 1e-5


def test_hi_nve_conserves_energy(cph):
    """gamma = 0 with mobile lambda: the HI correction's lambda derivative and forces are the
    gradient of its energy, so the total energy does not drift."""
    s = small_system()
    R = 4
    vel = np.stack([make_velocities(s, 70 + r) for r in range(R)])
    lam0 = np.tile([0.3, 0.6, 0.4], (R, 1))
    eq = cph.cph_create(s, np.full(R, 5.0), replica_seeds(2, R), lambda0=lam0, vel_replicas=vel, hamiltonian=1,
                        gamma_atom=5.0, gamma_lambda=5.0, barrier=2.0)
    eq.cph_step(3000)
    blob = eq.cph_get_state_all()
    ctx = cph.cph_create(s, np.full(R, 5.0), replica_seeds(2, R), lambda0=lam0, vel_replicas=vel, hamiltonian=1,
                         gamma_atom=0.0, gamma_lambda=0.0, barrier=2.0, nstenergy=10)
    ctx.cph_set_state_all(blob)
    e0 = np.array([ctx.cph_get_energies(r)["total"] for r in range(R)])
    tr = []
    for _ in range(40):
        ctx.cph_step(100)
        tr.append(np.array([ctx.cph_get_energies(r)["total"] for r in range(R)]) - e0)
    tr = np.array(tr)
    t = np.arange(1, 41) * 100 * 0.002
    slope = np.polyfit(t, tr.mean(1), 1)[0]
    print("HI NVE drift kJ/mol/ps", slope, "max |dE|", np.abs(tr).max())
    assert abs(slope) < 0.05 and np.abs(tr).max() < 1.0

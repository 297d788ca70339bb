"""Bussi thermostat on the GPU vs the oracle, and its temperature."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle.engine import OracleReplica  # noqa: E402
from oracle.units import kT  # noqa: E402
from synthetic.systems import make_velocities, replica_seeds, small_system  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def test_bussi_short_horizon_trajectory_matches_oracle(cph):
    """Same Philox streams (R28): the rescaled atom and lambda trajectories agree."""
    s = small_system()
    lam0 = np.array([[0.3, 0.6, 0.4]])
    vel = make_velocities(s, 5)[None]
    ctx = cph.cph_create(s, [5.0], [1234], lambda0=lam0, vel_replicas=vel, thermostat="bussi")
    ref = OracleReplica(s, 5.0, 1234, lam0=lam0[0], vel0=vel[0], params=dict(thermostat="bussi"))
    for n in (1, 4, 5):
        ctx.cph_step(n)
        for _ in range(n):
            ref.step()
        x, v = ctx.cph_get_positions(0)
        lam, lamv = ctx.cph_get_lambdas(0)
        d = x - ref.x
        d -= s.box * np.round(d / s.box)
        print("step", ref.step_index, "max|dx|", np.abs(d).max(), "max|dv|", np.abs(v - ref.v).max(),
              "max|dlam|", np.abs(lam - ref.lam).max(), "max|dlamv|", np.abs(lamv - ref.lamv).max())
        assert np.abs(d).max() < 1e-4 and np.abs(lam - ref.lam).max() < 1e-5
        assert np.abs(lamv - ref.lamv).max() < 1e-3


def test_bussi_temperature_atoms_and_lambda(cph):
    """Canonical kinetic energies: atoms 3 N_mobile kT/2, lambda C kT/2 per replica.  The
    replicas are first relaxed with strong Langevin friction: from the lattice / end-state
    start the lambda particles release tens of kJ/mol, which a weak global thermostat
    (tau_lambda = 1 ps, 3 degrees of freedom) takes several ps to remove."""
    s = small_system()
    R = 128
    vel = np.stack([make_velocities(s, 60 + r) for r in range(R)])
    pH = np.full(R, 4.4)
    seeds = replica_seeds(21, R)
    eq = cph.cph_create(s, pH, seeds, vel_replicas=vel, lambda0=np.tile([0.2, 0.8, 0.3], (R, 1)), barrier=2.0,
                        gamma_atom=5.0, gamma_lambda=5.0)
    eq.cph_step(5000)
    blob = eq.cph_get_state_all()
    ctx = cph.cph_create(s, pH, seeds, vel_replicas=vel, thermostat="bussi", nstenergy=10, barrier=2.0)
    ctx.cph_set_state_all(blob)
    ctx.cph_step(5000)        # 10 ps under Bussi before sampling: tau_lambda = 1 ps over 3 degrees of freedom
    ka, kl = [], []
    for _ in range(100):
        ctx.cph_step(40)
        for r in range(R):
            e = ctx.cph_get_energies(r)
            ka.append(e["KE_atoms"])
            kl.append(e["KE_lambda"])
    nf = 3 * int(np.count_nonzero(s.mass > 0))
    t_atoms = 2 * np.mean(ka) / (nf * kT(1.0))
    t_lam = 2 * np.mean(kl) / (3 * kT(1.0))
    print("T atoms", t_atoms, "T lambda", t_lam)
    assert abs(t_atoms - 300.0) < 3.0
    assert abs(t_lam - 300.0) < 25.0

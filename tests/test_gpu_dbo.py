"""DBO + censoring on the GPU (libcph.so through the C ABI) vs the oracle."""
import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import dbo as ODBO  # noqa: E402
from oracle import pfc as OPFC  # noqa: E402
from oracle.engine import OracleReplica  # noqa: E402
from synthetic.systems import make_velocities, replica_seeds, small_system  # noqa: E402
from tests.parity import ETOL, RTOL, compare_snapshot  # noqa: E402

KIND = {"well0": ODBO.WELL0, "well1": ODBO.WELL1, "barrier": ODBO.BARRIER,
        "barrier_t_prot": ODBO.BARRIER_T_PROT, "barrier_t_deprot": ODBO.BARRIER_T_DEPROT}


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def test_dbo_parameters_snapshot_and_pfc_parity(cph):
    """Shifted wells and protonation-keyed tautomer barriers: PFC depths, bias derivatives
    (including the barrier's lambda_p dependence) and energies match the oracle."""
    s = small_system()
    lam0 = np.array([[0.04, 0.7, 0.35], [0.93, 0.45, 0.8]])
    pH = np.array([4.0, 6.6])
    seeds = replica_seeds(5, 2)
    vel = np.stack([make_velocities(s, 30 + r) for r in range(2)])
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel)
    dbo = [np.array([[0.05, 0.94, 4.0, 4.0], [-0.03, 1.06, 9.0, 9.0], [0.02, 0.97, 2.0, 8.0]]),
           np.array([[-0.08, 1.08, 1.0, 1.0], [0.0, 1.0, 6.0, 6.0], [0.06, 1.0, 12.0, 3.0]])]
    for r in range(2):
        ctx.cph_set_dbo_params(r, dbo[r])
        np.testing.assert_array_equal(ctx.cph_get_dbo_params(r), dbo[r])
    for r in range(2):
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam0[r], vel0=vel[r], dbo_params=dbo[r])
        np.testing.assert_allclose(ctx.cph_get_bias_params(r), ref.d1, atol=1e-8)
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        print(r, {k: v for k, v in err.items() if k != "E_terms"})
        assert err["dvdl_bias"] <= 1e-9
        assert err["dvdl_coul"] <= RTOL and err["force"] <= RTOL
        assert err["E_total"] <= ETOL, err["E_terms"]
    # out-of-range parameters are rejected
    bad = dbo[0].copy()
    bad[0, 2] = 5.0                   # lambda_p coordinate with h_prot != h_deprot
    with pytest.raises(cph.CphError):
        ctx.cph_set_dbo_params(0, bad)


def test_dbo_short_run_events_censor_and_trajectory_match_oracle(cph):
    """Tiny blocks (well 20, barrier 30 steps) so every rule fires within 60 steps; the
    adjustment log, the block statistics, the censor flags and the lambda trajectory (which
    runs on the adjusted bias after each block end) agree with the oracle."""
    s = small_system()
    lam0 = np.array([[0.1, 0.9, 0.5]])
    vel = make_velocities(s, 5)[None]
    cfg = dict(well_steps=20, barrier_steps=30, censor_steps=10)
    ctx = cph.cph_create(s, [5.0], [1234], lambda0=lam0, vel_replicas=vel, nstout=1, frame_capacity=256,
                         dbo_well=1, dbo_barrier=1, dbo_well_steps=20, dbo_barrier_steps=30, dbo_censor_steps=10)
    ref = OracleReplica(s, 5.0, 1234, lam0=lam0[0], vel0=vel[0], dbo=dict(well=True, barrier=True, **cfg))
    # block statistics part-way through the first block
    ctx.cph_step(15)
    for _ in range(15):
        ref.step()
    w, b = ctx.cph_get_dbo_stats(0)
    np.testing.assert_array_equal(w[:, [0, 1, 3]], ref.stats_well.well[:, [0, 1, 3]])
    np.testing.assert_allclose(w[:, [2, 4]], ref.stats_well.well[:, [2, 4]], atol=1e-4)
    np.testing.assert_array_equal(b, ref.stats_barrier.barrier)
    ctx.cph_step(45)
    for _ in range(45):
        ref.step()
    ev = ctx.cph_get_dbo_events()
    print("gpu events", ev)
    print("oracle events", ref.events)
    assert len(ev) == len(ref.events) and len(ev) >= 4
    kinds = set()
    for (st, r, c, kind, old, new), (st_o, c_o, kind_o, old_o, new_o) in zip(ev, ref.events):
        assert (st, r, c, KIND[kind]) == (st_o, 0, c_o, kind_o)
        assert abs(old - old_o) < 1e-5 and abs(new - new_o) < 1e-5
        kinds.add(kind)
    assert {"well0", "well1", "barrier"} <= kinds
    np.testing.assert_allclose(ctx.cph_get_dbo_params(0), ref.dbo_params, atol=1e-5)
    np.testing.assert_allclose(ctx.cph_get_bias_params(0), ref.d1, atol=1e-4)
    # frames: steps 0..60 (nstout 1), censor flags per the oracle's rule on the site's events
    fr, cens, steps, _, dropped = ctx.cph_get_frames_ex(0)
    assert dropped == 0 and np.array_equal(steps, np.arange(61))
    group_of = np.array([0, 1, 1])
    for c in range(3):
        adj = [S for g, S in ref.censor if g == group_of[c]]
        np.testing.assert_array_equal(cens[:, c], ODBO.censor_flags(steps, adj, cfg["censor_steps"]))
    assert cens.any()
    lam, _ = ctx.cph_get_lambdas(0)
    print("max|dlam|", np.abs(lam - ref.lam).max())
    assert np.abs(lam - ref.lam).max() < 1e-4
    e = ctx.cph_get_energies(0)
    assert abs(e["total"] - ref.energies()["total"]) <= 1e-5 * abs(ref.energies()["total"])


def test_dbo_regulates_transitions_and_keeps_populations(cph):
    """Bias-only lambda dynamics (equal state charges): with both DBO controllers on, the
    barrier heights settle where about 25 % of the frames are in transition
    and every parameter stays within the paper's bounds; then, with the regulated wells and
    barriers frozen (DBO off, same states), the deprotonated fractions follow
    Henderson-Hasselbalch: the PFC recomputed for the adjusted potential
    keeps the populations.  (During regulation with 5-ps blocks the populations carry the
    relaxation after each adjustment, which censoring only partly removes.)"""
    s = copy.deepcopy(small_system())
    s.state_q[:, 2] = s.state_q[:, 0]
    s.state_q[:, 3] = s.state_q[:, 0]
    s.vmm[:] = 0.0
    levels = np.array([3.9, 4.4, 4.9])
    per = 192                        # standard error of each fraction ~0.011 (tools/diag_dbo_pop.py)
    pH = np.repeat(levels, per)
    R = len(pH)
    rng = np.random.default_rng(9)
    p_glu = 1.0 / (10 ** (4.4 - pH) + 1.0)
    w = np.stack([np.ones(R), 10 ** (pH - 6.53), 10 ** (pH - 6.92)], 1)
    his_state = np.array([rng.choice(3, p=wi / wi.sum()) for wi in w])
    lam0 = np.stack([(rng.random(R) < p_glu).astype(float), (his_state > 0).astype(float),
                     (his_state == 2).astype(float)], 1)
    vel = np.stack([make_velocities(s, r) for r in range(R)])
    seeds = replica_seeds(11, R)
    blk = 2500                                              # 5 ps blocks for both controllers
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, nstout=10, frame_capacity=8192, vel_replicas=vel,
                         dbo_well=1, dbo_barrier=1, dbo_well_steps=blk, dbo_barrier_steps=blk,
                         dbo_censor_steps=500)
    ctx.cph_step(30 * blk)                                  # regulate (150 ps)
    for r in range(R):
        ctx.cph_get_frames_ex(r)
    ev0 = ctx.cph_get_dbo_events()
    ctx.cph_step(20 * blk)                                  # 100 ps, still regulating
    ev1 = ctx.cph_get_dbo_events()
    print("events while regulating", len(ev0), "afterwards", len(ev1))
    trans = []
    params = []
    for r in range(R):
        fr, cens, steps, _, dropped = ctx.cph_get_frames_ex(r)
        assert dropped == 0
        prm = ctx.cph_get_dbo_params(r)
        assert np.all(np.abs(prm[:, 0]) <= 0.08 + 1e-12) and np.all(np.abs(prm[:, 1] - 1) <= 0.08 + 1e-12)
        assert np.all((prm[:, 2:] >= 1.0) & (prm[:, 2:] <= 20.0))
        trans.append(np.mean((fr[:, 0] > 0.2) & (fr[:, 0] < 0.8)))
        params.append(prm)
    print("in-transition fraction (Glu)", np.mean(trans))
    assert 0.15 <= np.mean(trans) <= 0.35
    # populations under the regulated (frozen) potential
    blob = ctx.cph_get_state_all()
    eq = cph.cph_create(s, pH, seeds, lambda0=lam0, nstout=10, frame_capacity=8192, vel_replicas=vel)
    for r in range(R):
        eq.cph_set_dbo_params(r, params[r])
    eq.cph_set_state_all(blob)
    eq.cph_step(2500)
    for r in range(R):
        eq.cph_get_frames(r)
    eq.cph_step(40000)
    glu = np.zeros(len(levels))
    for k in range(len(levels)):
        x = [eq.cph_get_frames(r)[0][:, 0] for r in range(k * per, (k + 1) * per)]
        glu[k] = np.mean(np.concatenate(x) >= 0.5)
    hh = 1.0 / (10 ** (4.4 - levels) + 1.0)
    print("glu (regulated potential)", glu, "HH", hh)
    assert np.all(np.abs(glu - hh) < 0.04)

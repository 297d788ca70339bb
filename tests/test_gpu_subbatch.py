"""Replica sub-batches (cph_params.sub_batches): a context split into S concurrently stepped
batches computes what one batch computes.  Every random number is keyed on (replica seed,
step, atom) and every kernel works per replica, so the split changes nothing but the batch
count of the cuFFT plans (whose fp32 rounding may depend on it): trajectories, energies and
frames agree with S = 1 to fp32 rounding, replica-exchange decisions, DBO events and frame
steps exactly, and the snapshot of a replica in the last batch matches the oracle."""
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


def _inputs(s, R, seed):
    rng = np.random.default_rng(seed)
    lam0 = rng.uniform(0.0, 1.0, (R, s.n_coords))
    pH = np.linspace(3.0, 7.0, R)
    seeds = replica_seeds(77, R, seed)
    vel = np.stack([make_velocities(s, 200 + r) for r in range(R)])
    return lam0, pH, seeds, vel


def _snapshot(ctx, R):
    out = []
    for r in range(R):
        pos, vel = ctx.cph_get_positions(r)
        lam, lv = ctx.cph_get_lambdas(r)
        e = ctx.cph_get_energies(r)
        fr, cens, steps, _, dropped = ctx.cph_get_frames_ex(r)
        out.append((pos, vel, lam, lv, np.array([e[k] for k in sorted(e)]), fr, steps, dropped))
    return out


def _assert_close(a, b, tol=2e-5):
    """pos, vel, lambda, lambda velocity, energies, frames to fp32 rounding; frame steps and
    drop counts exactly."""
    worst = 0.0
    for ra, rb in zip(a, b):
        for k, (xa, xb) in enumerate(zip(ra, rb)):
            xa, xb = np.asarray(xa, np.float64), np.asarray(xb, np.float64)
            assert xa.shape == xb.shape
            if k >= 6:
                assert np.array_equal(xa, xb)
                continue
            scale = np.maximum(1.0, np.abs(xb)) if k == 4 else 1.0
            d = float(np.max(np.abs(xa - xb) / scale)) if xa.size else 0.0
            worst = max(worst, d)
            assert d <= tol, (k, d)
    return worst


def test_sub_batches_equal_one_batch(cph):
    s = make_system(1)
    R = 5
    lam0, pH, seeds, vel = _inputs(s, R, 3)
    runs = {}
    for S in (1, 2, 3):
        ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, deterministic=1, sub_batches=S,
                             nstout=5)
        assert ctx.R == R
        if S == 3:      # replica 4 lives in the last batch (sizes 2, 2, 1)
            ref = OracleReplica(s, pH[4], int(seeds[4]), lam0=lam0[4], vel0=vel[4])
            err = compare_snapshot(ctx, 4, ref, lam_atoms=s.group_atoms)
            assert err["force"] <= RTOL and err["force_atom"] <= RTOL and err["dvdl_coul"] <= RTOL
            assert err["E_total"] <= ETOL
        f0 = [ctx.cph_get_forces(r)[0] for r in range(R)]
        if S == 1:
            f_one = f0
        else:     # step 0: same forces up to the FFT's rounding
            print("step-0 force max |diff|", S, max(float(np.abs(fa - fb).max()) for fa, fb in zip(f0, f_one)))
            for fa, fb in zip(f0, f_one):
                assert np.linalg.norm(fa - fb) <= 1e-6 * np.linalg.norm(fb)
        ctx.cph_step(13)
        ctx.cph_step(24)            # crosses rebuilds at 20 and 30 off the block phase
        assert ctx.cph_current_step() == 37
        assert ctx.cph_launch_count() > 0
        runs[S] = _snapshot(ctx, R)
        ctx.close()
    print("max deviation S=2", _assert_close(runs[2], runs[1]), "S=3", _assert_close(runs[3], runs[1]))


def test_sub_batches_checkpoint_moves_between_layouts(cph):
    """A checkpoint of a 2-batch context restores into a 1-batch context (and back) and both
    continue identically."""
    s = small_system()
    R = 4
    lam0, pH, seeds, vel = _inputs(s, R, 5)
    a = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, deterministic=1, sub_batches=2)
    a.cph_step(23)
    blob = a.cph_get_state_all()
    b = cph.cph_create(s, pH, seeds, deterministic=1, sub_batches=1)
    b.cph_set_state_all(blob)
    c = cph.cph_create(s, pH, seeds, deterministic=1, sub_batches=3)
    c.cph_set_state_all(b.cph_get_state_all())
    for ctx in (a, b, c):
        assert ctx.cph_current_step() == 23
        ctx.cph_step(17)
    sa, sb, sc = (_snapshot(x, R) for x in (a, b, c))
    _assert_close([r[:5] for r in sa], [r[:5] for r in sb])
    _assert_close([r[:5] for r in sa], [r[:5] for r in sc])
    # a single-replica restore into the split context goes to the right batch
    one = b.cph_get_state(3)
    a.cph_set_state(3, one)
    np.testing.assert_array_equal(a.cph_get_positions(3)[0], b.cph_get_positions(3)[0])   # restored bits
    with pytest.raises(cph.CphError):
        a.cph_get_lambdas(4)


def test_sub_batches_replica_exchange_across_batches(cph):
    """Ladders that straddle sub-batches (R = 6, P = 3, S = 4: batches 2, 2, 1, 1) take the
    decisions of one batch, through cph_exchange and through the row-buffer calls."""
    import torch
    s = small_system()
    levels = np.array([4.0, 4.5, 5.0])
    labels = np.array([2, 0, 1, 1, 2, 0])
    rng = np.random.default_rng(21)
    lam0 = rng.uniform(0.0, 1.0, (6, s.n_coords))
    seeds = replica_seeds(9, 6)
    one = cph.cph_create(s, levels[labels], seeds, lambda0=lam0, ph_levels=levels, deterministic=1, sub_batches=1)
    four = cph.cph_create(s, levels[labels], seeds, lambda0=lam0, ph_levels=levels, deterministic=1, sub_batches=4)
    for attempt in range(10):
        one.cph_step(10)
        four.cph_step(10)
        one.cph_exchange(3, attempt)
        if attempt % 2:
            four.cph_exchange(3, attempt)
        else:
            rows = torch.empty(6 * 4, dtype=torch.float64, device="cuda")
            four.exchange_energies_into(rows)
            four.exchange_apply_from(rows, 3, attempt)
        np.testing.assert_array_equal(one.cph_get_labels(), four.cph_get_labels())
    for r in range(6):
        np.testing.assert_allclose(one.cph_get_lambdas(r)[0], four.cph_get_lambdas(r)[0], atol=2e-5)
    s1, c1 = one.cph_get_exchange_stats(2)
    s4, c4 = four.cph_get_exchange_stats(2)
    np.testing.assert_array_equal(s1, s4)
    np.testing.assert_array_equal(c1, c4)
    assert c1.sum() > 0


def test_sub_batches_dbo_events_merged(cph):
    """DBO with two identical replicas in two batches: each replica's adjustment log is the
    single-batch one, and the merged log is ordered by (step, replica)."""
    s = small_system()
    lam0 = np.array([[0.1, 0.9, 0.5]] * 2)
    vel = np.stack([make_velocities(s, 5)] * 2)
    kw = dict(lambda0=lam0, vel_replicas=vel, nstout=1, frame_capacity=256, dbo_well=1, dbo_barrier=1,
              dbo_well_steps=20, dbo_barrier_steps=30, dbo_censor_steps=10, deterministic=1)
    one = cph.cph_create(s, [5.0, 5.0], [1234, 1234], sub_batches=1, **kw)
    two = cph.cph_create(s, [5.0, 5.0], [1234, 1234], sub_batches=2, **kw)
    one.cph_step(60)
    two.cph_step(60)
    e1, e2 = one.cph_get_dbo_events(), two.cph_get_dbo_events()
    assert len(e1) >= 8 and len(e1) == len(e2)
    for a, b in zip(e1, e2):
        assert a[:4] == b[:4] and abs(a[4] - b[4]) < 1e-5 and abs(a[5] - b[5]) < 1e-5
    assert [(e[0], e[1]) for e in e2] == sorted((e[0], e[1]) for e in e2)
    for r in range(2):
        assert [e[2:4] for e in e2 if e[1] == r] == [e[2:4] for e in e2 if e[1] == 0]
        np.testing.assert_allclose(one.cph_get_dbo_params(r), two.cph_get_dbo_params(r), atol=1e-5)
        f1, c1, *_ = one.cph_get_frames_ex(r)
        f2, c2, *_ = two.cph_get_frames_ex(r)
        assert np.allclose(f1, f2, atol=2e-5) and np.array_equal(c1, c2)


def test_sub_batches_profile_and_default(cph):
    """Automatic split (R * N >= 24000 -> 4 batches) runs; cph_profile_steps sums the batches."""
    s = make_system(2)
    R = 8
    lam0, pH, seeds, vel = _inputs(s, R, 8)
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel)
    ms, cnt = ctx.cph_profile_steps(10)
    ref = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, sub_batches=1)
    ms1, cnt1 = ref.cph_profile_steps(10)
    # four batches launch every per-step kernel four times
    assert cnt["nonbonded"] == 4 * cnt1["nonbonded"] and cnt["gather"] == 4 * cnt1["gather"]
    assert ctx.cph_current_step() == 10
    for r in range(R):
        np.testing.assert_allclose(ctx.cph_get_lambdas(r)[0], ref.cph_get_lambdas(r)[0], atol=1e-5)


@pytest.mark.parametrize("variant", ["bussi", "hamiltonian", "ti"])
def test_sub_batches_with_thermostat_hi_and_ti(cph, variant):
    """The Bussi thermostat (per-replica kinetic-energy reductions), Hamiltonian interpolation
    (per-group corrections) and fixed-lambda TI (per-replica accumulators) give one batch's
    results in three sub-batches."""
    s = make_system(1) if variant != "hamiltonian" else small_system()
    R = 5
    lam0, pH, seeds, vel = _inputs(s, R, 9)
    kw = {"bussi": dict(thermostat="bussi"), "hamiltonian": dict(hamiltonian=1), "ti": dict(mode=1)}[variant]
    out = []
    for S in (1, 3):
        ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, deterministic=1, sub_batches=S, **kw)
        ctx.cph_step(25)
        snap = _snapshot(ctx, R)
        ti = [ctx.cph_get_ti_means(r) for r in range(R)] if variant == "ti" else None
        out.append((snap, ti))
        ctx.close()
    _assert_close(out[1][0], out[0][0])
    if variant == "ti":
        for (m1, n1), (m3, n3) in zip(out[0][1], out[1][1]):
            assert n1 == n3 and n1 > 0
            np.testing.assert_allclose(m3, m1, rtol=1e-6, atol=1e-9)

"""pH replica exchange on the GPU vs the oracle."""
import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import pfc as OPFC  # noqa: E402
from oracle import remd as OR  # noqa: E402
from oracle.charges import coord_ptr  # noqa: E402
from oracle.units import kT  # noqa: E402
from synthetic.systems import make_velocities, replica_seeds, small_system  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def _level_d1(s, levels):
    return [np.array([OPFC.pfc_2state(6.0, s.pKa[0, 0], pH, 300.0, 1e6),
                      *OPFC.pfc_3state(6.0, s.pKa[1], pH, 300.0, 1e6)]) for pH in levels]


def test_exchange_energy_rows_match_oracle(cph):
    import torch
    s = small_system()
    levels = np.array([3.5, 4.5, 5.5, 6.5])
    R = 4
    rng = np.random.default_rng(2)
    lam0 = rng.uniform(-0.05, 1.05, (R, 3))
    ctx = cph.cph_create(s, levels[[2, 0, 3, 1]], replica_seeds(3, R), lambda0=lam0, ph_levels=levels)
    rows = torch.zeros(R * 5, dtype=torch.float64, device="cuda")
    ctx.exchange_energies_into(rows)
    rows = rows.cpu().numpy().reshape(R, 5)
    np.testing.assert_array_equal(rows[:, 0], [2, 0, 3, 1])
    np.testing.assert_array_equal(ctx.cph_get_labels(), [2, 0, 3, 1])
    d1 = _level_d1(s, levels)
    cptr = coord_ptr(s.group_kind)
    for r in range(R):
        for p in range(4):
            ref = OR.ph_energy(s, lam0[r], levels[p], d1[p], 300.0, 6.0, 1e6, cptr)
            assert abs(rows[r, 1 + p] - ref) <= 1e-7 * max(1.0, abs(ref)), (r, p, rows[r, 1 + p], ref)
        np.testing.assert_allclose(ctx.cph_get_bias_params(r), d1[[2, 0, 3, 1][r]], atol=1e-8)


def test_exchange_decisions_match_oracle_bit_for_bit(cph):
    """Synthetic energy rows through cph_exchange_apply: the same fp64 inputs and Philox
    counters give exactly the oracle's swaps; labels, level tables and statistics follow."""
    import torch
    s = small_system()
    P, L = 3, 2
    levels = np.array([4.0, 5.0, 6.0])
    R = P * L
    labels = np.array([1, 0, 2, 2, 1, 0])
    ctx = cph.cph_create(s, levels[labels], replica_seeds(4, R), ph_levels=levels)
    d1 = _level_d1(s, levels)
    rng = np.random.default_rng(8)
    att = np.zeros((L, P - 1), int)
    acc = np.zeros((L, P - 1), int)
    cur = labels.copy()
    for attempt in range(40):
        E = rng.normal(0.0, 1.2 * kT(300.0), (R, P))
        rows = np.concatenate([cur[:, None].astype(float), E], 1).reshape(-1)
        t = torch.from_numpy(rows).cuda()
        ctx.exchange_apply_from(t, 77, attempt)
        cur, dec = OR.decide(E, cur, P, kT(300.0), 77, attempt)
        for l, p, a in dec:
            att[l, p] += 1
            acc[l, p] += a
        np.testing.assert_array_equal(ctx.cph_get_labels(), cur)
    a, b = ctx.cph_get_exchange_stats(L)
    np.testing.assert_array_equal(a, att)
    np.testing.assert_array_equal(b, acc)
    assert 0 < acc.sum() < att.sum()
    for r in range(R):
        np.testing.assert_allclose(ctx.cph_get_bias_params(r), d1[cur[r]], atol=1e-8)


def test_replica_exchange_sampling_keeps_per_ph_populations(cph):
    """Bias-only lambda dynamics with exchanges every 100 steps: the frames collected at
    each pH level (by label) still follow Henderson-Hasselbalch, and swaps are accepted."""
    from paper_2410_01626_b200 import remd
    s = copy.deepcopy(small_system())
    s.state_q[:, 2] = s.state_q[:, 0]
    s.state_q[:, 3] = s.state_q[:, 0]
    s.vmm[:] = 0.0
    levels = np.array([3.4, 3.9, 4.4, 4.9, 5.4])
    P, L = len(levels), 48
    R = P * L
    labels = np.tile(np.arange(P), L)
    pH = levels[labels]
    rng = np.random.default_rng(5)
    lam0 = np.stack([(rng.random(R) < 1.0 / (10 ** (4.4 - pH) + 1.0)).astype(float), np.zeros(R), np.zeros(R)], 1)
    ctx = cph.cph_create(s, pH, replica_seeds(13, R), lambda0=lam0, ph_levels=levels, barrier=2.0, nstout=20,
                         frame_capacity=8192, vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    nxt = remd.run(ctx, 5000, 100, seed=99)
    for r in range(R):
        ctx.cph_get_frames_ex(r)
    remd.run(ctx, 80000, 100, seed=99, first_attempt=nxt)
    frac = np.zeros(P)
    cnt = np.zeros(P)
    for r in range(R):
        fr, _, _, lab, dropped = ctx.cph_get_frames_ex(r)
        assert dropped == 0
        for p in range(P):
            sel = lab == p
            frac[p] += np.count_nonzero(fr[sel, 0] >= 0.5)
            cnt[p] += np.count_nonzero(sel)
    frac /= cnt
    hh = 1.0 / (10 ** (4.4 - levels) + 1.0)
    a, b = ctx.cph_get_exchange_stats(L)
    print("per-level fraction", frac, "HH", hh, "acceptance", b.sum(0) / a.sum(0))
    # standard errors over ladders are ~0.01 at this length (tools/diag_remd_pop.py)
    assert np.all(np.abs(frac - hh) < 0.04)
    assert np.all(b.sum(0) > 0.1 * a.sum(0))


def test_two_contexts_exchange_like_one(cph):
    """The multi-GPU layout on one device: two contexts holding replicas [0, 3) and [3, 6) of
    one 6-replica ladder (remd_first / remd_total), rows concatenated as the NCCL all-gather
    would, take exactly the decisions of a single context holding all six."""
    import torch
    s = small_system()
    levels = np.array([3.5, 4.0, 4.5, 5.0, 5.5, 6.0])
    labels = np.array([2, 0, 5, 1, 4, 3])
    rng = np.random.default_rng(12)
    lam0 = rng.uniform(0.0, 1.0, (6, 3))
    seeds = replica_seeds(8, 6)
    one = cph.cph_create(s, levels[labels], seeds, lambda0=lam0, ph_levels=levels)
    a = cph.cph_create(s, levels[labels[:3]], seeds[:3], lambda0=lam0[:3], ph_levels=levels, remd_first=0,
                       remd_total=6)
    b = cph.cph_create(s, levels[labels[3:]], seeds[3:], lambda0=lam0[3:], ph_levels=levels, remd_first=3,
                       remd_total=6)
    for attempt in range(12):
        rows = torch.empty(6 * 7, dtype=torch.float64, device="cuda")
        a.exchange_energies_into(rows[:21])
        b.exchange_energies_into(rows[21:])
        a.exchange_apply_from(rows, 5, attempt)
        b.exchange_apply_from(rows, 5, attempt)
        one.cph_exchange(5, attempt)
        np.testing.assert_array_equal(np.concatenate([a.cph_get_labels(), b.cph_get_labels()]),
                                      one.cph_get_labels())
    sa, ca = a.cph_get_exchange_stats(1)
    so, co = one.cph_get_exchange_stats(1)
    np.testing.assert_array_equal(sa, so)
    np.testing.assert_array_equal(ca, co)
    assert co.sum() > 0

"""The cluster-pair path (cph_params.pair_list = 2: half cluster-pair list with per-i-cluster
interaction masks) against the fp64 oracle and against the per-atom path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import pairlist as OPL  # noqa: E402
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


def _ctx(cph, s, R, pair_list, seed=1):
    rng = np.random.default_rng(seed)
    lam0 = rng.uniform(-0.1, 1.1, (R, s.n_coords))
    pH = np.linspace(3.0, 7.0, R)
    seeds = replica_seeds(98, R, seed)
    vel = np.stack([make_velocities(s, 100 + r) for r in range(R)])
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel, pair_list=pair_list)
    return ctx, lam0, pH, seeds, vel


@pytest.mark.parametrize("which", ["tiny", "c1", "c2"])
def test_cluster_snapshot_parity(cph, which):
    s = small_system() if which == "tiny" else make_system(1 if which == "c1" else 2)
    ctx, lam0, pH, seeds, vel = _ctx(cph, s, 2, pair_list=2)
    for r in range(2):
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam0[r], vel0=vel[r])
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        print(which, r, {k: v for k, v in err.items() if k != "E_terms"})
        for k in ("force", "phi", "force_atom", "phi_atom", "phi_lambda_atoms", "dvdl_coul"):
            assert err[k] <= RTOL, (k, err[k])
        assert err["E_total"] <= ETOL, err["E_terms"]


@pytest.mark.parametrize("which", ["tiny", "c1", "c3"])
def test_cluster_pairlist_bit_exact(cph, which):
    """The set bits of the cluster masks are exactly the canonical pair set, each pair once
    (the directed getter reports both orientations: one evaluation acts on both atoms)."""
    s = small_system() if which == "tiny" else make_system({"c1": 1, "c3": 3}[which])
    ctx, *_ = _ctx(cph, s, 1, pair_list=2)
    ref = OPL.canonical_pairs(s.pos, s.box, s.params["rlist"], s.excl)
    got = ctx.cph_get_pairlist(0)
    assert got.shape == ref.shape and np.array_equal(got, ref)
    dirs = ctx.cph_get_pairlist_directed(0)
    both = np.concatenate([ref, ref[:, ::-1]])
    both = both[np.lexsort((both[:, 1], both[:, 0]))]
    assert dirs.shape == both.shape and np.array_equal(dirs, both)
    # after a rebuild, against the positions the device holds
    ctx.cph_step(s.params["nstlist"])
    pos, _ = ctx.cph_get_positions(0)
    ref2 = OPL.canonical_pairs(pos, s.box, s.params["rlist"], s.excl)
    got2 = ctx.cph_get_pairlist(0)
    assert got2.shape == ref2.shape and np.array_equal(got2, ref2)


def test_cluster_matches_atom_path_over_steps(cph):
    """Both layouts step the same trajectory to rounding (same Philox stream, same pair decisions)."""
    s = make_system(2)
    A, *_ = _ctx(cph, s, 2, pair_list=1)
    B, *_ = _ctx(cph, s, 2, pair_list=2)
    A.cph_step(2 * s.params["nstlist"])      # ends on a rebuild: the lists are those of the current positions
    B.cph_step(2 * s.params["nstlist"])
    for r in range(2):
        la, _ = A.cph_get_lambdas(r)
        lb, _ = B.cph_get_lambdas(r)
        fa, pa = A.cph_get_forces(r)
        fb, pb = B.cph_get_forces(r)
        assert np.max(np.abs(la - lb)) < 1e-4
        assert np.linalg.norm(fb - fa) / np.linalg.norm(fa) < 1e-4
        # rounding-level differences move a few pairs across r_list at the rebuilds: each
        # list is the canonical set of its own positions
        for ctx in (A, B):
            x, _ = ctx.cph_get_positions(r)
            assert np.array_equal(ctx.cph_get_pairlist(r), OPL.canonical_pairs(x, s.box, s.params["rlist"], s.excl))


def test_deterministic_rejects_cluster(cph):
    s = small_system()
    with pytest.raises(cph.CphError):
        cph.cph_create(s, [4.0], [1], pair_list=2, deterministic=1)


def test_cluster_pairlist_rows_c4(cph):
    """C4 (40k atoms, the bench config): sampled full rows of the cluster list (2000 atoms incl.
    every lambda atom and solute exclusions) against the oracle's canonical rows, at create and
    after a rebuild."""
    s = make_system(4)
    ctx = cph.cph_create(s, [5.0], [11], vel_replicas=make_velocities(s, 3)[None], pair_list=2)
    rng = np.random.default_rng(4)
    idx = np.unique(np.concatenate([s.group_atoms, s.excl[:200, 0], rng.choice(s.n_atoms, 1800, replace=False)]))
    for stage in range(2):
        x = s.pos if stage == 0 else ctx.cph_get_positions(0)[0]
        got = ctx.cph_get_pairlist_rows(0, idx)
        ref = OPL.canonical_partners(x, s.box, s.params["rlist"], s.excl, idx)
        bad = [int(i) for i, a, b in zip(idx, got, ref) if not np.array_equal(a, b)]
        assert not bad, bad[:10]
        ctx.cph_step(s.params["nstlist"])

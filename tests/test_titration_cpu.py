"""Host titration bookkeeping: replica assignment, the one
all-gather of lambda frames over torch.distributed (gloo, world size 2, on CPU), and the
H-H / Hill fits against the oracle's independent SciPy fits."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import analysis as OA
from paper_2410_01626_b200 import titration as T


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R = [3, 2][rank]                              # uneven replica counts per rank
    local = np.full((R, 5, 2), rank, np.float32) + np.arange(R, dtype=np.float32)[:, None, None] * 10
    got = T.gather_frames(local)
    out[rank] = got
    dist.destroy_process_group()


def test_gather_frames_gloo_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    a, b = out[0], out[1]
    assert a.shape == (5, 5, 2) and np.array_equal(a, b)
    np.testing.assert_array_equal(a[:, 0, 0], [0, 10, 20, 1, 11])


def test_assign_replicas_round_robin():
    parts = [T.assign_replicas(17, 8, r) for r in range(8)]
    assert sorted(sum(parts, [])) == list(range(17))
    assert parts[0] == [0, 8, 16] and parts[7] == [7, 15]


def test_fraction_and_fits_match_oracle():
    assert T.deprotonated_fraction([0.5, 0.49, 0.9, 0.1]) == 0.5          # lambda_p >= 0.5 (R1)
    # censored frames (DBO) do not count
    assert T.deprotonated_fraction([0.5, 0.49, 0.9, 0.1], censored=[0, 0, 1, 0]) == 1 / 3
    rng = np.random.default_rng(3)
    pH = np.repeat(np.linspace(2.0, 8.0, 13), 4)
    x = np.clip(OA.hh(pH, 4.4, 0.9) + rng.normal(0, 0.02, pH.size), 0, 1)
    assert abs(T.fit_curve(pH, x) - OA.fit_hh(pH, x)) < 1e-7
    pk, n = T.fit_curve(pH, x, hill=True)
    pk2, n2 = OA.fit_hill(pH, x)
    assert abs(pk - pk2) < 1e-6 and abs(n - n2) < 1e-6
    exact = OA.hh(np.linspace(2.5, 5.5, 7), 4.0)
    assert abs(T.fit_curve(np.linspace(2.5, 5.5, 7), exact) - 4.0) < 1e-9


def test_bootstrap_interval_contains_truth():
    rng = np.random.default_rng(0)
    levels = np.linspace(3.0, 6.0, 7)
    fr = np.clip(OA.hh(levels, 4.5)[:, None] + rng.normal(0, 0.03, (7, 10)), 0, 1)
    est, lo, hi = T.bootstrap(levels, fr, B=300, seed=1)
    assert lo <= 4.5 <= hi and hi - lo < 0.2
    with pytest.raises(ValueError):
        T.fit_curve([1.0, 2.0], [1.0, 1.0])


def test_fit_vmm_matches_oracle_fit():
    from oracle import bias as OB
    from oracle.calibration import vmm_from_ti
    rng = np.random.default_rng(8)
    c = rng.normal(size=36)
    c[0] = 0.0
    LP, LT = np.meshgrid(T.TI_GRID, T.TI_GRID, indexing="ij")
    lp, lt = LP.ravel(), LT.ravel()
    g = np.array([OB.vmm(c, a, b)[1:] for a, b in zip(lp, lt)]) + rng.normal(0, 0.1, (lp.size, 2))
    np.testing.assert_allclose(T.fit_vmm(3, lp, lt, g), vmm_from_ti(3, lp, lt, g), atol=1e-9)
    g1 = g[:14, :1]
    x = np.array(T.TI_GRID)
    np.testing.assert_allclose(T.fit_vmm(2, x, None, g1), vmm_from_ti(2, x, None, g1), atol=1e-9)


def test_his_micro_pka_recovered_from_exact_populations():
    """3-state His populations at Table 2 micro pKa values (6.53, 6.92):
    the micro ratios of PAPER.md:982-983 are H-H curves in the micro pKa, so fitting them
    returns the inputs (closed form); the library's counting matches the oracle's."""
    pk_d, pk_e = 6.53, 6.92
    levels = np.linspace(5.5, 8.0, 6)
    xd, xe = [], []
    for pH in levels:
        w = np.array([1.0, 10 ** (pH - pk_d), 10 ** (pH - pk_e)])
        n = np.round(w / w.sum() * 200000).astype(int)
        lp = np.concatenate([np.zeros(n[0]), np.ones(n[1] + n[2])])
        lt = np.concatenate([np.full(n[0], 0.3), np.zeros(n[1]), np.ones(n[2])])
        a, b = T.micro_fractions(lp, lt)
        assert (a, b) == OA.micro_fractions(lp, lt)
        xd.append(a)
        xe.append(b)
    assert abs(T.fit_curve(levels, np.array(xd)) - pk_d) < 1e-3
    assert abs(T.fit_curve(levels, np.array(xe)) - pk_e) < 1e-3

"""His microscopic pKa analysis on GPU-sampled frames."""
import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from synthetic.systems import make_velocities, replica_seeds, small_system  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def test_his_micro_pka_from_bias_only_sampling(cph):
    """Coulomb-free lambda dynamics with PFC: the micro ratios of the sampled frames fitted
    with H-H give the Table 2 micro pKa values the bias was built from (6.53, 6.92)."""
    from paper_2410_01626_b200 import titration as T
    s = copy.deepcopy(small_system())
    s.state_q[:, 2] = s.state_q[:, 0]
    s.state_q[:, 3] = s.state_q[:, 0]
    s.vmm[:] = 0.0
    levels = np.linspace(5.5, 8.0, 6)
    per = 128
    pH = np.repeat(levels, per)
    R = len(pH)
    rng = np.random.default_rng(17)
    w = np.stack([np.ones(R), 10 ** (pH - 6.53), 10 ** (pH - 6.92)], 1)
    st = np.array([rng.choice(3, p=wi / wi.sum()) for wi in w])
    lam0 = np.stack([np.zeros(R), (st > 0).astype(float), (st == 2).astype(float)], 1)
    ctx = cph.cph_create(s, pH, replica_seeds(31, R), lambda0=lam0, barrier=2.0, nstout=20, frame_capacity=8192,
                         vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    ctx.cph_step(5000)
    for r in range(R):
        ctx.cph_get_frames(r)
    ctx.cph_step(60000)
    xd, xe = [], []
    for k in range(len(levels)):
        lp, lt = [], []
        for r in range(k * per, (k + 1) * per):
            fr, _ = ctx.cph_get_frames(r)
            lp.append(fr[:, 1])
            lt.append(fr[:, 2])
        a, b = T.micro_fractions(np.concatenate(lp), np.concatenate(lt))
        xd.append(a)
        xe.append(b)
    pk_d = T.fit_curve(levels, np.array(xd))
    pk_e = T.fit_curve(levels, np.array(xe))
    print("micro pKa delta", pk_d, "eps", pk_e)
    assert abs(pk_d - 6.53) < 0.1 and abs(pk_e - 6.92) < 0.1

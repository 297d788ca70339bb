"""End to end with electrostatics on: fixed-lambda TI on the GPU (mode 1) -> V_mm fit
 -> lambda dynamics -> titration fit (SURVEY §8 a11 + a12).

With every atom frozen, the Coulomb energy is a fixed polynomial of the lambdas (charges are
bilinear in (lp, lt) by Eq. 2 and E is quadratic in the charges), so the TI means are its exact
derivative, the degree-5 fit reproduces it exactly and V_coul + V_mm is flat: the sampled
populations must follow the closed forms of the bias alone (Eq. 4 and the His micro pKa
values) although the compensated Coulomb free energy is hundreds of kJ/mol.  Glu is made
Coulomb-free so that the His calibration is not coupled to another site.

(With mobile solvent the same loop needs the long TI runs of PAPER.md:705-712: the synthetic
ionic solvent relaxes diffusively.)"""
import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from synthetic.systems import replica_seeds, small_system  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def test_gpu_ti_calibration_flattens_coulomb(cph):
    from paper_2410_01626_b200 import titration as T
    s = copy.deepcopy(small_system())
    s.mass[:] = 0.0                                  # frozen environment
    s.state_q[:7, 2] = s.state_q[:7, 0]              # Glu (group 0, 7 site atoms + buffer): equal states
    s.state_q[:7, 3] = s.state_q[:7, 0]
    s.state_q[7, :] = s.state_q[7, 0]                # ... and its buffer
    s.vmm[:] = 0.0
    grid = np.array(T.TI_GRID)
    lp, lt = [a.reshape(-1) for a in np.meshgrid(grid, grid, indexing="ij")]
    R = len(lp)
    lam0 = np.stack([np.zeros(R), lp, lt], 1)
    ti = cph.cph_create(s, np.full(R, 7.0), replica_seeds(3, R), lambda0=lam0, mode=1)
    ti.cph_step(4)
    means = np.array([ti.cph_get_ti_means(r)[0] for r in range(R)])
    assert np.all(np.abs(means[:, 0]) < 1e-3)          # Coulomb-free Glu
    span = np.ptp(means[:, 1])
    print("His TI dV/dlp span", span, "dV/dlt span", np.ptp(means[:, 2]))
    assert span > 100.0                                 # a strong Coulomb dependence to cancel
    s.vmm[1] = T.fit_vmm(3, lp, lt, means[:, 1:])
    # V_coul + V_mm is flat: the residual derivative at the grid points is at rounding level
    chk = cph.cph_create(s, np.full(R, 7.0), replica_seeds(4, R), lambda0=lam0, mode=1)
    res = np.array([chk.cph_get_dvdl(r)[0][1:] for r in range(R)])
    vm = np.array([_vmm_grad(s.vmm[1], a, b) for a, b in zip(lp, lt)])
    print("max |dV_coul/dl + dV_mm/dl| on the grid", np.max(np.abs(res + vm)))
    assert np.max(np.abs(res + vm)) < 0.5                # kJ/mol, vs kT = 2.49

    levels = np.array([3.4, 4.4, 5.4, 6.5, 7.5])
    per = 192
    pH = np.repeat(levels, per)
    R2 = len(pH)
    rng = np.random.default_rng(9)
    p_glu = 1.0 / (10 ** (4.4 - pH) + 1.0)
    w = np.stack([np.ones(R2), 10 ** (pH - 6.53), 10 ** (pH - 6.92)], 1)
    his_state = np.array([rng.choice(3, p=wi / wi.sum()) for wi in w])
    start = np.stack([(rng.random(R2) < p_glu).astype(float), (his_state > 0).astype(float),
                      (his_state == 2).astype(float)], 1)
    dyn = cph.cph_create(s, pH, replica_seeds(8, R2), lambda0=start, barrier=2.0, nstout=20,
                         frame_capacity=4096)
    dyn.cph_step(5000)
    for r in range(R2):
        dyn.cph_get_frames(r)
    dyn.cph_step(40000)
    glu, his_d, his_e = (np.zeros(len(levels)) for _ in range(3))
    for k in range(len(levels)):
        fr = np.concatenate([dyn.cph_get_frames(r)[0] for r in range(k * per, (k + 1) * per)])
        glu[k] = np.mean(fr[:, 0] >= 0.5)
        deprot = fr[:, 1] >= 0.5
        his_d[k] = np.mean(deprot & (fr[:, 2] < 0.5))
        his_e[k] = np.mean(deprot & (fr[:, 2] >= 0.5))
    hh = 1.0 / (10 ** (4.4 - levels) + 1.0)
    prot = 1.0 / (1 + 10 ** (levels - 6.53) + 10 ** (levels - 6.92))
    print("glu", glu, hh)
    print("his delta", his_d, prot * 10 ** (levels - 6.53), "eps", his_e, prot * 10 ** (levels - 6.92))
    assert np.all(np.abs(glu - hh) < 0.035)
    assert np.all(np.abs(his_d - prot * 10 ** (levels - 6.53)) < 0.035)
    assert np.all(np.abs(his_e - prot * 10 ** (levels - 6.92)) < 0.035)
    # macroscopic His pKa from the deprotonated fraction: -log10(10^-6.53 + 10^-6.92) = 6.38
    pka = T.fit_curve(levels, his_d + his_e)
    print("His macro pKa", pka)
    assert abs(pka - (-np.log10(10 ** -6.53 + 10 ** -6.92))) < 0.08


def _vmm_grad(c, lp, lt):
    c = np.asarray(c, np.float64).reshape(6, 6)
    dp = sum(a * c[a, b] * lp ** (a - 1) * lt ** b for a in range(1, 6) for b in range(6))
    dt = sum(b * c[a, b] * lp ** a * lt ** (b - 1) for a in range(6) for b in range(1, 6))
    return dp, dt

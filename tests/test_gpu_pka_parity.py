"""Electrostatics-on titration: GPU pKa vs the oracle's exact frozen-environment pKa.

C1 (one Glu-like site with its charge buffer in 1.5k atoms, BASELINE configs[0]) with every
atom frozen: only lambda moves, E_coul(lambda) = E0 + b lambda + c lambda^2 exactly (charge
interpolation), and the lambda dynamics samples exp(-V/kT) in 1-D.  The
oracle reads b, c off its own fp64 PME energies and integrates the density per pH
(oracle.titration_quadrature); the GPU runs the full step (pair kernel,
PME, lambda kernel, BAOAB) at each pH with independent replicas.  The two H-H pKa values
must agree within 0.05 pH units (BASELINE north star), with the GPU's bootstrap CI
 reported and narrower than that bar.

V_mm cancels 98 % of the Coulomb coupling (b = -380, c = -116 kJ/mol at C1) (the remainder moves the pKa by ~1 unit and
bends the landscape by the quadratic self term); the lambda mass is lowered to 10 u so the
lambda particle decorrelates in ~2 ps (the equilibrium density does not depend on it)."""
import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import titration_quadrature as TQ  # noqa: E402
from oracle.analysis import fit_hh  # noqa: E402
from oracle.engine import OracleReplica  # noqa: E402
from synthetic.systems import make_system, replica_seeds, small_system  # noqa: E402


@pytest.fixture(scope="module")
def cph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_01626_b200 as m
    return m


def test_electrostatics_on_pka_matches_oracle_quadrature(cph):
    from paper_2410_01626_b200 import titration as T
    s = copy.deepcopy(make_system(1))
    s.mass[:] = 0.0                                      # frozen environment
    s.vmm[:] = 0.0
    h, kw, temp = 2.0, 1e6, 300.0
    pKa = float(s.pKa[0, 0])
    rep = OracleReplica(s, pKa, 1, lam0=np.zeros(1))
    b, c, chk = TQ.coulomb_quadratic(rep, 0)
    print("oracle E_coul(l) - E_coul(0) = %.4f l + %.4f l^2 (quadratic check %.2e)" % (b, c, chk))
    assert chk < 1e-6 * max(1.0, abs(b))
    keep = 0.02
    s.vmm[0, 6] = -(1.0 - keep) * b                      # c_10 lambda_p
    s.vmm[0, 12] = -(1.0 - keep) * c                     # c_20 lambda_p^2
    # oracle: exact fractions on a fine pH grid -> its pKa; the GPU levels straddle it
    fine = np.linspace(pKa - 4.0, pKa + 4.0, 81)
    x_fine = TQ.titration_curve(pKa, fine, temp, h, kw, b=b, c=c, vmm=s.vmm[0])
    pka_or_fine = fit_hh(fine, x_fine)
    levels = np.round(pka_or_fine + np.array([-1.2, -0.8, -0.4, 0.0, 0.4, 0.8, 1.2]), 3)
    x_or = TQ.titration_curve(pKa, levels, temp, h, kw, b=b, c=c, vmm=s.vmm[0])
    pka_or = fit_hh(levels, x_or)
    print("oracle pKa %.4f (fine grid %.4f, set %.2f); fractions" % (pka_or, pka_or_fine, pKa), np.round(x_or, 4))

    per = 48
    pH = np.repeat(levels, per)
    R = len(pH)
    lam0 = (np.arange(R) % 2).astype(np.float64)[:, None]
    ctx = cph.cph_create(s, pH, replica_seeds(21, R), lambda0=lam0, barrier=h, lambda_mass=10.0,
                         nstout=25, frame_capacity=2048)
    ctx.cph_step(4000)                                    # 8 ps: the start is forgotten
    for r in range(R):
        ctx.cph_get_frames(r)
    ctx.cph_step(40000)                                   # 80 ps, 1600 frames per replica
    fr = np.stack([ctx.cph_get_frames(r)[0][:, 0] for r in range(R)])
    assert fr.shape[1] == 1600 and np.all(np.isfinite(fr))
    xr = (fr >= 0.5).mean(1).reshape(len(levels), per)  # per replica deprotonated fraction
    x_gpu = xr.mean(1)
    est, lo, hi = T.bootstrap(levels, xr, B=1000)
    print("GPU pKa %.4f  95%% CI [%.4f, %.4f]; fractions" % (est, lo, hi), np.round(x_gpu, 4))
    print("|dpKa| = %.4f" % abs(est - pka_or))
    assert abs(pka_or - pKa) > 0.3                        # the Coulomb remainder moves the pKa
    assert hi - lo < 0.05                                 # the test can resolve the bar
    assert abs(est - pka_or) <= 0.05
    assert np.all(np.abs(x_gpu - x_or) < 0.03)


def test_electrostatics_on_his_pka_matches_oracle_quadrature(cph):
    """The multisite case: the His group of the tiny system (HIP / HID / HIE, coordinates
    lambda_p, lambda_t) in a frozen environment, Glu made Coulomb-free.  E_coul
    is a polynomial of degree <= 2 in each of (lambda_p, lambda_t) (bilinear charges), read off
    the oracle on a 3 x 3 grid; V_mm cancels 92 % of it (the remainder's negative lambda_p^2
    curvature adds a ~2.8 kJ/mol hump, so the double-well barrier is lowered to 0.5 kJ/mol to
    keep transitions frequent).  The oracle's deprotonated / delta /
    eps fractions are 2-D quadratures of exp(-V/kT) with its own 3-state PFC depths; the GPU
    titration (full step, frozen atoms) must give the same macroscopic pKa within 0.05 and the
    tautomer populations within 0.03 per level."""
    from paper_2410_01626_b200 import titration as T
    s = copy.deepcopy(small_system())
    s.mass[:] = 0.0
    s.state_q[:7, 2] = s.state_q[:7, 0]              # Glu (group 0 + buffer): equal states
    s.state_q[:7, 3] = s.state_q[:7, 0]
    s.state_q[7, :] = s.state_q[7, 0]
    s.vmm[:] = 0.0
    h, kw, temp = 0.5, 1e6, 300.0
    pk = tuple(float(v) for v in s.pKa[1])
    rep = OracleReplica(s, pk[0], 1, lam0=np.zeros(3))
    c, chk = TQ.coulomb_biquadratic(rep, 1, 2)
    print("oracle E_coul polynomial c[a, b] (lp^a lt^b):", np.round(c, 4).tolist(), "check %.2e" % chk)
    assert chk < 1e-6 * max(1.0, np.abs(c).max())
    keep = 0.08
    for a in range(3):
        for b in range(3):
            s.vmm[1, a * 6 + b] = -(1.0 - keep) * c[a, b]
    levels = np.round(6.6 + np.array([-1.2, -0.8, -0.4, 0.0, 0.4, 0.8, 1.2]), 3)
    ref = np.array([TQ.his_fractions(pk, p, temp, h, kw, c=c, vmm=s.vmm[1], n=801) for p in levels])
    pka_or = fit_hh(levels, ref[:, 0])
    print("oracle macro pKa %.4f (set %.2f); deprot / delta / eps" % (pka_or, pk[0]), np.round(ref, 4).tolist())

    per = 128
    pH = np.repeat(levels, per)
    R = len(pH)
    lam0 = np.stack([np.zeros(R), (np.arange(R) % 2).astype(float), ((np.arange(R) // 2) % 2).astype(float)], 1)
    ctx = cph.cph_create(s, pH, replica_seeds(23, R), lambda0=lam0, barrier=h, lambda_mass=5.0,
                         nstout=25, frame_capacity=4096)
    ctx.cph_step(4000)
    for r in range(R):
        ctx.cph_get_frames(r)
    ctx.cph_step(60000)
    fr = np.stack([ctx.cph_get_frames(r)[0] for r in range(R)])          # [R, F, C]
    assert fr.shape[1] == 2400 and np.all(np.isfinite(fr))
    dep = fr[:, :, 1] >= 0.5
    xr = dep.mean(1).reshape(len(levels), per)
    xd = (dep & (fr[:, :, 2] < 0.5)).mean(1).reshape(len(levels), per).mean(1)
    xe = (dep & (fr[:, :, 2] >= 0.5)).mean(1).reshape(len(levels), per).mean(1)
    est, lo, hi = T.bootstrap(levels, xr, B=1000)
    print("GPU macro pKa %.4f  95%% CI [%.4f, %.4f]; |dpKa| = %.4f" % (est, lo, hi, abs(est - pka_or)))
    print("GPU deprot", np.round(xr.mean(1), 4).tolist(), "delta", np.round(xd, 4).tolist(), "eps", np.round(xe, 4).tolist())
    assert abs(pka_or - pk[0]) > 0.2                         # the Coulomb remainder moves the pKa
    assert hi - lo < 0.05
    assert abs(est - pka_or) <= 0.05
    assert np.all(np.abs(xd - ref[:, 1]) < 0.03) and np.all(np.abs(xe - ref[:, 2]) < 0.03)

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
from synthetic.systems import make_system, replica_seeds  # noqa: E402


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

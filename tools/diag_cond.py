"""Diagnostic: conditional mean of dV_coul/dlambda in lambda dynamics vs fixed-lambda TI means
(saved by diag_calib.py) for several integrator settings."""
import copy
import sys
import numpy as np
import paper_2410_01626_b200 as cph
from synthetic.systems import make_velocities, replica_seeds, small_system

z = np.load(sys.argv[1])
vmm, mean, grid = z["vmm"], z["mean"], z["grid"]
s = copy.deepcopy(small_system(his=False))
s.vmm[:] = 0.0
s.vmm[0] = vmm
R = 128
rng = np.random.default_rng(3)
lam_start = (rng.random(R) < 0.5).astype(float)[:, None]
vel = np.stack([make_velocities(s, 900 + r) for r in range(R)])
for label, kw in (("dt2", dict()), ("dt0.5", dict(dt=0.0005)), ("m600", dict(lambda_mass=600.0)),
                  ("gatom10", dict(gamma_atom=10.0))):
    nsub = int(round(0.002 / kw.get("dt", 0.002)))
    pre = cph.cph_create(s, np.full(R, 4.4), replica_seeds(63, R), lambda0=lam_start, mode=1, vel_replicas=vel, **kw)
    pre.cph_step(5000 * nsub)
    dyn = cph.cph_create(s, np.full(R, 4.4), replica_seeds(62, R), lambda0=lam_start, barrier=2.0, gamma_lambda=5.0, **kw)
    dyn.cph_set_state_all(pre.cph_get_state_all())
    del pre
    dyn.cph_step(10000 * nsub)
    L, D = [], []
    for _ in range(300):
        dyn.cph_step(50 * nsub)
        for r in range(R):
            L.append(dyn.cph_get_lambdas(r)[0][0])
            D.append(dyn.cph_get_dvdl(r)[0][0])
    L, D = np.array(L), np.array(D)
    row = []
    for g, m in zip(grid, mean):
        sel = np.abs(L - g) < 0.025
        row.append(round(float(D[sel].mean() - m), 1) if sel.sum() > 20 else None)
    print(label, "dyn - TI per grid point", row, flush=True)

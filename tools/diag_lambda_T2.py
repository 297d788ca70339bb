"""Diagnostic: lambda temperature vs time (Langevin, electrostatics on) and with a smaller dt."""
import sys
import numpy as np
import paper_2410_01626_b200 as cph
from synthetic.systems import make_velocities, replica_seeds, small_system

KT1 = 0.0083144626  # kJ/mol/K
s = small_system(his=False)
R = 64
vel = np.stack([make_velocities(s, 60 + r) for r in range(R)])
for label, kw in (("dt2", dict()), ("dt1", dict(dt=0.001)), ("dt0.5", dict(dt=0.0005)), ("gl10", dict(gamma_lambda=10.0))):
    ctx = cph.cph_create(s, np.full(R, 4.4), replica_seeds(21, R), vel_replicas=vel, nstenergy=10,
                         lambda0=np.tile([0.0], (R, 1)), **kw)
    nsub = int(round(0.002 / kw.get("dt", 0.002)))
    out = []
    for w in range(8):
        v2 = []
        ta = []
        for _ in range(100):
            ctx.cph_step(25 * nsub)
            for r in range(R):
                v2.append(ctx.cph_get_lambdas(r)[1] ** 2)
        out.append(round(float(s.lambda_mass if hasattr(s, "lambda_mass") else 60.0) * float(np.mean(v2)) / KT1, 0))
    print(label, "T_lambda per 5 ps window", out, flush=True)

"""Diagnostic: per-coordinate lambda temperature under Langevin / Bussi (small system)."""
import sys
import numpy as np
import paper_2410_01626_b200 as cph
from oracle.units import kT
from synthetic.systems import make_velocities, replica_seeds, small_system

s = small_system()
R = 48
vel = np.stack([make_velocities(s, 60 + r) for r in range(R)])
for label, kw in (("langevin", dict()), ("bussi", dict(thermostat="bussi")),
                  ("bussi tau_l=0.1", dict(thermostat="bussi", tau_lambda=0.1)),
                  ("langevin gamma_l=0.1", dict(gamma_lambda=0.1))):
    ctx = cph.cph_create(s, np.full(R, 4.4), replica_seeds(21, R), vel_replicas=vel, nstenergy=10, barrier=2.0,
                         lambda0=np.tile([0.2, 0.8, 0.3], (R, 1)), **kw)
    ctx.cph_step(2000)
    v2 = []
    ka = []
    for _ in range(150):
        ctx.cph_step(20)
        for r in range(R):
            lam, lamv = ctx.cph_get_lambdas(r)
            v2.append(lamv ** 2)
            ka.append(ctx.cph_get_energies(r)["KE_atoms"])
    t = 60.0 * np.mean(v2, 0) / kT(1.0)
    nf = 3 * int(np.count_nonzero(s.mass > 0))
    print(label, "T_lambda per coord", np.round(t, 1), "T atoms", round(2 * np.mean(ka) / (nf * kT(1.0)), 1), flush=True)

"""Diagnostic: NVE energy drift of the small system (atoms + lambda), dt 2 and 1 fs, lambda
free vs frozen; and lambda temperature with Coulomb-free lambda coupling."""
import copy
import numpy as np
import paper_2410_01626_b200 as cph
from oracle.units import kT
from synthetic.systems import make_velocities, replica_seeds, small_system

s = small_system()
R = 8
vel = np.stack([make_velocities(s, 60 + r) for r in range(R)])
eq = cph.cph_create(s, np.full(R, 4.4), replica_seeds(21, R), vel_replicas=vel, barrier=2.0,
                    lambda0=np.tile([0.2, 0.8, 0.3], (R, 1)), gamma_atom=5.0, gamma_lambda=5.0)
eq.cph_step(5000)
pos = np.stack([eq.cph_get_positions(r)[0] for r in range(R)])
vv = np.stack([eq.cph_get_positions(r)[1] for r in range(R)])
lam = np.stack([eq.cph_get_lambdas(r)[0] for r in range(R)])
for label, kw, nsteps in (("nve dt2", dict(dt=0.002), 5000), ("nve dt1", dict(dt=0.001), 10000),
                          ("nve dt2 lambda frozen", dict(dt=0.002, mode=1), 5000)):
    ctx = cph.cph_create(s, np.full(R, 4.4), replica_seeds(21, R), vel_replicas=vv, pos_replicas=pos, lambda0=lam,
                         barrier=2.0, gamma_atom=0.0, gamma_lambda=0.0, nstenergy=10, **kw)
    e0 = np.array([ctx.cph_get_energies(r)["total"] for r in range(R)])
    tr, kl = [], []
    for k in range(50):
        ctx.cph_step(nsteps // 50)
        tr.append(np.array([ctx.cph_get_energies(r)["total"] for r in range(R)]) - e0)
        kl.append(np.mean([ctx.cph_get_energies(r)["KE_lambda"] for r in range(R)]))
    tr = np.array(tr)
    t = np.arange(1, 51) * nsteps // 50 * kw["dt"]
    slope = np.polyfit(t, tr.mean(1), 1)[0]
    print(label, "drift kJ/mol/ps (mean over replicas)", round(slope, 3), "final dE", np.round(tr[-1], 2),
          "KE_lambda mean", round(np.mean(kl), 3), "(kT*3/2 =", round(1.5 * kT(300.0), 3), ")", flush=True)
# Coulomb-free lambda: equal state charges
s2 = copy.deepcopy(s)
s2.state_q[:, 2] = s2.state_q[:, 0]
s2.state_q[:, 3] = s2.state_q[:, 0]
ctx = cph.cph_create(s2, np.full(48, 4.4), replica_seeds(21, 48), barrier=2.0,
                     lambda0=np.tile([0.2, 0.8, 0.3], (48, 1)), gamma_lambda=0.1)
ctx.cph_step(2000)
v2 = []
for _ in range(100):
    ctx.cph_step(20)
    v2 += [ctx.cph_get_lambdas(r)[1] ** 2 for r in range(48)]
print("coulomb-free lambda T (gamma_l 0.1)", np.round(60.0 * np.mean(v2, 0) / kT(1.0), 1), flush=True)

"""Diagnostic: Glu deprotonated fraction at pH = pKa (Coulomb-free) for fixed DBO params."""
import copy
import numpy as np
import paper_2410_01626_b200 as cph
from synthetic.systems import make_velocities, replica_seeds, small_system

s = copy.deepcopy(small_system(his=False))
s.state_q[:, 2] = s.state_q[:, 0]
s.state_q[:, 3] = s.state_q[:, 0]
s.vmm[:] = 0.0
R = 192
for a0, a1, h in ((0.0, 1.0, 6.0), (0.0, 1.0, 1.0), (-0.06, 1.07, 1.0), (0.06, 0.93, 1.0), (-0.08, 1.08, 3.0)):
    rng = np.random.default_rng(1)
    lam0 = (rng.random((R, 1)) < 0.5).astype(float)
    ctx = cph.cph_create(s, np.full(R, 4.4), replica_seeds(5, R), lambda0=lam0, nstout=10, frame_capacity=8192,
                         vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    for r in range(R):
        ctx.cph_set_dbo_params(r, np.array([[a0, a1, h, h]]))
    ctx.cph_step(2500)
    for r in range(R):
        ctx.cph_get_frames(r)
    ctx.cph_step(50000)
    per = np.array([np.mean(ctx.cph_get_frames(r)[0][:, 0] >= 0.5) for r in range(R)])
    print(f"a0={a0} a1={a1} h={h}: fraction {per.mean():.4f} +- {per.std() / np.sqrt(R):.4f}  d1 {ctx.cph_get_bias_params(0)}", flush=True)

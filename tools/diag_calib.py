"""Diagnostic / end-to-end: fixed-lambda TI on the GPU -> V_mm fit -> lambda dynamics with
electrostatics on: the deprotonated fractions should follow H-H at the reference pKa."""
import copy
import sys
import numpy as np
import paper_2410_01626_b200 as cph
from paper_2410_01626_b200 import titration as T
from synthetic.systems import make_velocities, replica_seeds, small_system

per = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ti_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
s = copy.deepcopy(small_system(his=False))
s.vmm[:] = 0.0
grid = np.array(T.TI_GRID)
lam0 = np.repeat(grid, per)[:, None]
R = len(lam0)
vel = np.stack([make_velocities(s, 500 + r) for r in range(R)])
ti = cph.cph_create(s, np.full(R, 4.4), replica_seeds(61, R), lambda0=lam0, mode=1, vel_replicas=vel)
ti.cph_step(5000)
ti.cph_set_state_all(ti.cph_get_state_all())          # restart the TI accumulators after equilibration
ti.cph_step(ti_steps)
m = np.array([ti.cph_get_ti_means(r)[0][0] for r in range(R)]).reshape(len(grid), per)
mean, se = m.mean(1), m.std(1) / np.sqrt(per)
np.set_printoptions(linewidth=250)
print("TI <dV/dl>:", np.round(mean, 1))
print("se", np.round(se, 2))
vmm = T.fit_vmm(2, grid, None, mean[:, None])
import os
os.makedirs('gpurun_out', exist_ok=True)
np.savez('gpurun_out/calib.npz', vmm=vmm, mean=mean, grid=grid)
if os.environ.get('TI_ONLY'):
    sys.exit(0)
s2 = copy.deepcopy(s)
s2.vmm[0] = vmm
levels = np.array([3.9, 4.4, 4.9])
pr = 128
pH = np.repeat(levels, pr)
R2 = len(pH)
rng = np.random.default_rng(3)
lam_start = (rng.random(R2) < 1.0 / (10 ** (4.4 - pH) + 1.0)).astype(float)[:, None]
BAR = float(sys.argv[3]) if len(sys.argv) > 3 else 6.0
GL = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
NPROD = int(sys.argv[5]) if len(sys.argv) > 5 else 40000
pre = cph.cph_create(s2, pH, replica_seeds(63, R2), lambda0=lam_start, mode=1,
                     vel_replicas=np.stack([make_velocities(s2, 900 + r) for r in range(R2)]))
pre.cph_step(5000)                                   # solvent relaxed around each fixed start state
dyn = cph.cph_create(s2, pH, replica_seeds(62, R2), lambda0=lam_start, nstout=100, frame_capacity=8192,
                     barrier=BAR, gamma_lambda=GL)
dyn.cph_set_state_all(pre.cph_get_state_all())
del pre
dyn.cph_step(NPROD // 10)
for r in range(R2):
    dyn.cph_get_frames(r)
dyn.cph_step(NPROD)
lams = [dyn.cph_get_frames(r)[0][:, 0] for r in range(R2)]
trans = []
for l in lams:
    st = np.where(l < 0.2, 0, np.where(l > 0.8, 1, -1))
    st = st[st >= 0]
    trans.append(int(np.count_nonzero(np.diff(st))))
print("transitions per replica: mean", np.mean(trans), "replicas with none", int(np.sum(np.array(trans) == 0)), "of", R2)
lam_all = [np.concatenate(lams[k * pr:(k + 1) * pr]) for k in range(len(levels))]
frac = np.array([np.mean(l >= 0.5) for l in lam_all])
for k, l in enumerate(lam_all):
    h, _ = np.histogram(l, bins=12, range=(-0.1, 1.1))
    print("pH", levels[k], "hist", np.round(h / len(l), 3))
print("fractions", frac, "HH", 1.0 / (10 ** (4.4 - levels) + 1.0), "fitted pKa", T.fit_curve(levels, frac))
# conditional mean of dV_coul/dlambda in the dynamics vs the fixed-lambda TI means
L, D = [], []
for _ in range(200):
    dyn.cph_step(50)
    for r in range(R2):
        L.append(dyn.cph_get_lambdas(r)[0][0])
        D.append(dyn.cph_get_dvdl(r)[0][0])
L, D = np.array(L), np.array(D)
for g, m in zip(grid, mean):
    sel = np.abs(L - g) < 0.025
    if sel.sum() > 20:
        print(f"lambda {g:5.2f}  TI {m:8.1f}  dyn {D[sel].mean():8.1f} +- {D[sel].std() / np.sqrt(sel.sum()):.1f}  n={sel.sum()}")

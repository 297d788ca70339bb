"""Diagnostic: per-pH Glu deprotonated fraction, bias-only system, with and without pH
replica exchange; error bars from the spread over independent ladders."""
import copy
import numpy as np
import paper_2410_01626_b200 as cph
from paper_2410_01626_b200 import remd
from synthetic.systems import make_velocities, replica_seeds, small_system

s = copy.deepcopy(small_system())
s.state_q[:, 2] = s.state_q[:, 0]
s.state_q[:, 3] = s.state_q[:, 0]
s.vmm[:] = 0.0
levels = np.array([3.4, 3.9, 4.4, 4.9, 5.4])
P, L = len(levels), 48
R = P * L
labels = np.tile(np.arange(P), L)
pH = levels[labels]
hh = 1.0 / (10 ** (4.4 - levels) + 1.0)
for seed in (13, 14):
    for exch in (True, False):
        rng = np.random.default_rng(seed)
        lam0 = np.stack([(rng.random(R) < 1.0 / (10 ** (4.4 - pH) + 1.0)).astype(float), np.zeros(R), np.zeros(R)], 1)
        kw = dict(ph_levels=levels) if exch else {}
        ctx = cph.cph_create(s, pH, replica_seeds(seed, R), lambda0=lam0, barrier=2.0, nstout=20, frame_capacity=8192,
                             vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]), **kw)
        if exch:
            nxt = remd.run(ctx, 5000, 100, seed=99)
        else:
            ctx.cph_step(5000)
        for r in range(R):
            ctx.cph_get_frames_ex(r)
        if exch:
            remd.run(ctx, 80000, 100, seed=99, first_attempt=nxt)
        else:
            ctx.cph_step(80000)
        per_ladder = np.zeros((L, P))
        cnt = np.zeros((L, P))
        for r in range(R):
            fr, _, _, lab, dropped = ctx.cph_get_frames_ex(r)
            if not exch:
                lab = np.full(len(fr), labels[r])
            for p in range(P):
                sel = lab == p
                per_ladder[r // P, p] += np.count_nonzero(fr[sel, 0] >= 0.5)
                cnt[r // P, p] += np.count_nonzero(sel)
        frac = per_ladder.sum(0) / cnt.sum(0)
        se = (per_ladder / np.maximum(cnt, 1)).std(0) / np.sqrt(L)
        print("seed", seed, "exchange" if exch else "plain   ", "dev from HH", np.round(frac - hh, 4), "se", np.round(se, 4),
              flush=True)

#!/usr/bin/env python
"""Vmm calibration driver (SURVEY §8 a11, config 4 shape): one context batches every
(lambda_p, lambda_t) point of the SI grid as a replica in fixed-lambda TI mode,
collects <dV_coul/dlambda>, and fits the degree-5 polynomial.

    python tools/calibrate.py --config 2 --group 1 --steps 20000 --out vmm.json
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--group", type=int, default=0, help="lambda-group to calibrate (others held at 0)")
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--equil", type=int, default=500)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_2410_01626_b200 as cph
    from paper_2410_01626_b200 import titration as T
    from synthetic.systems import make_system, make_velocities, replica_seeds
    s = make_system(args.config)
    g = args.group
    kind = int(s.group_kind[g])
    cptr = np.concatenate([[0], np.cumsum([1 if k == 2 else 2 for k in s.group_kind])])
    grid = np.array(T.TI_GRID)
    if kind == 2:
        pts = [(a, 0.0) for a in grid]
    else:
        pts = [(a, b) for a in grid for b in grid]
    R = len(pts)
    lam0 = np.zeros((R, s.n_coords))
    for r, (a, b) in enumerate(pts):
        lam0[r, cptr[g]] = a
        if kind == 3:
            lam0[r, cptr[g] + 1] = b
    vel = np.stack([make_velocities(s, r) for r in range(R)])
    ctx = cph.cph_create(s, np.full(R, s.pKa[g, 0]), replica_seeds(100 + args.config, R), lambda0=lam0,
                         vel_replicas=vel, mode=1)
    ctx.cph_step(args.equil)
    ctx.cph_set_state_all(ctx.cph_get_state_all())     # restarts the TI accumulators
    ctx.cph_step(args.steps)
    means = np.array([ctx.cph_get_ti_means(r)[0][cptr[g]:cptr[g] + (1 if kind == 2 else 2)] for r in range(R)])
    lp = np.array([p[0] for p in pts])
    lt = np.array([p[1] for p in pts])
    vmm = T.fit_vmm(kind, lp, lt, means)
    res = {"config": args.config, "group": g, "kind": kind, "steps": args.steps, "grid": pts,
           "mean_dvdl_coul": means.tolist(), "vmm": vmm.tolist()}
    print(json.dumps({"group": g, "kind": kind, "points": R, "vmm_c10": vmm[6], "vmm_c01": vmm[1]}))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh)


if __name__ == "__main__":
    main()

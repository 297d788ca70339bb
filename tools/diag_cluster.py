"""Cluster-pair list (pair_list = 2) against the per-atom list (pair_list = 1): same pair set,
forces / phi / dV/dlambda / energies to rounding, and step timing (A/B on one box)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds, small_system  # noqa: E402


def make(s, R, mode, **kw):
    pH = np.resize(np.asarray(s.pH_grid if len(s.pH_grid) else (4.4,)), R)
    vel = np.stack([make_velocities(s, 100 + r) for r in range(R)])
    rng = np.random.default_rng(5)
    lam0 = rng.uniform(0.05, 0.95, (R, s.n_coords))
    return cph.cph_create(s, pH, [7 + r for r in range(R)], lambda0=lam0, vel_replicas=vel, pair_list=mode, **kw)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def compare(name, s, R=2, steps=0):
    A = make(s, R, 1)
    B = make(s, R, 2)
    if steps:
        A.cph_step(steps)
        B.cph_step(steps)
    for r in range(R):
        fa, pa = A.cph_get_forces(r)
        fb, pb = B.cph_get_forces(r)
        ca, _ = A.cph_get_dvdl(r)
        cb, _ = B.cph_get_dvdl(r)
        ea, eb = A.cph_get_energies(r), B.cph_get_energies(r)
        pla, plb = A.cph_get_pairlist(r), B.cph_get_pairlist(r)
        same = pla.shape == plb.shape and np.array_equal(pla, plb)
        da, db = A.cph_get_pairlist_directed(r), B.cph_get_pairlist_directed(r)
        samed = da.shape == db.shape and np.array_equal(da, db)
        fmax = np.max(np.abs(fa - fb)) / max(np.max(np.abs(fa)), 1e-30)
        print(f"{name} r{r} steps={steps}: pairs {pla.shape[0]} vs {plb.shape[0]} same={same} directed same={samed} "
              f"F rel {rel(fb, fa):.2e} Fmax {fmax:.2e} phi rel {rel(pb, pa):.2e} dvdl {np.abs(cb - ca).max():.3e} "
              f"(|dvdl| {np.abs(ca).max():.3e}) E {ea['total']:.6f} vs {eb['total']:.6f} "
              f"dE {abs(ea['total'] - eb['total']) / abs(ea['total']):.2e}", flush=True)
    A.close()
    B.close()


def timing(cfg, R, steps=200):
    s = make_system(cfg)
    out = {}
    for mode in (1, 2):
        ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid), R), replica_seeds(cfg, R),
                             vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]), pair_list=mode)
        ctx.cph_step(20)
        ctx.cph_sync()
        t0 = time.perf_counter()
        ctx.cph_step(steps)
        ctx.cph_sync()
        out[mode] = (time.perf_counter() - t0) / steps * 1e3
        prof = ctx.cph_profile_steps(20)
        print(f"C{cfg}x{R} pair_list={mode}: {out[mode]:.4f} ms/step; profile {prof}", flush=True)
        ctx.close()
    return out


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "parity"):
        compare("tiny", small_system(), R=2)
        compare("tiny", small_system(), R=2, steps=25)
        compare("C1", make_system(1), R=2)
        compare("C2", make_system(2), R=2, steps=12)
        compare("C3", make_system(3), R=1)
    if what in ("all", "time"):
        timing(2, 17)
        timing(4, 21)

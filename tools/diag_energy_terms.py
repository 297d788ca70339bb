import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2410_01626_b200 as cph
from oracle.engine import OracleReplica
from synthetic.systems import make_system, make_velocities, replica_seeds
from tests.parity import compare_snapshot
s = make_system(1)
for trial in range(3):
    R = 2
    rng = np.random.default_rng(0)
    lam0 = rng.uniform(0.0, 1.0, (R, s.n_coords))
    pH = np.linspace(3.0, 7.0, R)
    seeds = replica_seeds(99, R, 0)
    vel = np.stack([make_velocities(s, 100 + r) for r in range(R)])
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel)
    ctx.cph_step(37)
    for r in range(2):
        x, v = ctx.cph_get_positions(r)
        lam, lamv = ctx.cph_get_lambdas(r)
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam, vel0=v, pos0=x)
        ref.lamv = lamv
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        et = err["E_terms"]
        print(trial, r, "E_total", err["E_total"], {k: (round(a, 6), round(a - b, 6)) for k, (a, b) in et.items()})
    ctx.close()

"""Per-term energy differences GPU vs oracle at create on the tiny system (and C1, C2)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01626_b200 as cph  # noqa: E402
from oracle.engine import OracleReplica  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds, small_system  # noqa: E402
from tests.parity import compare_snapshot  # noqa: E402

for name, s in (("tiny", small_system()), ("c1", make_system(1))):
    R = 3
    rng = np.random.default_rng(1)
    lam0 = rng.uniform(-0.1, 1.1, (R, s.n_coords))
    pH = np.linspace(3.0, 7.0, R)
    seeds = replica_seeds(99, R, 1)
    vel = np.stack([make_velocities(s, 100 + r) for r in range(R)])
    ctx = cph.cph_create(s, pH, seeds, lambda0=lam0, vel_replicas=vel)
    for r in range(R):
        ref = OracleReplica(s, pH[r], int(seeds[r]), lam0=lam0[r], vel0=vel[r])
        err = compare_snapshot(ctx, r, ref, lam_atoms=s.group_atoms)
        print(name, r, "E_total", err["E_total"], {k: (round(a, 5), float(f"{a - b:.3e}")) for k, (a, b) in err["E_terms"].items()})
    ctx.close()

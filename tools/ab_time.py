"""Same-box A/B of two libcph.so builds (CPH_LIB=path selects one): ms/step over 300 steps after
30 warm-up steps, plus the pair-kernel and list-build class times, for C2 x 17 and C4 x 21.
usage: CPH_LIB=abtest/base.so python tools/ab_time.py base"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "cur"
for cfg, R in ((2, 17), (4, 21)):
    s = make_system(cfg)
    ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid), R), replica_seeds(cfg, R),
                         vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    ctx.cph_step(30)
    ctx.cph_sync()
    t0 = time.perf_counter()
    ctx.cph_step(300)
    ctx.cph_sync()
    ms = (time.perf_counter() - t0) / 300 * 1e3
    prof, _ = ctx.cph_profile_steps(20)
    print(f"{tag} C{cfg}x{R}: {ms:.4f} ms/step  nonbonded {prof['nonbonded'] / 20:.4f}  pairlist {prof['pairlist'] / 20:.4f}"
          f"  integrate {prof['integrate'] / 20:.4f}", flush=True)
    ctx.close()

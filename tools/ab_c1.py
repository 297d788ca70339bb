"""C1 x 64 / C1 x 256 ms per step (300 steps) for the A/B of the small-grid PME variants."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds  # noqa: E402

s = make_system(1)
for R in (64, 256):
    ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid), R), replica_seeds(1, R),
                         vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    ctx.cph_step(30)
    ctx.cph_sync()
    t0 = time.perf_counter()
    ctx.cph_step(300)
    ctx.cph_sync()
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'cur'} C1x{R}: {(time.perf_counter() - t0) / 300 * 1e3:.4f} ms/step", flush=True)
    ctx.close()

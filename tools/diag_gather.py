"""Brick-staged gather vs the global-load gather (CPH_GATHER=brick selects the brick kernel): forces after create and
after 15 steps must be bit-identical; per-class kernel times from cph_profile_steps.
usage: diag_gather.py {brick|global} out.npz  (then compare two files with: diag_gather.py cmp a b)"""
import os
import sys

import numpy as np

if sys.argv[1] == "brick":
    os.environ["CPH_GATHER"] = "brick"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        same = np.array_equal(a[k], b[k])
        print(k, "identical" if same else f"DIFFER max {np.max(np.abs(a[k] - b[k])):.3e}")
    sys.exit(0)

import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds, small_system  # noqa: E402

out = {}
for name, s, R in (("tiny", small_system(), 2), ("C1", make_system(1), 4), ("C2", make_system(2), 17),
                   ("C4", make_system(4), 21), ("C5", make_system(5), 8)):
    ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid if len(s.pH_grid) else (4.4,)), R), replica_seeds(7, R),
                         vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]))
    out[name + "_f0"] = ctx.cph_get_forces(R - 1)[0]
    ctx.cph_step(15)
    out[name + "_f15"] = ctx.cph_get_forces(R - 1)[0]
    out[name + "_lam"] = ctx.cph_get_lambdas(R - 1)[0]
    ms, cnt = ctx.cph_profile_steps(20)
    print(f"{name} x{R} {sys.argv[1]}: gather {ms['gather'] / 20:.4f} ms/step, spread {ms['spread'] / 20:.4f}, "
          f"nonbonded {ms['nonbonded'] / 20:.4f}", flush=True)
    ctx.close()
np.savez(sys.argv[2], **out)

"""Small driver for ncu captures: C2 workload (17 replicas), warm up, then a few steps."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds  # noqa: E402

cfg = int(os.environ.get("CPH_CFG", "2"))
R = int(os.environ.get("CPH_R", "17"))
s = make_system(cfg)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid), R), replica_seeds(cfg, R),
                     vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]), cuda_stream=st.cuda_stream)
ctx.cph_step(int(os.environ.get("CPH_STEPS", "20")))
ctx.cph_sync()
print("ok", ctx.cph_current_step())

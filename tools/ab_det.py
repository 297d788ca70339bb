"""Step time of the default (fp32-atomic) vs deterministic (fixed-point) PME spread, C4 x 21."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds  # noqa: E402

s = make_system(4)
R = 21
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for det in (0, 1, 0, 1):
    ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid), R), replica_seeds(4, R), deterministic=det,
                         vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]), cuda_stream=st.cuda_stream)
    ctx.cph_step(20)
    ctx.cph_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.cph_step(200)
    e1.record(st)
    torch.cuda.synchronize()
    prof, cnt = ctx.cph_profile_steps(20)
    print(f"deterministic={det}: {e0.elapsed_time(e1) / 200:.4f} ms/step, spread class {prof['spread'] / 20 * 1e3:.1f} us/step")
    ctx.close()

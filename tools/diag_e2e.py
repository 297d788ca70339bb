"""Diagnostic: time the phases of the bench's e2e loop (set_state_all / step / get_state_all)."""
import time
import numpy as np
import torch
import paper_2410_01626_b200 as cph
from synthetic.systems import make_system, make_velocities, replica_seeds

s = make_system(2)
R = 17
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = cph.cph_create(s, np.resize(np.asarray(s.pH_grid), R), replica_seeds(2, R),
                     vel_replicas=np.stack([make_velocities(s, r) for r in range(R)]), cuda_stream=st.cuda_stream)
ctx.cph_step(20)
blob = ctx.cph_get_state_all()
pin_in = torch.from_numpy(blob.copy()).pin_memory().numpy()
pin_out = torch.empty(blob.size, dtype=torch.uint8).pin_memory().numpy()
for it in range(3):
    t0 = time.perf_counter(); ctx.cph_set_state_all(pin_in); ctx.cph_sync(); t1 = time.perf_counter()
    ctx.cph_step(1); ctx.cph_sync(); t2 = time.perf_counter()
    ctx.cph_get_state_all(pin_out); t3 = time.perf_counter()
    print(f"set_state_all {1e3*(t1-t0):.2f} ms  step {1e3*(t2-t1):.2f} ms  get_state_all {1e3*(t3-t2):.2f} ms  blob {blob.size/1e6:.2f} MB")

"""ms/step of one context as a function of cph_params.sub_batches (replica sub-batches stepped
concurrently), per BASELINE operating point.  Usage: python tools/ab_subbatch.py [cfg:R ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds  # noqa: E402

K = int(os.environ.get("CPH_AB_STEPS", "200"))
points = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(4, 21), (2, 17), (2, 34), (1, 64), (3, 16),
                                                                         (5, 8), (4, 8)]


def time_ctx(s, pH, seeds, vel, S):
    st = torch.cuda.Stream()
    ctx = cph.cph_create(s, pH, seeds, vel_replicas=vel, cuda_stream=st.cuda_stream, sub_batches=S)
    ctx.cph_step(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.cph_step(K)
    e1.record(st)
    torch.cuda.synchronize()
    ctx.close()
    return e0.elapsed_time(e1) / K


for cfg, R in points:
    s = make_system(cfg)
    pH = np.resize(np.asarray(s.pH_grid), R)
    seeds = replica_seeds(cfg, R)
    vel = np.stack([make_velocities(s, r) for r in range(R)])
    res = {}
    for rep in range(2):
        for S in (1, 2, 3, 4):
            if S > R:
                continue
            res.setdefault(S, []).append(time_ctx(s, pH, seeds, vel, S))
    line = "  ".join(f"S={S}: {min(v):.4f}" for S, v in res.items())
    print(f"C{cfg} x {R}: ms/step  {line}", flush=True)

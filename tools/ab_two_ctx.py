"""Throughput of one context with R replicas vs two half contexts stepping concurrently on two
streams (the PME tail of one batch under the other batch's pair kernel), C4."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_01626_b200 as cph  # noqa: E402
from synthetic.systems import make_system, make_velocities, replica_seeds  # noqa: E402

cfg = int(os.environ.get("CPH_CFG", "4"))
R = int(os.environ.get("CPH_R", "21"))
K = 200
s = make_system(cfg)
pH = np.resize(np.asarray(s.pH_grid), R)
seeds = replica_seeds(cfg, R)
vel = np.stack([make_velocities(s, r) for r in range(R)])


def run(parts):
    streams = [torch.cuda.Stream() for _ in parts]
    ctxs = []
    for (a, b), st in zip(parts, streams):
        ctxs.append(cph.cph_create(s, pH[a:b], seeds[a:b], vel_replicas=vel[a:b], cuda_stream=st.cuda_stream))
    for c in ctxs:
        c.cph_step(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for st in streams:
        st.wait_event(e0)
    for c in ctxs:
        c.cph_step(K)
    for st in streams:
        ev = torch.cuda.Event()
        ev.record(st)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    for c in ctxs:
        c.close()
    return ms


for _ in range(2):
    one = run([(0, R)])
    two = run([(0, R // 2 + R % 2), (R // 2 + R % 2, R)])
    print(f"C{cfg} R={R}: one context {one:.4f} ms/step, two half contexts concurrently {two:.4f} ms/step")

"""Host side of multi-GPU pH replica exchange (paper_2410_01626_b200.remd) on CPU: two gloo
ranks whose ladder spans both, with a stand-in context whose energies and decisions come
from the oracle, must reach exactly the labels of a single-process run (the all-gather
layout and the attempt sequence are the host logic under test; the device kernels are
covered by tests/test_gpu_remd.py)."""
import os
import socket

import numpy as np
import torch
import torch.multiprocessing as mp

from oracle import remd as OR
from paper_2410_01626_b200 import remd as RE

P, R_PER_RANK, KT, SEED = 4, 2, 2.494, 1234


def _energy(g, p):
    return float(np.sin(1.7 * g + 0.9 * p) * 3.0 + 0.4 * g * p)


class FakeCtx:
    """Oracle-backed stand-in with the Context exchange interface (CPU tensors)."""

    def __init__(self, first, R):
        self.R, self.P, self.first = R, P, first
        self.labels = np.array([(first + r) % P for r in range(R)])
        self.steps = 0

    def cph_step(self, n):
        self.steps += n

    def exchange_device(self):
        return torch.device("cpu")

    def exchange_energies_into(self, t):
        rows = np.zeros((self.R, P + 1))
        for r in range(self.R):
            rows[r, 0] = self.labels[r]
            rows[r, 1:] = [_energy(self.first + r, p) for p in range(P)]
        t.copy_(torch.from_numpy(rows.reshape(-1)))

    def exchange_apply_from(self, t, seed, attempt):
        rows = t.numpy().reshape(-1, P + 1)
        new, _ = OR.decide(rows[:, 1:], rows[:, 0].astype(int), P, KT, seed, attempt)
        self.labels = new[self.first:self.first + self.R]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = FakeCtx(rank * R_PER_RANK, R_PER_RANK)
    nxt = RE.run(ctx, 250, 10, SEED)
    out[rank] = (ctx.labels.tolist(), nxt, ctx.steps)
    dist.destroy_process_group()


def test_exchange_over_two_gloo_ranks_matches_single_process():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    single = FakeCtx(0, 2 * R_PER_RANK)
    nxt = RE.run(single, 250, 10, SEED)
    assert out[0][1] == out[1][1] == nxt == 25 and out[0][2] == 250
    assert out[0][0] + out[1][0] == single.labels.tolist()
    assert sorted(single.labels.tolist()) == list(range(P))
    assert single.labels.tolist() != list(range(P))           # some swaps happened

"""Electrostatics-off lambda dynamics: many independent single-site replicas advanced by
the same BAOAB + Philox + bias + PFC as oracle.engine, vectorised over replicas.
Used for the closed-form pins of §8(c) P7/P9 (Henderson-Hasselbalch populations,
equipartition).  Step order and noise streams are identical to OracleReplica.step
for a system whose only force on lambda is the bias."""
import math

import numpy as np

from . import bias as B
from .philox import philox4x32
from .units import kT


def _normals_per_replica(seeds, step, stream, coord=0):
    M = len(seeds)
    ctr = np.zeros((M, 4), dtype=np.uint64)
    ctr[:, 0] = np.uint64(step)
    ctr[:, 1] = np.uint64(coord)
    ctr[:, 2] = np.uint64(stream)
    key = np.stack([seeds & np.uint64(0xFFFFFFFF), seeds >> np.uint64(32)], -1)
    x = philox4x32(ctr, key).astype(np.float64)
    u = (x + 0.5) * 2.0 ** -32
    return np.sqrt(-2.0 * np.log(u[:, 0])) * np.cos(2.0 * math.pi * u[:, 1])


def run_2state(seeds, lam0, pKa, pH, n_steps, h_barrier=6.0, d1=0.0, T=300.0, kw=1e6,
               dt=0.002, gamma=1.0, mass=60.0, record_every=10, vmm=None):
    seeds = np.asarray(seeds, dtype=np.uint64)
    M = len(seeds)
    lam = np.asarray(lam0, np.float64).copy()
    vel = np.zeros(M)
    kt = kT(T)
    c1 = math.exp(-gamma * dt)
    sd = math.sqrt((1 - c1 * c1) * kt / mass)
    vdw = lambda l: B.vdw(l, h_barrier, 0.0, d1, kw)[1]
    g = B.delta_g(np.asarray(pKa, np.float64), np.asarray(pH, np.float64), T)   # scalar or per replica
    d1 = np.asarray(d1, np.float64)

    def force(l):
        f = -(vdw(l) + g)
        if vmm is not None:
            f = f - B.vmm(vmm, l, 0.0)[1]
        return f
    F = force(lam)
    frames = []
    vframes = []
    for n in range(n_steps):
        xi = _normals_per_replica(seeds, n, 1)
        vel = vel + 0.5 * dt * F / mass
        lam = lam + 0.5 * dt * vel
        vel = c1 * vel + sd * xi
        lam = lam + 0.5 * dt * vel
        F = force(lam)
        vel = vel + 0.5 * dt * F / mass
        if (n + 1) % record_every == 0:
            frames.append(lam.copy())
            vframes.append(vel.copy())
    return np.array(frames), np.array(vframes)

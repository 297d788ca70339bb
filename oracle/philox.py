"""Philox4x32-10 counter-based RNG (Salmon et al., SC'11 / Random123) and Box-Muller,
plain numpy (reading R17: the noise of the BAOAB O-step, PAPER.md:902-907
names a stochastic thermostat).

Stream layout (both sides implement it independently):
  key  = (seed & 0xffffffff, seed >> 32)           seed = 64-bit replica seed
  atom noise      ctr = (step, atom_index, 0, 0)   -> normals z0, z1, z2 for x, y, z
  lambda noise    ctr = (step, coord_index, 1, 0)  -> normal z0
uniform u_k = (x_k + 0.5) * 2^-32 ; Box-Muller
  z0 = sqrt(-2 ln u0) cos(2 pi u1), z1 = sqrt(-2 ln u0) sin(2 pi u1), z2/z3 from (u2, u3).
Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt).
"""
import math

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
_MASK = 0xFFFFFFFF


def philox4x32(ctr, key, rounds=10):
    """ctr: (..., 4) uint64-valued array of 32-bit words; key: (..., 2). Returns (..., 4)."""
    c = [np.asarray(ctr[..., i], dtype=np.uint64) for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint64)
    k1 = np.asarray(key[..., 1], dtype=np.uint64)
    for r in range(rounds):
        if r > 0:
            k0 = (k0 + np.uint64(W0)) & np.uint64(_MASK)
            k1 = (k1 + np.uint64(W1)) & np.uint64(_MASK)
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(_MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(_MASK)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return np.stack(c, -1)


def _key(seed):
    seed = int(seed)
    return np.array([seed & _MASK, (seed >> 32) & _MASK], dtype=np.uint64)


def normals(seed, step, index, stream):
    """4 standard normals per index: array (len(index), 4)."""
    index = np.asarray(index, dtype=np.uint64)
    ctr = np.zeros((len(index), 4), dtype=np.uint64)
    ctr[:, 0] = np.uint64(step & _MASK)
    ctr[:, 1] = index
    ctr[:, 2] = np.uint64(stream)
    key = np.broadcast_to(_key(seed), (len(index), 2))
    x = philox4x32(ctr, key).astype(np.float64)
    u = (x + 0.5) * 2.0 ** -32
    r0 = np.sqrt(-2.0 * np.log(u[:, 0]))
    r1 = np.sqrt(-2.0 * np.log(u[:, 2]))
    t0 = 2.0 * math.pi * u[:, 1]
    t1 = 2.0 * math.pi * u[:, 3]
    return np.stack([r0 * np.cos(t0), r0 * np.sin(t0), r1 * np.cos(t1), r1 * np.sin(t1)], -1)

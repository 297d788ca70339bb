"""Dynamic Barrier and Well Optimization (DBO) and censoring.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): written from the paper, shares no code
with the CUDA path.

Well algorithm: per coordinate, in blocks of 40 ps, count the time with
lambda < 0.2 (near well 0) and lambda > 0.8 (near well 1) and the mean lambda there.  At the
block end, if more than 70 % of the block was spent near one well and |mean - ideal| > 0.03,
the well centre moves by 0.5 (ideal - mean) (reading R23: opposite the observed deviation),
the accumulated shift capped at +-0.08.

Barrier algorithm: per coordinate, in blocks of 1 ns, the fraction of
frames in transition (0.2 < lambda < 0.8); below 25 % - 5 % the barrier drops by 1 kJ/mol,
above 25 % + 5 % it rises by 1 kJ/mol, kept within [1, 20] kJ/mol, start 6 kJ/mol.  The
tautomer coordinate has two barriers keyed by the protonation of the site (lambda_p < 0.5:
protonated), each regulated on the frames of its own state (reading R25).

Censoring: after an adjustment of a site at the end of step S, its
frames at steps S < t <= S + 10 ps are tagged (reading R26).

Statistics are taken every step (reading R24: "time spent" = steps).
"""
import numpy as np

WELL_NEAR = 0.2          # lambda < 0.2 near well 0, lambda > 1 - 0.2 near well 1
RESIDENCY = 0.70
WELL_TOL = 0.03
WELL_GAIN = 0.5
WELL_CAP = 0.08
TRANS_LO, TRANS_HI = 0.2, 0.8
TRANS_TARGET = 0.25
TRANS_TOL = 0.05
BARRIER_STEP = 1.0
BARRIER_MIN, BARRIER_MAX = 1.0, 20.0

# event kinds (same numbering as the library's event log)
WELL0, WELL1, BARRIER, BARRIER_T_PROT, BARRIER_T_DEPROT = 0, 1, 2, 3, 4


def well_block_decide(shift, n, n_near, sum_near, ideal):
    """New lateral shift of one well (ideal 0 or 1) from one block's statistics.

    shift: current accumulated shift of the well centre; n: steps in the block; n_near,
    sum_near: steps near this well and the sum of lambda over them."""
    if n <= 0 or n_near <= 0 or not (n_near / n > RESIDENCY):
        return shift
    diff = ideal - sum_near / n_near
    if not (abs(diff) > WELL_TOL):
        return shift
    return float(np.clip(shift + WELL_GAIN * diff, -WELL_CAP, WELL_CAP))


def barrier_block_decide(h, n_frames, n_trans):
    """New barrier height from one block's in-transition fraction (no frames: unchanged)."""
    if n_frames <= 0:
        return h
    frac = n_trans / n_frames
    if frac < TRANS_TARGET - TRANS_TOL:
        return max(BARRIER_MIN, h - BARRIER_STEP)
    if frac > TRANS_TARGET + TRANS_TOL:
        return min(BARRIER_MAX, h + BARRIER_STEP)
    return h


class BlockStats:
    """Per-coordinate block accumulators of one replica.

    well: [n, n0, s0, n1, s1]; barrier: [n_A, trans_A, n_B, trans_B] where class A is
    'all frames' for lambda_p coordinates and 'protonated' (lambda_p < 0.5) for tautomer
    coordinates, class B 'deprotonated' for tautomer coordinates."""

    def __init__(self, n_coords):
        self.well = np.zeros((n_coords, 5))
        self.barrier = np.zeros((n_coords, 4))

    def add(self, lam, lp_of):
        """lam: lambda after a completed step; lp_of[c]: index of the lambda_p coordinate of
        c's site if c is a tautomer coordinate, else -1."""
        for c, l in enumerate(lam):
            w = self.well[c]
            w[0] += 1
            if l < WELL_NEAR:
                w[1] += 1
                w[2] += l
            elif l > 1.0 - WELL_NEAR:
                w[3] += 1
                w[4] += l
            cls = 0 if lp_of[c] < 0 or lam[lp_of[c]] < 0.5 else 1
            self.barrier[c, 2 * cls] += 1
            self.barrier[c, 2 * cls + 1] += 1 if TRANS_LO < l < TRANS_HI else 0


def well_update(dbo, stats):
    """Apply the well rule to every coordinate; returns events (coord, kind, old, new) and
    updates dbo rows (a0, a1, h_prot, h_deprot) in place."""
    ev = []
    for c in range(len(dbo)):
        n, n0, s0, n1, s1 = stats.well[c]
        a0 = well_block_decide(dbo[c][0], n, n0, s0, 0.0)
        a1 = 1.0 + well_block_decide(dbo[c][1] - 1.0, n, n1, s1, 1.0)
        if a0 != dbo[c][0]:
            ev.append((c, WELL0, dbo[c][0], a0))
            dbo[c][0] = a0
        if a1 != dbo[c][1]:
            ev.append((c, WELL1, dbo[c][1], a1))
            dbo[c][1] = a1
    return ev


def barrier_update(dbo, stats, lp_of):
    ev = []
    for c in range(len(dbo)):
        nA, tA, nB, tB = stats.barrier[c]
        if lp_of[c] < 0:
            h = barrier_block_decide(dbo[c][2], nA, tA)
            if h != dbo[c][2]:
                ev.append((c, BARRIER, dbo[c][2], h))
                dbo[c][2] = dbo[c][3] = h
        else:
            hp = barrier_block_decide(dbo[c][2], nA, tA)
            hd = barrier_block_decide(dbo[c][3], nB, tB)
            if hp != dbo[c][2]:
                ev.append((c, BARRIER_T_PROT, dbo[c][2], hp))
                dbo[c][2] = hp
            if hd != dbo[c][3]:
                ev.append((c, BARRIER_T_DEPROT, dbo[c][3], hd))
                dbo[c][3] = hd
    return ev


def censor_flags(frame_steps, adjust_steps, censor_steps):
    """Boolean per frame: True iff S < t <= S + censor_steps for an adjustment at step S."""
    t = np.asarray(frame_steps)
    out = np.zeros(t.shape, bool)
    for S in adjust_steps:
        out |= (t > S) & (t <= S + censor_steps)
    return out

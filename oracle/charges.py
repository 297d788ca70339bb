"""lambda -> atomic charges.

Eq. 2: H(lp, lt) = (1-lp)[(1-lt) H_A + lt H_B] + lp[(1-lt) H_C + lt H_D].
Only charges differ between forms, and under charge
interpolation (reading R7) each atom's charge carries the same
weights: q_i = sum_s w_s(lp, lt) q_i^s.  2-state sites have A = B and C = D
 so lt drops out; they own one coordinate (lp), 3-state (His)
sites own two (lp, lt).  The buffer oxygen is a member of its site's group with
states (-0.834, -0.834, +0.166, +0.166).
"""
import numpy as np


def eq2_weights(lp, lt):
    """Weights (w_A, w_B, w_C, w_D) of Eq. 2."""
    return ((1.0 - lp) * (1.0 - lt), (1.0 - lp) * lt, lp * (1.0 - lt), lp * lt)


def coord_ptr(group_kind):
    """Offsets of each group's coordinates in the flat lambda vector:
    kind 2 -> [lp], kind 3 -> [lp, lt]."""
    ptr = [0]
    for k in group_kind:
        ptr.append(ptr[-1] + (1 if int(k) == 2 else 2))
    return np.array(ptr, dtype=np.int64)


def group_lambdas(group_kind, lam):
    """(lp, lt) per group; lt = 0 for 2-state groups (value irrelevant there)."""
    cp = coord_ptr(group_kind)
    lp = np.array([lam[cp[g]] for g in range(len(group_kind))], dtype=np.float64)
    lt = np.array([lam[cp[g] + 1] if int(group_kind[g]) == 3 else 0.0
                   for g in range(len(group_kind))], dtype=np.float64)
    return lp, lt


def charges(sys, lam):
    """Full charge vector q(lambda) (float64) and dq/dlambda for every lambda atom.

    Returns q (N,), dq (n_lambda, 2) with columns d/dlp, d/dlt:
      dq/dlp = (1-lt)(q^C - q^A) + lt (q^D - q^B)
      dq/dlt = (1-lp)(q^B - q^A) + lp (q^D - q^C)   (derivatives of Eq. 2 weights)
    """
    q = sys.charge.astype(np.float64).copy()
    lp, lt = group_lambdas(sys.group_kind, lam)
    dq = np.zeros((len(sys.group_atoms), 2))
    for g in range(len(sys.group_kind)):
        for k in range(sys.group_ptr[g], sys.group_ptr[g + 1]):
            qa, qb, qc, qd = sys.state_q[k]
            w = eq2_weights(lp[g], lt[g])
            q[sys.group_atoms[k]] = w[0] * qa + w[1] * qb + w[2] * qc + w[3] * qd
            dq[k, 0] = (1.0 - lt[g]) * (qc - qa) + lt[g] * (qd - qb)
            dq[k, 1] = (1.0 - lp[g]) * (qb - qa) + lp[g] * (qd - qc)
    return q, dq

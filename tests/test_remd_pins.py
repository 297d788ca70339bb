"""Pins of the pH replica-exchange oracle (oracle.remd): the alternating neighbour pairs,
the Metropolis acceptance probability, and detailed balance of the label chain (the
stationary distribution over label permutations is Boltzmann in sum_g E[g, label_g])."""
import itertools
import math

import numpy as np

from oracle import remd

KT = 2.494


def test_alternating_pairs():
    assert remd.pairs(0, 6) == [0, 2, 4] and remd.pairs(1, 6) == [1, 3]
    assert remd.pairs(0, 2) == [0] and remd.pairs(1, 2) == []
    assert remd.pairs(3, 1) == []


def test_metropolis_acceptance_probability():
    E = np.array([[0.0, math.log(4.0) * KT], [0.0, 0.0]])   # swap costs Delta = ln 4 kT
    acc = [remd.decide(E, [0, 1], 2, KT, 99, 2 * k)[1][0][2] for k in range(6000)]
    assert abs(np.mean(acc) - 0.25) < 4 * math.sqrt(0.25 * 0.75 / 6000)
    # downhill swaps are always accepted
    E2 = np.array([[0.0, -1.0], [0.0, 0.0]])
    assert all(remd.decide(E2, [0, 1], 2, KT, 99, 2 * k)[1][0][2] for k in range(50))


def test_label_chain_detailed_balance():
    """Two ladders of P = 3: the empirical distribution of label permutations matches
    exp(-sum_g E[g, label_g] / kT) (a sign or index error in Delta breaks it), and the
    ladders evolve independently."""
    rng = np.random.default_rng(4)
    P = 3
    E = rng.normal(0.0, 0.6 * KT, (2 * P, P))
    labels = np.array([0, 1, 2, 2, 0, 1])
    counts = [dict(), dict()]
    n = 12000
    for k in range(n):
        labels, _ = remd.decide(E, labels, P, KT, 7, k)
        for l in range(2):
            key = tuple(labels[l * P:(l + 1) * P])
            counts[l][key] = counts[l].get(key, 0) + 1
    for l in range(2):
        perms = list(itertools.permutations(range(P)))
        w = np.array([math.exp(-sum(E[l * P + g, pp[g]] for g in range(P)) / KT) for pp in perms])
        w /= w.sum()
        emp = np.array([counts[l].get(pp, 0) / n for pp in perms])
        print(l, np.round(w, 3), np.round(emp, 3))
        assert np.max(np.abs(emp - w)) < 0.02

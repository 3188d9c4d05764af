"""Brute-force pins of the oracle's decision, G and correctness (CPU).

* Decision: for C <= 12 every subset of labels is made the API output (all 2^C
  subsets), with tie-heavy confidences and random, overlapping lists.  The
  oracle's literal sort-and-scan must equal the
  independent arg-max characterisation: the first mapped label in confidence
  order is the lexicographic max of (z, -c) over mapped labels, if it is above
  the threshold.
* Correctness (Eq. goal; reading A7): Decision(ŷ) is the set of
  branches the application reaches when the API returns exactly the
  ground-truth labels, over every order of them; the oracle's G / correct must
  agree with that enumeration for every GT subset of small label spaces.
"""
import itertools

import numpy as np

from oracle import Oracle


def random_lists(rng, C, max_lists=4, overlap=True):
    D = int(rng.integers(0, max_lists + 1))
    lists = []
    pool = list(range(C))
    for _ in range(D):
        n = int(rng.integers(0, min(C, 5) + 1))
        if overlap:
            lists.append(sorted(set(rng.choice(C, size=n, replace=True).tolist())) if n else [])
        else:
            rng.shuffle(pool)
            lists.append(sorted(pool[:n]))
            pool = pool[n:]
    return lists


def first_list(lists, c):
    for j, W in enumerate(lists):
        if c in W:
            return j
    return -1


def argmax_form(lists, z, tau):
    best = None
    for c in range(len(z)):
        if first_list(lists, c) < 0:
            continue
        if best is None or z[c] > z[best]:  # ascending c: strict > keeps the smaller id on ties
            best = c
    if best is None or not z[best] > tau:
        return len(lists)
    return first_list(lists, best)


def test_decision_all_subsets_C_le_12():
    rng = np.random.default_rng(10)
    tau = 0.0
    n_cases = 0
    for C in (1, 2, 3, 5, 8, 12):
        for rep in range(3 if C == 12 else 6):
            lists = random_lists(rng, C, overlap=bool(rep % 2))
            orc = Oracle(C, [lists], tau=tau)
            levels = rng.integers(1, 4, size=C).astype(np.float64)  # few levels -> many ties
            below = rng.choice([-1.0, 0.0], size=C)                  # 0.0 == tau is NOT output
            for s in range(1 << C):
                z = np.where([(s >> c) & 1 for c in range(C)], levels, below)
                assert orc.decide(z) == argmax_form(lists, z, tau), (C, lists, z)
                n_cases += 1
    assert n_cases > 4096 * 3


def app_decision(lists, outputs):
    """Generic form of the listing: walk outputs, lists in code order."""
    for c in outputs:
        for j, W in enumerate(lists):
            if c in W:
                return j
    return len(lists)


def test_gt_set_and_correctness_by_enumeration():
    rng = np.random.default_rng(11)
    for C in (3, 5, 7):
        for rep in range(8):
            lists = random_lists(rng, C, overlap=bool(rep % 2))
            orc = Oracle(C, [lists])
            D = len(lists)
            for s in range(1 << C):
                gt = [c for c in range(C) if (s >> c) & 1]
                if len(gt) > 4:
                    continue
                reachable = {app_decision(lists, order) for order in itertools.permutations(gt)}
                G = orc.gt_set(gt)
                for d in range(D + 1):
                    assert orc.correct(G, d) == (d in reachable), (lists, gt, d)


def test_decision_invariant_under_label_permutation():
    """Relabelling the label ids consistently (lists and logits) leaves the decision unchanged
    when confidences are distinct."""
    rng = np.random.default_rng(12)
    for trial in range(300):
        C = int(rng.integers(2, 30))
        lists = random_lists(rng, C, overlap=False)
        z = rng.permutation(C).astype(np.float64) - C / 2 + 0.5  # distinct
        p = rng.permutation(C)
        lists_p = [[int(p[c]) for c in W] for W in lists]
        zp = np.empty(C)
        zp[p] = z
        assert Oracle(C, [lists]).decide(z) == Oracle(C, [lists_p]).decide(zp)

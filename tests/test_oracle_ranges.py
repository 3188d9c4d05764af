"""Pins of the value-ranges oracle, CPU.

* The decision is the application's if-chain over its ranges, run verbatim here.
* k -> inf: the loss is 1 exactly when the score lies outside the ground-truth range
  ("the penalty ... will be low only when the API output score lies in the ground-truth
  value ranges"), 0 inside (away from the bounds).
* Finite differences of dL/dO; weights M/N_r reduce to inverse range frequency.
"""
import numpy as np
import pytest

from oracle import RangesOracle

# e.g. a sentiment application: negative / neutral / positive
LO, HI = [-1.0, -0.25, 0.25], [-0.25, 0.25, 1.0]


def app(score):
    """if -1.0 <= s <= -0.25: return 'negative' ... (code order), else default."""
    if LO[0] <= score <= HI[0]:
        return 0
    if LO[1] <= score <= HI[1]:
        return 1
    if LO[2] <= score <= HI[2]:
        return 2
    return 3


def test_range_decision_is_the_program():
    orc = RangesOracle(LO, HI)
    rng = np.random.default_rng(60)
    for s in list(rng.uniform(-1.5, 1.5, 3000)) + [-1.0, -0.25, 0.25, 1.0, 1.0001, -1.0001]:
        assert orc.range_of(s) == app(s)


def test_range_step_limit():
    orc = RangesOracle(LO, HI, k=1e7)
    rng = np.random.default_rng(61)
    for trial in range(3000):
        s, t = rng.uniform(-1.2, 1.2, 2)
        r = orc.range_of(t)
        if r == 3 or min(abs(s - b) for b in LO + HI) < 1e-4:
            continue
        L, _ = orc.loss(r, s)
        assert L == pytest.approx(float(orc.range_of(s) != r), abs=1e-6)


def test_range_gradient_fd():
    rng = np.random.default_rng(62)
    for trial in range(500):
        orc = RangesOracle(LO, HI, k=float(rng.choice([1.0, 10.0])))
        s = rng.uniform(-1.2, 1.2)
        r = int(rng.integers(0, 3))
        w = rng.uniform(0.5, 2)
        h = 1e-6
        L1, _ = orc.loss(r, s + h, w)
        L0, _ = orc.loss(r, s - h, w)
        _, dL = orc.loss(r, s, w)
        assert (L1 - L0) / (2 * h) == pytest.approx(dL, rel=1e-6, abs=1e-9)
    assert RangesOracle(LO, HI).loss(3, 0.0) == (0.0, 0.0)  # no target range


def test_range_weights_inverse_frequency():
    orc = RangesOracle(LO, HI)
    rng = np.random.default_rng(63)
    gt = rng.uniform(-1.3, 1.3, 1000).astype(np.float32)
    r = orc.eval(np.zeros(1000, np.float32), gt)
    H = r["hist_gt"]
    w = orc.weights(H)
    for b in range(4):
        assert w[b] == pytest.approx(1000 / H[b]) if H[b] else w[b] == 0

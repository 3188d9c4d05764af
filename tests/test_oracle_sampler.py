"""Pins of the rebalanced sampler (reading A24), CPU.

* Exact law: the measure of uniforms (u1, u2) mapped to each row equals q_i = w_i / Σw —
  checked on a fine grid of u1 x u2 against the closed form.
* Balance: with one list and w = M/N_1, M/(M-N_1), target and non-target
  inputs each receive exactly half of the probability mass; with disjoint singleton classes
  every class receives the same mass.
* Monte-Carlo frequencies within 5 sigma of q_i.
"""
import numpy as np
import pytest

import oracle
from oracle import Oracle


def q_of(mask, w):
    wi = np.asarray(w, dtype=np.float32).astype(np.float64)[mask]
    return wi / wi.sum()


def test_exact_law_on_grid():
    rng = np.random.default_rng(70)
    rows = 37
    mask = rng.choice([0, 1, 2, 5], size=rows).astype(np.uint8)
    w = np.zeros(256)
    w[[0, 1, 2, 5]] = [1.5, 4.0, 0.25, 3.0]
    g = 2000
    u1 = (np.arange(g) + 0.5) / g
    u2 = (np.arange(g) + 0.5) / g
    U1, U2 = np.meshgrid(u1, u2, indexing="ij")
    idx = oracle.sample(mask, w, U1.ravel(), U2.ravel())
    freq = np.bincount(idx, minlength=rows) / idx.size
    np.testing.assert_allclose(freq, q_of(mask, w), atol=2.0 / g)


def test_balance_true_false_and_singletons():
    rng = np.random.default_rng(71)
    C = 20
    orc = Oracle(C, [[[1, 2, 3]]])
    M = 501
    n = rng.integers(1, 4, size=M)
    off = np.zeros(M + 1, dtype=np.int64)
    off[1:] = np.cumsum(n)
    lab = rng.integers(0, C, size=int(off[-1])).astype(np.int32)
    r = orc.eval(np.zeros((M, C), np.float32), off, lab, want_loss=False)
    w = Oracle.weights_by_mask(r["hist_gt"])[0].astype(np.float32)
    q = q_of(r["gt_mask"], w)
    assert q[r["gt_mask"] == 1].sum() == pytest.approx(0.5, abs=1e-6)
    # disjoint singleton classes: equal mass per class
    orc = Oracle(6, [[[0], [1], [2], [3]]])
    cls = rng.integers(0, 6, size=M)
    r = orc.eval(np.zeros((M, 6), np.float32), np.arange(M + 1, dtype=np.int64), cls.astype(np.int32), want_loss=False)
    w = Oracle.weights_by_mask(r["hist_gt"])[0].astype(np.float32)
    q = q_of(r["gt_mask"], w)
    masses = [q[r["gt_mask"] == m].sum() for m in sorted(set(r["gt_mask"].tolist()))]
    np.testing.assert_allclose(masses, 1.0 / len(masses), atol=1e-6)


def test_monte_carlo_frequencies():
    rng = np.random.default_rng(72)
    rows = 60
    mask = rng.integers(0, 8, size=rows).astype(np.uint8)
    w = np.zeros(256)
    w[:8] = rng.uniform(0.1, 5.0, 8)
    n = 400000
    idx = oracle.sample(mask, w, rng.random(n), rng.random(n))
    q = q_of(mask, w)
    freq = np.bincount(idx, minlength=rows) / n
    sigma = np.sqrt(q * (1 - q) / n)
    assert np.all(np.abs(freq - q) <= 5 * sigma + 1e-12)


def test_zero_weight_masks_never_drawn():
    mask = np.array([0, 1, 1, 2, 0], dtype=np.uint8)
    w = np.zeros(256)
    w[1] = 2.0
    idx = oracle.sample(mask, w, np.linspace(0, 0.999, 50), np.linspace(0, 0.999, 50))
    assert set(idx.tolist()) <= {1, 2}
    with pytest.raises(ValueError):
        oracle.sample(mask, np.zeros(256), [0.5], [0.5])

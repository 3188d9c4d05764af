"""Pins of the rebalancing weights M/N_i, CPU.

* O(M^2) literal recount of N_i over the inputs vs the per-mask evaluation the
  oracle uses at full size (rows with equal G_i have equal N_i).
* True-False special case (Eq. loss): one list gives weights
  M/N_1 for target inputs and M/(M - N_1) for the others, N_1 counted straight
  from the ground-truth labels.
* Disjoint single-class ground truths reduce to textbook inverse class frequency.
"""
import numpy as np
import pytest

from oracle import Oracle


def rand_gt(rng, M, C, max_n=4):
    n = rng.integers(0, max_n + 1, size=M)
    off = np.zeros(M + 1, dtype=np.int64)
    off[1:] = np.cumsum(n)
    lab = rng.integers(0, C, size=int(off[-1])).astype(np.int32)
    return off, lab


def mask_hist(orc, off, lab):
    H = np.zeros(256, dtype=np.uint64)
    G = []
    for i in range(len(off) - 1):
        g = orc.gt_set(lab[off[i]:off[i + 1]])
        G.append(g)
        H[g] += 1
    return H, G


def test_literal_vs_by_mask():
    rng = np.random.default_rng(30)
    for trial in range(40):
        C = int(rng.integers(4, 30))
        D = int(rng.integers(1, 9))
        lists = [sorted(set(rng.integers(0, C, size=int(rng.integers(1, 5))).tolist())) for _ in range(D)]
        orc = Oracle(C, [lists])
        M = int(rng.integers(1, 250))
        off, lab = rand_gt(rng, M, C)
        w_lit = orc.weights_literal(off, lab)
        H, G = mask_hist(orc, off, lab)
        w_mask = Oracle.weights_by_mask(H)[0]
        np.testing.assert_allclose(w_lit, w_mask[G], rtol=1e-15)
        assert np.all(w_lit >= 1.0)


def test_true_false_weights():
    rng = np.random.default_rng(31)
    for trial in range(30):
        C = int(rng.integers(3, 40))
        W1 = sorted(set(rng.integers(0, C, size=int(rng.integers(1, C))).tolist()))
        orc = Oracle(C, [[W1]])
        M = int(rng.integers(2, 200))
        off, lab = rand_gt(rng, M, C)
        target = [bool(set(lab[off[i]:off[i + 1]].tolist()) & set(W1)) for i in range(M)]
        N1 = sum(target)
        w = orc.weights_literal(off, lab)
        for i in range(M):
            want = M / N1 if target[i] else M / (M - N1)
            assert w[i] == pytest.approx(want, rel=1e-15)


def test_inverse_class_frequency():
    rng = np.random.default_rng(32)
    lists = [[0], [1], [2], [3]]
    orc = Oracle(6, [lists])
    M = 500
    cls = rng.integers(0, 6, size=M)  # 4, 5 are unmapped -> non-target class
    off = np.arange(M + 1, dtype=np.int64)
    lab = cls.astype(np.int32)
    w = orc.weights_literal(off, lab)
    for i in range(M):
        c = cls[i]
        count = np.sum(cls == c) if c < 4 else np.sum(cls >= 4)
        assert w[i] == pytest.approx(M / count, rel=1e-15)


def test_absent_mask_weight_zero():
    H = np.zeros(256, dtype=np.uint64)
    H[0], H[1] = 10, 5
    w = Oracle.weights_by_mask(H)[0]
    assert w[0] == pytest.approx(15 / 10) and w[1] == pytest.approx(15 / 5)
    assert w[2] == 0.0          # no input touches class 1 alone -> N = 0 -> w = 0 (reading A13)
    assert w[3] == pytest.approx(15 / 5)  # {0,1} intersects the five {0} inputs


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_gt_hist_pass_agrees_with_full_pass(cfg):
    """orc_gt_hist (ground truth only, used to build the full-size tests' weights) gives the
    same G_i and mask histogram as the full pass, for every decision pattern."""
    import synth
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg)
    b = wl.host_batch(1234, 600)
    g = wl.host_gt(1234, 600)
    for k in ("gt_off", "gt_lab", "app"):
        np.testing.assert_array_equal(b[k], g[k])
    app = b["app"] if spec.n_apps > 1 else None
    for order in (0, 1, 2):
        orc = Oracle.from_spec(spec, order=order)
        r = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=app, want_loss=False)
        gm, H = orc.gt_hist(g["gt_off"], g["gt_lab"], app=app)
        np.testing.assert_array_equal(gm, r["gt_mask"])
        np.testing.assert_array_equal(H, r["hist_gt"])

"""Pins of the oracle's other decision patterns, CPU.

* Multi-Choice, application-choice order: the application checks its
  lists in code order and, for each, the output labels (the loop nesting of
  PAPER.md:2154-2156).  Pinned against that program run verbatim, against the closed
  form "lowest first-list among output labels", and the ground-truth decision's
  independence of the output order.
* Multi-Select: every list with an output label is selected.
  Pinned against the program, and the k -> inf limit of Eq. multi-select equals the
  Hamming distance between the selected and the ground-truth list sets ("only if the
  application decisions ... exactly match ... the penalty will be low").
* True-False: with one list all three patterns reduce to Eq. loss,
  y S(θ − P_1) + (1 − y) S(P_1 − θ) — a different equation from the three it pins.
* Central finite differences of both new losses; literal O(M^2) weights per pattern.
"""
import itertools

import numpy as np
import pytest

from oracle import API_OUTPUT, APP_CHOICE, MULTI_SELECT, Oracle


def random_lists(rng, C, overlap=True, max_lists=6):
    D = int(rng.integers(1, max_lists + 1))
    if overlap:
        return [sorted(set(rng.integers(0, C, size=int(rng.integers(0, 5))).tolist())) for _ in range(D)]
    perm = rng.permutation(C).tolist()
    out = []
    for _ in range(D):
        n = int(rng.integers(0, 4))
        out.append(sorted(perm[:n]))
        perm = perm[n:]
    return out


def app_choice_program(lists, outputs):
    """for W in lists: for obj in outputs: if obj in W: return W  (application-choice order)."""
    for j, W in enumerate(lists):
        for obj in outputs:
            if obj in W:
                return j
    return len(lists)


def multi_select_program(lists, outputs):
    """selected = [W for W in lists if any(obj in W for obj in outputs)]"""
    m = 0
    for j, W in enumerate(lists):
        if any(obj in W for obj in outputs):
            m |= 1 << j
    return m


def api_output(z, tau):
    ids = [c for c in range(len(z)) if z[c] > tau]
    ids.sort(key=lambda c: (-z[c], c))
    return ids


def sig(x):
    return 1.0 / (1.0 + np.exp(-x))


@pytest.mark.parametrize("overlap", [False, True])
def test_app_choice_decision_program_and_closed_form(overlap):
    rng = np.random.default_rng(40)
    for trial in range(1500):
        C = int(rng.integers(1, 14))
        lists = random_lists(rng, C, overlap)
        tau = float(rng.choice([0.0, -0.5]))
        orc = Oracle(C, [lists], tau=tau, order=APP_CHOICE)
        z = rng.integers(-2, 3, size=C).astype(np.float64)
        d = orc.decide(z)
        assert d == app_choice_program(lists, api_output(z, tau))
        firsts = [orc.first_list(c) for c in range(C) if z[c] > tau and orc.first_list(c) >= 0]
        assert d == (min(firsts) if firsts else len(lists))


def test_app_choice_ground_truth_decision_is_order_free():
    rng = np.random.default_rng(41)
    for trial in range(400):
        C = int(rng.integers(2, 10))
        lists = random_lists(rng, C, True)
        orc = Oracle(C, [lists], order=APP_CHOICE)
        gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
        k = orc.gt_decision_app_choice(gt)
        assert {app_choice_program(lists, p) for p in itertools.permutations(gt)} == {k}
        G = orc.gt_mask(gt)
        assert k == (int(G & -G).bit_length() - 1 if G else len(lists))  # lowest list hit = first set bit of G


@pytest.mark.parametrize("overlap", [False, True])
def test_multi_select_decision_program(overlap):
    rng = np.random.default_rng(42)
    for trial in range(1500):
        C = int(rng.integers(1, 14))
        lists = random_lists(rng, C, overlap)
        orc = Oracle(C, [lists], tau=0.0, order=MULTI_SELECT)
        z = rng.integers(-2, 3, size=C).astype(np.float64)
        assert orc.decide(z) == multi_select_program(lists, api_output(z, 0.0))
        gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
        assert orc.gt_set_raw(gt) == multi_select_program(lists, gt)


def tie_free(z, tau, gap=1e-4):
    vals = np.concatenate([sig(z), [sig(tau)]])
    d = np.abs(vals[:, None] - vals[None, :])[np.triu_indices(len(vals), 1)]
    return d.size == 0 or d.min() > gap


def test_multi_select_step_limit_is_hamming_distance():
    rng = np.random.default_rng(43)
    checked = 0
    for trial in range(3000):
        C = int(rng.integers(2, 14))
        lists = random_lists(rng, C, bool(trial % 2))
        tau = float(rng.choice([0.0, 0.7]))
        orc = Oracle(C, [lists], tau=tau, k=1e7, order=MULTI_SELECT)
        z = rng.normal(tau, 3.0, size=C)
        if not tie_free(z, tau):
            continue
        gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
        G = orc.gt_set_raw(gt)
        d = orc.decide(z)
        nonempty = sum(1 << j for j, W in enumerate(lists) if W)
        hamming = bin((d ^ G) & nonempty).count("1")
        assert orc.loss_row(z, G)["ell"] == pytest.approx(hamming, abs=1e-6)
        checked += 1
    assert checked > 1000


def test_app_choice_step_limit():
    """k -> inf: step = 1 implies an incorrect decision; a correct decision has step 0; and
    whenever no higher-priority list is above the threshold the two coincide exactly.
    (Eq. app_choice does not penalise a higher-priority list whose max lies between θ and
    P_k — reading A21; the decision there is incorrect but the step is 0.)"""
    rng = np.random.default_rng(44)
    checked = exact = 0
    for trial in range(4000):
        C = int(rng.integers(2, 14))
        lists = random_lists(rng, C, bool(trial % 2))
        tau = float(rng.choice([0.0, 0.5]))
        orc = Oracle(C, [lists], tau=tau, k=1e7, order=APP_CHOICE)
        z = rng.normal(tau, 3.0, size=C)
        if not tie_free(z, tau):
            continue
        gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
        G = orc.gt_mask(gt)
        d = orc.decide(z)
        correct = orc.is_correct(gt, d)
        step = orc.loss_row(z, G)["ell"]
        assert step == pytest.approx(round(step), abs=1e-6)
        if round(step) == 1:
            assert not correct
        if correct:
            assert round(step) == 0
        k = orc.gt_decision_app_choice(gt)
        higher = [c for c in range(C) if 0 <= orc.first_list(c) < k]
        if G == 0 or not any(z[c] > tau for c in higher):
            assert round(step) == int(not correct)
            exact += 1
        checked += 1
    assert checked > 1000 and exact > 500


def test_true_false_all_patterns_reduce_to_eq_loss():
    rng = np.random.default_rng(45)
    for trial in range(500):
        C = int(rng.integers(2, 20))
        W1 = sorted(set(rng.integers(0, C, size=int(rng.integers(1, C))).tolist()))
        tau = float(rng.choice([0.0, -1.0, 1.0]))
        kk = float(rng.choice([1.0, 10.0]))
        z = rng.normal(0, 2.5, size=C)
        gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
        y = int(bool(set(gt) & set(W1)))
        P1 = sig(max(z[c] for c in W1))
        theta = sig(tau)
        eq_loss = y * sig(kk * (theta - P1)) + (1 - y) * sig(kk * (P1 - theta))   # Eq. loss
        decision = 0 if any(z[c] > tau for c in W1) else 1
        for order in (API_OUTPUT, APP_CHOICE, MULTI_SELECT):
            orc = Oracle(C, [[W1]], tau=tau, k=kk, order=order)
            d = orc.decide(z)
            assert (d == 1 if order == MULTI_SELECT else d == 0) == (decision == 0)
            G = orc.gt_mask(gt)
            assert G == y
            assert orc.loss_row(z, G)["ell"] == pytest.approx(eq_loss, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("order", [APP_CHOICE, MULTI_SELECT])
def test_new_losses_gradients_match_central_differences(order):
    rng = np.random.default_rng(46 + order)
    h = 1e-6
    for trial in range(300):
        C = int(rng.integers(2, 16))
        lists = random_lists(rng, C, bool(trial % 2))
        tau = float(rng.choice([0.0, 0.5]))
        orc = Oracle(C, [lists], tau=tau, k=float(rng.choice([1.0, 10.0])), order=order)
        z = rng.normal(tau, 3.0, size=C)
        zs = np.sort(z)
        if np.min(np.diff(zs)) < 1e-3 or np.min(np.abs(z - tau)) < 1e-3:
            continue
        gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
        G = orc.gt_mask(gt)
        w = float(rng.uniform(0.5, 2.0))
        r = orc.loss_row(z, G, w)
        for c in range(C):
            zp, zn = z.copy(), z.copy()
            zp[c] += h
            zn[c] -= h
            fd = (orc.loss_row(zp, G, w)["L"] - orc.loss_row(zn, G, w)["L"]) / (2 * h)
            an = r["grads"].get(c, 0.0)
            assert abs(fd - an) <= 1e-5 * max(abs(an), 1e-3) + 1e-8, (order, c, fd, an)


@pytest.mark.parametrize("order", [API_OUTPUT, APP_CHOICE, MULTI_SELECT])
def test_pattern_weights_literal_vs_by_mask(order):
    rng = np.random.default_rng(50 + order)
    for trial in range(20):
        C = int(rng.integers(4, 24))
        lists = random_lists(rng, C, True)
        orc = Oracle(C, [lists], order=order)
        M = int(rng.integers(1, 150))
        n = rng.integers(0, 5, size=M)
        off = np.zeros(M + 1, dtype=np.int64)
        off[1:] = np.cumsum(n)
        lab = rng.integers(0, C, size=int(off[-1])).astype(np.int32)
        r = orc.eval(np.zeros((M, C), dtype=np.float32), off, lab, want_loss=False)
        w_mask = Oracle.weights_by_mask(r["hist_gt"])[0]
        np.testing.assert_allclose(orc.weights_literal_pattern(off, lab), w_mask[r["gt_mask"]], rtol=1e-15)

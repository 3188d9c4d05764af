"""Pins of the oracle against what the paper itself fixes (CPU, no GPU).

* The worked example with the Heapsortcypher lists
  (PAPER.md:123-125): decision Recycle, correct branch Compost, precision 80 %,
  recall 100 %.
* The non-critical Snack/Food confusion.
* The paper's own application code executed verbatim on
  random API outputs, against the oracle's decision.
* The True-False special case: one list, decision = "some
  W_1 label is output".
"""
import json
import os

import numpy as np
import pytest

from oracle import Oracle
from synth import HEAPSORT_NAMES

NAME_TO_ID = {n: i for i, n in enumerate(HEAPSORT_NAMES)}
BRANCHES = ["Recycle", "Compost", "Donate", "default"]


def heapsort_oracle(tau=0.0, k=10.0):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "heapsortcypher_worked_example.json")))
    lists = [[NAME_TO_ID[n] for n in g["lists_code_order"][b]] for b in ("Recycle", "Compost", "Donate")]
    return Oracle(32, [lists], tau, k), g


# --- the application code of Fig. app_example, verbatim (names as data) ---
Recycle = ['plastic', 'wood', 'glass', 'paper', 'cardboard', 'metal', 'aluminum', 'tin', 'carton']
Compost = ['food', 'produce', 'snack']
Donate = ['clothing', 'jacket', 'shirt', 'pants', 'footwear', 'shoe']


class _Obj:
    def __init__(self, name):
        self.name = name


def heapsortcypher(label_annotations):
    for obj in label_annotations:
        if obj.name in Recycle:
            return 'Recycle'
        if obj.name in Compost:
            return 'Compost'
        if obj.name in Donate:
            return 'Donate'
    return 'default'  # falls off the loop (reading A6)


def api_output(z, tau):
    """label_detection's response: labels above the threshold, ranked by
    descending confidence; equal confidence -> smaller id first (reading A4)."""
    ids = [c for c in range(len(z)) if z[c] > tau]
    ids.sort(key=lambda c: (-z[c], c))
    return [_Obj(HEAPSORT_NAMES[c]) for c in ids]


def worked_example_logits(g, rng=None):
    order = [NAME_TO_ID[n] for n in g["api_output_descending_confidence"]]
    z = np.full(32, -5.0)
    vals = [5.0, 4.0, 3.0, 2.0, 1.0] if rng is None else sorted(rng.uniform(0.01, 9.0, 5), reverse=True)
    for c, v in zip(order, vals):
        z[c] = v
    return z


def test_worked_example_decision_and_metrics():
    orc, g = heapsort_oracle()
    out_ids = [NAME_TO_ID[n] for n in g["api_output_descending_confidence"]]
    gt = [NAME_TO_ID[n] for n in ("candy", "snack", "confectionery", "lollipop")]
    # the GT set reproduces the printed precision / recall exactly
    tp = len(set(out_ids) & set(gt))
    assert tp / len(out_ids) == g["printed"]["precision"]
    assert tp / len(gt) == g["printed"]["recall"]
    # ... and is the only 4-subset of the output meeting the printed constraints
    cands = []
    for drop in out_ids:
        s = [c for c in out_ids if c != drop]
        gset = orc.gt_set(s)
        if gset == (1 << 1):  # only Compost intersects
            cands.append(drop)
    assert cands == [NAME_TO_ID["glass"]]
    rng = np.random.default_rng(0)
    for trial in range(50):
        z = worked_example_logits(g, None if trial == 0 else rng)
        d = orc.decide(z)
        assert BRANCHES[d] == g["printed"]["executed_branch"]
        G = orc.gt_set(gt)
        assert [BRANCHES[j] for j in range(3) if G >> j & 1] == [g["printed"]["correct_branch"]]
        assert not orc.correct(G, d)


def test_worked_example_loss_pin():
    orc, g = heapsort_oracle()
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example_loss.json")))
    z = worked_example_logits(g)
    gt = [NAME_TO_ID[n] for n in ("candy", "snack", "confectionery", "lollipop")]
    r = orc.loss_row(z, orc.gt_set(gt), 1.0)
    assert r["L"] == pytest.approx(ref["L"], abs=1e-9)
    assert r["c_plus"] == NAME_TO_ID["snack"] and r["c_minus"] == NAME_TO_ID["glass"]
    assert r["g_plus"] == pytest.approx(ref["grad"]["snack"], rel=1e-8)
    assert r["g_minus"] == pytest.approx(ref["grad"]["glass"], rel=1e-8)


def test_non_critical_error():
    orc, _ = heapsort_oracle()
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "non_critical_error.json")))
    z = np.full(32, -5.0)
    for c, v in zip(g["api_output_descending_confidence"], [3.0, 2.0]):
        z[NAME_TO_ID[c]] = v
    d = orc.decide(z)
    G = orc.gt_set([NAME_TO_ID[n] for n in g["ground_truth"]])
    assert BRANCHES[d] == g["expected_branch"]
    assert orc.correct(G, d) == g["expected_correct"]
    # label-wise the output is wrong (food is not in the ground truth) ...
    assert "food" not in g["ground_truth"]
    # ... and the loss stays in its low regime (< 1/2): no critical error to penalise
    assert orc.loss_row(z, G)["ell"] < 0.5


@pytest.mark.parametrize("tau", [0.0, -1.0, 1.5])
def test_paper_listing_verbatim(tau):
    """The oracle's decision equals the paper's program run on the API output."""
    orc, _ = heapsort_oracle(tau)
    rng = np.random.default_rng(1)
    for trial in range(3000):
        if trial % 3 == 0:
            z = rng.integers(-3, 4, size=32).astype(np.float64)  # tie-heavy
        else:
            z = rng.normal(0, 2, size=32)
        want = heapsortcypher(api_output(z, tau))
        assert BRANCHES[orc.decide(z)] == want


def test_true_false_special_case():
    """One list (True-False): decision 0 iff some W_1 label is output."""
    rng = np.random.default_rng(2)
    for trial in range(200):
        C = int(rng.integers(1, 40))
        W1 = sorted(set(rng.integers(0, C, size=int(rng.integers(0, C + 1))).tolist()))
        orc = Oracle(C, [[W1]], tau=0.0)
        z = rng.normal(0, 1, size=C)
        expect = 0 if any(z[c] > 0.0 for c in W1) else 1
        assert orc.decide(z) == expect

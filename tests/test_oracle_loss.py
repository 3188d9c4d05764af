"""Pins of the oracle's loss and gradient (Eq. api_output), CPU.

* Hand-enumerated tiny cases (tests/golden/hand_cases.json): decisions by hand,
  losses and gradients are closed forms of Eq. api_output.
* Step-function limit: the paper builds S as a smooth stand-in for a step
   so that "only if the first output label encountered belonging
  to any of the target classes matches with the ground-truth class, the penalty
  will be low".  As k -> inf the per-input loss must equal the
  incorrect-decision indicator of Eq. goal on tie-free inputs.
* Central finite differences of the loss against the analytic gradient.
"""
import json
import os

import numpy as np
import pytest

from oracle import Oracle


def load_cases():
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))


@pytest.mark.parametrize("case", load_cases()["cases"], ids=lambda c: c["id"])
def test_hand_cases(case):
    common = load_cases()["common"]
    orc = Oracle(common["C"], [case["lists"]], tau=case["tau"], k=common["k"])
    z = np.array(case["z"], dtype=np.float64)
    d = orc.decide(z)
    G = orc.gt_set(case["gt"])
    assert d == case["decision"]
    assert G == case["G"]
    assert orc.correct(G, d) == case["correct"]
    r = orc.loss_row(z, G, common["w"])
    assert r["L"] == pytest.approx(case["L"], abs=2e-9)
    got = {}
    if r["c_plus"] >= 0:
        got[r["c_plus"]] = got.get(r["c_plus"], 0.0) + r["g_plus"]
    if r["c_minus"] >= 0:
        got[r["c_minus"]] = got.get(r["c_minus"], 0.0) + r["g_minus"]
    want = {int(c): v for c, v in case["grad"].items()}
    assert set(got) == set(want)
    for c in want:
        assert got[c] == pytest.approx(want[c], rel=2e-6)


def random_case(rng, C=None):
    C = C or int(rng.integers(2, 24))
    D = int(rng.integers(1, 5))
    perm = rng.permutation(C)
    lists, pos = [], 0
    for j in range(D):
        n = int(rng.integers(1, max(2, C // D)))
        lists.append(sorted(perm[pos:pos + n].tolist()))
        pos += n
    tau = float(rng.choice([0.0, -0.5, 1.0]))
    z = rng.normal(tau, 3.0, size=C)
    gt = sorted(set(rng.integers(0, C, size=int(rng.integers(0, 4))).tolist()))
    return C, lists, tau, z, gt


def test_step_limit_equals_incorrect_indicator():
    rng = np.random.default_rng(20)
    checked = 0
    for trial in range(4000):
        C, lists, tau, z, gt = random_case(rng)
        orc = Oracle(C, [lists], tau=tau, k=1e7)
        G = orc.gt_set(gt)
        d = orc.decide(z)
        # keep inputs whose probabilities are separated (no ties at the step)
        p = 1 / (1 + np.exp(-z))
        th = 1 / (1 + np.exp(-tau))
        vals = np.concatenate([p, [th]])
        gaps = np.abs(vals[:, None] - vals[None, :])[np.triu_indices(len(vals), 1)]
        if gaps.min() < 1e-5:
            continue
        ell = orc.loss_row(z, G, 1.0)["ell"]
        assert ell == pytest.approx(float(not orc.correct(G, d)), abs=1e-6), (lists, z, gt, tau)
        checked += 1
    assert checked > 1000


def test_gradient_matches_central_differences():
    rng = np.random.default_rng(21)
    h = 1e-6
    worst = 0.0
    for trial in range(600):
        C, lists, tau, z, gt = random_case(rng)
        orc = Oracle(C, [lists], tau=tau, k=float(rng.choice([1.0, 10.0, 30.0])))
        G = orc.gt_set(gt)
        w = float(rng.uniform(0.5, 3.0))
        r = orc.loss_row(z, G, w)
        # skip inputs within h of a kink (arg max switch or z- at the threshold)
        mapped = [c for c in range(C) if orc.first_list(c) >= 0]
        zm = np.sort(z[mapped]) if mapped else np.array([])
        if len(zm) > 1 and np.min(np.diff(zm)) < 1e-3:
            continue
        if mapped and np.min(np.abs(z[mapped] - tau)) < 1e-3:
            continue
        analytic = np.zeros(C)
        if r["c_plus"] >= 0:
            analytic[r["c_plus"]] += r["g_plus"]
        if r["c_minus"] >= 0:
            analytic[r["c_minus"]] += r["g_minus"]
        for c in range(C):
            zp, zn = z.copy(), z.copy()
            zp[c] += h
            zn[c] -= h
            fd = (orc.loss_row(zp, G, w)["L"] - orc.loss_row(zn, G, w)["L"]) / (2 * h)
            err = abs(fd - analytic[c]) / max(abs(analytic[c]), 1e-3)
            worst = max(worst, err)
            assert abs(fd - analytic[c]) <= 1e-5 * max(abs(analytic[c]), 1e-3) + 1e-8, (c, fd, analytic[c])
    assert worst < 1e-5


def test_loss_properties():
    """w scales L and g linearly; a row with no mapped label and y=0 has zero loss;
    the loss is in (0, w)."""
    rng = np.random.default_rng(22)
    for trial in range(300):
        C, lists, tau, z, gt = random_case(rng)
        orc = Oracle(C, [lists], tau=tau)
        G = orc.gt_set(gt)
        r1, r3 = orc.loss_row(z, G, 1.0), orc.loss_row(z, G, 3.0)
        assert r3["L"] == pytest.approx(3 * r1["L"], rel=1e-12)
        assert r3["g_plus"] == pytest.approx(3 * r1["g_plus"], rel=1e-12)
        assert 0.0 <= r1["L"] < 1.0
    orc = Oracle(5, [[]])
    r = orc.loss_row(np.zeros(5), 0)
    assert r["L"] == 0.0 and r["c_plus"] == -1 and r["c_minus"] == -1

"""Pins of the oracle's BATCH drivers (CPU): orc_eval, orc_gt_hist, orc_ranges_eval.

Every GPU parity test compares the kernels with these drivers, so their assembly —
which row goes to which counter, which weight multiplies which loss, which slot holds
which gradient — is pinned here against a plain Python loop over the per-row functions
that the other oracle tests pin (decide / gt_set / correct / loss_row / range_of /
range_loss).  The batch outputs are the sums and tables the paper defines:

* Eq. goal: n_incorrect[a] = #{i of app a : Decision(API(x_i)) is
  not correct for ŷ_i}; the per-app split is the multi-application batch of
  BASELINE.json configs[3] (one context per app).
* hist_gt[a][m] = #{i of app a : G_i = m}, whose entries give the N_i.
* Eq. api_output: loss_sum[a] = Σ_i (M/N_i)·ℓ_i, loss_row[i] =
  (M/N_i)·ℓ_i, with w = M/N_i looked up by (app, G_i); the gradient slots are the
  per-row derivatives times the caller's grad_scale (reading A14).
* Value ranges: decision = first containing range, n_incorrect
  counts decision != ground-truth range, histograms over the m+1 range ids.

The expected values are built from per-row oracle calls plus numpy bookkeeping written
here; bf16 inputs are widened by numpy (bits << 16), not by the oracle's own loader.
"""
import numpy as np
import pytest

from oracle import API_OUTPUT, APP_CHOICE, MULTI_SELECT, Oracle, RangesOracle


def _random_context(rng, C, n_apps, order):
    apps = []
    for _ in range(n_apps):
        D = int(rng.integers(1, 6))
        lists = []
        for _ in range(D):
            n = int(rng.integers(0, 6))
            lists.append(sorted(set(rng.integers(0, C, size=n).tolist())))  # may overlap (A5 / A23)
        apps.append(lists)
    return Oracle(C, apps, tau=float(rng.choice([0.0, 0.5, -0.25])), k=float(rng.choice([3.0, 10.0])), order=order)


def _random_batch(rng, C, rows, ld, n_apps, bf16):
    # integer-heavy logits so ties and values on tau occur; some continuous values too
    z = rng.integers(-3, 4, size=(rows, ld)).astype(np.float32) * np.float32(0.5)
    cont = rng.random((rows, ld)) < 0.3
    z[cont] = rng.normal(0, 3, size=int(cont.sum())).astype(np.float32)
    z[:, C:] = np.nan  # padding columns must never be read
    if bf16:
        bits = (z.view(np.uint32) >> 16).astype(np.uint16)  # truncation: any bf16 pattern will do
        logits = bits
        z_eff = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    else:
        logits = z
        z_eff = z.astype(np.float64)
    n_gt = rng.integers(0, 5, size=rows)
    gt_off = np.zeros(rows + 1, np.int64)
    gt_off[1:] = np.cumsum(n_gt)
    base = int(rng.integers(0, 7))  # any CSR base
    gt_off += base
    gt_lab = np.concatenate([rng.integers(0, C, size=base), rng.integers(0, C, size=int(n_gt.sum()))]).astype(np.int32)
    app = rng.integers(0, n_apps, size=rows).astype(np.uint16) if n_apps > 1 else None
    return logits, z_eff, gt_off, gt_lab, app


def _expected(orc, z_eff, gt_off, gt_lab, app, w, grad_scale):
    rows = z_eff.shape[0]
    C, na, S = orc.C, orc.n_apps, orc.grad_slots
    e = dict(decision=np.zeros(rows, np.uint8), gt_mask=np.zeros(rows, np.uint8), correct=np.zeros(rows, np.uint8),
             n_incorrect=np.zeros(na, np.uint64), hist_pred=np.zeros(na * 256, np.uint64),
             hist_gt=np.zeros(na * 256, np.uint64), loss_sum=np.zeros(na, np.float64),
             loss_row=np.zeros(rows, np.float64), grad_idx=np.full(S * rows, -1, np.int32),
             grad_val=np.zeros(S * rows, np.float64))
    for i in range(rows):
        a = int(app[i]) if app is not None else 0
        zi = z_eff[i, :C]
        labels = gt_lab[gt_off[i]:gt_off[i + 1]]
        d = orc.decide(zi, app=a)
        G = orc.gt_mask(labels, app=a)
        ok = orc.is_correct(labels, d, app=a)
        wi = float(w[a * 256 + G]) if w is not None else 1.0
        r = orc.loss_row(zi, G, w=wi, app=a)
        e["decision"][i] = d
        e["gt_mask"][i] = G
        e["correct"][i] = ok
        e["n_incorrect"][a] += np.uint64(not ok)
        e["hist_pred"][a * 256 + d] += np.uint64(1)
        e["hist_gt"][a * 256 + G] += np.uint64(1)
        e["loss_sum"][a] += r["L"]
        e["loss_row"][i] = r["L"]
        if orc.order == MULTI_SELECT:
            cs, gs = r["slots"]
            e["grad_idx"][S * i:S * i + S] = cs
            e["grad_val"][S * i:S * i + S] = gs * grad_scale
        else:
            e["grad_idx"][S * i] = r["c_plus"]
            e["grad_val"][S * i] = r["g_plus"] * grad_scale
            e["grad_idx"][S * i + 1] = r["c_minus"]
            e["grad_val"][S * i + 1] = r["g_minus"] * grad_scale
        assert abs(r["L"] - wi * r["ell"]) <= 1e-15 * max(1.0, abs(r["L"]))  # L = (M/N_i)·ℓ_i
    return e


@pytest.mark.parametrize("order", [API_OUTPUT, APP_CHOICE, MULTI_SELECT])
@pytest.mark.parametrize("n_apps", [1, 3])
@pytest.mark.parametrize("bf16", [False, True])
def test_eval_driver_equals_loop_over_pinned_rows(order, n_apps, bf16):
    rng = np.random.default_rng(1000 * order + 10 * n_apps + bf16)
    C = int(rng.integers(8, 40))
    ld = C + int(rng.integers(0, 5))
    rows = 257
    orc = _random_context(rng, C, n_apps, order)
    logits, z_eff, gt_off, gt_lab, app = _random_batch(rng, C, rows, ld, n_apps, bf16)
    # per-(app, mask) weights that differ from 1 and from each other: w[a*256+m]
    w = (0.25 + rng.random(n_apps * 256) * 3.0).astype(np.float64)
    grad_scale = 1.0 / 7.0
    got = orc.eval(logits, gt_off, gt_lab, app=app, w=w, grad_scale=grad_scale)
    exp = _expected(orc, z_eff, gt_off, gt_lab, app, w, grad_scale)
    for key in ("decision", "gt_mask", "correct", "n_incorrect", "hist_pred", "hist_gt", "grad_idx"):
        np.testing.assert_array_equal(got[key], exp[key], err_msg=key)
    for key in ("loss_row", "grad_val", "loss_sum"):
        np.testing.assert_allclose(got[key], exp[key], rtol=1e-13, atol=1e-300, err_msg=key)
    # the tables are the paper's counts: every row lands in exactly one bin of each
    assert int(got["hist_gt"].sum()) == rows and int(got["hist_pred"].sum()) == rows
    assert int(got["n_incorrect"].sum()) == rows - int(got["correct"].sum())


@pytest.mark.parametrize("order", [API_OUTPUT, APP_CHOICE, MULTI_SELECT])
def test_eval_driver_accumulates_and_defaults(order):
    """Counters ACCUMULATE (+=) across calls (chunked batches sum to the whole batch);
    w = NULL means weight 1; grad_scale defaults to 1."""
    rng = np.random.default_rng(77 + order)
    C = 23
    orc = _random_context(rng, C, 2, order)
    logits, z_eff, gt_off, gt_lab, app = _random_batch(rng, C, 200, C, 2, False)
    whole = orc.eval(logits, gt_off, gt_lab, app=app)
    exp = _expected(orc, z_eff, gt_off, gt_lab, app, None, 1.0)
    np.testing.assert_allclose(whole["loss_sum"], exp["loss_sum"], rtol=1e-13)
    np.testing.assert_allclose(whole["grad_val"], exp["grad_val"], rtol=1e-13, atol=1e-300)
    parts = [(0, 61), (61, 62), (62, 200)]
    acc = {k: np.zeros_like(whole[k]) for k in ("n_incorrect", "hist_pred", "hist_gt", "loss_sum")}
    for lo, hi in parts:
        r = orc.eval(logits[lo:hi], gt_off[lo:hi + 1], gt_lab, app=app[lo:hi])
        for k in acc:
            acc[k] += r[k]
    for k in ("n_incorrect", "hist_pred", "hist_gt"):
        np.testing.assert_array_equal(acc[k], whole[k], err_msg=k)
    np.testing.assert_allclose(acc["loss_sum"], whole["loss_sum"], rtol=1e-13)


@pytest.mark.parametrize("order", [API_OUTPUT, MULTI_SELECT])
def test_gt_hist_driver_equals_loop(order):
    rng = np.random.default_rng(5 + order)
    C = 31
    orc = _random_context(rng, C, 3, order)
    _, _, gt_off, gt_lab, app = _random_batch(rng, C, 300, C, 3, False)
    gm, H = orc.gt_hist(gt_off, gt_lab, app=app)
    exp_gm = np.zeros(300, np.uint8)
    exp_H = np.zeros(3 * 256, np.uint64)
    for i in range(300):
        a = int(app[i])
        G = orc.gt_mask(gt_lab[gt_off[i]:gt_off[i + 1]], app=a)
        exp_gm[i] = G
        exp_H[a * 256 + G] += np.uint64(1)
    np.testing.assert_array_equal(gm, exp_gm)
    np.testing.assert_array_equal(H, exp_H)


def test_eval_driver_bf16_equals_widened_f32():
    """The bf16 loader widens bit patterns exactly: the bf16 batch and the same values
    given as f32 produce identical outputs."""
    rng = np.random.default_rng(9)
    C = 29
    orc = _random_context(rng, C, 1, API_OUTPUT)
    bits, z_eff, gt_off, gt_lab, _ = _random_batch(rng, C, 150, C + 3, 1, True)
    a = orc.eval(bits, gt_off, gt_lab, w=None)
    f = z_eff.astype(np.float32)
    f[:, C:] = np.nan
    b = orc.eval(f, gt_off, gt_lab, w=None)
    for key in a:
        np.testing.assert_array_equal(a[key], b[key], err_msg=key)


@pytest.mark.parametrize("with_w", [False, True])
def test_ranges_driver_equals_loop(with_w):
    rng = np.random.default_rng(11 + with_w)
    lo = np.array([-1.0, -0.2, 0.3, 0.3, 0.9])
    hi = np.array([-0.3, 0.25, 0.5, 0.8, 1.5])
    orc = RangesOracle(lo, hi, k=7.0)
    rows = 400
    score = rng.uniform(-1.6, 1.8, size=rows).astype(np.float32)
    gt = rng.uniform(-1.6, 1.8, size=rows).astype(np.float32)
    gt[:20] = hi[[0, 1, 2, 3, 4] * 4].astype(np.float32)  # ground truth on bounds
    score[20:40] = lo[[0, 1, 2, 3, 4] * 4].astype(np.float32)
    m = len(lo)
    w = (0.5 + rng.random(m + 1)) if with_w else None
    gs = 0.125
    got = orc.eval(score, gt, w=w, grad_scale=gs)
    e_dec = np.zeros(rows, np.uint8)
    e_gt = np.zeros(rows, np.uint8)
    e_hp = np.zeros(m + 1, np.uint64)
    e_hg = np.zeros(m + 1, np.uint64)
    e_lr = np.zeros(rows)
    e_g = np.zeros(rows)
    n_inc = 0
    loss = 0.0
    for i in range(rows):
        d = orc.range_of(float(score[i]))
        r = orc.range_of(float(gt[i]))
        L, dL = orc.loss(r, float(score[i]), w=float(w[r]) if with_w else 1.0)
        e_dec[i], e_gt[i] = d, r
        e_hp[d] += np.uint64(1)
        e_hg[r] += np.uint64(1)
        n_inc += d != r
        loss += L
        e_lr[i] = L
        e_g[i] = dL * gs
    np.testing.assert_array_equal(got["decision"], e_dec)
    np.testing.assert_array_equal(got["gt_range"], e_gt)
    np.testing.assert_array_equal(got["hist_pred"], e_hp)
    np.testing.assert_array_equal(got["hist_gt"], e_hg)
    assert int(got["n_incorrect"][0]) == n_inc
    np.testing.assert_allclose(got["loss_row"], e_lr, rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(got["grad"], e_g, rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(got["loss_sum"][0], loss, rtol=1e-13)
    assert 0 < n_inc < rows  # the batch exercises both outcomes

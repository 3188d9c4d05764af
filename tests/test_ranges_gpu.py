"""GPU parity of the value-ranges path against the oracle."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("m,rows,off,overlap", [(1, 1, 0, False), (3, 100003, 0, False), (7, 5000, 0, True),
                                                (7, 5000, 1, True), (7, 30001, 0, False), (20, 70001, 0, True),
                                                (20, 70001, 0, False), (40, 20000, 0, True), (40, 20000, 3, False),
                                                (200, 9000, 0, False), (7, 30001, 0, "gaps"), (7, 30001, 0, "cluster"),
                                                (200, 9000, 0, "cluster"), (1, 5000, 0, "point"),
                                                (3, 30001, 0, "deep"), (7, 30001, 1, "deep"), (20, 20001, 0, "deep")])
def test_ranges_parity(m, rows, off, overlap):
    # 2-8 bins: packed counters, 21: ballot, 41: match; off: unaligned (scalar) accesses;
    # overlap False: ranges in ascending order that touch (binary-search lookup when m > 16);
    # "gaps": ascending ranges with holes between them; "cluster": most bounds packed into
    # [0, 1e-3]; "point": one degenerate range lo == hi
    import torch
    import paper_2310_07240_b200 as sc
    from oracle import RangesOracle
    rng = np.random.default_rng(m * 1000 + rows)
    edges = np.sort(rng.uniform(-1, 1, size=m + 1)).astype(np.float32)
    lo, hi = edges[:-1].copy(), edges[1:].copy()
    if overlap is True:  # overlapping ranges: the first containing range wins
        hi[1] = np.float32(min(1.0, hi[1] + 0.2))
    elif overlap == "gaps":  # hi[j] < lo[j+1]
        hi = (lo + np.float32(0.6) * (hi - lo)).astype(np.float32)
    elif overlap == "cluster":  # m - 1 tiny touching ranges in [0, 1e-3], then one up to 1
        edges = np.concatenate([np.sort(rng.uniform(0, 1e-3, size=m)), [1.0]]).astype(np.float32)
        lo, hi = edges[:-1].copy(), edges[1:].copy()
    elif overlap == "point":
        lo = hi = np.array([0.25], dtype=np.float32)
    k = 10.0
    span = 1.2
    if overlap == "deep":  # wide ranges: |k(l - O)|, |k(O - h)| up to ~300, S arguments past fp32's exp range
        lo, hi = (lo * np.float32(12)).astype(np.float32), (hi * np.float32(12)).astype(np.float32)
        span = 14.4
    score = rng.uniform(-span, span, rows).astype(np.float32)
    score[: rows // 10] = lo[rng.integers(0, m, rows // 10)]  # exactly on a bound
    score[rows // 10: rows // 5] = hi[rng.integers(0, m, rows // 5 - rows // 10)]
    if overlap == "cluster":
        score[rows // 5: rows // 2] = rng.uniform(-1e-4, 1.1e-3, rows // 2 - rows // 5).astype(np.float32)
    gt = rng.uniform(-span, span, rows).astype(np.float32)
    gt[: rows // 2] = rng.permutation(score[: rows // 2])  # GT on bounds / inside the clusters as well
    orc = RangesOracle(lo.astype(np.float64), hi.astype(np.float64), k)
    pre = orc.eval(score, gt)
    w_ref = orc.weights(pre["hist_gt"])
    ref = orc.eval(score, gt, w=w_ref, grad_scale=1.0 / rows)

    r = sc.Ranges(lo, hi, k)
    # off > 0: the device arrays start `off` elements into a larger allocation (not 16-B aligned)
    d_score = torch.cat([torch.zeros(off), torch.from_numpy(score)]).cuda()[off:]
    d_gt = torch.cat([torch.zeros(off), torch.from_numpy(gt)]).cuda()[off:]
    hist = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
    def buf(dt):  # outputs shifted by `off` elements as well
        return torch.empty(rows + off, dtype=dt, device="cuda")[off:]

    gtr = buf(torch.uint8)
    sc.sc_ranges_hist(r, d_gt, hist_gt=hist, gt_range_out=gtr)
    w = torch.empty(m + 1, dtype=torch.float32, device="cuda")
    sc.sc_ranges_weights(r, hist, w)
    out = dict(loss_sum=torch.zeros(1, dtype=torch.float64, device="cuda"),
               loss_row=buf(torch.float32), grad=buf(torch.float32), decision=buf(torch.uint8),
               n_incorrect=torch.zeros(1, dtype=torch.int64, device="cuda"),
               hist_pred=torch.zeros(m + 1, dtype=torch.int64, device="cuda"))
    sc.sc_ranges_loss_fwd_bwd(r, d_score, gtr, w=w, grad_scale=1.0 / rows, **out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hist.cpu().numpy().astype(np.uint64), pre["hist_gt"])
    np.testing.assert_array_equal(gtr.cpu().numpy(), ref["gt_range"])
    np.testing.assert_allclose(w.cpu().numpy(), w_ref, rtol=1e-7)
    np.testing.assert_array_equal(out["decision"].cpu().numpy(), ref["decision"])
    np.testing.assert_array_equal(out["n_incorrect"].cpu().numpy().astype(np.uint64), ref["n_incorrect"])
    np.testing.assert_array_equal(out["hist_pred"].cpu().numpy().astype(np.uint64), ref["hist_pred"])
    # 1e-5 relative; SURVEY.md §8(c)9's absolute rule below 1e-30 (subnormal fp32 results)
    lr, lr_ref = out["loss_row"].cpu().numpy().astype(np.float64), ref["loss_row"]
    assert np.all(np.abs(lr - lr_ref) <= 1e-5 * np.maximum(np.abs(lr_ref), 1e-30))
    # dL/dO = w k (σ'(k(O − hi)) − σ'(k(lo − O))): the two terms can cancel, so the bar is
    # 1e-5 of the terms' magnitude (a tolerance bound only; the reference value is the oracle's)
    r_i = ref["gt_range"].astype(np.int64)
    ok = r_i < m
    dsg = lambda x: np.exp(-np.abs(x)) / (1 + np.exp(-np.abs(x))) ** 2
    mag = np.zeros(rows)
    lo64, hi64, s64 = lo.astype(np.float64), hi.astype(np.float64), score.astype(np.float64)
    mag[ok] = w_ref[r_i[ok]] * k * (dsg(k * (lo64[r_i[ok]] - s64[ok])) + dsg(k * (s64[ok] - hi64[r_i[ok]]))) / rows
    assert np.all(np.abs(out["grad"].cpu().numpy() - ref["grad"]) <= 1e-5 * np.maximum(mag, 1e-30))
    np.testing.assert_allclose(out["loss_sum"].cpu().numpy(), ref["loss_sum"], rtol=1e-5)

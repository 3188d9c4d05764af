"""GPU parity: libsc (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): decisions, G_i, counts and histograms bit-exact;
loss and gradients within 1e-5 relative (DESIGN.md §5 derives why fp32 meets it).
Inputs are the seeded synthetic workloads of synth/ (host generator here, so the
CUDA generator is not on the parity path), at sizes that span several stages /
tiles and a ragged tail, plus edge cases.
"""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

RTOL = 1e-5


def _mods():
    import torch
    import paper_2310_07240_b200 as sc
    import synth
    from oracle import Oracle
    return torch, sc, synth, Oracle


def to_dev(b, dtype):
    torch, *_ = _mods()
    lg = b["logits"]
    if dtype == "bf16":
        t = torch.from_numpy(np.ascontiguousarray(lg).view(np.int16)).cuda().view(torch.bfloat16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(lg)).cuda()
    out = dict(logits=t, gt_off=torch.from_numpy(b["gt_off"]).cuda(),
               gt_lab=torch.from_numpy(b["gt_lab"] if len(b["gt_lab"]) else np.zeros(1, np.int32)).cuda())
    if "app" in b and b["app"] is not None:
        out["app"] = torch.from_numpy(np.ascontiguousarray(b["app"]).view(np.int16)).cuda()
    return out


def run_gpu(ctxspec, d, mode="mask", dense=False, with_app=False, order=0, compact=False, host=None):
    """hist pre-pass -> weights -> fused loss pass; returns numpy dict.  compact: the logits
    are column-compacted rows of a sc_context_load_compact context.  host = (mode, stager
    chunk bytes): the loss pass reads the logits from pinned host memory
    (sc_loss_fwd_bwd_host); res["host_mode"] = the mode libsc took."""
    torch, sc, _, _ = _mods()
    ctx = sc.Context(ctxspec.C, ctxspec.lists, ctxspec.tau, ctxspec.k, order=order, multi_app=True, compact=compact)
    rows, na = d["logits"].shape[0], ctxspec.n_apps
    S = ctx.grad_slots
    app = d.get("app") if with_app else None
    hist = torch.zeros(na * 256, dtype=torch.int64, device="cuda")
    gmask = torch.empty(rows + 16, dtype=torch.uint8, device="cuda")
    sc.sc_decision_hist(ctx, sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], app=app, rows=rows),
                        hist_gt=hist, gt_mask_out=gmask)
    w = torch.empty(na * 256, dtype=torch.float32, device="cuda")
    sc.sc_weights_from_hist(ctx, hist, w)
    o = dict(
        decision=torch.full((rows,), 77, dtype=torch.uint8, device="cuda"),
        n_incorrect=torch.zeros(na, dtype=torch.int64, device="cuda"),
        hist_pred=torch.zeros(na * 256, dtype=torch.int64, device="cuda"),
        hist_gt=torch.zeros(na * 256, dtype=torch.int64, device="cuda"),
        loss_sum=torch.zeros(na, dtype=torch.float64, device="cuda"),
        loss_row=torch.full((rows,), -1.0, dtype=torch.float32, device="cuda"),
        grad_idx=torch.full((S * rows,), -7, dtype=torch.int32, device="cuda"),
        grad_val=torch.full((S * rows,), -7.0, dtype=torch.float32, device="cuda"),
    )
    ld = d["logits"].stride(0)
    if dense:
        o["grad_dense"] = torch.full((rows * ld,), 3.0, dtype=torch.float32, device="cuda")
    if mode == "mask":
        batch = sc.Batch(logits=d["logits"], gt_mask=gmask, app=app)
    else:
        batch = sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"], app=app)
    grad_scale = 1.0 / max(rows, 1)
    used = None
    if host is None:
        sc.sc_loss_fwd_bwd(ctx, batch, w=w, grad_scale=grad_scale, **o)
    else:
        hmode, chunk = host
        batch.logits = d["logits"].cpu().pin_memory()
        stager = sc.Stager(chunk) if chunk else None
        used = sc.sc_loss_fwd_bwd_host(ctx, stager, batch, mode=hmode, w=w, grad_scale=grad_scale, **o)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in o.items()}
    res["host_mode"] = used
    res["hist_pre"] = hist.cpu().numpy()
    res["gt_mask"] = gmask[:rows].cpu().numpy()
    res["w"] = w.cpu().numpy()
    res["grad_scale"] = grad_scale
    res["ld"] = ld
    res["S"] = S
    return res


def run_oracle(ctxspec, b, grad_scale, with_app=False, order=0):
    *_, Oracle = _mods()
    orc = Oracle.from_spec(ctxspec, order)
    app = b.get("app") if with_app else None
    pre = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=app, want_loss=False)
    w = Oracle.weights_by_mask(pre["hist_gt"])
    return orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=app, w=w, grad_scale=grad_scale), w


def assert_rel(got, ref, rtol=RTOL, floor=1e-30, err_msg=""):
    """|got - ref| <= rtol * max(|ref|, floor): relative, except for entries below `floor`
    (gradient entries with |g_ref| < 1e-30 are compared absolutely — fp32
    cannot hold them to 1e-5 relative once they are subnormal, e.g. σ'(z) for |z| > 87)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    bound = rtol * np.maximum(np.abs(ref), floor)
    bad = ~(np.abs(got - ref) <= bound)
    assert not bad.any(), (f"{err_msg}: {int(bad.sum())} entries off, first at {np.nonzero(bad)[0][:5]}: "
                           f"got {got[bad][:5]} ref {ref[bad][:5]}")


def compare(g, o, w_orc, rows):
    np.testing.assert_array_equal(g["gt_mask"], o["gt_mask"])
    np.testing.assert_array_equal(g["hist_pre"].astype(np.uint64), o["hist_gt"])
    np.testing.assert_array_equal(g["hist_gt"].astype(np.uint64), o["hist_gt"])
    np.testing.assert_array_equal(g["decision"], o["decision"])
    np.testing.assert_array_equal(g["hist_pred"].astype(np.uint64), o["hist_pred"])
    np.testing.assert_array_equal(g["n_incorrect"].astype(np.uint64), o["n_incorrect"])
    np.testing.assert_allclose(g["w"], w_orc.reshape(-1), rtol=1e-7)
    np.testing.assert_array_equal(g["grad_idx"], o["grad_idx"])
    assert_rel(g["loss_row"], o["loss_row"], err_msg="loss_row")
    assert_rel(g["grad_val"], o["grad_val"], err_msg="grad_val")
    np.testing.assert_allclose(g["loss_sum"], o["loss_sum"], rtol=RTOL, atol=0)
    if "grad_dense" in g:
        ld, S = g["ld"], g["S"]
        dense = np.zeros((rows, ld), dtype=np.float64)
        mag = np.zeros((rows, ld), dtype=np.float64)  # Σ|terms|: bound for sums that cancel (Multi-Select)
        gi, gv = o["grad_idx"].reshape(rows, S), o["grad_val"].reshape(rows, S)
        for s in range(S):
            m = gi[:, s] >= 0
            dense[np.nonzero(m)[0], gi[m, s]] += gv[m, s]
            mag[np.nonzero(m)[0], gi[m, s]] += np.abs(gv[m, s])
        got = g["grad_dense"].reshape(rows, ld).astype(np.float64)
        bound = RTOL * np.maximum(mag, 1e-30)
        assert np.all(np.abs(got - dense) <= bound), np.max(np.abs(got - dense) - bound)


CASES = [
    # (config, dtype, row0, rows, mode, ld_extra, layout)
    (1, "f32", 0, 4096, "mask", 0, 0),
    (1, "f32", 0, 4096, "csr", 0, 0),
    (1, "bf16", 0, 4096, "mask", 8, 0),
    (2, "f32", 777, 3001, "mask", 0, 0),
    (2, "f32", 5, 1203, "csr", 4, 0),
    (2, "bf16", 123, 2049, "mask", 0, 0),
    (3, "f32", 31, 203, "mask", 0, 0),
    (3, "bf16", 0, 150, "csr", 8, 0),
    (4, "f32", (1 << 18) - 700, 1500, "mask", 0, 0),
    (4, "f32", 10, 1500, "mask", 0, 1),
    (4, "bf16", 10, 999, "csr", 0, 1),
]


@pytest.fixture(params=["tma", "gather"])
def kernel(request, monkeypatch):
    """Both eval kernels (dense TMA ring / sector-sparse gather) must meet the same bar."""
    monkeypatch.setenv("SC_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("cfg,dtype,row0,rows,mode,ld_extra,layout", CASES)
def test_parity_configs(cfg, dtype, row0, rows, mode, ld_extra, layout, kernel):
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(cfg)
    ld = synth.default_ld(spec.C, dtype) + ld_extra
    wl = synth.Workload(spec, seed=cfg, dtype=dtype, ld=ld, layout=layout)
    b = wl.host_batch(row0, rows)
    multi = spec.n_apps > 1
    g = run_gpu(spec, to_dev(b, dtype), mode=mode, dense=(cfg in (1, 2)), with_app=multi)
    o, w = run_oracle(spec, b, g["grad_scale"], with_app=multi)
    compare(g, o, w, rows)


def tie_heavy_batch(rng, C, rows, ld, lists, tau):
    z = rng.integers(-2, 3, size=(rows, C)).astype(np.float32)
    z[rng.random((rows, C)) < 0.1] = np.float32(tau)          # exactly at the threshold
    z[rng.random((rows, C)) < 0.05] = np.float32(-0.0)
    lg = np.full((rows, ld), np.nan, dtype=np.float32)
    lg[:, :C] = z
    n = rng.integers(0, 5, size=rows)
    off = np.zeros(rows + 1, dtype=np.int64)
    off[1:] = np.cumsum(n)
    lab = rng.integers(0, C, size=int(off[-1])).astype(np.int32)
    return dict(logits=lg, gt_off=off, gt_lab=lab)


@pytest.mark.parametrize("C,ld,rows", [(1, 4, 100), (4, 4, 333), (37, 40, 1000), (64, 64, 4097), (300, 300, 777),
                                       (4097, 4100, 97), (12000, 12000, 40)])
def test_parity_tie_heavy_overlapping(C, ld, rows, kernel):
    _, _, synth, _ = _mods()
    rng = np.random.default_rng(C * 7 + rows)
    for tau in (0.0, -1.0):
        D = int(rng.integers(0, 9))
        lists = [sorted(set(rng.integers(0, C, size=int(rng.integers(0, min(C, 40) + 1))).tolist())) for _ in range(D)]
        spec = synth.ContextSpec(C, [lists], tau=tau, k=float(rng.choice([1.0, 10.0, 25.0])))
        b = tie_heavy_batch(rng, C, rows, ld, lists, tau)
        g = run_gpu(spec, to_dev(b, "f32"), mode="mask" if tau == 0 else "csr", dense=C < 1000)
        o, w = run_oracle(spec, b, g["grad_scale"])
        compare(g, o, w, rows)


def test_hand_cases_through_gpu(golden_dir, kernel):
    import json, os
    torch, sc, synth, Oracle = _mods()
    cases = json.load(open(os.path.join(golden_dir, "hand_cases.json")))
    for case in cases["cases"]:
        spec = synth.ContextSpec(4, [case["lists"]], tau=case["tau"], k=cases["common"]["k"])
        gt = case["gt"]
        b = dict(logits=np.array([case["z"]], dtype=np.float32),
                 gt_off=np.array([0, len(gt)], dtype=np.int64), gt_lab=np.array(gt, dtype=np.int32))
        d = to_dev(b, "f32")
        ctx = sc.Context(4, [case["lists"]], case["tau"], cases["common"]["k"], multi_app=True)
        dec = torch.empty(1, dtype=torch.uint8, device="cuda")
        lr = torch.empty(1, dtype=torch.float32, device="cuda")
        gi = torch.empty(2, dtype=torch.int32, device="cuda")
        gv = torch.empty(2, dtype=torch.float32, device="cuda")
        sc.sc_loss_fwd_bwd(ctx, sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"]),
                           loss_row=lr, grad_idx=gi, grad_val=gv, decision=dec)
        assert int(dec.item()) == case["decision"], case["id"]
        assert float(lr.item()) == pytest.approx(case["L"], rel=RTOL, abs=1e-7), case["id"]
        got = {}
        for c, v in zip(gi.cpu().tolist(), gv.cpu().tolist()):
            if c >= 0:
                got[c] = got.get(c, 0.0) + v
        want = {int(c): v for c, v in case["grad"].items()}
        assert set(got) == set(want), case["id"]
        for c in want:
            assert got[c] == pytest.approx(want[c], rel=2e-6), case["id"]


def test_accumulate_and_chunking(kernel):
    """Outputs accumulate (+=): two half-batches equal one whole batch (the shard algebra)."""
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(2)
    wl = synth.Workload(spec, seed=2)
    d = to_dev(wl.host_batch(0, 2000), "f32")
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)

    def agg(parts):
        ni = torch.zeros(1, dtype=torch.int64, device="cuda")
        hp = torch.zeros(256, dtype=torch.int64, device="cuda")
        hg = torch.zeros(256, dtype=torch.int64, device="cuda")
        ls = torch.zeros(1, dtype=torch.float64, device="cuda")
        for lo, hi in parts:
            off = d["gt_off"][lo:hi + 1]
            sc.sc_loss_fwd_bwd(ctx, sc.Batch(logits=d["logits"][lo:hi], gt_off=off, gt_lab=d["gt_lab"]),
                               loss_sum=ls, n_incorrect=ni, hist_pred=hp, hist_gt=hg)
        torch.cuda.synchronize()
        return ni.cpu(), hp.cpu(), hg.cpu(), ls.cpu()

    whole = agg([(0, 2000)])
    parts = agg([(0, 613), (613, 1500), (1500, 2000)])
    for a, b in zip(whole[:3], parts[:3]):
        assert torch.equal(a, b)
    assert float(parts[3]) == pytest.approx(float(whole[3]), rel=1e-12)


def test_edge_cases_and_errors():
    torch, sc, synth, _ = _mods()
    ctx = sc.Context(10, [[1, 2], [3]])
    lg = torch.zeros(0, 12, dtype=torch.float32, device="cuda")
    sc.sc_decide(ctx, sc.Batch(logits=lg))  # rows = 0: no-op
    with pytest.raises(sc.ScError):  # counters without GT
        sc.sc_decide(ctx, sc.Batch(logits=torch.zeros(4, 12, device="cuda")),
                     n_incorrect=torch.zeros(1, dtype=torch.int64, device="cuda"))
    with pytest.raises(sc.ScError):  # ld*4 % 16 != 0
        sc.sc_decide(ctx, sc.Batch(logits=torch.zeros(4, 10, device="cuda")))
    with pytest.raises(sc.ScError):  # ld < C
        sc.sc_decide(ctx, sc.Batch(logits=torch.zeros(4, 8, device="cuda")))
    with pytest.raises(sc.ScError):
        sc.Context(10, [[1, 10]])  # label out of range
    with pytest.raises(sc.ScError):
        sc.Context(10, [[1]] * 9)  # > 8 lists
    with pytest.raises(sc.ScError):
        sc.Context(10, [[1]], order=7)
    with pytest.raises(ValueError):
        sc.sc_decide(ctx, sc.Batch(logits=torch.zeros(4, 12)))  # CPU tensor: no fallback
    # decisions only (no GT) on one row
    dec = torch.empty(1, dtype=torch.uint8, device="cuda")
    z = torch.full((1, 12), -1.0, device="cuda")
    z[0, 3] = 2.0
    z[0, 1] = 1.0
    sc.sc_decide(ctx, sc.Batch(logits=z), decision=dec)
    assert int(dec.item()) == 1


def test_evaluator_step_matches_oracle():
    torch, sc, synth, Oracle = _mods()
    from paper_2310_07240_b200.step import Evaluator
    spec = synth.config_context(2)
    wl = synth.Workload(spec, seed=2)
    b = wl.host_batch(4242, 4000)
    d = to_dev(b, "f32")
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    ev = Evaluator(ctx, 4000, want_loss_row=True)
    o = ev.step(d["logits"], d["gt_off"], d["gt_lab"])
    torch.cuda.synchronize()
    ref, _ = run_oracle(spec, b, 1.0 / 4000)
    np.testing.assert_array_equal(o.decision[:4000].cpu().numpy(), ref["decision"])
    np.testing.assert_array_equal(o.hist_gt.cpu().numpy().astype(np.uint64), ref["hist_gt"])
    np.testing.assert_array_equal(o.n_incorrect(1).cpu().numpy().astype(np.uint64), ref["n_incorrect"])
    np.testing.assert_array_equal(o.hist_pred(1).cpu().numpy().reshape(-1).astype(np.uint64), ref["hist_pred"])
    np.testing.assert_allclose(o.loss_sum.cpu().numpy(), ref["loss_sum"], rtol=RTOL)
    np.testing.assert_allclose(o.grad_val[:8000].cpu().numpy(), ref["grad_val"], rtol=RTOL, atol=0)


def test_step_host_matches_device_step():
    """The end-to-end API (pinned host buffers, chunked H2D overlapped with the kernel)
    returns exactly what the device-resident step returns."""
    torch, sc, synth, _ = _mods()
    from paper_2310_07240_b200.step import Evaluator
    spec = synth.config_context(4)
    wl = synth.Workload(spec, seed=4, layout=1)
    rows = 20000
    b = wl.host_batch(0, rows)
    d = to_dev(b, "f32")
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    ev = Evaluator(ctx, rows)
    o = ev.step(d["logits"], d["gt_off"], d["gt_lab"], app=d["app"])
    torch.cuda.synchronize()
    ref = {k: getattr(o, k)[: (2 * rows if k.startswith("grad") else rows)].clone()
           for k in ("decision", "grad_idx", "grad_val")}
    ref_counts, ref_hist, ref_loss = o.counts.clone(), o.hist_gt.clone(), o.loss_sum.clone()
    h_logits = torch.from_numpy(b["logits"]).pin_memory()
    h_off = torch.from_numpy(b["gt_off"]).pin_memory()
    h_lab = torch.from_numpy(b["gt_lab"]).pin_memory()
    h_app = torch.from_numpy(b["app"].view(np.int16)).pin_memory()
    out = ev.host_outputs(rows)
    ev.step_host(h_logits, h_off, h_lab, out, h_app=h_app, chunk_rows=3000)
    assert torch.equal(out["decision"][:rows], ref["decision"].cpu())
    assert torch.equal(out["grad_idx"][: 2 * rows], ref["grad_idx"].cpu())
    assert torch.equal(out["grad_val"][: 2 * rows], ref["grad_val"].cpu())
    assert torch.equal(out["counts"], ref_counts.cpu())
    assert torch.equal(out["hist_gt"], ref_hist.cpu())
    np.testing.assert_allclose(out["loss_sum"].numpy(), ref_loss.cpu().numpy(), rtol=1e-12)


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_fused_hist_weights_matches_two_launches(cfg):
    """sc_decision_hist_weights (weights from the pre-pass's last CTA) == hist + weights kernels;
    repeated calls reuse the context's completion counter."""
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg, layout=1)
    b = wl.host_batch(0, 5000)
    d = to_dev(b, "f32")
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    na = spec.n_apps
    app = d.get("app")
    batch = sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], app=app, rows=5000)
    h1 = torch.zeros(na * 256, dtype=torch.int64, device="cuda")
    w1 = torch.empty(na * 256, dtype=torch.float32, device="cuda")
    m1 = torch.empty(5000, dtype=torch.uint8, device="cuda")
    sc.sc_decision_hist(ctx, batch, hist_gt=h1, gt_mask_out=m1)
    sc.sc_weights_from_hist(ctx, h1, w1)
    for rep in range(3):
        h2 = torch.zeros(na * 256, dtype=torch.int64, device="cuda")
        w2 = torch.full((na * 256,), -1.0, dtype=torch.float32, device="cuda")
        m2 = torch.empty(5000, dtype=torch.uint8, device="cuda")
        sc.sc_decision_hist_weights(ctx, batch, h2, w2, gt_mask_out=m2)
        torch.cuda.synchronize()
        assert torch.equal(h1, h2) and torch.equal(m1, m2) and torch.equal(w1, w2)


def test_hist_weights_concurrent_streams():
    """sc_decision_hist_weights on two streams at once with one context: each stream has its
    own completion counter, so both get the weights of their own histogram."""
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(2)
    wl = synth.Workload(spec, seed=2)
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    streams = [torch.cuda.Stream() for _ in range(3)]
    batches = []
    for i, rows in enumerate((50000, 70001, 1)):
        b = wl.host_batch(1000 * i, rows)
        d = to_dev(b, "f32")
        batches.append(sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], rows=rows))
    ref = []
    for bt in batches:  # two launches, one at a time
        h = torch.zeros(256, dtype=torch.int64, device="cuda")
        w = torch.empty(256, dtype=torch.float32, device="cuda")
        sc.sc_decision_hist(ctx, bt, hist_gt=h)
        sc.sc_weights_from_hist(ctx, h, w)
        ref.append((h, w))
    torch.cuda.synchronize()
    for rep in range(20):
        outs = []
        for st, bt in zip(streams, batches):
            with torch.cuda.stream(st):
                h = torch.zeros(256, dtype=torch.int64, device="cuda")
                w = torch.full((256,), -1.0, dtype=torch.float32, device="cuda")
                sc.sc_decision_hist_weights(ctx, bt, h, w)
                outs.append((h, w))
        torch.cuda.synchronize()
        for (h, w), (hr, wr) in zip(outs, ref):
            assert torch.equal(h, hr) and torch.equal(w, wr), rep


@pytest.mark.parametrize("mask_off,app_off", [(0, 0), (3, 1), (15, 7), (1, 0)])
def test_unaligned_side_bands(mask_off, app_off, kernel):
    """gt_mask / app at any offset: the ring bulk-copies only the 16-B-aligned interior of
    each unit's window and reads the ragged rows from global memory (no byte outside the
    arrays is read; compute-sanitizer memcheck runs this test)."""
    torch, sc, synth, Oracle = _mods()
    spec = synth.config_context(4)
    wl = synth.Workload(spec, seed=4, layout=1)
    rows = 3001
    b = wl.host_batch(77, rows)
    d = to_dev(b, "f32")
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    gbuf = torch.empty(rows + mask_off, dtype=torch.uint8, device="cuda")
    gm = gbuf[mask_off:]
    abuf = torch.empty(rows + app_off, dtype=torch.int16, device="cuda")
    ap = abuf[app_off:]
    ap.copy_(d["app"])
    h = torch.zeros(spec.n_apps * 256, dtype=torch.int64, device="cuda")
    sc.sc_decision_hist(ctx, sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], app=ap, rows=rows), hist_gt=h,
                        gt_mask_out=gm)
    w = torch.empty(spec.n_apps * 256, dtype=torch.float32, device="cuda")
    sc.sc_weights_from_hist(ctx, h, w)
    dec = torch.empty(rows, dtype=torch.uint8, device="cuda")
    ni = torch.zeros(spec.n_apps, dtype=torch.int64, device="cuda")
    ls = torch.zeros(spec.n_apps, dtype=torch.float64, device="cuda")
    gi = torch.empty(2 * rows, dtype=torch.int32, device="cuda")
    gv = torch.empty(2 * rows, dtype=torch.float32, device="cuda")
    sc.sc_loss_fwd_bwd(ctx, sc.Batch(logits=d["logits"], gt_mask=gm, app=ap), w=w, grad_scale=1.0 / rows,
                       loss_sum=ls, grad_idx=gi, grad_val=gv, decision=dec, n_incorrect=ni)
    torch.cuda.synchronize()
    o, _ = run_oracle(spec, b, 1.0 / rows, with_app=True)
    np.testing.assert_array_equal(dec.cpu().numpy(), o["decision"])
    np.testing.assert_array_equal(ni.cpu().numpy().astype(np.uint64), o["n_incorrect"])
    np.testing.assert_array_equal(gi.cpu().numpy(), o["grad_idx"])
    assert_rel(gv.cpu().numpy(), o["grad_val"], err_msg="grad_val")
    np.testing.assert_allclose(ls.cpu().numpy(), o["loss_sum"], rtol=RTOL)


@pytest.mark.parametrize("cfg,dtype,rows,mode,host_mode,chunk_rows,expect", [
    (2, "f32", 5000, "mask", 0, 1234, 1),     # dense context: AUTO copies (ragged last chunk)
    (2, "bf16", 3001, "csr", 1, 1000, 1),
    (3, "f32", 700, "mask", 0, 300, 2),       # sparse context (cfg3): AUTO reads the pinned rows in place
    (3, "bf16", 650, "csr", 1, 200, 1),
    (1, "f32", 4096, "csr", 2, 0, 2),         # ZERO_COPY needs no stager
    (4, "f32", 2000, "mask", 1, 512, 1),      # 256 applications, per-row app ids
])
def test_loss_fwd_bwd_host(cfg, dtype, rows, mode, host_mode, chunk_rows, expect):
    """sc_loss_fwd_bwd_host (C ABI, logits in pinned host memory): chunked double-buffered
    copies inside libsc, or zero copy, give exactly the oracle's outputs (same bar as the
    device path; dense gradients written chunk by chunk)."""
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg, dtype=dtype, layout=1)
    b = wl.host_batch(17, rows)
    multi = spec.n_apps > 1
    elt = 4 if dtype == "f32" else 2
    chunk = chunk_rows * synth.default_ld(spec.C, dtype) * elt
    g = run_gpu(spec, to_dev(b, dtype), mode=mode, dense=(cfg in (1, 2)), with_app=multi, host=(host_mode, chunk))
    assert g["host_mode"] == expect
    o, w = run_oracle(spec, b, g["grad_scale"], with_app=multi)
    compare(g, o, w, rows)


def test_loss_fwd_bwd_host_errors():
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(2)
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    lg = torch.zeros((64, 1000), dtype=torch.float32)  # pageable
    gm = torch.zeros(64, dtype=torch.uint8, device="cuda")
    dec = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(sc.ScError, match="page-locked"):
        sc.sc_loss_fwd_bwd_host(ctx, None, sc.Batch(logits=lg, gt_mask=gm), mode=sc.SC_HOST_ZERO_COPY, decision=dec)
    with pytest.raises(sc.ScError, match="stager"):
        sc.sc_loss_fwd_bwd_host(ctx, None, sc.Batch(logits=lg.pin_memory(), gt_mask=gm), mode=sc.SC_HOST_COPY,
                                decision=dec)
    with pytest.raises(sc.ScError, match="wider"):
        sc.sc_loss_fwd_bwd_host(ctx, sc.Stager(1024), sc.Batch(logits=lg.pin_memory(), gt_mask=gm),
                                mode=sc.SC_HOST_COPY, decision=dec)
    with pytest.raises(ValueError):  # device logits are not host logits
        sc.sc_loss_fwd_bwd_host(ctx, sc.Stager(1 << 20), sc.Batch(logits=lg.cuda(), gt_mask=gm), decision=dec)
    # pageable rows still work through the copy path (synchronous copies)
    used = sc.sc_loss_fwd_bwd_host(ctx, sc.Stager(1 << 20), sc.Batch(logits=lg, gt_mask=gm), decision=dec)
    torch.cuda.synchronize()
    assert used == sc.SC_HOST_COPY

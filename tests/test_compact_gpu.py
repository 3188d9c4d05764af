"""GPU parity of column-compacted logit rows (sc_context_load_compact).

For a sparse context (the OpenImages-shaped cfg3: |𝕎| = 1000 of C = 20000 labels)
a producer that writes only the mapped columns hands the path 20x fewer bytes.  Unmapped
labels never reach a decision, a count or the loss, and their gradient is exactly 0 (Eq.
api_output), so the outputs must be identical to the dense path's.  The
reference is the oracle on the DENSE rows (it knows nothing of compaction): the compacted
row is dense[:, cols] with cols = sc_context_columns.  Bar as everywhere: decisions,
counters, gradient indices (label ids) exact; loss / gradients 1e-5 relative.
"""
import numpy as np
import pytest

from conftest import gpu_available
from test_parity_gpu import assert_rel, compare, kernel, run_gpu, run_oracle, to_dev  # noqa: F401 (fixture)

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def compact_rows(b, cols, dtype):
    import synth
    n = len(cols)
    ldc = synth.default_ld(n, dtype)
    lg = b["logits"]
    out = np.full((lg.shape[0], ldc), np.nan if dtype == "f32" else 0x7FC0,
                  dtype=np.float32 if dtype == "f32" else np.uint16)
    out[:, :n] = lg[:, cols]
    c = dict(b)
    c["logits"] = out
    return c


def union_cols(spec):
    return np.nonzero(spec.mapped().any(axis=0))[0].astype(np.int32)


@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("cfg,dtype,row0,rows,mode", [
    (3, "f32", 31, 333, "mask"),
    (3, "bf16", 7, 250, "csr"),
    (2, "f32", 777, 2001, "mask"),
    (1, "f32", 0, 4096, "csr"),
    (4, "f32", (1 << 18) - 300, 700, "mask"),
])
def test_compact_equals_dense_oracle(order, cfg, dtype, row0, rows, mode, kernel):
    import paper_2310_07240_b200 as sc
    import synth
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg, dtype=dtype)
    b = wl.host_batch(row0, rows)
    cols = union_cols(spec)
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=order, multi_app=True, compact=True)
    np.testing.assert_array_equal(ctx.columns(), cols)
    bc = compact_rows(b, cols, dtype)
    multi = spec.n_apps > 1
    g = run_gpu(spec, to_dev(bc, dtype), mode=mode, with_app=multi, order=order, compact=True)
    o, w = run_oracle(spec, b, g["grad_scale"], with_app=multi, order=order)
    compare(g, o, w, rows)


def test_compact_dense_gradient_layout():
    """grad_dense of a compacted batch is laid out like its rows: column j = label cols[j]."""
    import torch
    import paper_2310_07240_b200 as sc
    import synth
    spec = synth.config_context(3)
    b = synth.Workload(spec, seed=3).host_batch(100, 200)
    cols = union_cols(spec)
    bc = compact_rows(b, cols, "f32")
    g = run_gpu(spec, to_dev(bc, "f32"), mode="csr", dense=False, compact=True)
    o, _ = run_oracle(spec, b, g["grad_scale"])
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, multi_app=True, compact=True)
    d = to_dev(bc, "f32")
    rows, ldc = bc["logits"].shape
    hist = torch.zeros(256, dtype=torch.int64, device="cuda")
    w = torch.empty(256, dtype=torch.float32, device="cuda")
    sc.sc_decision_hist_weights(ctx, sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], rows=rows), hist, w)
    gd = torch.full((rows * ldc,), 5.0, dtype=torch.float32, device="cuda")
    sc.sc_loss_fwd_bwd(ctx, sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"]), w=w,
                       grad_scale=g["grad_scale"], grad_dense=gd)
    torch.cuda.synchronize()
    pos = np.full(spec.C, -1, np.int64)
    pos[cols] = np.arange(len(cols))
    want = np.zeros((rows, ldc))
    gi, gv = o["grad_idx"].reshape(rows, 2), o["grad_val"].reshape(rows, 2)
    for s in range(2):
        m = gi[:, s] >= 0
        want[np.nonzero(m)[0], pos[gi[m, s]]] += gv[m, s]
    got = gd.cpu().numpy().reshape(rows, ldc)
    assert_rel(got.reshape(-1), want.reshape(-1), err_msg="grad_dense")


def test_compact_head_and_errors():
    """The fused head accepts a compacted context (its W rows are looked up by label);
    the all-apps pass (dense rows only) rejects it; ld must cover the compacted columns."""
    import torch
    import paper_2310_07240_b200 as sc
    import synth
    spec = synth.config_context(2)
    ctx = sc.Context(spec.C, spec.lists, multi_app=True, compact=True)
    assert len(ctx.columns()) == 180
    lg = torch.zeros(4, 176, device="cuda")
    with pytest.raises(sc.ScError):
        sc.sc_decide(ctx, sc.Batch(logits=lg))
    ctx4 = sc.Context(1000, synth.config_context(4).lists[:3], multi_app=True, compact=True)
    with pytest.raises(sc.ScError):
        sc.sc_decide_all_apps(ctx4, sc.Batch(logits=torch.zeros(4, 1000, device="cuda"),
                                             gt_off=torch.zeros(5, dtype=torch.int64, device="cuda"),
                                             gt_lab=torch.zeros(1, dtype=torch.int32, device="cuda")),
                              n_incorrect=torch.zeros(3, dtype=torch.int64, device="cuda"))
    from test_head_gpu import compare_exact, gt_for, oracle_eval, weights
    rows, d = 300, 128
    x, W, bias = synth.head_operands(spec.C, d, rows, seed=4, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, 4)
    wv = weights(spec, gt_off, gt_lab)
    head = sc.Head(ctx, torch.from_numpy(W.view(np.int16)).cuda().view(torch.bfloat16), torch.from_numpy(bias).cuda())
    o = dict(decision=torch.empty(rows, dtype=torch.uint8, device="cuda"),
             n_incorrect=torch.zeros(1, dtype=torch.int64, device="cuda"),
             hist_pred=torch.zeros(256, dtype=torch.int64, device="cuda"),
             hist_gt=torch.zeros(256, dtype=torch.int64, device="cuda"),
             loss_sum=torch.zeros(1, dtype=torch.float64, device="cuda"),
             loss_row=torch.empty(rows, dtype=torch.float32, device="cuda"),
             grad_idx=torch.empty(2 * rows, dtype=torch.int32, device="cuda"),
             grad_val=torch.empty(2 * rows, dtype=torch.float32, device="cuda"))
    sc.sc_head_loss_fwd_bwd(ctx, head, torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16),
                            gt_off=torch.from_numpy(gt_off).cuda(), gt_lab=torch.from_numpy(gt_lab).cuda(),
                            w=torch.from_numpy(wv).cuda(), grad_scale=1.0 / rows, **o)
    torch.cuda.synchronize()
    ref, _, _ = oracle_eval(spec, x, W, bias, gt_off, gt_lab, w=wv, grad_scale=1.0 / rows)
    compare_exact({k: v.cpu().numpy() for k, v in o.items()}, ref)


@pytest.mark.parametrize("C,dtype,rows", [(1, "f32", 100), (4, "f32", 333), (37, "f32", 1000), (128, "f32", 700),
                                          (129, "f32", 513), (257, "f32", 600), (1000, "f32", 999), (1024, "f32", 300),
                                          (8, "bf16", 257), (300, "bf16", 333), (1000, "bf16", 640),
                                          (1024, "bf16", 300)])
def test_dense_mapped_rows(C, dtype, rows, monkeypatch):
    """Rows whose every column is a mapped label of the one application (what a compacted
    context produces, and any context that maps every label) take the dense-mapped kernel
    (16-B vector loads per lane, winners tracked by slot index): tie-heavy values (integers,
    exactly tau, -0.0), every label mapped, overlapping lists, ragged last groups."""
    import paper_2310_07240_b200 as sc
    import synth
    from test_parity_gpu import tie_heavy_batch
    rng = np.random.default_rng(C * 13 + rows)
    if C <= 256:  # below the automatic threshold the lane-resident path runs: force the dense-mapped one
        monkeypatch.setenv("SC_DM", "2")
    for tau in (0.0, -1.0):
        D = int(rng.integers(1, 9))
        owner = rng.integers(0, D, size=C)
        lists = [sorted(np.nonzero(owner == j)[0].tolist()) for j in range(D)]
        for j in range(D):  # overlaps: a few labels repeated in a later list (first list wins, A5)
            lists[j] = sorted(set(lists[j]) | set(rng.integers(0, C, size=3).tolist()))
        spec = synth.ContextSpec(C, [lists], tau=tau, k=10.0)
        ld = synth.default_ld(C, dtype)
        b = tie_heavy_batch(rng, C, rows, ld, lists, tau)
        if dtype == "bf16":
            b["logits"] = synth.f32_to_bf16_bits(b["logits"])
        g = run_gpu(spec, to_dev(b, dtype), mode="mask" if tau == 0 else "csr", dense=True)
        assert sc.sc_last_kernel().startswith("tma_ring_dense_nv"), sc.sc_last_kernel()
        o, w = run_oracle(spec, b, g["grad_scale"])
        compare(g, o, w, rows)

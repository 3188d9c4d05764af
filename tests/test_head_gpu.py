"""GPU parity of the fused classifier head (sc_head_loss_fwd_bwd, NEXT f4) against the oracle.

The oracle computes the full logits z = x Wᵀ + b over all C labels (oracle.head_logits,
fp64) and evaluates them (Oracle.eval); the kernel computes only the |𝕎| mapped columns on
the tensor cores and evaluates them in the GEMM epilogue.

* Integer-valued operands (synth.head_operands kind="int"): every fp32 summation order
  gives the exact logits, so the bar is the path's own: decisions, G-dependent counters and
  histograms bit-exact, loss / gradients within 1e-5 relative, ties included (frequent).
* Gaussian operands (kind="normal"): the kernel's fp32 tensor-core sums and the oracle's
  fp64 sums differ by rounding; rows whose decision-relevant margins are below a rounding
  bound are set aside (< 3%), every other row must agree exactly on decision and gradient
  index and within 1e-4 relative on loss and gradient (reading A25).
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
    import oracle
    return torch, sc, synth, oracle


def bits_to_dev(bits, ld=None):
    torch, *_ = _mods()
    bits = np.ascontiguousarray(bits)
    if ld is not None and ld != bits.shape[1]:
        pad = np.zeros((bits.shape[0], ld), dtype=np.uint16)
        pad[:, : bits.shape[1]] = bits
        t = torch.from_numpy(pad.view(np.int16)).cuda().view(torch.bfloat16)
        return t[:, : bits.shape[1]]
    return torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)


def run_head(spec, x, W, b, gt_off, gt_lab, w=None, mode="csr", ldx=None, grad_scale=1.0, outputs=None, order=0):
    torch, sc, _, _ = _mods()
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=order, multi_app=True)
    S = ctx.grad_slots
    head = sc.Head(ctx, bits_to_dev(W), torch.from_numpy(b).cuda() if b is not None else None)
    rows = x.shape[0]
    xd = bits_to_dev(x, ldx)
    o = dict(
        decision=torch.full((rows,), 77, dtype=torch.uint8, device="cuda"),
        n_incorrect=torch.zeros(1, dtype=torch.int64, device="cuda"),
        hist_pred=torch.zeros(256, dtype=torch.int64, device="cuda"),
        hist_gt=torch.zeros(256, dtype=torch.int64, device="cuda"),
        loss_sum=torch.zeros(1, dtype=torch.float64, device="cuda"),
        loss_row=torch.full((rows,), -1.0, dtype=torch.float32, device="cuda"),
        grad_idx=torch.full((S * rows,), -7, dtype=torch.int32, device="cuda"),
        grad_val=torch.full((S * rows,), -7.0, dtype=torch.float32, device="cuda"),
    )
    if outputs is not None:
        o = {k: v for k, v in o.items() if k in outputs}
    go = torch.from_numpy(gt_off).cuda()
    gl = torch.from_numpy(gt_lab if len(gt_lab) else np.zeros(1, np.int32)).cuda()
    gmask = None
    if mode == "mask":
        gmask = torch.empty(rows, dtype=torch.uint8, device="cuda")
        sc.sc_decision_hist(ctx, sc.Batch(gt_off=go, gt_lab=gl, rows=rows), gt_mask_out=gmask)
        go = gl = None
    wd = torch.from_numpy(np.asarray(w, dtype=np.float32).reshape(-1)).cuda() if w is not None else None
    sc.sc_head_loss_fwd_bwd(ctx, head, xd, gt_off=go, gt_lab=gl, gt_mask=gmask, w=wd, grad_scale=grad_scale, **o)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in o.items()}
    res["n_cols"] = head.info()[1]
    return res


def oracle_eval(spec, x, W, b, gt_off, gt_lab, w=None, grad_scale=1.0, order=0):
    *_, oracle = _mods()
    z = oracle.head_logits(x, W, b)
    z32 = z.astype(np.float32)
    orc = oracle.Oracle.from_spec(spec, order)
    wo = None if w is None else np.asarray(w, dtype=np.float32).astype(np.float64)
    return orc.eval(z32, gt_off, gt_lab, w=wo, grad_scale=grad_scale), z, orc


def weights(spec, gt_off, gt_lab, order=0):
    *_, oracle = _mods()
    orc = oracle.Oracle.from_spec(spec, order)
    rows = len(gt_off) - 1
    pre = orc.eval(np.zeros((rows, spec.C), np.float32), gt_off, gt_lab, want_loss=False)
    return oracle.Oracle.weights_by_mask(pre["hist_gt"]).astype(np.float32).reshape(-1)


def compare_exact(g, o):
    np.testing.assert_array_equal(g["decision"], o["decision"])
    np.testing.assert_array_equal(g["hist_pred"].astype(np.uint64), o["hist_pred"][:256])
    np.testing.assert_array_equal(g["hist_gt"].astype(np.uint64), o["hist_gt"][:256])
    np.testing.assert_array_equal(g["n_incorrect"].astype(np.uint64), o["n_incorrect"])
    np.testing.assert_array_equal(g["grad_idx"], o["grad_idx"])
    np.testing.assert_allclose(g["loss_row"], o["loss_row"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(g["grad_val"], o["grad_val"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(g["loss_sum"], o["loss_sum"], rtol=RTOL, atol=0)


def custom_spec(C, sizes, seed):
    _, _, synth, _ = _mods()
    return synth.ContextSpec(C, [synth.placed_context(C, sizes, seed)], 0.0, 10.0)


def gt_for(spec, rows, seed):
    _, _, synth, _ = _mods()
    hb = synth.Workload(spec, seed=seed).host_batch(0, rows)
    return hb["gt_off"], hb["gt_lab"]


def explicit_spec(C, lists):
    _, _, synth, _ = _mods()
    return synth.ContextSpec(C, [[np.asarray(l, dtype=np.int32) for l in lists]], 0.0, 10.0)


# head columns: each list padded to 16, the total to 32 (sc_head_info)
SPECS = {
    "cfg1": lambda s: s.config_context(1),                      # (9,3,6) -> 16+16+16 -> 64 columns
    "cfg2": lambda s: s.config_context(2),                      # (90,30,60) -> 96+32+64 = 192
    "w256": lambda s: custom_spec(1000, (96, 96, 64), 9),       # 256 columns, one MMA, 2 accumulators
    "w300": lambda s: custom_spec(1000, (120, 100, 80), 10),    # 128+112+80 = 320: two MMAs of 160, one accumulator
    "w512": lambda s: custom_spec(1000, (192, 144, 96, 62), 11),  # 496 -> 512: two MMAs of 256
    "d8": lambda s: custom_spec(1000, (10, 20, 30, 5, 7, 3, 50, 1), 12),  # D' = 8 lists
    # overlapping lists (reading A5): list 1 keeps only 41..60, list 2 is empty, list 3 after it
    "ovl": lambda s: explicit_spec(300, [list(range(0, 41)), list(range(20, 61)), list(range(5, 30)),
                                         list(range(100, 117)) + [3]]),
}


@pytest.mark.parametrize("name,d,rows,mode", [
    ("cfg2", 2048, 1000, "csr"),
    ("cfg2", 2048, 1000, "mask"),
    ("cfg2", 64, 777, "csr"),
    ("cfg2", 200, 129, "csr"),
    ("cfg1", 512, 4096, "mask"),
    ("cfg1", 8, 300, "csr"),
    ("w256", 1024, 700, "csr"),
    ("w300", 1024, 700, "csr"),
    ("w512", 512, 513, "mask"),
    ("cfg2", 2048, 1, "csr"),
    ("d8", 256, 1500, "csr"),
    ("ovl", 192, 900, "mask"),
])
def test_head_exact(name, d, rows, mode):
    torch, sc, synth, _ = _mods()
    spec = SPECS[name](synth)
    x, W, b = synth.head_operands(spec.C, d, rows, seed=rows + d, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, seed=5)
    w = weights(spec, gt_off, gt_lab)
    gs = 1.0 / rows
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w, mode=mode, grad_scale=gs)
    o, z, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w, grad_scale=gs)
    assert np.all(z.astype(np.float32).astype(np.float64) == z)  # exact logits
    compare_exact(g, o)


def test_head_ties_pick_smallest_label():
    """All features zero: every logit equals its bias; biases with many equal values."""
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(2)
    rows, d = 300, 128
    x = np.zeros((rows, d), dtype=np.uint16)
    _, W, _ = synth.head_operands(spec.C, d, 1, seed=1, kind="int")
    rng = np.random.default_rng(3)
    b = (rng.integers(-2, 3, size=spec.C) / 4).astype(np.float32)
    gt_off, gt_lab = gt_for(spec, rows, seed=6)
    g = run_head(spec, x, W, b, gt_off, gt_lab)
    o, _, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab)
    compare_exact(g, o)


def test_head_ldx_padding_and_partial_outputs():
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(2)
    rows, d = 500, 136
    x, W, b = synth.head_operands(spec.C, d, rows, seed=8, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, seed=7)
    g = run_head(spec, x, W, b, gt_off, gt_lab, ldx=200)
    o, _, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab)
    compare_exact(g, o)
    # decisions only, no ground truth
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, multi_app=True)
    head = sc.Head(ctx, bits_to_dev(W), torch.from_numpy(b).cuda())
    dec = torch.zeros(rows, dtype=torch.uint8, device="cuda")
    hp = torch.zeros(256, dtype=torch.int64, device="cuda")
    sc.sc_head_loss_fwd_bwd(ctx, head, bits_to_dev(x), decision=dec, hist_pred=hp)
    np.testing.assert_array_equal(dec.cpu().numpy(), o["decision"])
    np.testing.assert_array_equal(hp.cpu().numpy().astype(np.uint64), o["hist_pred"][:256])
    # no bias: the oracle with b = 0
    head0 = sc.Head(ctx, bits_to_dev(W), None)
    sc.sc_head_loss_fwd_bwd(ctx, head0, bits_to_dev(x), decision=dec)
    o0, _, _ = oracle_eval(spec, x, W, None, gt_off, gt_lab)
    np.testing.assert_array_equal(dec.cpu().numpy(), o0["decision"])


def test_head_errors():
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(2)
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, multi_app=True)
    _, W, b = synth.head_operands(spec.C, 64, 1, seed=1, kind="int")
    head = sc.Head(ctx, bits_to_dev(W), torch.from_numpy(b).cuda())
    assert head.info() == (64, 192)
    assert sc.Head(ctx, bits_to_dev(synth.head_operands(spec.C, 8, 1, seed=1)[1]), None).info() == (8, 192)
    x = torch.zeros((10, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(sc.ScError):  # loss without ground truth
        sc.sc_head_loss_fwd_bwd(ctx, head, x, loss_row=torch.zeros(10, device="cuda"))
    with pytest.raises(sc.ScError):  # ldx % 8 != 0
        xb = torch.zeros((10, 67), dtype=torch.bfloat16, device="cuda")[:, :64]
        sc.sc_head_loss_fwd_bwd(ctx, head, xb, decision=torch.zeros(10, dtype=torch.uint8, device="cuda"))
    # empty batch is a no-op
    sc.sc_head_loss_fwd_bwd(ctx, head, x[:0], decision=torch.zeros(1, dtype=torch.uint8, device="cuda"))
    # a head compiled for one order, used with a context of another
    ctx_ac = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=sc.SC_ORDER_APP_CHOICE, multi_app=True)
    with pytest.raises(sc.ScError, match="INVALID"):
        sc.sc_head_loss_fwd_bwd(ctx_ac, head, x, decision=torch.zeros(10, dtype=torch.uint8, device="cuda"))
    # unsupported: several applications, more than 4096 head columns
    spec4 = synth.config_context(4)
    ctx4 = sc.Context(spec4.C, spec4.lists, spec4.tau, spec4.k, multi_app=True)
    with pytest.raises(sc.ScError, match="UNSUPPORTED"):
        sc.Head(ctx4, bits_to_dev(W), None)
    big = custom_spec(5000, (2500, 1700), 3)
    ctxb = sc.Context(big.C, big.lists, big.tau, big.k, multi_app=True)
    _, Wb, _ = synth.head_operands(big.C, 64, 1, seed=1, kind="int")
    with pytest.raises(sc.ScError, match="UNSUPPORTED"):
        sc.Head(ctxb, bits_to_dev(Wb), None)


@pytest.mark.parametrize("q", [1, 2, "2t2"])
@pytest.mark.parametrize("name,rows", [("cfg2", 148 * 128 * 2 + 1000), ("w300", 5000), ("cfg1", 300), ("w512", 700),
                                       ("cfg2", 148 * 512 + 777)])
def test_head_single_and_pair(q, name, rows, monkeypatch):
    """Lone CTAs (cta_group::1, M = 128, forced with SC_HEAD_CLUSTER=1) and CTA pairs
    (cta_group::2, M = 256, W halves in the two CTAs) with one row tile (SC_HEAD_PAIR_T2=0) or
    two ("2t2", the default where pairs fit: 512 rows per pass over W); unit counts that leave some CTAs without rows in the last step, odd tile
    counts (a pair's second CTA past the end)."""
    if q == "2t2":
        monkeypatch.setenv("SC_HEAD_PAIR_T2", "1")
        q = 2
    elif q == 2:
        monkeypatch.setenv("SC_HEAD_PAIR_T2", "0")  # pairs with one tile (double-buffered accumulators)
    torch, sc, synth, _ = _mods()
    spec = SPECS[name](synth)
    d = 320
    x, W, b = synth.head_operands(spec.C, d, rows, seed=q + rows, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, seed=q)
    w = weights(spec, gt_off, gt_lab)
    monkeypatch.setenv("SC_HEAD_CLUSTER", str(q))
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w, mode="mask", grad_scale=1.0 / rows)
    assert sc.sc_last_kernel() == ("head_tcgen05_pair" if q == 2 else "head_tcgen05")
    o, _, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w, grad_scale=1.0 / rows)
    compare_exact(g, o)


def margins_fragile(z, spec, G, tau, eps):
    """Rows where a decision-relevant comparison of mapped logits is within eps (per row)."""
    mapped = np.nonzero(spec.mapped()[0])[0]
    cat = {}
    for j, lst in enumerate(spec.lists[0]):
        for c in lst:
            cat.setdefault(int(c), j)
    cats = np.array([cat[int(c)] for c in mapped])
    zm = z[:, mapped]
    fragile = np.zeros(z.shape[0], dtype=bool)
    for i in range(z.shape[0]):
        plus = ((G[i] >> cats) & 1).astype(bool)
        vals = []
        for side in (plus, ~plus):
            s = np.sort(zm[i, side])[::-1]
            if len(s) >= 2 and s[0] - s[1] <= 2 * eps[i]:
                fragile[i] = True
            if len(s):
                vals.append(s[0])
        vals.append(tau)
        v = np.array(vals)
        dif = np.abs(v[:, None] - v[None, :])[np.triu_indices(len(v), 1)]
        if np.any(dif <= 2 * eps[i]):
            fragile[i] = True
    return fragile


def accumulation_bound(oracle, x, W, spec):
    """Per-row bound on |z_fp32 - z_exact| over the mapped columns: the MMA adds exact bf16
    products in groups of K = 16 into the fp32 accumulator, so at most d/16 + 16 roundings
    (a factor 2 allows truncation) of partial sums bounded by Σ_t |x_t w_t|, plus the bias add."""
    d = x.shape[1]
    absprod = np.abs(oracle.bf16_to_f64(x)) @ np.abs(oracle.bf16_to_f64(W)).T
    return (d / 16 + 32) * 2.0 ** -23 * absprod[:, spec.mapped()[0].astype(bool)].max(axis=1) + 1e-6


def test_head_normal_operands_margin_aware():
    torch, sc, synth, oracle = _mods()
    spec = synth.config_context(2)
    rows, d = 4096, 2048
    x, W, b = synth.head_operands(spec.C, d, rows, seed=21, kind="normal")
    gt_off, gt_lab = gt_for(spec, rows, seed=8)
    w = weights(spec, gt_off, gt_lab)
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w)
    o, z, orc = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w)
    eps = accumulation_bound(oracle, x, W, spec)
    fragile = margins_fragile(z, spec, o["gt_mask"], spec.tau, eps)
    assert fragile.mean() < 0.03, fragile.mean()
    ok = ~fragile
    np.testing.assert_array_equal(g["decision"][ok], o["decision"][ok])
    gi, oi = g["grad_idx"].reshape(rows, 2), o["grad_idx"].reshape(rows, 2)
    np.testing.assert_array_equal(gi[ok], oi[ok])
    np.testing.assert_allclose(g["loss_row"][ok], o["loss_row"][ok], rtol=1e-4, atol=1e-7)
    gv, ov = g["grad_val"].reshape(rows, 2), o["grad_val"].reshape(rows, 2)
    np.testing.assert_allclose(gv[ok], ov[ok], rtol=1e-4, atol=1e-7)
    # counters are consistent with the kernel's own decisions
    np.testing.assert_array_equal(g["hist_pred"], np.bincount(g["decision"], minlength=256))
    inc = sum(not orc.correct(int(G), int(dd)) for G, dd in zip(o["gt_mask"], g["decision"]))
    assert int(g["n_incorrect"][0]) == inc
    np.testing.assert_array_equal(g["hist_gt"].astype(np.uint64), o["hist_gt"][:256])


def test_head_fullsize_sampled():
    """1M rows x d=2048 (the bench's launch): sampled rows against the oracle, counters by
    consistency with the kernel's decisions and the oracle's G_i."""
    torch, sc, synth, oracle = _mods()
    spec = synth.config_context(2)
    rows, d = 1 << 20, 2048
    xd, Wd, bd = synth.head_operands_device(spec.C, d, rows, seed=2)
    wl = synth.Workload(spec, seed=2)
    dev = wl.device_batch(0, rows)
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, multi_app=True)
    head = sc.Head(ctx, Wd, bd)
    dec = torch.empty(rows, dtype=torch.uint8, device="cuda")
    lr = torch.empty(rows, dtype=torch.float32, device="cuda")
    gi = torch.empty(2 * rows, dtype=torch.int32, device="cuda")
    gv = torch.empty(2 * rows, dtype=torch.float32, device="cuda")
    ninc = torch.zeros(1, dtype=torch.int64, device="cuda")
    hp = torch.zeros(256, dtype=torch.int64, device="cuda")
    hg = torch.zeros(256, dtype=torch.int64, device="cuda")
    sc.sc_head_loss_fwd_bwd(ctx, head, xd, gt_off=dev["gt_off"], gt_lab=dev["gt_lab"], loss_row=lr, grad_idx=gi,
                            grad_val=gv, decision=dec, n_incorrect=ninc, hist_pred=hp, hist_gt=hg)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    idx = np.sort(np.concatenate([rng.choice(rows, 1500, replace=False), np.arange(rows - 200, rows)]))
    xs = xd[idx].view(torch.int16).cpu().numpy().view(np.uint16)
    Ws = Wd.view(torch.int16).cpu().numpy().view(np.uint16)
    bs = bd.cpu().numpy()
    hb = wl.host_batch(0, 1)  # noqa: F841 (warms the host generator)
    go = dev["gt_off"].cpu().numpy()
    gl = dev["gt_lab"].cpu().numpy()
    s_off = np.zeros(len(idx) + 1, dtype=np.int64)
    s_lab = []
    for j, i in enumerate(idx):
        s_lab.extend(gl[go[i]:go[i + 1]].tolist())
        s_off[j + 1] = len(s_lab)
    s_lab = np.asarray(s_lab, dtype=np.int32)
    o, z, orc = oracle_eval(spec, xs, Ws, bs, s_off, s_lab)
    ok = ~margins_fragile(z, spec, o["gt_mask"], spec.tau, accumulation_bound(oracle, xs, Ws, spec))
    assert ok.mean() > 0.97
    np.testing.assert_array_equal(dec.cpu().numpy()[idx][ok], o["decision"][ok])
    np.testing.assert_array_equal(gi.view(-1, 2).cpu().numpy()[idx][ok], o["grad_idx"].reshape(-1, 2)[ok])
    np.testing.assert_allclose(lr.cpu().numpy()[idx][ok], o["loss_row"][ok], rtol=1e-4, atol=1e-7)
    d_all = dec.cpu().numpy()
    np.testing.assert_array_equal(hp.cpu().numpy(), np.bincount(d_all, minlength=256))
    assert int(hg.sum()) == rows and int(hp.sum()) == rows


# more columns than TMEM holds: equal column passes of <= 256 columns, per-list maxima carried
# across passes (lists straddle pass boundaries)
WIDE = {
    "w560": lambda s: custom_spec(1000, (300, 250), 3),                    # 304+256 = 560 -> 3 passes x 192
    "cfg3": lambda s: s.config_context(3),                                 # |W| = 1000 of C = 20000: 1056 -> 5 x 224
    "w1100": lambda s: custom_spec(3000, (700, 10, 390), 4),               # 704+16+400 -> 5 passes x 224
}


@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("name,d,rows,mode", [
    ("cfg2", 256, 700, "mask"),
    ("cfg1", 64, 300, "csr"),
    ("ovl", 192, 900, "mask"),      # overlapping lists: Multi-Select columns repeat a label per list
    ("d8", 128, 1100, "csr"),
    ("w560", 128, 600, "mask"),
    ("cfg3", 192, 400, "mask"),
    ("w1100", 64, 333, "csr"),
])
def test_head_patterns_and_passes(order, name, d, rows, mode):
    """The head under every decision pattern (API-output order, application-choice order,
    Multi-Select) and with column passes (|𝕎| up to the OpenImages-shaped
    1000 mapped labels): exact integer logits, so the path's full bar."""
    torch, sc, synth, _ = _mods()
    spec = {**SPECS, **WIDE}[name](synth)
    x, W, b = synth.head_operands(spec.C, d, rows, seed=rows + d + order, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, seed=5 + order)
    w = weights(spec, gt_off, gt_lab, order)
    gs = 1.0 / rows
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w, mode=mode, grad_scale=gs, order=order)
    o, z, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w, grad_scale=gs, order=order)
    assert np.all(z.astype(np.float32).astype(np.float64) == z)  # exact logits
    if name in WIDE:
        assert g["n_cols"] > 512
    compare_exact(g, o)


@pytest.mark.parametrize("nchunk", [1, 2, 4])
@pytest.mark.parametrize("name,rows,q", [("cfg2", 5000, 1), ("w300", 3000, 1), ("w512", 700, 1), ("cfg2", 3000, 2),
                                         ("cfg1", 300, 1)])
def test_head_mma_chunks(nchunk, name, rows, q, monkeypatch):
    """The head's columns split into 1, 2 or 4 MMA chunks (SC_HEAD_NCHUNK), each its own
    accumulator chain: the same exact results (integer operands)."""
    torch, sc, synth, _ = _mods()
    spec = SPECS[name](synth)
    d = 192
    x, W, b = synth.head_operands(spec.C, d, rows, seed=nchunk + rows, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, seed=nchunk)
    w = weights(spec, gt_off, gt_lab)
    monkeypatch.setenv("SC_HEAD_NCHUNK", str(nchunk))
    monkeypatch.setenv("SC_HEAD_CLUSTER", str(q))
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w, mode="mask", grad_scale=1.0 / rows)
    o, _, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w, grad_scale=1.0 / rows)
    compare_exact(g, o)


@pytest.mark.parametrize("nchunk", [1, 2])
def test_head_mma_chunks_passes(nchunk, monkeypatch):
    torch, sc, synth, _ = _mods()
    spec = synth.config_context(3)
    rows, d = 300, 128
    x, W, b = synth.head_operands(spec.C, d, rows, seed=3 + nchunk, kind="int")
    gt_off, gt_lab = gt_for(spec, rows, seed=3)
    w = weights(spec, gt_off, gt_lab)
    monkeypatch.setenv("SC_HEAD_NCHUNK", str(nchunk))
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w, mode="mask", grad_scale=1.0 / rows)
    o, _, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w, grad_scale=1.0 / rows)
    compare_exact(g, o)

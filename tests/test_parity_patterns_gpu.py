"""GPU parity of the other decision patterns against the oracle:
Multi-Choice application-choice order (Eq. app_choice) and Multi-Select (Eq. multi-select).
Both kernels (the TMA ring with lane-resident entries, the sector-sparse gather) meet the
same bar as the hot path: decisions, G, counters and gradient indices bit-exact; loss and
gradient values within 1e-5 relative; overlapping lists exercise the two membership rules
(first list for the choice orders, every list for Multi-Select)."""
import numpy as np
import pytest

from conftest import gpu_available
from test_parity_gpu import compare, kernel, run_gpu, run_oracle, tie_heavy_batch, to_dev  # noqa: F401 (fixture)

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

APP_CHOICE, MULTI_SELECT = 1, 2


@pytest.mark.parametrize("order", [APP_CHOICE, MULTI_SELECT])
@pytest.mark.parametrize("cfg,dtype,row0,rows,mode,layout", [
    (1, "f32", 0, 4096, "mask", 0),
    (1, "bf16", 0, 4096, "csr", 0),
    (2, "f32", 777, 3001, "mask", 0),
    (2, "bf16", 5, 2049, "csr", 0),
    (3, "f32", 31, 203, "mask", 0),
    (4, "f32", (1 << 18) - 700, 1500, "mask", 0),
    (4, "bf16", 10, 999, "mask", 1),
])
def test_patterns_configs(order, cfg, dtype, row0, rows, mode, layout, kernel):
    import synth
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg, dtype=dtype, layout=layout)
    b = wl.host_batch(row0, rows)
    multi = spec.n_apps > 1
    g = run_gpu(spec, to_dev(b, dtype), mode=mode, dense=(cfg in (1, 2)), with_app=multi, order=order)
    o, w = run_oracle(spec, b, g["grad_scale"], with_app=multi, order=order)
    compare(g, o, w, rows)


@pytest.mark.parametrize("order", [APP_CHOICE, MULTI_SELECT])
@pytest.mark.parametrize("C,ld,rows", [(1, 4, 100), (4, 4, 333), (37, 40, 1000), (300, 300, 777), (4097, 4100, 97)])
def test_patterns_tie_heavy_overlapping(order, C, ld, rows, kernel):
    import synth
    rng = np.random.default_rng(C * 11 + rows + order)
    for tau in (0.0, -1.0):
        D = int(rng.integers(1, 9))
        lists = [sorted(set(rng.integers(0, C, size=int(rng.integers(0, min(C, 40) + 1))).tolist()))
                 for _ in range(D)]
        spec = synth.ContextSpec(C, [lists], tau=tau, k=float(rng.choice([1.0, 10.0, 25.0])))
        b = tie_heavy_batch(rng, C, rows, ld, lists, tau)
        g = run_gpu(spec, to_dev(b, "f32"), mode="mask" if tau == 0 else "csr", dense=C < 1000, order=order)
        o, w = run_oracle(spec, b, g["grad_scale"], order=order)
        compare(g, o, w, rows)


def test_true_false_patterns_agree_on_gpu(kernel):
    """One list: the three patterns give the same decisions (list 0 / its mask) and losses."""
    import torch
    import synth
    rng = np.random.default_rng(5)
    C, rows = 64, 2000
    W1 = sorted(set(rng.integers(0, C, size=12).tolist()))
    spec = synth.ContextSpec(C, [[W1]], tau=0.0, k=10.0)
    b = tie_heavy_batch(rng, C, rows, C, [W1], 0.0)
    res = {o: run_gpu(spec, to_dev(b, "f32"), order=o) for o in (0, APP_CHOICE, MULTI_SELECT)}
    d0 = res[0]["decision"]
    np.testing.assert_array_equal(res[APP_CHOICE]["decision"], d0)
    np.testing.assert_array_equal(res[MULTI_SELECT]["decision"], (d0 == 0).astype(np.uint8))
    for o in (APP_CHOICE, MULTI_SELECT):
        np.testing.assert_allclose(res[o]["loss_row"], res[0]["loss_row"], rtol=1e-6, atol=0)
        np.testing.assert_array_equal(res[o]["n_incorrect"], res[0]["n_incorrect"])


@pytest.mark.parametrize("order", [APP_CHOICE, MULTI_SELECT])
@pytest.mark.parametrize("sizes,shared", [
    ((32, 32, 32, 32, 32, 32, 32, 32), 0),   # exactly 8 list-major slots: the TMA ring's limit
    ((33, 1, 64, 31, 30), 0),                # 2 + 1 + 2 + 1 + 1 = 7 slots, ragged padding
    ((40, 40, 40, 40, 40), 0),               # 10 slots: falls back to the gather kernel
    ((30, 30, 30), 20),                      # overlapping lists: Multi-Select labels in several slots
])
def test_patterns_slot_layouts(order, sizes, shared, monkeypatch):
    """List-major slots (DevContext::lent): lists padded to 32 labels per slot, <= 8 slots on
    the TMA ring, more on the gather kernel; overlaps follow each pattern's membership rule."""
    import paper_2310_07240_b200 as sc
    import synth
    monkeypatch.setenv("SC_KERNEL", "tma")
    rng = np.random.default_rng(sum(sizes) * 7 + shared + order)
    C, rows = 700, 1500
    perm = rng.permutation(C)
    lists, pos = [], 0
    common = sorted(perm[:shared].tolist())
    pos = shared
    for n in sizes:
        own = perm[pos:pos + n].tolist()
        pos += n
        lists.append(sorted(set(own) | set(common)))
    spec = synth.ContextSpec(C, [lists], tau=0.0, k=10.0)
    b = tie_heavy_batch(rng, C, rows, C, lists, 0.0)
    g = run_gpu(spec, to_dev(b, "f32"), order=order)
    o, w = run_oracle(spec, b, g["grad_scale"], order=order)
    compare(g, o, w, rows)
    n_slots = sum((len(l) + 31) // 32 for l in lists) if order == MULTI_SELECT else None
    if order == MULTI_SELECT:
        want = "tma_ring_lists" if n_slots <= 8 else "gather_lists"
        assert sc.sc_last_kernel().startswith(want), (sc.sc_last_kernel(), n_slots)


@pytest.mark.parametrize("order", [0, APP_CHOICE, MULTI_SELECT])
@pytest.mark.parametrize("cfg,dtype,rows", [(2, "f32", 3000), (2, "bf16", 2001), (4, "f32", 1500)])
def test_decide_only_all_patterns(order, cfg, dtype, rows, kernel):
    """sc_decide (no loss): decisions and counters of every pattern on both kernels, with the
    ground truth as CSR (G built in the pass) — the epilogues' want_loss = 0 branch."""
    import torch
    import paper_2310_07240_b200 as sc
    import synth
    from oracle import Oracle
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg, dtype=dtype)
    b = wl.host_batch((1 << 18) - 500 if cfg == 4 else 99, rows)
    d = to_dev(b, dtype)
    multi = spec.n_apps > 1
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=order, multi_app=True)
    na = spec.n_apps
    dec = torch.full((rows,), 77, dtype=torch.uint8, device="cuda")
    ni = torch.zeros(na, dtype=torch.int64, device="cuda")
    hp = torch.zeros(na * 256, dtype=torch.int64, device="cuda")
    hg = torch.zeros(na * 256, dtype=torch.int64, device="cuda")
    sc.sc_decide(ctx, sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"],
                               app=d.get("app") if multi else None),
                 decision=dec, n_incorrect=ni, hist_pred=hp, hist_gt=hg)
    torch.cuda.synchronize()
    ref = Oracle.from_spec(spec, order).eval(b["logits"], b["gt_off"], b["gt_lab"], app=b["app"] if multi else None,
                                             want_loss=False)
    np.testing.assert_array_equal(dec.cpu().numpy(), ref["decision"])
    np.testing.assert_array_equal(ni.cpu().numpy().astype(np.uint64), ref["n_incorrect"])
    np.testing.assert_array_equal(hp.cpu().numpy().astype(np.uint64), ref["hist_pred"])
    np.testing.assert_array_equal(hg.cpu().numpy().astype(np.uint64), ref["hist_gt"])

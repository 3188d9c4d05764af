"""GPU parity of "one read, many contexts" (sc_decide_all_apps, NEXT f3): the decisions
of every row under every application equal the oracle's evaluation of each application
separately; counters exact."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def random_apps_spec(A, C, seed):
    """A applications with 0..8 overlapping lists of 0..60 labels (some with no mapped label)."""
    import synth
    rng = np.random.default_rng(seed)
    apps = []
    for _ in range(A):
        D = int(rng.integers(0, 9))
        apps.append([sorted(set(rng.integers(0, C, size=int(rng.integers(0, 61))).tolist())) for _ in range(D)])
    return synth.ContextSpec(C, apps, 0.0, 10.0)


@pytest.mark.parametrize("impl", ["rows", "lane", "warp"])
@pytest.mark.parametrize("cfg,dtype,rows", [(4, "f32", 600), (4, "bf16", 301), (4, "f32", 603),  # ragged unit tails
                                            ("r300", "f32", 257), ("r300", "bf16", 130), ("r33", "f32", 999),
                                            ("r40c1024", "f32", 95), ("r40c1024", "bf16", 64), ("r17c31", "bf16", 33)])
def test_all_apps_parity(impl, cfg, dtype, rows, monkeypatch):
    """The three kernels: lane per row (default for C <= 1024: 32-row units transposed in
    shared memory, applications in size order; C = 1024 fills the staging registers, odd C the
    bf16 column pairs), lane per application (SC_ALLAPPS=lane; applications grouped 32 at a
    time by size, a partial last group with cfg "r300" / "r33", applications with no mapped
    label) and warp per application (SC_ALLAPPS=warp)."""
    import torch
    import paper_2310_07240_b200 as sc
    import synth
    from oracle import Oracle
    from test_parity_gpu import to_dev
    if impl != "rows":
        monkeypatch.setenv("SC_ALLAPPS", impl)
    if cfg == 4:
        spec = synth.config_context(4)
    else:
        A, _, C = cfg[1:].partition("c")
        spec = random_apps_spec(int(A), int(C) if C else 997, seed=rows)
    wl = synth.Workload(spec, seed=4, dtype=dtype, layout=1)
    b = wl.host_batch(1234, rows)
    d = to_dev(b, dtype)
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    A = spec.n_apps
    ni = torch.zeros(A, dtype=torch.int64, device="cuda")
    hp = torch.zeros(A * 256, dtype=torch.int64, device="cuda")
    dec = torch.empty(rows * A, dtype=torch.uint8, device="cuda")
    sc.sc_decide_all_apps(ctx, sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"]),
                          n_incorrect=ni, hist_pred=hp, decision=dec)
    torch.cuda.synchronize()
    assert sc.sc_last_kernel() == "all_apps_" + impl
    dec = dec.cpu().numpy().reshape(rows, A)
    orc = Oracle.from_spec(spec)
    ni_ref = np.zeros(A, np.uint64)
    hp_ref = np.zeros(A * 256, np.uint64)
    for a in range(0, A, 1):
        r = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=np.full(rows, a, np.uint16), want_loss=False)
        np.testing.assert_array_equal(dec[:, a], r["decision"], err_msg=f"app {a}")
        ni_ref += r["n_incorrect"]
        hp_ref += r["hist_pred"]
    np.testing.assert_array_equal(ni.cpu().numpy().astype(np.uint64), ni_ref)
    np.testing.assert_array_equal(hp.cpu().numpy().astype(np.uint64), hp_ref)


def test_all_apps_wide_rows_fall_back():
    """C > 1024 columns: the lane-per-row kernel's staging does not hold a row, so the default
    is the lane-per-application kernel; same decisions."""
    import torch
    import paper_2310_07240_b200 as sc
    import synth
    from oracle import Oracle
    from test_parity_gpu import to_dev
    spec = random_apps_spec(20, 1500, seed=7)
    rows = 70
    wl = synth.Workload(spec, seed=4, dtype="f32", layout=1)
    b = wl.host_batch(0, rows)
    d = to_dev(b, "f32")
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    A = spec.n_apps
    ni = torch.zeros(A, dtype=torch.int64, device="cuda")
    hp = torch.zeros(A * 256, dtype=torch.int64, device="cuda")
    dec = torch.empty(rows * A, dtype=torch.uint8, device="cuda")
    sc.sc_decide_all_apps(ctx, sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"]),
                          n_incorrect=ni, hist_pred=hp, decision=dec)
    torch.cuda.synchronize()
    assert sc.sc_last_kernel() == "all_apps_lane"
    dec = dec.cpu().numpy().reshape(rows, A)
    orc = Oracle.from_spec(spec)
    for a in range(A):
        r = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=np.full(rows, a, np.uint16), want_loss=False)
        np.testing.assert_array_equal(dec[:, a], r["decision"], err_msg=f"app {a}")

"""GPU parity on large-magnitude logits: the σ-saturation regime ("what's missing" 5).

Why it matters: in fp32 σ(20) = σ(25) = 1.0f, so taking P⁺ / P⁻ as a max over p instead
of over z would move the arg max (reading A8); and σ'(z) = e^{-|z|}/(1+
e^{-|z|})² underflows to subnormals for |z| > ~87 and to 0 above ~104.  Mapped logits here
span ±[16, 120] (integers and bf16-exact values, so ties are frequent, including
σ-saturated ties such as z⁺ = 20 vs z⁻ = 25), mixed with small values so every branch of
the loss is reached.  Bar: decisions, G, counters and gradient indices bit-exact; loss and
gradient values 1e-5 relative, with SURVEY.md §8(c)9's absolute rule for entries whose
reference magnitude is below 1e-30 (`assert_rel` in test_parity_gpu.py).  Both eval
kernels, all three decision patterns, f32 and bf16; and the fused head (NEXT f4) with
integer operands plus a large bias, where every fp32 summation order is exact.
"""
import numpy as np
import pytest

from conftest import gpu_available
from test_parity_gpu import compare, kernel, run_gpu, run_oracle, to_dev  # noqa: F401 (fixture)

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

LARGE = np.array([16, 20, 25, 40, 64, 87, 88, 89, 100, 103, 104, 105, 110, 120], dtype=np.float32)


def large_batch(rng, C, rows, ld, dtype):
    kind = rng.random((rows, C))
    z = rng.integers(-2, 3, size=(rows, C)).astype(np.float32)            # small, tie-heavy
    sign = np.where(rng.random((rows, C)) < 0.5, -1.0, 1.0).astype(np.float32)
    m1 = kind < 0.45
    z[m1] = (sign * LARGE[rng.integers(0, len(LARGE), size=(rows, C))])[m1]   # exact large values: ties
    m2 = (kind >= 0.45) & (kind < 0.75)
    # uniform magnitudes in [16, 120) on a 1/16 grid
    z[m2] = (sign * (16 + rng.integers(0, 104 * 16, size=(rows, C)) / 16.0).astype(np.float32))[m2]
    if dtype == "bf16":  # keep the bf16-representable part (spacing 1/8 .. 1/2 above 16)
        z = (z.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    lg = np.full((rows, ld), np.nan, dtype=np.float32)
    lg[:, :C] = z
    n = rng.integers(0, 5, size=rows)
    off = np.zeros(rows + 1, dtype=np.int64)
    off[1:] = np.cumsum(n)
    lab = rng.integers(0, C, size=int(off[-1])).astype(np.int32)
    if dtype == "bf16":
        u = np.ascontiguousarray(lg).view(np.uint32)
        assert np.all((u[:, :C] & 0xFFFF) == 0), "values chosen bf16-exact"
        lg = (u >> 16).astype(np.uint16)
    return dict(logits=lg, gt_off=off, gt_lab=lab)


@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("C,rows", [(37, 3001), (300, 1500), (1000, 700)])
def test_large_logits_all_patterns(order, dtype, C, rows, kernel):
    import synth
    rng = np.random.default_rng(C * 31 + rows + 7 * order + (dtype == "bf16"))
    ld = synth.default_ld(C, dtype) + (8 if C == 37 else 0)
    tiny = False
    for tau in (0.0, 3.0, -1.0):
        D = int(rng.integers(1, 8))
        lists = [sorted(set(rng.integers(0, C, size=int(rng.integers(1, min(C, 60) + 1))).tolist()))
                 for _ in range(D)]
        spec = synth.ContextSpec(C, [lists], tau=tau, k=float(rng.choice([1.0, 10.0])))
        b = large_batch(rng, C, rows, ld, dtype)
        g = run_gpu(spec, to_dev(b, dtype), mode="mask" if tau == 0 else "csr", dense=(C < 1000 and dtype == "f32"),
                    order=order)
        o, w = run_oracle(spec, b, g["grad_scale"], order=order)
        compare(g, o, w, rows)
        # the regime is really exercised: gradients of saturated winners are subnormal or 0
        live = o["grad_idx"] >= 0
        tiny |= bool(np.any(np.abs(o["grad_val"][live]) < 1e-38))
    assert tiny


def test_sigma_saturated_tie_on_both_sides(kernel):
    """z⁺ = 20, z⁻ = 25 (σ(20) = σ(25) = 1.0f): the arg max over z picks the competitor, the
    decision follows it and the gradient goes to those two labels (reading A8)."""
    import synth
    C = 8
    spec = synth.ContextSpec(C, [[[0, 1], [2, 3]]], tau=0.0, k=10.0)
    z = np.full((4, C), -30.0, dtype=np.float32)
    z[0, 1], z[0, 2] = 20.0, 25.0   # GT list 0, competitor list 1 larger: incorrect
    z[1, 1], z[1, 2] = 25.0, 20.0   # GT list 0 larger: correct
    z[2, 0], z[2, 3] = 100.0, 100.0  # exact tie across lists: smaller id (0) wins
    z[3, 0], z[3, 2] = 120.0, -120.0
    off = np.array([0, 1, 2, 3, 4], dtype=np.int64)
    lab = np.array([0, 0, 3, 2], dtype=np.int32)
    b = dict(logits=z, gt_off=off, gt_lab=lab)
    g = run_gpu(spec, to_dev(b, "f32"), mode="csr", dense=True)
    o, w = run_oracle(spec, b, g["grad_scale"])
    compare(g, o, w, 4)
    assert list(g["decision"]) == [1, 0, 0, 0]
    assert list(g["grad_idx"][:2]) == [1, 2]


def test_head_large_bias():
    """Fused head (NEXT f4) with logits in ±[16, 120]: integer-valued operands and a large
    integer bias keep every fp32 summation order exact, so the bar is the path's own."""
    import synth
    from test_head_gpu import compare_exact, gt_for, oracle_eval, run_head, weights
    rng = np.random.default_rng(3)
    spec = synth.config_context(2)
    rows, d = 1000, 256
    x, W, b = synth.head_operands(spec.C, d, rows, seed=5, kind="int")
    b = (np.where(rng.random(spec.C) < 0.5, -1, 1) * rng.integers(16, 121, size=spec.C)).astype(np.float32)
    b[rng.random(spec.C) < 0.3] = 20.0  # many equal saturated logits: ties broken by label id
    gt_off, gt_lab = gt_for(spec, rows, 5)
    w = weights(spec, gt_off, gt_lab)
    g = run_head(spec, x, W, b, gt_off, gt_lab, w=w, mode="csr", grad_scale=1.0 / rows)
    o, z, _ = oracle_eval(spec, x, W, b, gt_off, gt_lab, w=w, grad_scale=1.0 / rows)
    assert np.abs(z[:, :]).max() > 100
    from test_parity_gpu import assert_rel
    np.testing.assert_array_equal(g["decision"], o["decision"])
    np.testing.assert_array_equal(g["grad_idx"], o["grad_idx"])
    np.testing.assert_array_equal(g["n_incorrect"].astype(np.uint64), o["n_incorrect"])
    np.testing.assert_array_equal(g["hist_pred"].astype(np.uint64), o["hist_pred"][:256])
    assert_rel(g["loss_row"], o["loss_row"], err_msg="loss_row")
    assert_rel(g["grad_val"], o["grad_val"], err_msg="grad_val")
    np.testing.assert_allclose(g["loss_sum"], o["loss_sum"], rtol=1e-5)
    del compare_exact

"""Pins of the classifier-head oracle, CPU.

* bf16 decoding: fixed bit patterns with known values (IEEE binary32 upper halves).
* head_logits: one-hot features give W's columns plus the bias (closed form); a triple
  loop over tiny shapes (brute force); the integer workload is exact in fp32 in any order.
* The property the fused kernel rests on: the evaluation depends on the logits of mapped
  labels only (labels in no list never decide; Eq. api_output
  reads maxima over 𝕎) — arbitrary values in unmapped columns leave
  every output unchanged.
"""
import numpy as np
import pytest

import synth
from oracle import API_OUTPUT, APP_CHOICE, MULTI_SELECT, Oracle, bf16_to_f64, head_logits


def test_bf16_decode_known_values():
    bits = np.array([0x3F80, 0xC020, 0x0000, 0x8000, 0x3E00, 0x4049, 0x7F80, 0xFF80], dtype=np.uint16)
    want = [1.0, -2.5, 0.0, -0.0, 0.125, 3.140625, np.inf, -np.inf]
    np.testing.assert_array_equal(bf16_to_f64(bits), want)
    assert np.signbit(bf16_to_f64(bits))[3]


def test_bf16_rounding_of_generator_is_nearest_even():
    vals = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -9, 3.0e-3], dtype=np.float32)
    got = bf16_to_f64(synth.f32_to_bf16_bits(vals))
    # 1+2^-8 is a tie between 1 and 1+2^-7 -> even (1); 1+3·2^-8 ties up to 1+2^-6
    np.testing.assert_array_equal(got[:4], [1.0, 1.0, 1.0 + 2 ** -6, -1.0])
    assert abs(got[4] - 3.0e-3) <= 3.0e-3 * 2 ** -8


def test_head_logits_one_hot_features_give_weight_columns():
    C, d = 13, 40
    _, W, b = synth.head_operands(C, d, 1, seed=3, kind="normal")
    one = synth.f32_to_bf16_bits(np.eye(d, dtype=np.float32))
    z = head_logits(one, W, b)
    np.testing.assert_array_equal(z, bf16_to_f64(W).T + b.astype(np.float64)[None, :])
    np.testing.assert_array_equal(head_logits(one, W), bf16_to_f64(W).T)


def test_head_logits_brute_force_tiny():
    rng = np.random.default_rng(7)
    for trial in range(20):
        rows, C, d = (int(v) for v in rng.integers(1, 6, size=3))
        x, W, b = synth.head_operands(C, d, rows, seed=100 + trial, kind="normal")
        xf, Wf = bf16_to_f64(x), bf16_to_f64(W)
        z = head_logits(x, W, b)
        for i in range(rows):
            for c in range(C):
                s = 0.0
                for t in range(d):
                    s += xf[i, t] * Wf[c, t]
                assert z[i, c] == pytest.approx(s + float(b[c]), rel=1e-12, abs=1e-12)


def test_integer_workload_is_exact_in_fp32_in_any_order():
    C, d, rows = 24, 2048, 6
    x, W, b = synth.head_operands(C, d, rows, seed=5, kind="int")
    z = head_logits(x, W, b)
    xf, Wf = bf16_to_f64(x).astype(np.float32), bf16_to_f64(W).astype(np.float32)
    rng = np.random.default_rng(0)
    for order in (np.arange(d), np.arange(d)[::-1], rng.permutation(d)):
        acc = np.zeros((rows, C), dtype=np.float32)
        for t in order:
            acc += xf[:, t : t + 1] * Wf[None, :, t]
        acc += b[None, :]
        np.testing.assert_array_equal(acc.astype(np.float64), z)
    assert np.all(z * 128 == np.round(z * 128))


@pytest.mark.parametrize("order", [API_OUTPUT, APP_CHOICE, MULTI_SELECT])
def test_evaluation_reads_mapped_columns_only(order):
    spec = synth.config_context(2)
    orc = Oracle.from_spec(spec, order=order)
    wl = synth.Workload(spec, seed=11)
    hb = wl.host_batch(0, 300)
    z = np.array(hb["logits"], dtype=np.float32)
    mapped = spec.mapped()[0].astype(bool)
    rng = np.random.default_rng(1)
    z2 = z.copy()
    z2[:, ~mapped] = rng.normal(0, 50, size=(z.shape[0], int((~mapped).sum()))).astype(np.float32)
    r1 = orc.eval(z, hb["gt_off"], hb["gt_lab"])
    r2 = orc.eval(z2, hb["gt_off"], hb["gt_lab"])
    for key in r1:
        np.testing.assert_array_equal(r1[key], r2[key], err_msg=key)
    # and the mapped columns do matter
    z3 = z.copy()
    z3[:, mapped] = rng.normal(0, 50, size=(z.shape[0], int(mapped.sum()))).astype(np.float32)
    assert not np.array_equal(orc.eval(z3, hb["gt_off"], hb["gt_lab"])["loss_row"], r1["loss_row"])

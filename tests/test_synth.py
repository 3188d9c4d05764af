"""The seeded input generator (harness): recipe properties on CPU, and the two
independent implementations (synth_host.c / synth_cuda.cu) agreeing bit for bit on GPU."""
import numpy as np
import pytest

import synth
from conftest import gpu_available


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_host_recipe_properties(dtype):
    ctx = synth.config_context(2)
    wl = synth.Workload(ctx, seed=2, dtype=dtype, ld=1008)
    b = wl.host_batch(0, 300)
    lg = b["logits"]
    if dtype == "bf16":
        lg = (lg.astype(np.uint32) << 16).view(np.float32)
    assert np.all(np.isnan(lg[:, 1000:]))
    z = lg[:, :1000].astype(np.float64)
    assert np.all(np.isfinite(z))
    step = 2.0 ** -12 if dtype == "f32" else 1.0 / 16
    assert np.all(np.abs(z / step - np.round(z / step)) == 0)
    lo = -12 if dtype == "f32" else -8
    assert z.min() >= lo and z.max() < (4 if dtype == "f32" else 8) + 8
    n = np.diff(b["gt_off"])
    assert n.min() >= 1 and n.max() <= 4
    assert b["gt_lab"].min() >= 0 and b["gt_lab"].max() < 1000
    mapped = ctx.mapped()[0]
    first = b["gt_lab"][b["gt_off"][:-1]]
    frac = mapped[first].mean()
    assert 0.4 < frac < 0.75  # 0.5 drawn from W plus 0.5 * 180/1000 by chance


def test_host_chunking_is_deterministic():
    wl = synth.Workload(synth.config_context(4), seed=4, layout=1)
    a = wl.host_batch(100, 64)
    b1, b2 = wl.host_batch(100, 30), wl.host_batch(130, 34)
    np.testing.assert_array_equal(a["logits"], np.concatenate([b1["logits"], b2["logits"]]))
    np.testing.assert_array_equal(a["gt_lab"], np.concatenate([b1["gt_lab"], b2["gt_lab"]]))
    np.testing.assert_array_equal(a["app"], np.arange(100, 164) % 256)


def test_heapsort_context_is_the_paper_listing():
    ctx = synth.heapsort_context()
    names = [[synth.HEAPSORT_NAMES[c] for c in l] for l in ctx.lists[0]]
    assert names[0] == ['plastic', 'wood', 'glass', 'paper', 'cardboard', 'metal', 'aluminum', 'tin', 'carton']
    assert names[1] == ['food', 'produce', 'snack']
    assert names[2] == ['clothing', 'jacket', 'shirt', 'pants', 'footwear', 'shoe']


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs CUDA")
@pytest.mark.parametrize("cfg,dtype,layout", [(1, "f32", 0), (2, "f32", 0), (2, "bf16", 0), (4, "f32", 1), (3, "bf16", 0)])
def test_cuda_generator_matches_host(cfg, dtype, layout):
    wl = synth.Workload(synth.config_context(cfg), seed=cfg, dtype=dtype, layout=layout)
    row0, n = 12345, 257
    h = wl.host_batch(row0, n)
    d = wl.device_batch(row0, n, with_app=True)
    np.testing.assert_array_equal(d["gt_off"].cpu().numpy(), h["gt_off"])
    np.testing.assert_array_equal(d["gt_lab"].cpu().numpy(), h["gt_lab"])
    np.testing.assert_array_equal(d["app"].cpu().numpy().view(np.uint16), h["app"])
    dl = d["logits"].cpu()
    dl = dl.numpy() if dtype == "f32" else dl.view(__import__("torch").int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(dl.view(np.uint32 if dtype == "f32" else np.uint16),
                                  h["logits"].view(np.uint32 if dtype == "f32" else np.uint16))

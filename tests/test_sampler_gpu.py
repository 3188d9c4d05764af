"""GPU parity of the rebalanced sampler (reading A24): for the same
uniforms the kernel draws exactly the oracle's rows (integer work: bit-exact)."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("rows,n,nmasks", [(1, 10, 1), (4097, 20000, 8), (100003, 300000, 256), (1 << 20, 1 << 20, 5)])
def test_sampler_bit_exact(rows, n, nmasks):
    import torch
    import oracle
    import paper_2310_07240_b200 as sc
    rng = np.random.default_rng(rows + n)
    mask = rng.integers(0, nmasks, size=rows).astype(np.uint8)
    w = np.zeros(256, dtype=np.float32)
    w[:nmasks] = rng.uniform(0.0, 5.0, nmasks).astype(np.float32)
    w[0] = 0.0 if nmasks > 2 else w[0]  # a zero-weight mask is never drawn
    if nmasks == 1:
        w[0] = 1.0
    u = rng.random(2 * n)
    ref = oracle.sample(mask, w, u[0::2], u[1::2])
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    sc.sc_rebalance_sample(torch.from_numpy(mask).cuda(), torch.from_numpy(w).cuda(), torch.from_numpy(u).cuda(), out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), ref)

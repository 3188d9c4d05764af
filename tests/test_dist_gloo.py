"""N > 1 host logic on CPU: world_size-2 gloo process group.

The multi-GPU step shards rows contiguously (step.shard_range), allreduces the
mask histogram before the weights (the global N_i of PAPER.md:2029) and the
aggregates after the loss pass (step.allreduce_).  Here each rank computes its
shard's per-rank partials with the CPU oracle (the kernels need a GPU) and the
product's shard/allreduce code combines them; the result must equal the
single-process evaluation of the whole batch (integers exactly, loss to 1e-12).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import Oracle
        from paper_2310_07240_b200.step import allreduce_, shard_range
        spec = synth.config_context(1)
        wl = synth.Workload(spec, seed=1)
        lo, hi = shard_range(rows, rank, world)
        b = wl.host_batch(lo, hi - lo)
        orc = Oracle.from_spec(spec)
        pre = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], want_loss=False)
        H = torch.from_numpy(pre["hist_gt"].astype(np.int64))
        allreduce_(H)                                       # global histogram before the weights
        w = Oracle.weights_by_mask(H.numpy().astype(np.uint64))
        r = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], w=w, grad_scale=1.0 / rows)
        counts = torch.from_numpy(np.concatenate([r["n_incorrect"], r["hist_pred"]]).astype(np.int64))
        loss = torch.from_numpy(r["loss_sum"].copy())
        allreduce_(counts)
        allreduce_(loss)
        if rank == 0:
            q.put((H.numpy(), counts.numpy(), loss.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2310_07240_b200.step import shard_range
    for rows in (0, 1, 7, 4096, 1 << 20):
        for world in (1, 2, 3, 8):
            parts = [shard_range(rows, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == rows
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_step_equals_single_process(world):
    import synth
    from oracle import Oracle
    rows = 3001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    H, counts, loss = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = synth.config_context(1)
    b = synth.Workload(spec, seed=1).host_batch(0, rows)
    orc = Oracle.from_spec(spec)
    pre = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], want_loss=False)
    w = Oracle.weights_by_mask(pre["hist_gt"])
    ref = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], w=w, grad_scale=1.0 / rows)
    np.testing.assert_array_equal(H.astype(np.uint64), ref["hist_gt"])
    np.testing.assert_array_equal(counts[:1].astype(np.uint64), ref["n_incorrect"])
    np.testing.assert_array_equal(counts[1:].astype(np.uint64), ref["hist_pred"])
    np.testing.assert_allclose(loss, ref["loss_sum"], rtol=1e-12)

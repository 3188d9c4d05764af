"""Multi-rank parity of the data-parallel step on the GPU.

World sizes 2 and 3 run as separate processes, all on cuda:0, over a gloo process
group with CUDA tensors (one GPU here; the step's collectives are the same calls as
over NCCL).  Each rank runs ``Evaluator.step`` (device buffers) or
``Evaluator.step_host`` (pinned host buffers) with the real libsc kernels on its
contiguous ``shard_range`` shard, ``global_rows`` = the whole batch.  The whole-batch
oracle is the reference:

* N_i counts over the whole training set, so every rank must end with
  the GLOBAL mask histogram and identical weights w = M/N;
* Eq. goal counts all inputs: n_incorrect, hist_pred and
  loss_sum (Eq. api_output) are global on every rank after the step;
* per-row outputs (decision, G_i, loss, gradient slots) concatenated over the ranks
  equal the whole-batch oracle's, element by element.

Bar: integers bit-exact, loss / gradients 1e-5 relative (north star).
"""
import os
import socket

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

RTOL = 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spec_and_workload(cfg, dtype):
    import synth
    spec = synth.config_context(cfg)
    # cfg4: 16 rows per application so a few thousand rows cover all 256 apps and the
    # shard boundaries fall inside an application's row block
    wl = synth.Workload(spec, seed=cfg, dtype=dtype, rows_per_app=16)
    return spec, wl


def _worker(rank, world, port, cfg, dtype, order, rows, mode, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_07240_b200 as sc
        from paper_2310_07240_b200.step import Evaluator, shard_range
        spec, wl = _spec_and_workload(cfg, dtype)
        lo, hi = shard_range(rows, rank, world)
        n = hi - lo
        b = wl.host_batch(lo, n)
        ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=order, multi_app=True)
        ev = Evaluator(ctx, n, want_loss_row=(mode == "step"))
        S = ctx.grad_slots
        if dtype == "bf16":
            h_logits = torch.from_numpy(np.ascontiguousarray(b["logits"]).view(np.int16)).view(torch.bfloat16)
        else:
            h_logits = torch.from_numpy(np.ascontiguousarray(b["logits"]))
        h_off = torch.from_numpy(b["gt_off"])
        h_lab = torch.from_numpy(b["gt_lab"] if len(b["gt_lab"]) else np.zeros(1, np.int32))
        h_app = torch.from_numpy(np.ascontiguousarray(b["app"]).view(np.int16)) if spec.n_apps > 1 else None
        na = spec.n_apps
        if mode == "step":
            o = ev.step(h_logits.cuda(), h_off.cuda(), h_lab.cuda(), app=None if h_app is None else h_app.cuda(),
                        global_rows=rows)
            torch.cuda.synchronize()
            res = dict(decision=o.decision[:n].cpu().numpy(), gt_mask=o.gt_mask[:n].cpu().numpy(),
                       grad_idx=o.grad_idx[:S * n].cpu().numpy(), grad_val=o.grad_val[:S * n].cpu().numpy(),
                       loss_row=o.loss_row[:n].cpu().numpy(), hist_gt=o.hist_gt.cpu().numpy(),
                       n_incorrect=o.n_incorrect(na).cpu().numpy(), hist_pred=o.hist_pred(na).cpu().numpy().reshape(-1),
                       loss_sum=o.loss_sum.cpu().numpy(), w=o.w.cpu().numpy())
        else:
            pin = lambda t: t.pin_memory()  # noqa: E731
            host_out = ev.host_outputs(max(n, 1))
            ev.step_host(pin(h_logits), pin(h_off), pin(h_lab), host_out,
                         h_app=None if h_app is None else pin(h_app), global_rows=rows, chunk_rows=1000)
            res = dict(decision=host_out["decision"][:n].numpy(), gt_mask=ev.out.gt_mask[:n].cpu().numpy(),
                       grad_idx=host_out["grad_idx"][:S * n].numpy(), grad_val=host_out["grad_val"][:S * n].numpy(),
                       hist_gt=host_out["hist_gt"].numpy(), n_incorrect=host_out["counts"][:na].numpy(),
                       hist_pred=host_out["counts"][na:].numpy(), loss_sum=host_out["loss_sum"].numpy(),
                       w=ev.out.w.cpu().numpy())
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, cfg, dtype, order, rows, mode, tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, dtype, order, rows, mode, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0] * world, f"rank exit codes {codes}"
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


CASES = [
    # (world, cfg, dtype, order, rows, mode)
    (2, 1, "f32", 0, 3001, "step"),
    (3, 1, "f32", 0, 3001, "step"),
    (3, 1, "f32", 0, 3001, "host"),
    (2, 2, "bf16", 0, 2049, "step"),
    (3, 2, "f32", 1, 1537, "step"),       # application-choice order
    (2, 2, "f32", 2, 1025, "step"),       # Multi-Select (8 gradient slots)
    (3, 4, "f32", 0, 4099, "step"),       # 256 applications, shard edges inside app blocks
    (2, 4, "f32", 0, 4099, "host"),
    (3, 1, "f32", 0, 2, "step"),          # one rank owns no rows
]


@pytest.mark.parametrize("world,cfg,dtype,order,rows,mode", CASES)
def test_sharded_step_equals_whole_batch_oracle(world, cfg, dtype, order, rows, mode, tmp_path):
    from oracle import Oracle
    res = _run(world, cfg, dtype, order, rows, mode, tmp_path)
    spec, wl = _spec_and_workload(cfg, dtype)
    b = wl.host_batch(0, rows)
    orc = Oracle.from_spec(spec, order=order)
    app = b["app"] if spec.n_apps > 1 else None
    _, H = orc.gt_hist(b["gt_off"], b["gt_lab"], app=app)
    w = Oracle.weights_by_mask(H)
    ref = orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=app, w=w, grad_scale=1.0 / rows)
    # aggregates: global and identical on every rank
    for r, o in enumerate(res):
        np.testing.assert_array_equal(o["hist_gt"].astype(np.uint64), ref["hist_gt"], err_msg=f"hist_gt rank {r}")
        np.testing.assert_array_equal(o["n_incorrect"].astype(np.uint64), ref["n_incorrect"], err_msg=f"rank {r}")
        np.testing.assert_array_equal(o["hist_pred"].astype(np.uint64), ref["hist_pred"], err_msg=f"rank {r}")
        np.testing.assert_allclose(o["loss_sum"], ref["loss_sum"], rtol=RTOL, atol=0, err_msg=f"loss_sum rank {r}")
        np.testing.assert_allclose(o["w"], w.reshape(-1).astype(np.float32), rtol=1e-7, err_msg=f"w rank {r}")
        np.testing.assert_array_equal(o["w"], res[0]["w"])
    # per-row outputs: concatenation over the ranks = the whole batch
    cat = {k: np.concatenate([o[k] for o in res]) for k in ("decision", "gt_mask", "grad_idx", "grad_val")}
    np.testing.assert_array_equal(cat["decision"], ref["decision"])
    np.testing.assert_array_equal(cat["gt_mask"], ref["gt_mask"])
    np.testing.assert_array_equal(cat["grad_idx"], ref["grad_idx"])
    np.testing.assert_allclose(cat["grad_val"], ref["grad_val"], rtol=RTOL, atol=0)
    if mode == "step":
        lr = np.concatenate([o["loss_row"] for o in res])
        np.testing.assert_allclose(lr, ref["loss_row"], rtol=RTOL, atol=0)
    assert int(ref["hist_gt"].sum()) == rows

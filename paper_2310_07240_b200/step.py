"""One data-parallel step of the hot path over the C ABI.

    sc_decision_hist  (GT only: G_i per row + mask histogram)
    -> all_reduce(hist_gt)                      [N > 1: the global N_i, PAPER.md:2029]
    -> sc_weights_from_hist                     (M/N per mask, identical on every rank)
    -> sc_loss_fwd_bwd (one read of the logits: decision, counters, loss, gradient)
    -> all_reduce(n_incorrect, hist_pred), all_reduce(loss_sum)   [N > 1]

Rows shard contiguously across ranks (``shard_range``); per-row outputs stay on
their rank and only the aggregates cross GPUs.  torch.distributed (NCCL on GPUs,
gloo in the CPU tests) is plumbing; every step of the path runs in libsc kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import (SC_HOST_AUTO, Batch, Context, Stager, sc_decision_hist, sc_decision_hist_weights, sc_loss_fwd_bwd,
               sc_loss_fwd_bwd_host, sc_weights_from_hist)


def shard_range(rows: int, rank: int, world: int):
    """Contiguous row shard [lo, hi) of rank `rank` (sizes differ by at most one row)."""
    base, rem = divmod(rows, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def _pg_active(group) -> bool:
    """A process group with > 1 rank is active (SC_FORCE_DIST=1: any initialised group, so the
    N > 1 step — collectives included — can be run with one rank on one GPU)."""
    import os

    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return False
    return dist.get_world_size(group) > 1 or os.environ.get("SC_FORCE_DIST") == "1"


def allreduce_(t: torch.Tensor, group=None):
    """Sum-allreduce in place when a process group with >1 rank is active (exact for int64)."""
    if _pg_active(group):
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_many_(tensors, group=None):
    """Several sum-allreduces; tensors of one dtype are issued as one NCCL group."""
    if not _pg_active(group):
        return tensors
    return _allreduce_list_(tensors, group)


def _allreduce_list_(tensors, group=None):
    # NCCL's coalesced allreduce requires identical dtypes ("Tensors must have identical
    # type", measured with NCCL 2.28 / torch 2.11): coalesce per dtype, int64 counters and
    # the fp64 loss go as separate collectives.
    import torch.distributed as dist
    cm = getattr(dist, "_coalescing_manager", None)
    by_dtype = {}
    for t in tensors:
        by_dtype.setdefault(t.dtype, []).append(t)
    for ts in by_dtype.values():
        if len(ts) > 1 and cm is not None and ts[0].is_cuda and dist.get_backend(group) == "nccl":
            with cm(group=group, device=ts[0].device):
                for t in ts:
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        else:
            for t in ts:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return tensors


@dataclass
class StepOutputs:
    decision: torch.Tensor     # uint8 [rows]       (this rank's rows)
    gt_mask: torch.Tensor      # uint8 [rows]
    grad_idx: torch.Tensor     # int32 [rows*S]  (S = ctx.grad_slots: 2, or 8 for Multi-Select)
    grad_val: torch.Tensor     # float32 [rows*S]
    hist_gt: torch.Tensor      # int64 [n_apps*256]  global after the step
    counts: torch.Tensor       # int64 [n_apps*257]  n_incorrect | hist_pred(256), global
    loss_sum: torch.Tensor     # float64 [n_apps]    global
    w: torch.Tensor            # float32 [n_apps*256]
    loss_row: torch.Tensor | None = None
    grad_dense: torch.Tensor | None = None

    def n_incorrect(self, n_apps: int):
        return self.counts[:n_apps]

    def hist_pred(self, n_apps: int):
        return self.counts[n_apps:].view(n_apps, 256)


class Evaluator:
    """Preallocated buffers + the step sequence for batches of up to `max_rows` rows."""

    def __init__(self, ctx: Context, max_rows: int, device="cuda", want_loss_row=False, dense_ld: int = 0,
                 group=None):
        self.ctx, self.group = ctx, group
        na = ctx.n_apps
        dev = torch.device(device)
        r = max(int(max_rows), 1)
        S = ctx.grad_slots
        self.S = S
        # every accumulator in one buffer so a step clears them with a single memset:
        # [hist_gt n_apps*256 | n_incorrect n_apps | hist_pred n_apps*256 | loss_sum n_apps (f64 bits)]
        self._acc = torch.zeros(na * 256 + na * 257 + na, dtype=torch.int64, device=dev)
        self.out = StepOutputs(
            decision=torch.empty(r, dtype=torch.uint8, device=dev),
            gt_mask=torch.empty(r + 16, dtype=torch.uint8, device=dev),
            grad_idx=torch.empty(S * r, dtype=torch.int32, device=dev),
            grad_val=torch.empty(S * r, dtype=torch.float32, device=dev),
            hist_gt=self._acc[:na * 256],
            counts=self._acc[na * 256:na * 513],
            loss_sum=self._acc[na * 513:].view(torch.float64),
            w=torch.empty(na * 256, dtype=torch.float32, device=dev),
            loss_row=torch.empty(r, dtype=torch.float32, device=dev) if want_loss_row else None,
            grad_dense=torch.empty(r * dense_ld, dtype=torch.float32, device=dev) if dense_ld else None,
        )

    def step(self, logits, gt_off, gt_lab, app=None, grad_scale: float | None = None, global_rows: int | None = None):
        o, ctx, na = self.out, self.ctx, self.ctx.n_apps
        rows = logits.shape[0]
        if grad_scale is None:
            grad_scale = 1.0 / max(1, global_rows if global_rows is not None else rows)
        self._acc.zero_()
        gt_batch = Batch(logits=None, gt_off=gt_off, gt_lab=gt_lab, app=app, rows=rows)
        if _pg_active(self.group) or na > 1:  # N_i needs the global histogram: allreduce in between
            sc_decision_hist(ctx, gt_batch, hist_gt=o.hist_gt, gt_mask_out=o.gt_mask)
            allreduce_(o.hist_gt, self.group)
            sc_weights_from_hist(ctx, o.hist_gt, o.w)  # one CTA per application
        else:                                  # one GPU, one app: weights from the pre-pass launch
            sc_decision_hist_weights(ctx, gt_batch, o.hist_gt, o.w, gt_mask_out=o.gt_mask)
        sc_loss_fwd_bwd(ctx, Batch(logits=logits, gt_mask=o.gt_mask, app=app), w=o.w, grad_scale=grad_scale,
                        loss_sum=o.loss_sum, loss_row=o.loss_row, grad_idx=o.grad_idx, grad_val=o.grad_val,
                        grad_dense=o.grad_dense, decision=o.decision, n_incorrect=o.counts[:na],
                        hist_pred=o.counts[na:])
        allreduce_many_([o.counts, o.loss_sum], self.group)
        return o

    # ---------------------------------------------------------------- end to end (host buffers)

    def host_outputs(self, rows: int):
        """Pinned host buffers for step_host's per-row results and aggregates."""
        na = self.ctx.n_apps
        pin = dict(pin_memory=True)
        S = self.S
        return dict(decision=torch.empty(rows, dtype=torch.uint8, **pin),
                    grad_idx=torch.empty(S * rows, dtype=torch.int32, **pin),
                    grad_val=torch.empty(S * rows, dtype=torch.float32, **pin),
                    counts=torch.empty(na * 257, dtype=torch.int64, **pin),
                    hist_gt=torch.empty(na * 256, dtype=torch.int64, **pin),
                    loss_sum=torch.empty(na, dtype=torch.float64, **pin))

    def step_host(self, h_logits, h_gt_off, h_gt_lab, host_out, h_app=None, grad_scale=None,
                  global_rows=None, chunk_rows: int = 1 << 16, host_mode: int = SC_HOST_AUTO):
        """The same step with inputs and outputs in (pinned) host memory.

        The small ground truth goes first (pre-pass + weights need all of it); the logits are
        then evaluated from host memory by sc_loss_fwd_bwd_host (C ABI): chunked host->device
        copies double-buffered against the pass inside libsc, or the kernels reading the
        pinned rows in place (sparse contexts); per-row results and aggregates come back."""
        o, ctx, na = self.out, self.ctx, self.ctx.n_apps
        dev = o.decision.device
        rows, C = h_logits.shape
        if grad_scale is None:
            grad_scale = 1.0 / max(1, global_rows if global_rows is not None else rows)
        row_bytes = h_logits.stride(0) * h_logits.element_size()
        if getattr(self, "_stager", None) is None or self._stager.chunk_bytes < chunk_rows * row_bytes:
            self._stager = Stager(chunk_rows * row_bytes)
        if getattr(self, "_d_off", None) is None or self._d_off.numel() < rows + 1 or \
                self._d_lab.numel() < h_gt_lab.numel():
            self._d_off = torch.empty(rows + 1, dtype=torch.int64, device=dev)
            self._d_lab = torch.empty(max(1, h_gt_lab.numel()), dtype=torch.int32, device=dev)
        if h_app is not None and (getattr(self, "_d_app", None) is None or self._d_app.numel() < rows):
            self._d_app = torch.empty(max(1, rows), dtype=torch.int16, device=dev)
        d_off = self._d_off[:rows + 1]
        d_off.copy_(h_gt_off, non_blocking=True)
        d_lab = self._d_lab[:h_gt_lab.numel()]
        d_lab.copy_(h_gt_lab, non_blocking=True)
        d_app = None
        if h_app is not None:
            d_app = self._d_app[:rows]
            d_app.copy_(h_app, non_blocking=True)
        self._acc.zero_()
        sc_decision_hist(ctx, Batch(gt_off=d_off, gt_lab=d_lab, app=d_app, rows=rows), hist_gt=o.hist_gt,
                         gt_mask_out=o.gt_mask)
        allreduce_(o.hist_gt, self.group)
        sc_weights_from_hist(ctx, o.hist_gt, o.w)
        self.host_mode_used = sc_loss_fwd_bwd_host(
            ctx, self._stager, Batch(logits=h_logits, gt_mask=o.gt_mask[:rows], app=d_app), mode=host_mode, w=o.w,
            grad_scale=grad_scale, loss_sum=o.loss_sum, grad_idx=o.grad_idx[:self.S * rows],
            grad_val=o.grad_val[:self.S * rows], decision=o.decision[:rows], n_incorrect=o.counts[:na],
            hist_pred=o.counts[na:])
        allreduce_many_([o.counts, o.loss_sum], self.group)
        host_out["decision"][:rows].copy_(o.decision[:rows], non_blocking=True)
        S = self.S
        host_out["grad_idx"][:S * rows].copy_(o.grad_idx[:S * rows], non_blocking=True)
        host_out["grad_val"][:S * rows].copy_(o.grad_val[:S * rows], non_blocking=True)
        host_out["counts"].copy_(o.counts, non_blocking=True)
        host_out["hist_gt"].copy_(o.hist_gt, non_blocking=True)
        host_out["loss_sum"].copy_(o.loss_sum, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return host_out

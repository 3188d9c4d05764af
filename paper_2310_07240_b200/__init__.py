"""paper_2310_07240_b200 — B200-native software-context evaluation (thin Python binding).

The hot path runs entirely in ``libsc.so`` (hand-written sm_100a CUDA behind the
C ABI in ``include/sc.h``).  This module only marshals torch tensors into that
ABI: it passes ``data_ptr()`` values and the current CUDA stream.  There is no
CPU fallback: if ``libsc.so`` is missing or a tensor is not on a CUDA device,
calls raise.

Names follow the ABI: ``sc_context_load``, ``sc_decide``, ``sc_decision_hist``,
``sc_weights_from_hist``, ``sc_loss_fwd_bwd``, ``sc_last_error``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

from . import build as _build

__all__ = [
    "ScError", "Context", "Batch", "sc_context_load", "sc_context_load_compact", "sc_context_columns",
    "sc_context_free", "sc_decide", "sc_decision_hist",
    "sc_weights_from_hist", "sc_decision_hist_weights", "sc_loss_fwd_bwd", "Head", "sc_head_load",
    "sc_head_loss_fwd_bwd", "sc_last_error", "sc_launch_count", "sc_last_kernel", "library_path",
    "Stager", "sc_loss_fwd_bwd_host", "SC_HOST_AUTO", "SC_HOST_COPY", "SC_HOST_ZERO_COPY",
]

SC_OK, SC_ERR_INVALID_ARG, SC_ERR_OOM, SC_ERR_CUDA, SC_ERR_UNSUPPORTED = range(5)
_STATUS = {1: "SC_ERR_INVALID_ARG", 2: "SC_ERR_OOM", 3: "SC_ERR_CUDA", 4: "SC_ERR_UNSUPPORTED"}
SC_F32, SC_BF16 = 0, 1
SC_ORDER_API_OUTPUT, SC_ORDER_APP_CHOICE, SC_ORDER_MULTI_SELECT = 0, 1, 2


class ScError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class _CBatch(ctypes.Structure):
    _fields_ = [
        ("logits", ctypes.c_void_p),
        ("dtype", ctypes.c_int),
        ("rows", ctypes.c_int64),
        ("ld", ctypes.c_int64),
        ("gt_off", ctypes.c_void_p),
        ("gt_lab", ctypes.c_void_p),
        ("gt_mask", ctypes.c_void_p),
        ("app", ctypes.c_void_p),
    ]


class _CHeadBatch(ctypes.Structure):
    _fields_ = [
        ("x", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("ldx", ctypes.c_int64),
        ("gt_off", ctypes.c_void_p),
        ("gt_lab", ctypes.c_void_p),
        ("gt_mask", ctypes.c_void_p),
    ]


def library_path() -> str:
    return _build.SO


def _load():
    path = _build.SO
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing — build it with `python -m paper_2310_07240_b200.build` "
                          "or __graft_entry__.build(); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P, I32, I64, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    lib.sc_context_load.restype = ctypes.c_int
    lib.sc_context_load.argtypes = [I32, I32, P, P, P, F, F, ctypes.c_int, ctypes.POINTER(P)]
    lib.sc_context_load_compact.restype = ctypes.c_int
    lib.sc_context_load_compact.argtypes = [I32, I32, P, P, P, F, F, ctypes.c_int, ctypes.POINTER(P)]
    lib.sc_context_columns.restype = ctypes.c_int
    lib.sc_context_columns.argtypes = [P, P, ctypes.POINTER(I32)]
    lib.sc_context_free.restype = ctypes.c_int
    lib.sc_context_free.argtypes = [P]
    lib.sc_context_info.restype = ctypes.c_int
    lib.sc_context_info.argtypes = [P, I32, ctypes.POINTER(I32), ctypes.POINTER(I32)]
    lib.sc_context_order.restype = ctypes.c_int
    lib.sc_context_order.argtypes = [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(I32)]
    lib.sc_decide.restype = ctypes.c_int
    lib.sc_decide.argtypes = [P, ctypes.POINTER(_CBatch), P, P, P, P, P]
    lib.sc_decision_hist.restype = ctypes.c_int
    lib.sc_decision_hist.argtypes = [P, ctypes.POINTER(_CBatch), P, P, P]
    lib.sc_decision_hist_weights.restype = ctypes.c_int
    lib.sc_decision_hist_weights.argtypes = [P, ctypes.POINTER(_CBatch), P, P, P, P]
    lib.sc_decide_all_apps.restype = ctypes.c_int
    lib.sc_decide_all_apps.argtypes = [P, ctypes.POINTER(_CBatch), P, P, P, P]
    lib.sc_weights_from_hist.restype = ctypes.c_int
    lib.sc_weights_from_hist.argtypes = [P, P, P, P]
    lib.sc_loss_fwd_bwd.restype = ctypes.c_int
    lib.sc_loss_fwd_bwd.argtypes = [P, ctypes.POINTER(_CBatch), P, F, P, P, P, P, P, P, P, P, P, P]
    lib.sc_stager_create.restype = ctypes.c_int
    lib.sc_stager_create.argtypes = [I64, ctypes.POINTER(P)]
    lib.sc_stager_free.restype = ctypes.c_int
    lib.sc_stager_free.argtypes = [P]
    lib.sc_loss_fwd_bwd_host.restype = ctypes.c_int
    lib.sc_loss_fwd_bwd_host.argtypes = [P, P, ctypes.POINTER(_CBatch), I32, P, F, P, P, P, P, P, P, P, P, P,
                                         ctypes.POINTER(I32), P]
    lib.sc_last_error.restype = ctypes.c_char_p
    lib.sc_last_error.argtypes = []
    lib.sc_launch_count.restype = ctypes.c_uint64
    lib.sc_launch_count.argtypes = []
    lib.sc_last_kernel.restype = ctypes.c_char_p
    lib.sc_last_kernel.argtypes = []
    F32 = ctypes.c_float
    lib.sc_ranges_load.restype = ctypes.c_int
    lib.sc_ranges_load.argtypes = [I32, P, P, F32, ctypes.POINTER(P)]
    lib.sc_ranges_free.restype = ctypes.c_int
    lib.sc_ranges_free.argtypes = [P]
    lib.sc_ranges_hist.restype = ctypes.c_int
    lib.sc_ranges_hist.argtypes = [P, P, I64, P, P, P]
    lib.sc_ranges_weights.restype = ctypes.c_int
    lib.sc_ranges_weights.argtypes = [P, P, P, P]
    lib.sc_ranges_loss_fwd_bwd.restype = ctypes.c_int
    lib.sc_ranges_loss_fwd_bwd.argtypes = [P, P, P, I64, P, F32, P, P, P, P, P, P, P]
    lib.sc_ranges_last_error.restype = ctypes.c_char_p
    lib.sc_ranges_last_error.argtypes = []
    lib.sc_sample_workspace_bytes.restype = ctypes.c_size_t
    lib.sc_sample_workspace_bytes.argtypes = [I64]
    lib.sc_rebalance_sample.restype = ctypes.c_int
    lib.sc_rebalance_sample.argtypes = [P, I64, P, P, I64, P, P, ctypes.c_size_t, P]
    lib.sc_sample_last_error.restype = ctypes.c_char_p
    lib.sc_sample_last_error.argtypes = []
    lib.sc_head_load.restype = ctypes.c_int
    lib.sc_head_load.argtypes = [P, P, I64, I64, P, P, ctypes.POINTER(P)]
    lib.sc_head_free.restype = ctypes.c_int
    lib.sc_head_free.argtypes = [P]
    lib.sc_head_info.restype = ctypes.c_int
    lib.sc_head_info.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I32)]
    lib.sc_head_loss_fwd_bwd.restype = ctypes.c_int
    lib.sc_head_loss_fwd_bwd.argtypes = [P, P, ctypes.POINTER(_CHeadBatch), P, F, P, P, P, P, P, P, P, P, P]
    return lib


_lib = _load()


def sc_last_error() -> str:
    return _lib.sc_last_error().decode()


def sc_launch_count() -> int:
    return int(_lib.sc_launch_count())


def sc_last_kernel() -> str:
    return _lib.sc_last_kernel().decode()


def _check(status: int):
    if status != SC_OK:
        raise ScError(status, sc_last_error())


# ------------------------------------------------------------------ marshalling helpers

def _torch():
    import torch
    return torch


def _dev_ptr(t, name: str, dtypes, numel: Optional[int] = None):
    """data_ptr() of a CUDA tensor after checking dtype / device / contiguity; None -> NULL."""
    if t is None:
        return None
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype not in dtypes:
        raise TypeError(f"{name}: dtype {t.dtype} not in {dtypes}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {numel}")
    return t.data_ptr()


def _stream(stream):
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ------------------------------------------------------------------ context

def _nesting(x) -> int:
    """1 + depth of the first non-empty nesting (labels are depth 1)."""
    if isinstance(x, (list, tuple)) or hasattr(x, "__len__") and not isinstance(x, (str, bytes)) and hasattr(x, "__iter__"):
        for e in x:
            return 1 + _nesting(e)
        return 1
    return 0


class Context:
    """Handle to an uploaded software context (``sc_context``).

    ``lists[a][j]`` are the label ids of list W_j of application a, in code order
    (e.g. Heapsortcypher: Recycle, Compost, Donate).  For a single
    application ``lists`` may be given as a list of lists."""

    def __init__(self, C: int, lists, tau: float = 0.0, k: float = 10.0, order: int = SC_ORDER_API_OUTPUT,
                 multi_app: Optional[bool] = None, compact: bool = False):
        if multi_app is None:
            multi_app = _nesting(lists) >= 3
        if not multi_app:
            lists = [lists]
        n_lists, off, labels = [], [], []
        pos = 0
        for app in lists:
            n_lists.append(len(app))
            off.append(pos)
            for l in app:
                labels.extend(int(c) for c in l)
                pos += len(l)
                off.append(pos)
        self.C, self.n_apps, self.tau, self.k = int(C), len(lists), float(tau), float(k)
        self.order = int(order)
        self.lists = lists
        a_n = (ctypes.c_int32 * max(1, len(n_lists)))(*n_lists)
        a_off = (ctypes.c_int64 * max(1, len(off)))(*off)
        a_lab = (ctypes.c_int32 * max(1, len(labels)))(*labels)
        h = ctypes.c_void_p()
        load = _lib.sc_context_load_compact if compact else _lib.sc_context_load
        _check(load(self.C, self.n_apps, a_n, a_off, a_lab, self.tau, self.k, order, ctypes.byref(h)))
        self._h = h
        self.compact = bool(compact)

    def columns(self):
        """Labels of the logit columns a batch row holds (sc_context_columns): arange(C) for a
        dense context, the ascending union of the mapped labels for a compacted one."""
        import numpy as np
        n = ctypes.c_int32()
        _check(_lib.sc_context_columns(self._h, None, ctypes.byref(n)))
        cols = np.empty(max(n.value, 1), dtype=np.int32)
        _check(_lib.sc_context_columns(self._h, cols.ctypes.data, ctypes.byref(n)))
        return cols[: n.value]

    @property
    def handle(self):
        return self._h

    @property
    def grad_slots(self) -> int:
        """Sparse-gradient entries per row: 2 (Multi-Choice orders) or 8 (Multi-Select)."""
        o, g = ctypes.c_int(), ctypes.c_int32()
        _check(_lib.sc_context_order(self._h, ctypes.byref(o), ctypes.byref(g)))
        return g.value

    def n_lists(self, app: int = 0) -> int:
        n, m = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.sc_context_info(self._h, app, ctypes.byref(n), ctypes.byref(m)))
        return n.value

    def n_mapped(self, app: int = 0) -> int:
        n, m = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.sc_context_info(self._h, app, ctypes.byref(n), ctypes.byref(m)))
        return m.value

    def free(self):
        if getattr(self, "_h", None):
            _lib.sc_context_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sc_context_load(C: int, lists, tau: float = 0.0, k: float = 10.0, order: int = SC_ORDER_API_OUTPUT,
                    multi_app: Optional[bool] = None) -> Context:
    return Context(C, lists, tau, k, order, multi_app)


def sc_context_load_compact(C: int, lists, tau: float = 0.0, k: float = 10.0, order: int = SC_ORDER_API_OUTPUT,
                            multi_app: Optional[bool] = None) -> Context:
    """Context for column-compacted rows: column j = label Context.columns()[j]."""
    return Context(C, lists, tau, k, order, multi_app, compact=True)


def sc_context_columns(ctx: Context):
    return ctx.columns()


def sc_context_free(ctx: Context):
    ctx.free()


@dataclass
class Batch:
    """Device tensors of one batch (see sc_batch in include/sc.h).

    logits: [rows, C] float32 or bfloat16 CUDA tensor with unit column stride; its row
    stride is the ABI's ``ld``.  gt_off int64 [rows+1] / gt_lab int32: ground-truth CSR.
    gt_mask uint8 [rows]: precomputed G_i (from sc_decision_hist).  app int16/uint16 [rows]."""
    logits: object = None
    gt_off: object = None
    gt_lab: object = None
    gt_mask: object = None
    app: object = None
    rows: Optional[int] = None

    def _c(self) -> _CBatch:
        torch = _torch()
        cb = _CBatch()
        rows = self.rows
        if self.logits is not None:
            lg = self.logits
            if not lg.is_cuda:
                raise ValueError("logits must be a CUDA tensor (no CPU fallback)")
            if lg.dim() != 2 or lg.stride(1) != 1:
                raise ValueError("logits must be 2-D with unit column stride")
            if lg.dtype == torch.float32:
                cb.dtype = SC_F32
            elif lg.dtype == torch.bfloat16:
                cb.dtype = SC_BF16
            else:
                raise TypeError("logits dtype must be float32 or bfloat16")
            cb.logits = lg.data_ptr()
            cb.ld = lg.stride(0) if lg.size(0) > 1 else max(lg.stride(0), lg.size(1))
            rows = lg.size(0) if rows is None else rows
        if rows is None:
            if self.gt_off is not None:
                rows = self.gt_off.numel() - 1
            elif self.gt_mask is not None:
                rows = self.gt_mask.numel()
            else:
                raise ValueError("cannot infer rows")
        cb.rows = int(rows)
        cb.gt_off = _dev_ptr(self.gt_off, "gt_off", (torch.int64,), rows + 1)
        cb.gt_lab = _dev_ptr(self.gt_lab, "gt_lab", (torch.int32,))
        cb.gt_mask = _dev_ptr(self.gt_mask, "gt_mask", (torch.uint8,), rows)
        cb.app = _dev_ptr(self.app, "app", (torch.int16, torch.uint16), rows)
        return cb


def _u64(t, name, n):
    torch = _torch()
    return _dev_ptr(t, name, (torch.int64, torch.uint64), n)


def sc_decide(ctx: Context, batch: Batch, decision=None, n_incorrect=None, hist_pred=None, hist_gt=None,
              stream=None):
    """Decisions and counters of a batch (no loss).  Counters accumulate (+=)."""
    torch = _torch()
    cb = batch._c()
    _check(_lib.sc_decide(ctx.handle, ctypes.byref(cb),
                          _dev_ptr(decision, "decision", (torch.uint8,), cb.rows),
                          _u64(n_incorrect, "n_incorrect", ctx.n_apps),
                          _u64(hist_pred, "hist_pred", ctx.n_apps * 256),
                          _u64(hist_gt, "hist_gt", ctx.n_apps * 256), _stream(stream)))


def sc_decision_hist(ctx: Context, batch: Batch, hist_gt=None, gt_mask_out=None, stream=None):
    """Ground-truth-only pre-pass: mask histogram (+=) and optional per-row G_i."""
    torch = _torch()
    cb = batch._c()
    _check(_lib.sc_decision_hist(ctx.handle, ctypes.byref(cb), _u64(hist_gt, "hist_gt", ctx.n_apps * 256),
                                 _dev_ptr(gt_mask_out, "gt_mask_out", (torch.uint8,), cb.rows), _stream(stream)))


def sc_decide_all_apps(ctx: Context, batch: Batch, n_incorrect=None, hist_pred=None, decision=None, stream=None):
    """One read of the logits, every application of the context (provider what-if)."""
    torch = _torch()
    cb = batch._c()
    cb.app = None
    cb.gt_mask = None
    _check(_lib.sc_decide_all_apps(ctx.handle, ctypes.byref(cb), _u64(n_incorrect, "n_incorrect", ctx.n_apps),
                                   _u64(hist_pred, "hist_pred", ctx.n_apps * 256),
                                   _dev_ptr(decision, "decision", (torch.uint8,), cb.rows * ctx.n_apps),
                                   _stream(stream)))


def sc_decision_hist_weights(ctx: Context, batch: Batch, hist_gt, w, gt_mask_out=None, stream=None):
    """Pre-pass + weights in one launch (whole dataset on one GPU; hist_gt must start at 0)."""
    torch = _torch()
    cb = batch._c()
    _check(_lib.sc_decision_hist_weights(ctx.handle, ctypes.byref(cb), _u64(hist_gt, "hist_gt", ctx.n_apps * 256),
                                         _dev_ptr(gt_mask_out, "gt_mask_out", (torch.uint8,), cb.rows),
                                         _dev_ptr(w, "w", (torch.float32,), ctx.n_apps * 256), _stream(stream)))


def sc_weights_from_hist(ctx: Context, hist_gt, w, stream=None):
    """Rebalancing weights M/N(m) from the global mask histogram (overwrites w)."""
    torch = _torch()
    _check(_lib.sc_weights_from_hist(ctx.handle, _u64(hist_gt, "hist_gt", ctx.n_apps * 256),
                                     _dev_ptr(w, "w", (torch.float32,), ctx.n_apps * 256), _stream(stream)))


def sc_loss_fwd_bwd(ctx: Context, batch: Batch, w=None, grad_scale: float = 1.0, loss_sum=None, loss_row=None,
                    grad_idx=None, grad_val=None, grad_dense=None, decision=None, n_incorrect=None,
                    hist_pred=None, hist_gt=None, stream=None):
    """The fused pass: decisions, counters and Eq. api_output forward + backward."""
    torch = _torch()
    cb = batch._c()
    ld = cb.ld
    _check(_lib.sc_loss_fwd_bwd(
        ctx.handle, ctypes.byref(cb),
        _dev_ptr(w, "w", (torch.float32,), ctx.n_apps * 256), float(grad_scale),
        _dev_ptr(loss_sum, "loss_sum", (torch.float64,), ctx.n_apps),
        _dev_ptr(loss_row, "loss_row", (torch.float32,), cb.rows),
        _dev_ptr(grad_idx, "grad_idx", (torch.int32,), ctx.grad_slots * cb.rows),
        _dev_ptr(grad_val, "grad_val", (torch.float32,), ctx.grad_slots * cb.rows),
        _dev_ptr(grad_dense, "grad_dense", (torch.float32,), cb.rows * ld),
        _dev_ptr(decision, "decision", (torch.uint8,), cb.rows),
        _u64(n_incorrect, "n_incorrect", ctx.n_apps),
        _u64(hist_pred, "hist_pred", ctx.n_apps * 256),
        _u64(hist_gt, "hist_gt", ctx.n_apps * 256), _stream(stream)))


# ------------------------------------------------------------------ host-resident batches

SC_HOST_AUTO, SC_HOST_COPY, SC_HOST_ZERO_COPY = 0, 1, 2


class Stager:
    """Handle to an ``sc_stager``: device staging (two chunks of ``chunk_bytes``), a copy
    stream and its events, for sc_loss_fwd_bwd_host.  One call at a time per stager."""

    def __init__(self, chunk_bytes: int = 256 << 20):
        h = ctypes.c_void_p()
        _check(_lib.sc_stager_create(int(chunk_bytes), ctypes.byref(h)))
        self._h = h
        self.chunk_bytes = int(chunk_bytes)

    @property
    def handle(self):
        return self._h

    def free(self):
        if getattr(self, "_h", None):
            _lib.sc_stager_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sc_loss_fwd_bwd_host(ctx: Context, stager: Optional[Stager], batch: Batch, mode: int = SC_HOST_AUTO, w=None,
                         grad_scale: float = 1.0, loss_sum=None, loss_row=None, grad_idx=None, grad_val=None,
                         grad_dense=None, decision=None, n_incorrect=None, hist_pred=None, hist_gt=None,
                         stream=None) -> int:
    """sc_loss_fwd_bwd over HOST logits (batch.logits: a pinned CPU tensor; everything else on
    the device).  Returns the sc_host_mode taken (COPY: chunked, double-buffered H2D inside
    libsc; ZERO_COPY: the kernels read the pinned rows in place)."""
    torch = _torch()
    lg = batch.logits
    if lg is None or lg.is_cuda or lg.dim() != 2 or lg.stride(1) != 1:
        raise ValueError("batch.logits must be a 2-D host tensor with unit column stride")
    if lg.dtype not in (torch.float32, torch.bfloat16):
        raise TypeError("logits dtype must be float32 or bfloat16")
    gpu_part = Batch(logits=None, gt_off=batch.gt_off, gt_lab=batch.gt_lab, gt_mask=batch.gt_mask, app=batch.app,
                     rows=lg.size(0))
    cb = gpu_part._c()
    cb.logits = lg.data_ptr()
    cb.dtype = SC_F32 if lg.dtype == torch.float32 else SC_BF16
    cb.ld = lg.stride(0) if lg.size(0) > 1 else max(lg.stride(0), lg.size(1))
    used = ctypes.c_int32(-1)
    _check(_lib.sc_loss_fwd_bwd_host(
        ctx.handle, stager.handle if stager is not None else None, ctypes.byref(cb), int(mode),
        _dev_ptr(w, "w", (torch.float32,), ctx.n_apps * 256), float(grad_scale),
        _dev_ptr(loss_sum, "loss_sum", (torch.float64,), ctx.n_apps),
        _dev_ptr(loss_row, "loss_row", (torch.float32,), cb.rows),
        _dev_ptr(grad_idx, "grad_idx", (torch.int32,), ctx.grad_slots * cb.rows),
        _dev_ptr(grad_val, "grad_val", (torch.float32,), ctx.grad_slots * cb.rows),
        _dev_ptr(grad_dense, "grad_dense", (torch.float32,), cb.rows * cb.ld),
        _dev_ptr(decision, "decision", (torch.uint8,), cb.rows),
        _u64(n_incorrect, "n_incorrect", ctx.n_apps),
        _u64(hist_pred, "hist_pred", ctx.n_apps * 256),
        _u64(hist_gt, "hist_gt", ctx.n_apps * 256), ctypes.byref(used), _stream(stream)))
    return used.value


# ------------------------------------------------------------------ classifier head (NEXT f4)

class Head:
    """Handle to a compiled classifier head (``sc_head``): the mapped rows of W (bf16,
    [C, d]) and their bias, for the fused head GEMM + evaluation."""

    def __init__(self, ctx: Context, weight, bias=None, stream=None):
        torch = _torch()
        if weight.dim() != 2 or weight.shape[0] != ctx.C:
            raise ValueError("weight must be [C, d]")
        if weight.stride(1) != 1:
            raise ValueError("weight rows must be contiguous")
        h = ctypes.c_void_p()
        _check(_lib.sc_head_load(ctx.handle, _dev_ptr(weight, "weight", (torch.bfloat16,)), weight.stride(0),
                                 weight.shape[1], _dev_ptr(bias, "bias", (torch.float32,), ctx.C),
                                 _stream(stream), ctypes.byref(h)))
        self._h = h
        self.ctx = ctx

    @property
    def handle(self):
        return self._h

    def info(self):
        """-> (d, n_cols): feature width and head columns computed per row."""
        d, n = ctypes.c_int64(), ctypes.c_int32()
        _check(_lib.sc_head_info(self._h, ctypes.byref(d), ctypes.byref(n)))
        return d.value, n.value

    def free(self):
        if getattr(self, "_h", None):
            _lib.sc_head_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sc_head_load(ctx: Context, weight, bias=None, stream=None) -> Head:
    return Head(ctx, weight, bias, stream)


def sc_head_loss_fwd_bwd(ctx: Context, head: Head, x, gt_off=None, gt_lab=None, gt_mask=None, w=None,
                         grad_scale: float = 1.0, loss_sum=None, loss_row=None, grad_idx=None, grad_val=None,
                         decision=None, n_incorrect=None, hist_pred=None, hist_gt=None, stream=None):
    """Head GEMM (tcgen05) with the evaluation in its epilogue: x bf16 [rows, d]."""
    torch = _torch()
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("x must be a 2-D bf16 tensor with contiguous rows")
    if not x.is_cuda or x.dtype != torch.bfloat16:
        raise TypeError("x must be a CUDA bf16 tensor (no CPU fallback)")
    rows = x.shape[0]
    cb = _CHeadBatch(x.data_ptr(), rows, x.stride(0) if rows > 1 else max(x.stride(0), x.shape[1]),
                     _dev_ptr(gt_off, "gt_off", (torch.int64,), rows + 1) if gt_off is not None else None,
                     _dev_ptr(gt_lab, "gt_lab", (torch.int32,)) if gt_lab is not None else None,
                     _dev_ptr(gt_mask, "gt_mask", (torch.uint8,), rows) if gt_mask is not None else None)
    _check(_lib.sc_head_loss_fwd_bwd(
        ctx.handle, head.handle, ctypes.byref(cb),
        _dev_ptr(w, "w", (torch.float32,), 256), float(grad_scale),
        _dev_ptr(loss_sum, "loss_sum", (torch.float64,), 1),
        _dev_ptr(loss_row, "loss_row", (torch.float32,), rows),
        _dev_ptr(grad_idx, "grad_idx", (torch.int32,), ctx.grad_slots * rows),
        _dev_ptr(grad_val, "grad_val", (torch.float32,), ctx.grad_slots * rows),
        _dev_ptr(decision, "decision", (torch.uint8,), rows),
        _u64(n_incorrect, "n_incorrect", 1), _u64(hist_pred, "hist_pred", 256), _u64(hist_gt, "hist_gt", 256),
        _stream(stream)))


# ------------------------------------------------------------------ value ranges

def _rcheck(status: int):
    if status != SC_OK:
        raise ScError(status, _lib.sc_ranges_last_error().decode())


class Ranges:
    """Handle to a value-ranges application (sc_ranges): ranges [lo_j, hi_j] in code order."""

    def __init__(self, lo, hi, k: float = 10.0):
        self.m = len(lo)
        a_lo = (ctypes.c_float * max(1, self.m))(*[float(x) for x in lo])
        a_hi = (ctypes.c_float * max(1, len(hi)))(*[float(x) for x in hi])
        if len(hi) != self.m:
            raise ValueError("lo and hi must have the same length")
        h = ctypes.c_void_p()
        _rcheck(_lib.sc_ranges_load(self.m, a_lo, a_hi, float(k), ctypes.byref(h)))
        self._h = h

    def free(self):
        if getattr(self, "_h", None):
            _lib.sc_ranges_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sc_ranges_hist(r: Ranges, gt_score, hist_gt=None, gt_range_out=None, stream=None):
    torch = _torch()
    n = gt_score.numel()
    _rcheck(_lib.sc_ranges_hist(r._h, _dev_ptr(gt_score, "gt_score", (torch.float32,)), n,
                                _u64(hist_gt, "hist_gt", r.m + 1),
                                _dev_ptr(gt_range_out, "gt_range_out", (torch.uint8,), n), _stream(stream)))


def sc_ranges_weights(r: Ranges, hist_gt, w, stream=None):
    torch = _torch()
    _rcheck(_lib.sc_ranges_weights(r._h, _u64(hist_gt, "hist_gt", r.m + 1),
                                   _dev_ptr(w, "w", (torch.float32,), r.m + 1), _stream(stream)))


def sc_ranges_loss_fwd_bwd(r: Ranges, score, gt_range, w=None, grad_scale: float = 1.0, loss_sum=None,
                           loss_row=None, grad=None, decision=None, n_incorrect=None, hist_pred=None, stream=None):
    torch = _torch()
    n = score.numel()
    _rcheck(_lib.sc_ranges_loss_fwd_bwd(
        r._h, _dev_ptr(score, "score", (torch.float32,)), _dev_ptr(gt_range, "gt_range", (torch.uint8,), n), n,
        _dev_ptr(w, "w", (torch.float32,), r.m + 1), float(grad_scale),
        _dev_ptr(loss_sum, "loss_sum", (torch.float64,), 1), _dev_ptr(loss_row, "loss_row", (torch.float32,), n),
        _dev_ptr(grad, "grad", (torch.float32,), n), _dev_ptr(decision, "decision", (torch.uint8,), n),
        _u64(n_incorrect, "n_incorrect", 1), _u64(hist_pred, "hist_pred", r.m + 1), _stream(stream)))


# ------------------------------------------------------------------ rebalanced sampler

def sc_sample_workspace_bytes(rows: int) -> int:
    return int(_lib.sc_sample_workspace_bytes(int(rows)))


def sc_rebalance_sample(gt_mask, w, u, out, workspace=None, stream=None):
    """Draw out.numel() rows with probability ∝ w[G_i] (u: float64 [2n] uniforms)."""
    torch = _torch()
    rows, n = gt_mask.numel(), out.numel()
    if workspace is None:
        workspace = torch.empty(sc_sample_workspace_bytes(rows), dtype=torch.uint8, device=gt_mask.device)
    st = _lib.sc_rebalance_sample(_dev_ptr(gt_mask, "gt_mask", (torch.uint8,), rows), rows,
                                  _dev_ptr(w, "w", (torch.float32,), 256), _dev_ptr(u, "u", (torch.float64,), 2 * n),
                                  n, _dev_ptr(out, "out", (torch.int64,), n),
                                  _dev_ptr(workspace, "workspace", (torch.uint8,)), workspace.numel(), _stream(stream))
    if st != SC_OK:
        raise ScError(st, _lib.sc_sample_last_error().decode())
    return out

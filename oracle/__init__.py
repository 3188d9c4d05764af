"""CPU oracle for the software-context hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
``paper_2310_07240_b200`` never imports it and shares no code with it.

The arithmetic lives in ``sc_oracle.c`` (plain C, double precision, one
function per step of the paper; see that file's header for citations and
pins).  This module only marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_DIR, "liboracle.so")
_SRC = os.path.join(_DIR, "sc_oracle.c")


def build(force: bool = False) -> str:
    if os.environ.get("ORACLE_SO"):  # mutation testing of the pins (tests/mutate_oracle.py)
        return os.environ["ORACLE_SO"]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


class _Ctx(ctypes.Structure):
    _fields_ = [
        ("C", ctypes.c_int32),
        ("n_apps", ctypes.c_int32),
        ("n_lists", ctypes.c_void_p),
        ("list_off", ctypes.c_void_p),
        ("list_labels", ctypes.c_void_p),
        ("tau", ctypes.c_double),
        ("k", ctypes.c_double),
        ("order", ctypes.c_int32),
    ]


API_OUTPUT, APP_CHOICE, MULTI_SELECT = 0, 1, 2


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.orc_first_list.restype = I32
        L.orc_first_list.argtypes = [P, I32, I32]
        L.orc_compile.argtypes = [P, I32, P]
        L.orc_decide.restype = I32
        L.orc_decide.argtypes = [P, I32, P, P, P]
        L.orc_gt_set.restype = ctypes.c_uint32
        L.orc_gt_set.argtypes = [P, P, I64]
        L.orc_correct.restype = I32
        L.orc_correct.argtypes = [ctypes.c_uint32, I32, I32]
        L.orc_loss_row.argtypes = [P, P, P, ctypes.c_uint32, D, P, P, P, P, P, P]
        L.orc_weights_literal.argtypes = [P, I64, P, P, P]
        L.orc_weights_by_mask.argtypes = [I32, P, P]
        L.orc_label_lists.restype = ctypes.c_uint32
        L.orc_label_lists.argtypes = [P, I32, I32]
        L.orc_gt_set_raw.restype = ctypes.c_uint32
        L.orc_gt_set_raw.argtypes = [P, I32, P, I64]
        L.orc_decide_app_choice.restype = I32
        L.orc_decide_app_choice.argtypes = [P, I32, P]
        L.orc_gt_decision_app_choice.restype = I32
        L.orc_gt_decision_app_choice.argtypes = [P, I32, P, I64]
        L.orc_decide_multi_select.restype = ctypes.c_uint32
        L.orc_decide_multi_select.argtypes = [P, I32, P]
        L.orc_loss_row_app_choice.argtypes = [P, P, P, ctypes.c_uint32, D, P, P, P, P, P, P]
        L.orc_loss_row_multi_select.argtypes = [P, I32, P, ctypes.c_uint32, D, P, P, P, P]
        L.orc_weights_literal_masks.argtypes = [P, I64, P, P, P]
        L.orc_range_of.restype = I32
        L.orc_range_of.argtypes = [I32, P, P, D]
        L.orc_range_loss.argtypes = [I32, P, P, D, I32, D, D, P, P]
        L.orc_ranges_eval.argtypes = [I32, P, P, D, I64, P, P, P, D] + [P] * 8
        L.orc_ranges_weights.argtypes = [I32, P, P]
        L.orc_sample.restype = ctypes.c_int
        L.orc_sample.argtypes = [P, I64, P, I64, P, P, P]
        L.orc_gt_hist.restype = ctypes.c_int
        L.orc_gt_hist.argtypes = [P, I64, P, P, P, P, P]
        L.orc_eval.restype = ctypes.c_int
        L.orc_eval.argtypes = [P, I64, I64, I32, P, P, P, P, P, D] + [P] * 10
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class Oracle:
    """Oracle bound to one context: ``lists[a][j]`` are the label ids of W_j of app a."""

    def __init__(self, C: int, lists, tau: float = 0.0, k: float = 10.0, order: int = API_OUTPUT):
        self.C, self.tau, self.k, self.order = int(C), float(tau), float(k), int(order)
        self.lists = [[list(map(int, l)) for l in app] for app in lists]
        n_lists, off, labels = [], [], []
        pos = 0
        for app in self.lists:
            n_lists.append(len(app))
            off.append(pos)
            for l in app:
                labels.extend(l)
                pos += len(l)
                off.append(pos)
        self._n_lists = np.asarray(n_lists, dtype=np.int32)
        self._off = np.asarray(off, dtype=np.int64)
        self._labels = np.asarray(labels if labels else [0], dtype=np.int32)
        self._ctx = _Ctx(self.C, len(self.lists), self._n_lists.ctypes.data, self._off.ctypes.data,
                         self._labels.ctypes.data, self.tau, self.k, self.order)

    @classmethod
    def from_spec(cls, spec, order: int = API_OUTPUT):
        return cls(spec.C, spec.lists, spec.tau, spec.k, order)

    @property
    def grad_slots(self) -> int:
        return 8 if self.order == MULTI_SELECT else 2

    @property
    def n_apps(self):
        return len(self.lists)

    def n_lists(self, app: int = 0) -> int:
        return len(self.lists[app])

    # ---- single steps ----
    def first_list(self, c: int, app: int = 0) -> int:
        return int(lib().orc_first_list(ctypes.byref(self._ctx), app, c))

    def compile(self, app: int = 0) -> np.ndarray:
        cat = np.empty(self.C, dtype=np.int8)
        lib().orc_compile(ctypes.byref(self._ctx), app, cat.ctypes.data)
        return cat

    def decide(self, z, app: int = 0) -> int:
        """Decision(API(x)) for the context's pattern (a list mask for Multi-Select)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        if self.order == APP_CHOICE:
            return int(lib().orc_decide_app_choice(ctypes.byref(self._ctx), app, z.ctypes.data))
        if self.order == MULTI_SELECT:
            return int(lib().orc_decide_multi_select(ctypes.byref(self._ctx), app, z.ctypes.data))
        scratch = np.empty(self.C, dtype=np.int32)
        return int(lib().orc_decide(ctypes.byref(self._ctx), app, self.compile(app).ctypes.data,
                                    z.ctypes.data, scratch.ctypes.data))

    def label_lists(self, c: int, app: int = 0) -> int:
        return int(lib().orc_label_lists(ctypes.byref(self._ctx), app, c))

    def gt_set_raw(self, labels, app: int = 0) -> int:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        return int(lib().orc_gt_set_raw(ctypes.byref(self._ctx), app, labels.ctypes.data, len(labels)))

    def gt_decision_app_choice(self, labels, app: int = 0) -> int:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        return int(lib().orc_gt_decision_app_choice(ctypes.byref(self._ctx), app, labels.ctypes.data, len(labels)))

    def gt_mask(self, labels, app: int = 0) -> int:
        """G_i as the pattern defines it (compiled first list for the choice orders)."""
        return self.gt_set_raw(labels, app) if self.order == MULTI_SELECT else self.gt_set(labels, app)

    def is_correct(self, labels, d: int, app: int = 0) -> bool:
        if self.order == APP_CHOICE:
            return d == self.gt_decision_app_choice(labels, app)
        if self.order == MULTI_SELECT:
            return d == self.gt_set_raw(labels, app)
        return self.correct(self.gt_set(labels, app), d, app)

    def gt_set(self, labels, app: int = 0) -> int:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        return int(lib().orc_gt_set(self.compile(app).ctypes.data, labels.ctypes.data, len(labels)))

    def correct(self, G: int, d: int, app: int = 0) -> bool:
        return bool(lib().orc_correct(G, d, self.n_lists(app)))

    def loss_row(self, z, G: int, w: float = 1.0, app: int = 0):
        """-> dict(ell, L, c_plus, g_plus, c_minus, g_minus, grads={label: dL/dz}) (unscaled).
        For Multi-Select c_plus/c_minus are unused (-1) and grads holds one entry per list."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        ell, L = ctypes.c_double(), ctypes.c_double()
        if self.order == MULTI_SELECT:
            cs = np.full(8, -1, dtype=np.int32)
            gs = np.zeros(8, dtype=np.float64)
            lib().orc_loss_row_multi_select(ctypes.byref(self._ctx), app, z.ctypes.data, G, w, ctypes.byref(ell),
                                            ctypes.byref(L), cs.ctypes.data, gs.ctypes.data)
            grads = {}
            for c, g in zip(cs.tolist(), gs.tolist()):
                if c >= 0:
                    grads[c] = grads.get(c, 0.0) + g
            return dict(ell=ell.value, L=L.value, c_plus=-1, g_plus=0.0, c_minus=-1, g_minus=0.0, grads=grads,
                        slots=(cs, gs))
        gp, gm = ctypes.c_double(), ctypes.c_double()
        cp, cm = ctypes.c_int32(), ctypes.c_int32()
        fn = lib().orc_loss_row_app_choice if self.order == APP_CHOICE else lib().orc_loss_row
        fn(ctypes.byref(self._ctx), self.compile(app).ctypes.data, z.ctypes.data, G, w,
           ctypes.byref(ell), ctypes.byref(L), ctypes.byref(cp), ctypes.byref(gp), ctypes.byref(cm), ctypes.byref(gm))
        grads = {}
        for c, g in ((cp.value, gp.value), (cm.value, gm.value)):
            if c >= 0:
                grads[c] = grads.get(c, 0.0) + g
        return dict(ell=ell.value, L=L.value, c_plus=cp.value, g_plus=gp.value,
                    c_minus=cm.value, g_minus=gm.value, grads=grads)

    def weights_literal(self, gt_off, gt_lab, app: int = 0) -> np.ndarray:
        gt_off = np.ascontiguousarray(gt_off, dtype=np.int64)
        gt_lab = np.ascontiguousarray(gt_lab if len(gt_lab) else [0], dtype=np.int32)
        M = len(gt_off) - 1
        w = np.empty(max(M, 1), dtype=np.float64)
        lib().orc_weights_literal(self.compile(app).ctypes.data, M, gt_off.ctypes.data, gt_lab.ctypes.data,
                                  w.ctypes.data)
        return w[:M]

    def weights_literal_pattern(self, gt_off, gt_lab, app: int = 0) -> np.ndarray:
        """Literal O(M^2) N_i with the pattern's label->lists map (first list / every list)."""
        gt_off = np.ascontiguousarray(gt_off, dtype=np.int64)
        gt_lab = np.ascontiguousarray(gt_lab if len(gt_lab) else [0], dtype=np.int32)
        if self.order == MULTI_SELECT:
            lm = np.array([self.label_lists(c, app) for c in range(self.C)], dtype=np.uint8)
        else:
            cat = self.compile(app)
            lm = np.where(cat >= 0, 1 << np.maximum(cat, 0).astype(np.int64), 0).astype(np.uint8)
        M = len(gt_off) - 1
        w = np.empty(max(M, 1), dtype=np.float64)
        lib().orc_weights_literal_masks(lm.ctypes.data, M, gt_off.ctypes.data, gt_lab.ctypes.data, w.ctypes.data)
        return w[:M]

    @staticmethod
    def weights_by_mask(H) -> np.ndarray:
        H = np.ascontiguousarray(H, dtype=np.uint64).reshape(-1, 256)
        w = np.empty(H.shape, dtype=np.float64)
        lib().orc_weights_by_mask(H.shape[0], H.ctypes.data, w.ctypes.data)
        return w

    # ---- whole batch ----
    def gt_hist(self, gt_off, gt_lab, app=None):
        """Ground truth only: (gt_mask [rows], hist_gt [n_apps*256]) — orc_gt_hist."""
        gt_off = np.ascontiguousarray(gt_off, dtype=np.int64)
        rows = len(gt_off) - 1
        gt_lab = np.ascontiguousarray(gt_lab if len(gt_lab) else [0], dtype=np.int32)
        if app is not None:
            app = np.ascontiguousarray(app, dtype=np.uint16)
        gm = np.zeros(max(rows, 1), np.uint8)
        H = np.zeros(self.n_apps * 256, np.uint64)
        if lib().orc_gt_hist(ctypes.byref(self._ctx), rows, _p(gt_off), _p(gt_lab), _p(app), _p(gm), _p(H)) != 0:
            raise ValueError("oracle rejected the ground truth (out-of-range id)")
        return gm[:rows], H

    def eval(self, logits, gt_off=None, gt_lab=None, app=None, w=None, grad_scale: float = 1.0,
             want_loss: bool = True):
        """All outputs for a batch.  logits: float32 [rows, ld] or uint16 (bf16 bits).
        gt_off is a CSR offset array with rows+1 entries (any base)."""
        logits = np.ascontiguousarray(logits)
        rows, ld = logits.shape
        dtype = 0 if logits.dtype == np.float32 else 1
        if dtype == 1 and logits.dtype != np.uint16:
            raise TypeError("bf16 logits must be passed as uint16 bit patterns")
        has_gt = gt_off is not None
        if has_gt:
            gt_off = np.ascontiguousarray(gt_off, dtype=np.int64)
            gt_lab = np.ascontiguousarray(gt_lab if len(gt_lab) else [0], dtype=np.int32)
        if app is not None:
            app = np.ascontiguousarray(app, dtype=np.uint16)
        if w is not None:
            w = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
        na = self.n_apps
        r1 = max(rows, 1)
        S = self.grad_slots
        out = dict(decision=np.zeros(r1, np.uint8), hist_pred=np.zeros(na * 256, np.uint64))
        if has_gt:
            out.update(gt_mask=np.zeros(r1, np.uint8), correct=np.zeros(r1, np.uint8),
                       n_incorrect=np.zeros(na, np.uint64), hist_gt=np.zeros(na * 256, np.uint64))
            if want_loss:
                out.update(loss_sum=np.zeros(na, np.float64), loss_row=np.zeros(r1, np.float64),
                           grad_idx=np.full(S * r1, -1, np.int32), grad_val=np.zeros(S * r1, np.float64))
        g = out.get
        rc = lib().orc_eval(ctypes.byref(self._ctx), rows, ld, dtype, logits.ctypes.data,
                            _p(gt_off), _p(gt_lab), _p(app), _p(w), grad_scale,
                            _p(g("decision")), _p(g("gt_mask")), _p(g("correct")), _p(g("n_incorrect")),
                            _p(g("hist_pred")), _p(g("hist_gt")), _p(g("loss_sum")), _p(g("loss_row")),
                            _p(g("grad_idx")), _p(g("grad_val")))
        if rc != 0:
            raise ValueError("oracle rejected the batch (non-finite logit or out-of-range id)")
        for key in ("decision", "gt_mask", "correct", "loss_row"):
            if key in out:
                out[key] = out[key][:rows]
        for key in ("grad_idx", "grad_val"):
            if key in out:
                out[key] = out[key][: S * rows]
        return out


class RangesOracle:
    """Value-ranges applications: ranges [lo_j, hi_j] in code order."""

    def __init__(self, lo, hi, k: float = 10.0):
        self.lo = np.ascontiguousarray(lo, dtype=np.float64)
        self.hi = np.ascontiguousarray(hi, dtype=np.float64)
        self.m, self.k = len(self.lo), float(k)

    def range_of(self, score: float) -> int:
        return int(lib().orc_range_of(self.m, self.lo.ctypes.data, self.hi.ctypes.data, float(score)))

    def loss(self, r: int, score: float, w: float = 1.0):
        L, dL = ctypes.c_double(), ctypes.c_double()
        lib().orc_range_loss(self.m, self.lo.ctypes.data, self.hi.ctypes.data, self.k, r, float(score), w,
                             ctypes.byref(L), ctypes.byref(dL))
        return L.value, dL.value

    def weights(self, H) -> np.ndarray:
        H = np.ascontiguousarray(H, dtype=np.uint64)
        w = np.empty(self.m + 1, dtype=np.float64)
        lib().orc_ranges_weights(self.m, H.ctypes.data, w.ctypes.data)
        return w

    def eval(self, score, gt_score, w=None, grad_scale: float = 1.0):
        score = np.ascontiguousarray(score, dtype=np.float32)
        gt_score = np.ascontiguousarray(gt_score, dtype=np.float32)
        rows = len(score)
        r1 = max(rows, 1)
        out = dict(decision=np.zeros(r1, np.uint8), gt_range=np.zeros(r1, np.uint8),
                   n_incorrect=np.zeros(1, np.uint64), hist_pred=np.zeros(self.m + 1, np.uint64),
                   hist_gt=np.zeros(self.m + 1, np.uint64), loss_sum=np.zeros(1, np.float64),
                   loss_row=np.zeros(r1, np.float64), grad=np.zeros(r1, np.float64))
        wp = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        g = out.get
        lib().orc_ranges_eval(self.m, self.lo.ctypes.data, self.hi.ctypes.data, self.k, rows, score.ctypes.data,
                              gt_score.ctypes.data, _p(wp), grad_scale, _p(g("decision")), _p(g("gt_range")),
                              _p(g("n_incorrect")), _p(g("hist_pred")), _p(g("hist_gt")), _p(g("loss_sum")),
                              _p(g("loss_row")), _p(g("grad")))
        for key in ("decision", "gt_range", "loss_row", "grad"):
            out[key] = out[key][:rows]
        return out


def sample(gt_mask, w, u1, u2):
    """Rebalanced sampler (reading A24): indices for the uniforms (u1, u2).
    gt_mask: uint8 [rows]; w: per-mask weights [256] (the kernel's f32 values)."""
    gt_mask = np.ascontiguousarray(gt_mask, dtype=np.uint8)
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float32).astype(np.float64))
    u1 = np.ascontiguousarray(u1, dtype=np.float64)
    u2 = np.ascontiguousarray(u2, dtype=np.float64)
    out = np.empty(max(len(u1), 1), dtype=np.int64)
    rc = lib().orc_sample(gt_mask.ctypes.data if len(gt_mask) else None, len(gt_mask), w.ctypes.data, len(u1),
                          u1.ctypes.data, u2.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise ValueError("every weight is zero")
    return out[: len(u1)]


# ------------------------------------------------------------------ classifier head (NEXT f4)

def bf16_to_f64(bits) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float64: a bf16 is the upper half of an IEEE binary32."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def head_logits(x_bits, w_bits, bias=None) -> np.ndarray:
    """z = x Wᵀ + b over ALL C labels — the linear classifier head whose outputs are the
    API's confidences (the API output the application reads,
    PAPER.md:862).  x [rows, d] and W [C, d] are bf16 bit patterns, bias [C] float or None.
    Plain fp64: the products of two bf16 are exact in fp64 and the sum is a library matmul
    (for the integer-valued workloads of synth.head_operands(kind="int") it is exact).
    The fused GPU path computes only the mapped columns; the oracle keeps the definition."""
    x = bf16_to_f64(x_bits)
    W = bf16_to_f64(w_bits)
    z = x @ W.T
    if bias is not None:
        z = z + np.asarray(bias, dtype=np.float64)[None, :]
    return z

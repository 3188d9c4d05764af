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
    ]


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
        L.orc_eval.restype = ctypes.c_int
        L.orc_eval.argtypes = [P, I64, I64, I32, P, P, P, P, P, D] + [P] * 10
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class Oracle:
    """Oracle bound to one context: ``lists[a][j]`` are the label ids of W_j of app a."""

    def __init__(self, C: int, lists, tau: float = 0.0, k: float = 10.0):
        self.C, self.tau, self.k = int(C), float(tau), float(k)
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
                         self._labels.ctypes.data, self.tau, self.k)

    @classmethod
    def from_spec(cls, spec):
        return cls(spec.C, spec.lists, spec.tau, spec.k)

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
        z = np.ascontiguousarray(z, dtype=np.float64)
        scratch = np.empty(self.C, dtype=np.int32)
        return int(lib().orc_decide(ctypes.byref(self._ctx), app, self.compile(app).ctypes.data,
                                    z.ctypes.data, scratch.ctypes.data))

    def gt_set(self, labels, app: int = 0) -> int:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        return int(lib().orc_gt_set(self.compile(app).ctypes.data, labels.ctypes.data, len(labels)))

    def correct(self, G: int, d: int, app: int = 0) -> bool:
        return bool(lib().orc_correct(G, d, self.n_lists(app)))

    def loss_row(self, z, G: int, w: float = 1.0, app: int = 0):
        """-> dict(ell, L, c_plus, g_plus, c_minus, g_minus) (unscaled gradients)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        ell, L, gp, gm = (ctypes.c_double() for _ in range(4))
        cp, cm = ctypes.c_int32(), ctypes.c_int32()
        lib().orc_loss_row(ctypes.byref(self._ctx), self.compile(app).ctypes.data, z.ctypes.data, G, w,
                           ctypes.byref(ell), ctypes.byref(L), ctypes.byref(cp), ctypes.byref(gp),
                           ctypes.byref(cm), ctypes.byref(gm))
        return dict(ell=ell.value, L=L.value, c_plus=cp.value, g_plus=gp.value,
                    c_minus=cm.value, g_minus=gm.value)

    def weights_literal(self, gt_off, gt_lab, app: int = 0) -> np.ndarray:
        gt_off = np.ascontiguousarray(gt_off, dtype=np.int64)
        gt_lab = np.ascontiguousarray(gt_lab if len(gt_lab) else [0], dtype=np.int32)
        M = len(gt_off) - 1
        w = np.empty(max(M, 1), dtype=np.float64)
        lib().orc_weights_literal(self.compile(app).ctypes.data, M, gt_off.ctypes.data, gt_lab.ctypes.data,
                                  w.ctypes.data)
        return w[:M]

    @staticmethod
    def weights_by_mask(H) -> np.ndarray:
        H = np.ascontiguousarray(H, dtype=np.uint64).reshape(-1, 256)
        w = np.empty(H.shape, dtype=np.float64)
        lib().orc_weights_by_mask(H.shape[0], H.ctypes.data, w.ctypes.data)
        return w

    # ---- whole batch ----
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
        out = dict(decision=np.zeros(r1, np.uint8), hist_pred=np.zeros(na * 16, np.uint64))
        if has_gt:
            out.update(gt_mask=np.zeros(r1, np.uint8), correct=np.zeros(r1, np.uint8),
                       n_incorrect=np.zeros(na, np.uint64), hist_gt=np.zeros(na * 256, np.uint64))
            if want_loss:
                out.update(loss_sum=np.zeros(na, np.float64), loss_row=np.zeros(r1, np.float64),
                           grad_idx=np.full(2 * r1, -1, np.int32), grad_val=np.zeros(2 * r1, np.float64))
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
                out[key] = out[key][: 2 * rows]
        return out

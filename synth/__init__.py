"""Seeded synthetic workloads (harness module; holds none of the method's arithmetic).

Both the CUDA path and the oracle consume these inputs.  The recipe is in
``synth/synth.h`` and DESIGN.md §4; it has two independent implementations,
``synth_host.c`` (numpy-facing) and ``synth_cuda.cu`` (torch-facing), checked
against each other bit for bit in ``tests/test_synth.py``.

The contexts reproduce SURVEY.md §8(d):

* cfg1 — the paper's Heapsortcypher lists: ids 0-8 Recycle,
  9-11 Compost, 12-17 Donate, 18-31 distractors (18 candy, 19 confectionery,
  20 lollipop — the other labels of the worked example).
* cfg2/cfg5 — C=1000, list sizes (90, 30, 60) (Heapsortcypher x10), seeded placement.
* cfg3 — C=20000, seven lists (250, 200, 175, 150, 100, 75, 50).
* cfg4 — C=1000, 256 apps, app a has sizes (9, 3, 6) x (1 + a mod 10).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_DIR, "libsynth_host.so")
_CUDA_SO = os.path.join(_DIR, "libsynth_cuda.so")

HEAPSORT_NAMES = (
    ["plastic", "wood", "glass", "paper", "cardboard", "metal", "aluminum", "tin", "carton"]
    + ["food", "produce", "snack"]
    + ["clothing", "jacket", "shirt", "pants", "footwear", "shoe"]
    + ["candy", "confectionery", "lollipop"]
    + [f"label{i}" for i in range(21, 32)]
)


class _Spec(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("C", ctypes.c_int32),
        ("n_apps", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("rows_per_app", ctypes.c_int64),
        ("mapped", ctypes.c_void_p),
        ("wset_off", ctypes.c_void_p),
        ("wset_lab", ctypes.c_void_p),
    ]


def build_host(force: bool = False) -> str:
    src = os.path.join(_DIR, "synth_host.c")
    if force or not os.path.exists(_HOST_SO) or os.path.getmtime(_HOST_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-o", _HOST_SO, src])
    return _HOST_SO


def build_cuda(force: bool = False) -> str:
    src = os.path.join(_DIR, "synth_cuda.cu")
    if force or not os.path.exists(_CUDA_SO) or os.path.getmtime(_CUDA_SO) < os.path.getmtime(src):
        subprocess.check_call([
            "nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
            "-Xcompiler", "-fPIC", "-shared", "-o", _CUDA_SO, src])
    return _CUDA_SO


_host = None
_cuda = None


def _host_lib():
    global _host
    if _host is None:
        lib = ctypes.CDLL(build_host())
        P = ctypes.c_void_p
        lib.synth_hash.restype = ctypes.c_uint64
        lib.synth_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64]
        lib.synth_perm.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, P]
        lib.synth_host_apps.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P]
        lib.synth_host_gt_count.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P]
        lib.synth_host_gt_fill.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, P]
        lib.synth_host_logits.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P, P, P]
        _host = lib
    return _host


def _cuda_lib():
    global _cuda
    if _cuda is None:
        if not os.path.exists(_CUDA_SO):
            raise RuntimeError(f"{_CUDA_SO} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_CUDA_SO)
        P = ctypes.c_void_p
        lib.synth_cuda_apps.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, P]
        lib.synth_cuda_gt_count.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, P]
        lib.synth_cuda_gt_fill.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, P, P]
        lib.synth_cuda_logits.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P, P, P, P]
        _cuda = lib
    return _cuda


def synth_hash(seed: int, stream: int, a: int, b: int) -> int:
    return int(_host_lib().synth_hash(seed, stream, a, b))


def perm(seed: int, app: int, C: int) -> np.ndarray:
    out = np.empty(C, dtype=np.int32)
    _host_lib().synth_perm(seed, app, C, out.ctypes.data)
    return out


# ------------------------------------------------------------------ contexts

@dataclass
class ContextSpec:
    """An application's extracted software context: per app, the
    target-class label lists in code order.  ``lists[a][j]`` = label ids of W_j."""
    C: int
    lists: list  # list[app] -> list[list[int]]
    tau: float = 0.0
    k: float = 10.0

    @property
    def n_apps(self) -> int:
        return len(self.lists)

    def csr(self):
        """(n_lists int32[n_apps], list_off int64[], list_labels int32[]) in the sc.h layout."""
        n_lists, off, labels = [], [], []
        pos = 0
        for app_lists in self.lists:
            n_lists.append(len(app_lists))
            off.append(pos)
            for lst in app_lists:
                labels.extend(int(c) for c in lst)
                pos += len(lst)
                off.append(pos)
        return (np.asarray(n_lists, dtype=np.int32), np.asarray(off, dtype=np.int64),
                np.asarray(labels, dtype=np.int32))

    def mapped(self) -> np.ndarray:
        """uint8[n_apps, C]: 1 where the label is in some list of the app (set union only)."""
        m = np.zeros((self.n_apps, self.C), dtype=np.uint8)
        for a, app_lists in enumerate(self.lists):
            for lst in app_lists:
                m[a, np.asarray(lst, dtype=np.int64)] = 1
        return m

    def wset(self):
        m = self.mapped()
        labs = [np.nonzero(m[a])[0].astype(np.int32) for a in range(self.n_apps)]
        off = np.zeros(self.n_apps + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(x) for x in labs])
        lab = np.concatenate(labs) if labs and off[-1] > 0 else np.zeros(1, dtype=np.int32)
        return off, lab


def heapsort_context(tau: float = 0.0, k: float = 10.0) -> ContextSpec:
    """cfg1: Heapsortcypher (Fig. app_example), C = 32."""
    return ContextSpec(32, [[list(range(0, 9)), list(range(9, 12)), list(range(12, 18))]], tau, k)


def placed_context(C: int, sizes, seed: int, app: int = 0) -> list:
    p = perm(seed, app, C)
    out, pos = [], 0
    for s in sizes:
        out.append([int(c) for c in p[pos:pos + s]])
        pos += s
    return out


CONFIGS = {
    1: dict(name="cfg1_heapsortcypher", C=32, rows=4096, n_apps=1, seed=1),
    2: dict(name="cfg2_imagenet1k", C=1000, rows=1 << 20, n_apps=1, seed=2),
    3: dict(name="cfg3_openimages20k", C=20000, rows=4 << 20, n_apps=1, seed=3),
    4: dict(name="cfg4_multiapp256", C=1000, rows=256 << 18, n_apps=256, seed=4),
    5: dict(name="cfg5_rebalance64m", C=1000, rows=64 << 20, n_apps=1, seed=5),
}


def config_context(n: int, tau: float = 0.0, k: float = 10.0) -> ContextSpec:
    cfg = CONFIGS[n]
    if n == 1:
        return heapsort_context(tau, k)
    if n in (2, 5):
        return ContextSpec(1000, [placed_context(1000, (90, 30, 60), cfg["seed"])], tau, k)
    if n == 3:
        return ContextSpec(20000, [placed_context(20000, (250, 200, 175, 150, 100, 75, 50), cfg["seed"])], tau, k)
    if n == 4:
        lists = []
        for a in range(256):
            f = 1 + a % 10
            lists.append(placed_context(1000, (9 * f, 3 * f, 6 * f), cfg["seed"], app=a))
        return ContextSpec(1000, lists, tau, k)
    raise KeyError(n)


# ------------------------------------------------------------------ workloads

def default_ld(C: int, dtype: str) -> int:
    elt = 4 if dtype == "f32" else 2
    per16 = 16 // elt
    return (C + per16 - 1) // per16 * per16


@dataclass
class Workload:
    ctx: ContextSpec
    seed: int
    dtype: str = "f32"          # "f32" | "bf16"
    ld: int = 0                 # 0 -> default_ld
    layout: int = 0             # multi-app: 0 contiguous, 1 app = row % n_apps
    rows_per_app: int = 1 << 18
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        if self.ld == 0:
            self.ld = default_ld(self.ctx.C, self.dtype)
        self._mapped = np.ascontiguousarray(self.ctx.mapped().reshape(-1))
        self._woff, self._wlab = self.ctx.wset()

    @property
    def dtype_code(self) -> int:
        return 0 if self.dtype == "f32" else 1

    def _spec(self, mapped_ptr, woff_ptr, wlab_ptr) -> _Spec:
        return _Spec(self.seed, self.ctx.C, self.ctx.n_apps, self.layout, self.rows_per_app,
                     mapped_ptr, woff_ptr, wlab_ptr)

    # ---- host (numpy) ----
    def host_batch(self, row0: int, n: int):
        """Rows [row0, row0+n): dict of numpy arrays; gt_off is local (starts at 0)."""
        lib = _host_lib()
        sp = self._spec(self._mapped.ctypes.data, self._woff.ctypes.data, self._wlab.ctypes.data)
        cnt = np.empty(max(n, 1), dtype=np.int64)
        lib.synth_host_gt_count(ctypes.byref(sp), row0, n, cnt.ctypes.data)
        off = np.zeros(n + 1, dtype=np.int64)
        off[1:] = np.cumsum(cnt[:n])
        lab = np.empty(max(int(off[-1]), 1), dtype=np.int32)
        lib.synth_host_gt_fill(ctypes.byref(sp), row0, n, off.ctypes.data, lab.ctypes.data)
        app = np.empty(max(n, 1), dtype=np.uint16)
        lib.synth_host_apps(ctypes.byref(sp), row0, n, app.ctypes.data)
        logits = np.empty((max(n, 1), self.ld), dtype=np.float32 if self.dtype == "f32" else np.uint16)
        lib.synth_host_logits(ctypes.byref(sp), row0, n, self.ld, self.dtype_code,
                              off.ctypes.data, lab.ctypes.data, logits.ctypes.data)
        return dict(logits=logits[:n], gt_off=off, gt_lab=lab[: int(off[-1])], app=app[:n])

    def host_gt(self, row0: int, n: int):
        """Ground truth (and app ids) of rows [row0, row0+n) only — no logits."""
        lib = _host_lib()
        sp = self._spec(self._mapped.ctypes.data, self._woff.ctypes.data, self._wlab.ctypes.data)
        cnt = np.empty(max(n, 1), dtype=np.int64)
        lib.synth_host_gt_count(ctypes.byref(sp), row0, n, cnt.ctypes.data)
        off = np.zeros(n + 1, dtype=np.int64)
        off[1:] = np.cumsum(cnt[:n])
        lab = np.empty(max(int(off[-1]), 1), dtype=np.int32)
        lib.synth_host_gt_fill(ctypes.byref(sp), row0, n, off.ctypes.data, lab.ctypes.data)
        app = np.empty(max(n, 1), dtype=np.uint16)
        lib.synth_host_apps(ctypes.byref(sp), row0, n, app.ctypes.data)
        return dict(gt_off=off, gt_lab=lab[: int(off[-1])], app=app[:n])

    # ---- device (torch) ----
    def device_batch(self, row0: int, n: int, device="cuda", with_app: bool | None = None):
        """Rows [row0, row0+n) generated on the GPU by synth_cuda.cu (torch tensors)."""
        import torch
        lib = _cuda_lib()
        dev = torch.device(device)
        st = torch.cuda.current_stream(dev).cuda_stream
        mapped = torch.from_numpy(self._mapped).to(dev)
        woff = torch.from_numpy(self._woff).to(dev)
        wlab = torch.from_numpy(self._wlab).to(dev)
        sp = self._spec(mapped.data_ptr(), woff.data_ptr(), wlab.data_ptr())
        cnt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        _ck(lib.synth_cuda_gt_count(ctypes.byref(sp), row0, n, cnt.data_ptr(), st))
        off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        if n:
            torch.cumsum(cnt[:n], 0, out=off[1:])
        nnz = int(off[-1].item())
        lab = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        _ck(lib.synth_cuda_gt_fill(ctypes.byref(sp), row0, n, off.data_ptr(), lab.data_ptr(), st))
        tdt = torch.float32 if self.dtype == "f32" else torch.bfloat16
        logits = torch.empty((max(n, 1), self.ld), dtype=tdt, device=dev)
        _ck(lib.synth_cuda_logits(ctypes.byref(sp), row0, n, self.ld, self.dtype_code,
                                  off.data_ptr(), lab.data_ptr(), logits.data_ptr(), st))
        out = dict(logits=logits[:n], gt_off=off, gt_lab=lab[:nnz])
        if with_app or (with_app is None and self.ctx.n_apps > 1):
            app = torch.empty(max(n, 1), dtype=torch.int16, device=dev)
            _ck(lib.synth_cuda_apps(ctypes.byref(sp), row0, n, app.data_ptr(), st))
            out["app"] = app[:n]
        torch.cuda.current_stream(dev).synchronize()
        del mapped, woff, wlab
        return out


def _ck(rc: int):
    if rc != 0:
        raise RuntimeError(f"synth CUDA launch failed: cudaError {rc}")


# ------------------------------------------------------------------ classifier-head operands (NEXT f4)

def f32_to_bf16_bits(a) -> np.ndarray:
    """Round float32 to bf16 (round to nearest even) and return the bit patterns."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def head_operands(C: int, d: int, rows: int, seed: int, kind: str = "int"):
    """Seeded features x [rows, d] and head weights W [C, d] (bf16 bit patterns, uint16)
    and bias [C] (float32).

    kind "int":    x ∈ {-3..3}/8, W ∈ {-3..3}/16, bias ∈ {-64..64}/128.  Every product is a
                   multiple of 2^-7 and every partial sum stays below 2^17·2^-7, so all fp32
                   summation orders give the exact logits (and ties are frequent).
    kind "normal": x ~ N(0, 1), W ~ N(0, 1/d), bias ~ N(0, 0.1²), rounded to bf16.
    """
    rng = np.random.default_rng(seed)
    if kind == "int":
        x = rng.integers(-3, 4, size=(rows, d)).astype(np.float32) / 8
        W = rng.integers(-3, 4, size=(C, d)).astype(np.float32) / 16
        b = rng.integers(-64, 65, size=C).astype(np.float32) / 128
    elif kind == "normal":
        x = rng.standard_normal((rows, d), dtype=np.float32)
        W = rng.standard_normal((C, d), dtype=np.float32) / np.float32(np.sqrt(d))
        b = (rng.standard_normal(C, dtype=np.float32) * np.float32(0.1)).astype(np.float32)
    else:
        raise ValueError(kind)
    return f32_to_bf16_bits(x), f32_to_bf16_bits(W), b


def head_operands_device(C: int, d: int, rows: int, seed: int, device="cuda"):
    """Full-size "normal" operands generated on the GPU (torch generator; bench only)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn((rows, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    W = (torch.randn((C, d), generator=g, device=device, dtype=torch.float32) / d ** 0.5).to(torch.bfloat16)
    b = torch.randn((C,), generator=g, device=device, dtype=torch.float32) * 0.1
    return x, W, b

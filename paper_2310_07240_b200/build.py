"""Build libsc.so (the C-ABI library, sm_100a kernels) in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "libsc.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "sc.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc -c per translation unit (in parallel), then one nvcc -shared link."""
    if force or needs_build():
        from concurrent.futures import ThreadPoolExecutor
        objdir = os.path.join(PKG, "build")
        os.makedirs(objdir, exist_ok=True)
        compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

        def compile_one(src):
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            cmd = ["nvcc", *compile_flags, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
            r = subprocess.run(cmd, capture_output=True, text=True)
            return obj, r

        with ThreadPoolExecutor(max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
            results = list(ex.map(compile_one, sources()))
        for obj, r in results:
            if r.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
            if verbose:
                print(r.stderr)
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", SO,
               *[o for o, _ in results]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)

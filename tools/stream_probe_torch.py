"""Stream torch-allocated buffers with the stream_probe kernel: is the head's x slow to read?"""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "stream_probe.so"))
lib.stream_probe_ptr.restype = ctypes.c_float
lib.stream_probe_ptr.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int]
import synth
rows, d = 1 << 20, 2048
def rate(t, name):
    n = t.numel() * t.element_size()
    for layout in (0, 2):
        ms = lib.stream_probe_ptr(t.data_ptr(), n // 65536 * 65536, 65536, 3, layout)
        print(f"{name:40s} layout={layout} {n/1e9:.2f} GB {ms:.3f} ms {n/ms/1e9:.2f} TB/s", flush=True)
a = torch.empty(rows * d, dtype=torch.bfloat16, device="cuda"); a.fill_(1.0); rate(a, "torch.empty bf16 fill")
x, W, b = synth.head_operands_device(1000, d, rows, seed=2)
rate(x, "head_operands_device x")
x2 = x.clone(); rate(x2, "x.clone()")

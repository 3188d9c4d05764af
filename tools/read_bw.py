"""Calibrate the practical HBM read bandwidth on this B200 (torch reductions / copy)."""
import torch
import json
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n / 1e3
res = {}
for gb in (4, 16):
    x = torch.empty(gb << 28, dtype=torch.float32, device="cuda").normal_()
    y = torch.empty_like(x)
    dt = t(lambda: x.sum()); res[f"sum_{gb}GB_TBps"] = x.numel() * 4 / dt / 1e12
    dt = t(lambda: torch.amax(x)); res[f"amax_{gb}GB_TBps"] = x.numel() * 4 / dt / 1e12
    dt = t(lambda: y.copy_(x)); res[f"copy_{gb}GB_TBps(r+w)"] = 2 * x.numel() * 4 / dt / 1e12
    del y, x
    print(json.dumps(res), flush=True)

"""Time the GT pre-pass variants on cfg2 (CUDA events, 50 reps)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_07240_b200 as sc
import synth

spec = synth.config_context(2)
wl = synth.Workload(spec, seed=2)
rows = 1 << 20
d = wl.device_batch(0, rows)
ctx = sc.Context(spec.C, spec.lists, multi_app=True)
b = sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], rows=rows)
h = torch.zeros(256, dtype=torch.int64, device="cuda")
m = torch.empty(rows, dtype=torch.uint8, device="cuda")
w = torch.empty(256, dtype=torch.float32, device="cuda")

def t(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3

print("hist+mask      %.2f us" % t(lambda: sc.sc_decision_hist(ctx, b, hist_gt=h, gt_mask_out=m)))
print("mask only      %.2f us" % t(lambda: sc.sc_decision_hist(ctx, b, gt_mask_out=m)))
print("hist only      %.2f us" % t(lambda: sc.sc_decision_hist(ctx, b, hist_gt=h)))
print("weights        %.2f us" % t(lambda: sc.sc_weights_from_hist(ctx, h, w)))
print("zero 4KB       %.2f us" % t(lambda: h.zero_()))
h.zero_()
def fused():
    h.zero_(); sc.sc_decision_hist_weights(ctx, b, h, w, gt_mask_out=m)
print("zero+fused     %.2f us" % t(fused))
x = torch.empty(19 << 20, dtype=torch.uint8, device="cuda")
print("read 19MB sum  %.2f us" % t(lambda: x.sum(dtype=torch.int64)))

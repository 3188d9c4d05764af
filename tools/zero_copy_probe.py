"""Experiment: host-resident logits read by the kernels in place (UVA zero-copy) versus the
chunked H2D copy.  Does PCIe move only the sectors the gather kernel touches?

    python tools/zero_copy_probe.py [cfg] [rows]

Prints one line per variant: ms per pass and effective GB/s of *dense* logits."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2310_07240_b200 as sc  # noqa: E402
import synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 18)
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg)
    d = wl.device_batch(0, rows)
    lg = d["logits"]
    nbytes = lg.numel() * lg.element_size()
    h = torch.empty(lg.shape, dtype=lg.dtype, pin_memory=True)
    h.copy_(lg)
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, multi_app=True)
    gm = torch.empty(rows + 16, dtype=torch.uint8, device="cuda")
    hg = torch.zeros(256, dtype=torch.int64, device="cuda")
    w = torch.empty(256, dtype=torch.float32, device="cuda")
    sc.sc_decision_hist_weights(ctx, sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], rows=rows), hg, w, gt_mask_out=gm)
    out = dict(decision=torch.empty(rows, dtype=torch.uint8, device="cuda"),
               grad_idx=torch.empty(2 * rows, dtype=torch.int32, device="cuda"),
               grad_val=torch.empty(2 * rows, dtype=torch.float32, device="cuda"),
               loss_sum=torch.zeros(1, dtype=torch.float64, device="cuda"))

    def run(logits_tensor, host_ptr=None):
        b = sc.Batch(logits=logits_tensor, gt_mask=gm)
        if host_ptr is None:
            sc.sc_loss_fwd_bwd(ctx, b, w=w, **out)
            return
        cb = b._c()
        cb.logits = host_ptr
        st = torch.cuda.current_stream().cuda_stream
        rc = sc._lib.sc_loss_fwd_bwd(ctx.handle, ctypes.byref(cb), w.data_ptr(), ctypes.c_float(1.0),
                                     out["loss_sum"].data_ptr(), None, out["grad_idx"].data_ptr(),
                                     out["grad_val"].data_ptr(), None, out["decision"].data_ptr(), None, None, None, st)
        if rc:
            raise RuntimeError(sc.sc_last_error())

    def timeit(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps * 1e3

    ref_dec = None
    for kern in ("gather", "tma"):
        os.environ["SC_KERNEL"] = kern
        ms = timeit(lambda: run(lg))
        ref_dec = out["decision"].clone()
        print(f"cfg{cfg} rows={rows} device-resident {kern:6s}: {ms:8.3f} ms  {nbytes / ms / 1e6:8.1f} GB/s dense",
              flush=True)
    dst = torch.empty_like(lg)
    ms = timeit(lambda: dst.copy_(h, non_blocking=True))
    print(f"cfg{cfg} H2D copy alone          : {ms:8.3f} ms  {nbytes / ms / 1e6:8.1f} GB/s", flush=True)
    for kern in ("gather", "tma"):
        os.environ["SC_KERNEL"] = kern
        try:
            out["decision"].fill_(99)
            ms = timeit(lambda: run(lg, h.data_ptr()))
            ok = bool(torch.equal(out["decision"], ref_dec))
            print(f"cfg{cfg} zero-copy host   {kern:6s}: {ms:8.3f} ms  {nbytes / ms / 1e6:8.1f} GB/s dense-equiv  "
                  f"decisions_match={ok}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"cfg{cfg} zero-copy host {kern}: FAILED {e}", flush=True)
            return


if __name__ == "__main__":
    main()

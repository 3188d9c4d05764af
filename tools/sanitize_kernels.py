"""Every libsc kernel on tiny shapes, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  Run as

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_kernels.py

Covers: the eval kernel on the TMA ring (split maxima and list-major slots, EPL and generic
chunked paths), the sector gather kernel, both GT pre-pass kernels with and without the fused
weights, the weights kernel, the all-apps kernel, the value-ranges kernels (packed / ballot /
match counters, fast and far S arguments, unaligned arrays), the sampler, and the fused
classifier head.  Round 2 adds: the dense-mapped eval path (column-compacted rows, f32 /
bf16), the host-buffer entry (copy and zero copy), the lane-per-application all-apps kernel,
the head under every pattern and with column passes (CTA pairs with two row tiles too);
session 3: the lane-per-row all-apps kernel (f32 / bf16, ragged units) and the parked dense
gradient rows (every grad_dense step on the TMA ring).
Side bands at unaligned offsets and ragged row counts exercise the clamped TMA windows.  Outputs are checked against each other only lightly (the parity tests do the
real checking); the point is a clean sanitizer report.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_07240_b200 as sc  # noqa: E402
import synth  # noqa: E402


def dev_batch(b, dtype="f32"):
    lg = b["logits"]
    if dtype == "bf16":
        t = torch.from_numpy(np.ascontiguousarray(lg).view(np.int16)).cuda().view(torch.bfloat16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(lg)).cuda()
    out = dict(logits=t, gt_off=torch.from_numpy(b["gt_off"]).cuda(),
               gt_lab=torch.from_numpy(b["gt_lab"] if len(b["gt_lab"]) else np.zeros(1, np.int32)).cuda())
    out["app"] = torch.from_numpy(np.ascontiguousarray(b["app"]).view(np.int16)).cuda()
    return out


def step(spec, d, rows, order=0, app=False, mask_off=0, app_off=0, compact=False, host=None):
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=order, multi_app=True, compact=compact)
    na, S = spec.n_apps, ctx.grad_slots
    ap = None
    if app:
        abuf = torch.zeros(rows + app_off, dtype=torch.int16, device="cuda")
        ap = abuf[app_off:]
        ap.copy_(d["app"][:rows])
    gbuf = torch.zeros(rows + mask_off, dtype=torch.uint8, device="cuda")
    gm = gbuf[mask_off:]
    h = torch.zeros(na * 256, dtype=torch.int64, device="cuda")
    w = torch.empty(na * 256, dtype=torch.float32, device="cuda")
    gt = sc.Batch(gt_off=d["gt_off"], gt_lab=d["gt_lab"], app=ap, rows=rows)
    if na == 1:
        sc.sc_decision_hist_weights(ctx, gt, h, w, gt_mask_out=gm)
    sc.sc_decision_hist(ctx, gt, hist_gt=h.zero_(), gt_mask_out=gm)
    sc.sc_weights_from_hist(ctx, h, w)
    o = dict(loss_sum=torch.zeros(na, dtype=torch.float64, device="cuda"),
             loss_row=torch.empty(rows, dtype=torch.float32, device="cuda"),
             grad_idx=torch.empty(S * rows, dtype=torch.int32, device="cuda"),
             grad_val=torch.empty(S * rows, dtype=torch.float32, device="cuda"),
             decision=torch.empty(rows, dtype=torch.uint8, device="cuda"),
             n_incorrect=torch.zeros(na, dtype=torch.int64, device="cuda"),
             hist_pred=torch.zeros(na * 256, dtype=torch.int64, device="cuda"),
             hist_gt=torch.zeros(na * 256, dtype=torch.int64, device="cuda"))
    ld = d["logits"].stride(0)
    if spec.C <= 1000:
        o["grad_dense"] = torch.empty(rows * ld, dtype=torch.float32, device="cuda")
    if host is None:
        sc.sc_loss_fwd_bwd(ctx, sc.Batch(logits=d["logits"][:rows], gt_mask=gm, app=ap), w=w, grad_scale=1.0 / rows, **o)
    else:  # (mode, stager chunk rows): logits from pinned host memory
        hmode, crows = host
        hl = d["logits"][:rows].cpu().pin_memory()
        stg = sc.Stager(crows * hl.stride(0) * hl.element_size()) if crows else None
        sc.sc_loss_fwd_bwd_host(ctx, stg, sc.Batch(logits=hl, gt_mask=gm, app=ap), mode=hmode, w=w,
                                grad_scale=1.0 / rows, **o)
    sc.sc_decide(ctx, sc.Batch(logits=d["logits"][:rows], gt_off=d["gt_off"][:rows + 1], gt_lab=d["gt_lab"], app=ap),
                 decision=o["decision"], n_incorrect=o["n_incorrect"], hist_pred=o["hist_pred"], hist_gt=o["hist_gt"])
    torch.cuda.synchronize()
    assert int(o["hist_pred"].sum()) == 2 * rows
    return sc.sc_last_kernel()


def main():
    torch.cuda.set_device(0)
    seen = []
    for kernel in ("tma", "gather"):
        os.environ["SC_KERNEL"] = kernel
        for cfg, dtype, rows, order, app, mo, ao in [
            (1, "f32", 1000, 0, False, 0, 0), (1, "f32", 333, 0, False, 3, 0), (2, "f32", 517, 0, False, 5, 0),
            (2, "bf16", 300, 0, False, 1, 0), (2, "f32", 300, 1, False, 0, 0), (2, "f32", 300, 2, False, 7, 0),
            (3, "f32", 37, 0, False, 2, 0), (3, "bf16", 41, 1, False, 0, 0), (4, "f32", 701, 0, True, 3, 1),
            (4, "bf16", 257, 2, True, 0, 3)]:
            spec = synth.config_context(cfg)
            wl = synth.Workload(spec, seed=cfg, dtype=dtype, layout=1)
            b = wl.host_batch(11, rows)
            seen.append((kernel, cfg, dtype, order, step(spec, dev_batch(b, dtype), rows, order, app, mo, ao)))
    os.environ.pop("SC_KERNEL")
    # generic path: C > 1024 mapped labels / rows split into column chunks
    rng = np.random.default_rng(1)
    C = 30000
    spec = synth.ContextSpec(C, [[sorted(rng.choice(C, 800, replace=False).tolist()),
                                  sorted(rng.choice(C, 700, replace=False).tolist())]], 0.0, 10.0)
    b = synth.Workload(spec, seed=9).host_batch(0, 40)
    seen.append(("auto", "wide", "f32", 0, step(spec, dev_batch(b), 40)))
    os.environ["SC_HIST"] = "warp"
    spec = synth.config_context(2)
    b = synth.Workload(spec, seed=2).host_batch(0, 999)
    seen.append(("auto", "hist_warp", "f32", 0, step(spec, dev_batch(b), 999, mask_off=9)))
    os.environ.pop("SC_HIST")

    # column-compacted rows: the dense-mapped path (> 256 mapped columns), f32 and bf16
    for cfg, dtype, rows in ((3, "f32", 45), (3, "bf16", 70)):
        spec = synth.config_context(cfg)
        b = synth.Workload(spec, seed=cfg, dtype=dtype).host_batch(5, rows)
        cols = np.nonzero(spec.mapped().any(axis=0))[0]
        ldc = synth.default_ld(len(cols), dtype)
        lg = np.zeros((rows, ldc), dtype=b["logits"].dtype)
        lg[:, :len(cols)] = b["logits"][:, cols]
        bc = dict(b)
        bc["logits"] = lg
        seen.append(("compact", cfg, dtype, step(spec, dev_batch(bc, dtype), rows, compact=True)))
    # host-buffer entry: chunked copies (ragged last chunk) and zero copy
    spec = synth.config_context(2)
    b = synth.Workload(spec, seed=2).host_batch(3, 700)
    seen.append(("host_copy", step(spec, dev_batch(b), 700, host=(1, 256))))
    seen.append(("host_zero_copy", step(spec, dev_batch(b), 700, host=(2, 0))))

    # one read, every application
    spec = synth.config_context(4)
    b = synth.Workload(spec, seed=4, layout=1).host_batch(0, 77)
    d = dev_batch(b)
    ctx = sc.Context(spec.C, spec.lists, multi_app=True)
    ni = torch.zeros(256, dtype=torch.int64, device="cuda")
    hp = torch.zeros(256 * 256, dtype=torch.int64, device="cuda")
    dec = torch.empty(77 * 256, dtype=torch.uint8, device="cuda")
    for impl in ("rows", "lane", "warp"):
        if impl != "rows":
            os.environ["SC_ALLAPPS"] = impl
        sc.sc_decide_all_apps(ctx, sc.Batch(logits=d["logits"], gt_off=d["gt_off"], gt_lab=d["gt_lab"]),
                              n_incorrect=ni, hist_pred=hp, decision=dec)
        torch.cuda.synchronize()
        seen.append(("all_apps", sc.sc_last_kernel()))
    os.environ.pop("SC_ALLAPPS")
    bb = synth.Workload(spec, seed=4, dtype="bf16", layout=1).host_batch(0, 45)  # bf16 rows, ragged unit
    db = dev_batch(bb, "bf16")
    sc.sc_decide_all_apps(ctx, sc.Batch(logits=db["logits"], gt_off=db["gt_off"], gt_lab=db["gt_lab"]),
                          n_incorrect=ni, hist_pred=hp, decision=dec[:45 * 256])
    torch.cuda.synchronize()
    seen.append(("all_apps_bf16", sc.sc_last_kernel()))

    # value ranges: 2-8 bins packed, 21 ballot, 41 match; far S arguments; unaligned arrays
    for m, off, scale in ((7, 0, 1.0), (7, 1, 12.0), (20, 0, 1.0), (40, 3, 12.0)):
        edges = np.sort(rng.uniform(-1, 1, m + 1)).astype(np.float32) * np.float32(scale)
        r = sc.Ranges(edges[:-1], edges[1:], 10.0)
        n = 1003
        score = torch.cat([torch.zeros(off), torch.from_numpy(rng.uniform(-1.2, 1.2, n).astype(np.float32) * scale)]).cuda()[off:]
        gts = torch.cat([torch.zeros(off), torch.from_numpy(rng.uniform(-1.2, 1.2, n).astype(np.float32) * scale)]).cuda()[off:]
        hist = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
        gtr = torch.empty(n + off, dtype=torch.uint8, device="cuda")[off:]
        sc.sc_ranges_hist(r, gts, hist_gt=hist, gt_range_out=gtr)
        w = torch.empty(m + 1, dtype=torch.float32, device="cuda")
        sc.sc_ranges_weights(r, hist, w)
        out = dict(loss_sum=torch.zeros(1, dtype=torch.float64, device="cuda"),
                   loss_row=torch.empty(n + off, dtype=torch.float32, device="cuda")[off:],
                   grad=torch.empty(n + off, dtype=torch.float32, device="cuda")[off:],
                   decision=torch.empty(n + off, dtype=torch.uint8, device="cuda")[off:],
                   n_incorrect=torch.zeros(1, dtype=torch.int64, device="cuda"),
                   hist_pred=torch.zeros(m + 1, dtype=torch.int64, device="cuda"))
        sc.sc_ranges_loss_fwd_bwd(r, score, gtr, w=w, grad_scale=1.0 / n, **out)
        torch.cuda.synchronize()
        assert int(out["hist_pred"].sum()) == n
    seen.append(("ranges", 4))

    # sampler
    gm = torch.from_numpy(rng.integers(0, 8, 5000).astype(np.uint8)).cuda()
    w = torch.from_numpy(rng.uniform(0.5, 2, 256).astype(np.float32)).cuda()
    u = torch.from_numpy(rng.random(2 * 3001)).cuda()
    out = torch.empty(3001, dtype=torch.int64, device="cuda")
    sc.sc_rebalance_sample(gm, w, u, out)
    torch.cuda.synchronize()
    assert int(out.min()) >= 0 and int(out.max()) < 5000
    seen.append(("sampler",))

    # fused head: two tiles per unit (cfg2), one tile (w300), column passes (w560), the
    # per-list patterns, CTA pairs with two row tiles; ragged rows
    for sizes, d_, rows, order, env in (((90, 30, 60), 256, 300, 0, {}), ((120, 100, 80), 128, 129, 0, {}),
                                        ((300, 250), 64, 200, 1, {}), ((90, 30, 60), 128, 600, 2, {}),
                                        ((90, 30, 60), 128, 1100, 0, {"SC_HEAD_CLUSTER": "2", "SC_HEAD_PAIR_T2": "1"})):
        os.environ.update(env)
        spec = synth.ContextSpec(1000, [synth.placed_context(1000, sizes, 9)], 0.0, 10.0)
        x, W, bias = synth.head_operands(1000, d_, rows, seed=3, kind="int")
        ctx = sc.Context(spec.C, spec.lists, order=order, multi_app=True)
        S = ctx.grad_slots
        Wd = torch.from_numpy(W.view(np.int16)).cuda().view(torch.bfloat16)
        head = sc.Head(ctx, Wd, torch.from_numpy(bias).cuda())
        xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
        hb = synth.Workload(spec, seed=3).host_batch(0, rows)
        go, gl = torch.from_numpy(hb["gt_off"]).cuda(), torch.from_numpy(hb["gt_lab"]).cuda()
        o = dict(decision=torch.empty(rows, dtype=torch.uint8, device="cuda"),
                 loss_row=torch.empty(rows, dtype=torch.float32, device="cuda"),
                 grad_idx=torch.empty(S * rows, dtype=torch.int32, device="cuda"),
                 grad_val=torch.empty(S * rows, dtype=torch.float32, device="cuda"),
                 loss_sum=torch.zeros(1, dtype=torch.float64, device="cuda"),
                 n_incorrect=torch.zeros(1, dtype=torch.int64, device="cuda"),
                 hist_pred=torch.zeros(256, dtype=torch.int64, device="cuda"),
                 hist_gt=torch.zeros(256, dtype=torch.int64, device="cuda"))
        sc.sc_head_loss_fwd_bwd(ctx, head, xd, gt_off=go, gt_lab=gl, grad_scale=1.0 / rows, **o)
        torch.cuda.synchronize()
        assert int(o["hist_pred"].sum()) == rows
        seen.append(("head", order, sc.sc_last_kernel(), head.info()))
        for k in env:
            os.environ.pop(k)
    for s in seen:
        print(*s)
    print(f"sanitize_kernels: {sc.sc_launch_count()} libsc launches ok")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the hot path: batched software-context evaluation (decide + counters
+ rebalanced decision-aware loss fwd/bwd) on B200, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one pass of the whole hot path over one batch:
sc_decision_hist -> allreduce(hist) -> sc_weights_from_hist -> sc_loss_fwd_bwd ->
allreduce(aggregates).  Workload (BASELINE.json configs[1]): C = 1000 labels, 3 lists
+ default (D = 4), B = 2^20 rows per GPU, f32 logits, seeded synthetic data (synth/),
weak scaling (each rank owns its own 2^20 rows of one global dataset).

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (oracle/) on
this box's host cores instead (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/s for fused decide+loss fwd/bwd (1/2/4/8 B200); % of HBM roofline"
CFG = 2
ROWS_PER_GPU = 1 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (GPUs); without torchrun, N > 1 re-launches this script under torch.distributed.run")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=0, help="rows per GPU (default: 2^20 for cfg2)")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--config", type=int, default=CFG, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default 2, the metric's config; others for characterisation)")
    ap.add_argument("--kernel", default=None, choices=["tma", "gather"], help="force an eval kernel (default: auto)")
    ap.add_argument("--mode", default="step", choices=["step", "all_apps", "head", "sample", "ranges"],
                    help="step: the hot path; all_apps: one read, every application (NEXT f3, config 4); "
                         "head: classifier-head GEMM fused with the evaluation (NEXT f4); sample: the "
                         "rebalanced sampler (NEXT f2); ranges: the value-ranges pattern (NEXT f1)")
    ap.add_argument("--d", type=int, default=2048, help="--mode head: feature width (ResNet-50 penultimate = 2048)")
    ap.add_argument("--order", default="api_output", choices=["api_output", "app_choice", "multi_select"],
                    help="decision pattern (default: the north star's API-output order)")
    ap.add_argument("--compact", action="store_true",
                    help="column-compacted rows (sc_context_load_compact, NEXT f3): each row holds only the "
                         "mapped labels' logits, as a producer restricted to those columns emits them")
    ap.add_argument("--grad", default="sparse", choices=["sparse", "dense"],
                    help="gradient output: sparse slots (default) or the dense [rows, ld] f32 gradient "
                         "(SURVEY.md 8(d): reported separately, adds ld*4 B/row of writes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU work of the cpu_baseline sample")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers

def dist_on(world: int) -> bool:
    """Collectives in play: N > 1, or SC_FORCE_DIST=1 (the N > 1 path with one rank)."""
    return world > 1 or os.environ.get("SC_FORCE_DIST") == "1"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


WORKLOADS = {
    1: "cfg1_heapsortcypher: C=32 labels, D=4 (the paper's Recycle/Compost/Donate + default)",
    2: "cfg2_imagenet1k: C=1000 labels, D=4 (Recycle/Compost/Donate x10 + default)",
    3: "cfg3_openimages20k: C=20000 labels, D=8 (7 lists + default)",
    4: "cfg4_multiapp256: C=1000 labels, 256 applications (per-row app id), contiguous rows per app",
    5: "cfg5_rebalance64m: C=1000 labels, D=4 (cfg2's context), 64M rows over 8 GPUs",
}
DEFAULT_ROWS = {1: 4096, 2: 1 << 20, 3: 1 << 19, 4: 1 << 22, 5: 1 << 23}


def workload_name(cfg, dtype):
    return f"{WORKLOADS[cfg]}, {dtype} logits"


def touched_sector_bytes(spec, ld, elt, rows=None, layout_rows_per_app=1 << 18, columns=None, granule=32):
    """Mean bytes per row of the 32-B sectors holding at least one mapped label of the
    row's application (SURVEY.md §8(d)'s algorithmic minimum), row base addresses r*ld*elt.
    columns: the labels of a compacted row's columns (sc_context_columns), else column c = label c.
    granule=128: the same over 128-B lines, the unit HBM is read in for scattered sectors
    (lts__t_sectors_srcunit_tex_op_read = dram__sectors_read for the gather)."""
    import numpy as np
    m = spec.mapped()
    per_app = []
    for a in range(spec.n_apps):
        cols = np.nonzero(m[a])[0]
        if columns is not None:
            cols = np.searchsorted(columns, cols)
        if len(cols) == 0:
            per_app.append(0.0)
            continue
        if (ld * elt) % granule == 0:
            per_app.append(len(np.unique((cols * elt) // granule)) * float(granule))
        else:  # rows not granule aligned: average over the row phases (rows are 16-B aligned)
            phases = range(0, granule, 16)
            tot = 0
            for ph in phases:
                tot += len(np.unique((ph + cols * elt) // granule)) * granule
            per_app.append(tot / len(phases))
    if rows is None or spec.n_apps == 1:
        return float(np.mean(per_app))
    apps = (np.arange(rows) // layout_rows_per_app) % spec.n_apps
    return float(np.mean(np.asarray(per_app)[apps]))


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_traffic(cfg, dtype, kernel, rows, compact=False):
    """dram read+write bytes per launch of the eval kernel from the committed ncu summary
    (profiles/ncu_eval_cfg{cfg}[_compact]_{dtype}_{kernel}.json), scaled to this launch's rows."""
    tag = f"cfg{cfg}_compact" if compact else f"cfg{cfg}"
    path = os.path.join(ROOT, "profiles", f"ncu_eval_{tag}_{dtype}_{kernel}.json")
    try:
        d = json.load(open(path))
        return d["dram_bytes_per_row"] * rows, os.path.relpath(path, ROOT)
    except Exception:
        return None, None


# ------------------------------------------------------------------ CPU oracle timing

class OracleSample:
    """A bounded sample of the cfg2 workload on the host plus the oracle (as it stands)
    timed over it with `threads` host threads (512-row chunks; ctypes releases the GIL)."""

    chunk = 512

    def __init__(self, cpu_seconds: float, threads: int | None = None, seed_rows: int = 0):
        from concurrent.futures import ThreadPoolExecutor

        import synth
        from oracle import Oracle
        self.Oracle = Oracle
        spec = synth.config_context(CFG)
        self.wl = synth.Workload(spec, seed=CFG)
        self.orc = Oracle.from_spec(spec)
        self.threads = threads or os.cpu_count() or 1
        b = self.wl.host_batch(seed_rows, self.chunk)
        t = time.perf_counter()
        pre = self.orc.eval(b["logits"], b["gt_off"], b["gt_lab"], want_loss=False)
        self.orc.eval(b["logits"], b["gt_off"], b["gt_lab"], w=Oracle.weights_by_mask(pre["hist_gt"]))
        per_row = (time.perf_counter() - t) / self.chunk
        # ~cpu_seconds of oracle work in total (summed over threads)
        n_chunks = max(self.threads, int(cpu_seconds / (per_row * self.chunk)))
        n_chunks = min(n_chunks, (1 << 18) // self.chunk)  # <= 1 GB of host logits
        with ThreadPoolExecutor(self.threads) as ex:
            self.batches = list(ex.map(lambda i: self.wl.host_batch(seed_rows + i * self.chunk, self.chunk),
                                       range(n_chunks)))
        self.rows = n_chunks * self.chunk
        self.first_row = seed_rows

    def run(self):
        """One pass of the hot path over the sample: GT pre-pass, weights, full pass. -> seconds"""
        from concurrent.futures import ThreadPoolExecutor
        orc, Oracle, rows = self.orc, self.Oracle, self.rows

        def hist(bb):
            return orc.eval(bb["logits"], bb["gt_off"], bb["gt_lab"], want_loss=False)["hist_gt"]

        def full(args):
            bb, w = args
            return orc.eval(bb["logits"], bb["gt_off"], bb["gt_lab"], w=w, grad_scale=1.0 / rows)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            H = sum(ex.map(hist, self.batches))
            w = Oracle.weights_by_mask(H)
            list(ex.map(full, [(bb, w) for bb in self.batches]))
        return time.perf_counter() - t0

    def describe(self, dt):
        return (f"{self.rows} rows of cfg2 (rows {self.first_row}..{self.first_row + self.rows - 1}), GT pre-pass + "
                f"weights + full oracle pass, {self.threads} threads x {self.chunk}-row chunks, {dt:.2f} s wall")


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_oracle_rate(seconds: float, threads: int | None = None, seed_rows=0):
    """Oracle (as it stands) on host cores over a bounded sample of the same workload."""
    s = OracleSample(seconds, threads, seed_rows)
    dt = s.run()
    return s.rows / dt, s.rows, dt, s.threads, s


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    # each step: one oracle pass over a bounded sample, sized so warmup+steps end in ~2.5 minutes
    threads = os.cpu_count() or 1
    budget_wall = 150.0 / max(1, args.steps + args.warmup)
    sample = OracleSample(max(0.05, min(budget_wall, 10.0)) * threads)
    times = []
    for i in range(args.warmup + args.steps):
        dt = sample.run()
        if i >= args.warmup:
            times.append(dt)
    total_t = sum(times)
    value = sample.rows * len(times) / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / max(1, len(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(CFG, "f32"), "C": 1000, "rows_per_step": sample.rows,
                   "parallelism": f"{sample.threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": sample.threads, "kind": "oracle",
                         "sample": sample.describe(total_t / max(1, len(times))) + " per step"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def run_ours(args):
    import numpy as np
    import torch

    if args.kernel:
        os.environ["SC_KERNEL"] = args.kernel
    cfg = args.config

    world, rank, local = dist_env()
    # SC_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo (exercises the N > 1 path on one GPU)
    share = os.environ.get("SC_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    elif torch.cuda.device_count() < world:
        print(json.dumps({"error": f"{world} ranks but {torch.cuda.device_count()} visible GPUs "
                                   "(SC_BENCH_SHARE_GPU=1 runs every rank on cuda:0 over gloo)"}),
              file=sys.stderr, flush=True)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    # SC_FORCE_DIST=1: a process group (and the N > 1 step) even for one rank
    if dist_on(world):
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2310_07240_b200 as sc
    import synth
    from paper_2310_07240_b200.step import Evaluator

    spec = synth.config_context(cfg)
    B = args.rows or DEFAULT_ROWS[cfg]
    wl = synth.Workload(spec, seed=cfg, dtype=args.dtype, rows_per_app=1 << 18)
    order = {"api_output": 0, "app_choice": 1, "multi_select": 2}[args.order]
    ctx = sc.Context(spec.C, spec.lists, spec.tau, spec.k, order=order, multi_app=True, compact=args.compact)
    columns = None
    if args.compact:
        columns = ctx.columns()
        data = compact_device_batch(wl, rank * B, B, columns, dev)
    else:
        data = wl.device_batch(rank * B, B, device=dev)  # this rank's rows of the global dataset
    logits, gt_off, gt_lab = data["logits"], data["gt_off"], data["gt_lab"]
    app = data.get("app")
    ev = Evaluator(ctx, B, device=dev, group=group, dense_ld=logits.stride(0) if args.grad == "dense" else 0)
    global_rows = B * world

    def barrier():
        if dist_on(world):
            import torch.distributed as dist
            dist.barrier()

    stream = torch.cuda.current_stream(dev)
    if args.mode == "head":
        return run_head(args, sc, ctx, spec, gt_off, gt_lab, B, dev, stream, rank, data)
    if args.mode == "all_apps":
        return run_all_apps(args, sc, ctx, logits, gt_off, gt_lab, B, dev, stream, rank)
    if args.mode == "sample":
        return run_sample(args, sc, ev, logits, gt_off, gt_lab, B, dev, stream, rank)
    if args.mode == "ranges":
        del data, logits, gt_off, gt_lab
        return run_ranges(args, sc, dev, stream, rank)
    for _ in range(args.warmup):
        ev.step(logits, gt_off, gt_lab, app=app, global_rows=global_rows)
    torch.cuda.synchronize(dev)

    # instrumented step: CUDA events around each libsc call on the stream it is launched on
    import paper_2310_07240_b200.step as step_mod
    phases = ("sc_decision_hist", "sc_decision_hist_weights", "sc_weights_from_hist", "sc_loss_fwd_bwd")
    called = set()
    ev_s = {ph: [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] for ph in phases}
    ev_e = {ph: [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] for ph in phases}
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    idx = {"i": -1}
    origs = {ph: getattr(step_mod, ph) for ph in phases}

    def wrap(ph):
        def timed(*a, **kw):
            i = idx["i"]
            called.add(ph)
            ev_s[ph][i].record(stream)
            origs[ph](*a, **kw)
            ev_e[ph][i].record(stream)
        return timed

    for ph in phases:
        setattr(step_mod, ph, wrap(ph))
    k_start, k_end = ev_s["sc_loss_fwd_bwd"], ev_e["sc_loss_fwd_bwd"]
    launches0 = sc.sc_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        t_start.record(stream)
        for i in range(args.steps):
            idx["i"] = i
            ev.step(logits, gt_off, gt_lab, app=app, global_rows=global_rows)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    for ph in phases:
        setattr(step_mod, ph, origs[ph])
    launches = sc.sc_launch_count() - launches0
    phase_us = {ph: 1e3 * sum(a.elapsed_time(b) for a, b in zip(ev_s[ph], ev_e[ph])) / args.steps
                for ph in phases if ph in called}
    ms = t_start.elapsed_time(t_end)
    k_ms = sum(a.elapsed_time(b) for a, b in zip(k_start, k_end)) / args.steps
    if dist_on(world):
        import torch.distributed as dist
        t = torch.tensor([ms, k_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, k_ms = float(t[0]), float(t[1])
    ms_per_step = ms / args.steps
    value = global_rows / (ms_per_step / 1e3)

    # sanity: the outputs of the last step are self-consistent
    o = ev.out
    assert int(o.hist_gt.sum()) == global_rows and int(o.hist_pred(spec.n_apps).sum()) == global_rows

    # roofline of the dominant kernel (eval_kernel behind sc_loss_fwd_bwd)
    elt = 4 if args.dtype == "f32" else 2
    ld = logits.stride(0)
    sect = touched_sector_bytes(spec, ld, elt, rows=B, columns=columns)
    lines = touched_sector_bytes(spec, ld, elt, rows=B, columns=columns, granule=128)
    per_row = sect + 1 + 1 + 8 * ctx.grad_slots + (2 if app is not None else 0)  # sectors + G_i + decision + sparse grad (+ app)
    if args.grad == "dense":
        per_row += ld * 4  # the full f32 gradient row written
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = B * per_row / (k_ms / 1e3) / 1e9
    kname = sc.sc_last_kernel()
    traffic, tpath = load_traffic(cfg, args.dtype, kname, B, compact=args.compact)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "eval_kernel (sc_loss_fwd_bwd)", "kernel_ms": k_ms,
                "algorithmic_bytes_per_row": per_row, "dense_bytes_per_row": ld * elt + 18,
                "dense_frac": B * (ld * elt + 18) / (k_ms / 1e3) / 1e9 / peak,
                # the same with the 128-B lines holding a mapped label in place of the sectors
                "line_bytes_per_row": per_row - sect + lines,
                "line_frac": B * (per_row - sect + lines) / (k_ms / 1e3) / 1e9 / peak,
                "eval_kernel": kname, "traffic_source": tpath,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peaks else "fallback 6.65 TB/s"}

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.dtype), "C": spec.C, "rows_per_gpu": B, "global_batch": global_rows,
                   "parallelism": f"dp{world}", "l2": f"no flush: {B * ld * elt / 1e9:.2f} GB of logits per step per GPU > 126 MB L2",
                   "grad": (f"sparse ({ctx.grad_slots} slots/row)" if args.grad == "sparse"
                            else f"dense f32 [rows, {ld}] + sparse slots"), "order": args.order,
                   "layout": (f"column-compacted: {len(columns)} of {spec.C} label columns per row (sc_context_load_compact)"
                              if args.compact else "dense rows, column c = label c")},
        "roofline": roofline,
        "gpu_launches": int(launches),
        "phases_us": {k: round(v, 2) for k, v in phase_us.items()},
        "clocks": clk.summary(),
    }

    # e2e: same metric through the public API with host (pinned) buffers, copies inside the timed region
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, ev, data, global_rows, dev, barrier, world)
    del data, logits
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the oracle baseline: rank 0 at N = 1 only
        rate, rows, dt, threads, smp = cpu_oracle_rate(args.cpu_seconds)
        rate1, rows1, dt1, _, smp1 = cpu_oracle_rate(min(4.0, args.cpu_seconds / 3), threads=1)
        line["cpu_baseline"] = {"value": rate, "unit": "samples/s", "cores": threads, "kind": "oracle",
                                "sample": smp.describe(dt), "cpu_model": cpu_model(),
                                "single_thread": {"value": rate1, "unit": "samples/s", "sample": smp1.describe(dt1)},
                                "per_config": "profiles/r2_cpu_baseline_split.json (tools/cpu_baseline_split.py)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_on(world):
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def compact_device_batch(wl, row0, n, columns, dev, chunk=1 << 14):
    """Rows [row0, row0+n) of the workload with only the given label columns kept (the rows a
    producer restricted to the mapped labels emits): generated densely chunk by chunk on the
    GPU, then column-gathered (input preparation, outside every timed region)."""
    import torch
    import synth
    cols = torch.from_numpy(columns.astype("int64")).to(dev)
    ldc = synth.default_ld(len(columns), wl.dtype)
    tdt = torch.float32 if wl.dtype == "f32" else torch.bfloat16
    logits = torch.full((max(n, 1), ldc), float("nan"), dtype=tdt, device=dev)
    gt = wl.device_batch(row0, 0, device=dev) if n == 0 else None
    offs, labs, apps, base = [], [], [], 0
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        b = wl.device_batch(row0 + lo, hi - lo, device=dev)
        logits[lo:hi, :len(columns)] = b["logits"].index_select(1, cols)
        offs.append(b["gt_off"][:-1] + base if lo + chunk < n else b["gt_off"] + base)
        labs.append(b["gt_lab"])
        base += int(b["gt_off"][-1])
        if "app" in b:
            apps.append(b["app"])
        del b
    out = dict(logits=logits[:n])
    if n == 0:
        out.update(gt_off=gt["gt_off"], gt_lab=gt["gt_lab"])
    else:
        out.update(gt_off=torch.cat(offs), gt_lab=torch.cat(labs))
    if apps:
        out["app"] = torch.cat(apps)
    return out


def run_all_apps(args, sc, ctx, logits, gt_off, gt_lab, B, dev, stream, rank):
    """One read of the logits, every application (sc_decide_all_apps): row-app evaluations/s."""
    import torch
    A = ctx.n_apps
    ni = torch.zeros(A, dtype=torch.int64, device=dev)
    hp = torch.zeros(A * 256, dtype=torch.int64, device=dev)
    batch = sc.Batch(logits=logits, gt_off=gt_off, gt_lab=gt_lab)
    for _ in range(args.warmup):
        sc.sc_decide_all_apps(ctx, batch, n_incorrect=ni, hist_pred=hp)
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(args.steps):
        sc.sc_decide_all_apps(ctx, batch, n_incorrect=ni, hist_pred=hp)
    e.record(stream)
    torch.cuda.synchronize(dev)
    ms = s.elapsed_time(e) / args.steps
    # roofline: plain ALU work, at least one compare per (row, application, mapped label); the
    # peak is the ALU pipe (IADD3/LOP3/FMNMX: 16 lanes/clk per SM sub-partition, 4 per SM,
    # /opt/skills/guides/B300_MICROARCH.md "Pipe rates") x 148 SMs x the max SM clock
    import synth
    entries = int(synth.config_context(args.config).mapped().sum())
    ops = B * entries
    peak_ops = 148 * 64 * 1.965e9
    hbm = B * (logits.stride(0) * logits.element_size() + 18) / (ms / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({"metric": "row-application evaluations/s (one read, every application)",
                          "value": B * A / (ms / 1e3), "unit": "evaluations/s", "ms_per_step": ms, "rows": B,
                          "apps": A, "dtype": args.dtype, "config": {"workload": workload_name(args.config, args.dtype)},
                          "roofline": {"bound": "alu", "achieved": ops / (ms / 1e3) / 1e12, "peak": peak_ops / 1e12,
                                       "unit": "Tops/s (one compare per row x app x mapped label)",
                                       "frac": ops / (ms / 1e3) / peak_ops, "entries_per_row": entries,
                                       "hbm_gbs": hbm, "hbm_frac": hbm / _peak()},
                          "gpu_launches_per_step": 1}), flush=True)
    return 0


def _peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(path)).get("hbm_gbs", 6650.0) if os.path.exists(path) else 6650.0


def _timed(fn, steps, warmup, stream, dev):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        fn()
    e.record(stream)
    torch.cuda.synchronize(dev)
    return s.elapsed_time(e) / steps


def run_sample(args, sc, ev, logits, gt_off, gt_lab, B, dev, stream, rank):
    """Rebalanced training-data sampler (NEXT f2): B draws with probability
    proportional to w[G_i] over the batch's B rows (G_i and w from one step of the hot path)."""
    import torch
    o = ev.step(logits, gt_off, gt_lab)
    g = torch.Generator(device=dev)
    g.manual_seed(args.config)
    n = B
    u = torch.rand(2 * n, dtype=torch.float64, device=dev, generator=g)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    ws = torch.empty(sc.sc_sample_workspace_bytes(B), dtype=torch.uint8, device=dev)
    gm = o.gt_mask[:B]
    ms = _timed(lambda: sc.sc_rebalance_sample(gm, o.w, u, out, workspace=ws), args.steps, args.warmup, stream, dev)
    per = B * 1 + n * (16 + 8)  # masks read + uniforms read + indices written (algorithmic bytes)
    peak = _peak()
    ach = per / (ms / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({"metric": "rebalanced draws/s (NEXT f2)", "value": n / (ms / 1e3), "unit": "draws/s",
                          "ms_per_step": ms, "rows": B, "draws": n, "steps": args.steps, "warmup": args.warmup,
                          "config": {"workload": workload_name(args.config, args.dtype) + ", G_i / w from the step"},
                          "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                                       "algorithmic_bytes": per},
                          "gpu_launches_per_step": 5}), flush=True)
    return 0


def run_ranges(args, sc, dev, stream, rank):
    """Value-ranges pattern (NEXT f1): GT pre-pass + weights + fused loss
    pass over 2^26 scores (7 ranges over [-1, 1]; uniform scores and ground-truth scores)."""
    import torch
    rows = args.rows or (1 << 26)
    m = 7
    edges = torch.linspace(-1.0, 1.0, m + 1)
    r = sc.Ranges(edges[:-1].numpy().astype("float32"), edges[1:].numpy().astype("float32"), 10.0)
    g = torch.Generator(device=dev)
    g.manual_seed(args.config)
    score = (torch.rand(rows, device=dev, generator=g) * 2.4 - 1.2).float()
    gt = (torch.rand(rows, device=dev, generator=g) * 2.4 - 1.2).float()
    hist = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    gtr = torch.empty(rows, dtype=torch.uint8, device=dev)
    w = torch.empty(m + 1, dtype=torch.float32, device=dev)
    out = dict(loss_sum=torch.zeros(1, dtype=torch.float64, device=dev),
               loss_row=torch.empty(rows, dtype=torch.float32, device=dev),
               grad=torch.empty(rows, dtype=torch.float32, device=dev),
               decision=torch.empty(rows, dtype=torch.uint8, device=dev),
               n_incorrect=torch.zeros(1, dtype=torch.int64, device=dev),
               hist_pred=torch.zeros(m + 1, dtype=torch.int64, device=dev))

    def step():
        hist.zero_()
        sc.sc_ranges_hist(r, gt, hist_gt=hist, gt_range_out=gtr)
        sc.sc_ranges_weights(r, hist, w)
        sc.sc_ranges_loss_fwd_bwd(r, score, gtr, w=w, grad_scale=1.0 / rows, **out)

    ms = _timed(step, args.steps, args.warmup, stream, dev)
    per_row = (4 + 1) + (4 + 1 + 4 + 4 + 1)  # pre-pass: gt score in, range out; loss: score, range in, loss, grad, decision out
    peak = _peak()
    ach = rows * per_row / (ms / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({"metric": "samples/s, value-ranges decide+loss fwd/bwd (NEXT f1)", "value": rows / (ms / 1e3),
                          "unit": "samples/s", "ms_per_step": ms, "rows": rows, "ranges": m, "steps": args.steps,
                          "warmup": args.warmup, "dtype": "f32",
                          "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                                       "algorithmic_bytes_per_row": per_row}}), flush=True)
    return 0


def run_head(args, sc, ctx, spec, gt_off, gt_lab, B, dev, stream, rank, data):
    """Classifier head z = x W_𝕎ᵀ + b on tcgen05 with decide + loss fwd/bwd in the GEMM
    epilogue (sc_head_loss_fwd_bwd), against the unfused pair it replaces: a cuBLAS GEMM
    writing all C bf16 logits, then sc_loss_fwd_bwd reading them back."""
    import torch
    import synth
    del data["logits"]
    torch.cuda.empty_cache()
    x, W, b = synth.head_operands_device(spec.C, args.d, B, seed=args.config)
    head = sc.Head(ctx, W, b)
    d, n_cols = head.info()
    gm = torch.empty(B + 16, dtype=torch.uint8, device=dev)
    hg = torch.zeros(256, dtype=torch.int64, device=dev)
    w = torch.empty(256, dtype=torch.float32, device=dev)
    S = ctx.grad_slots
    out = dict(decision=torch.empty(B, dtype=torch.uint8, device=dev),
               grad_idx=torch.empty(S * B, dtype=torch.int32, device=dev),
               grad_val=torch.empty(S * B, dtype=torch.float32, device=dev),
               loss_sum=torch.zeros(1, dtype=torch.float64, device=dev),
               n_incorrect=torch.zeros(1, dtype=torch.int64, device=dev),
               hist_pred=torch.zeros(256, dtype=torch.int64, device=dev))

    def fused():
        hg.zero_()
        sc.sc_decision_hist_weights(ctx, sc.Batch(gt_off=gt_off, gt_lab=gt_lab, rows=B), hg, w, gt_mask_out=gm)
        sc.sc_head_loss_fwd_bwd(ctx, head, x, gt_mask=gm, w=w, grad_scale=1.0 / B, **out)

    logits = torch.empty((B, spec.C), dtype=torch.bfloat16, device=dev)

    def unfused():
        hg.zero_()
        sc.sc_decision_hist_weights(ctx, sc.Batch(gt_off=gt_off, gt_lab=gt_lab, rows=B), hg, w, gt_mask_out=gm)
        torch.addmm(b.to(torch.bfloat16), x, W.t(), out=logits)
        sc.sc_loss_fwd_bwd(ctx, sc.Batch(logits=logits, gt_mask=gm), w=w, grad_scale=1.0 / B, **out)

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(steps):
            fn()
        e.record(stream)
        torch.cuda.synchronize(dev)
        return s.elapsed_time(e) / steps

    # the head kernel's own time inside the timed steps: CUDA events around each launch on the
    # stream it is launched on
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kidx = {"i": 0}

    def fused_timed():
        hg.zero_()
        sc.sc_decision_hist_weights(ctx, sc.Batch(gt_off=gt_off, gt_lab=gt_lab, rows=B), hg, w, gt_mask_out=gm)
        i = kidx["i"]
        if i < len(kev):
            kev[i][0].record(stream)
        sc.sc_head_loss_fwd_bwd(ctx, head, x, gt_mask=gm, w=w, grad_scale=1.0 / B, **out)
        if i < len(kev):
            kev[i][1].record(stream)
        kidx["i"] = i + 1

    for _ in range(args.warmup):
        fused()
    torch.cuda.synchronize(dev)
    launches0 = sc.sc_launch_count()
    with ClockSampler(dev.index or 0) as clk:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            fused_timed()
        s1.record(stream)
        torch.cuda.synchronize(dev)
    ms = s0.elapsed_time(s1) / args.steps
    launches = sc.sc_launch_count() - launches0
    k_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    kname = sc.sc_last_kernel()
    un_ms = timed(unfused, max(3, args.steps // 4))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    tc = peaks.get("bf16_tflops", 1662.7)
    per_row = d * 2 + 1 + 1 + 8 * S  # features + G_i + decision + sparse gradient
    achieved = B * per_row / (k_ms / 1e3) / 1e9
    n_mapped = int(spec.mapped()[0].sum())
    tflops = B * 2.0 * d * n_mapped / (k_ms / 1e3) / 1e12
    # the bound: whichever floor is higher — x bytes at the HBM peak, or the mapped columns'
    # flops at the bf16 tensor peak (a wide context, e.g. cfg3's 1000 mapped labels)
    t_hbm = B * per_row / (hbm * 1e9)
    t_tc = B * 2.0 * d * n_mapped / (tc * 1e12)
    if t_tc > t_hbm:
        roof = {"bound": "tensor", "achieved": tflops, "peak": tc, "unit": "TFLOP/s", "frac": tflops / tc,
                "hbm": {"achieved_gbs": achieved, "peak_gbs": hbm, "frac": achieved / hbm}}
    else:
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "tensor": {"achieved_tflops": tflops, "peak_tflops": tc, "frac": tflops / tc}}
    roof.update({"kernel": kname, "kernel_ms": k_ms, "algorithmic_bytes_per_row": per_row,
                 "flops_per_row": 2 * d * n_mapped, "traffic": None,
                 "peak_source": "MEASURED_PEAKS.json (hbm_gbs copy, bf16_tflops cuBLAS burst)" if peaks else "fallback"})
    line = {
        "metric": "samples/s for the classifier head fused with decide+loss fwd/bwd (NEXT f4)",
        "value": B / (ms / 1e3), "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "dtype": "bf16 operands, f32 accumulate", "data": "synthetic",
        "config": {"workload": f"{WORKLOADS[args.config]}, bf16 features d={d}, head over the {n_mapped} mapped "
                               f"labels ({n_cols} columns)", "rows": B, "d": d, "order": args.order},
        "roofline": roof,
        "unfused": {"ms_per_step": un_ms, "what": f"cuBLAS addmm -> bf16 logits [B, {spec.C}] + sc_loss_fwd_bwd",
                    "speedup_fused": un_ms / ms},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_e2e(args, ev, data, global_rows, dev, barrier, world):
    import torch
    B = data["logits"].shape[0]
    h_logits = torch.empty(data["logits"].shape, dtype=data["logits"].dtype, pin_memory=True)
    h_logits.copy_(data["logits"])
    h_off = torch.empty(data["gt_off"].shape, dtype=torch.int64, pin_memory=True).copy_(data["gt_off"])
    h_lab = torch.empty(data["gt_lab"].shape, dtype=torch.int32, pin_memory=True).copy_(data["gt_lab"])
    host_out = ev.host_outputs(B)
    h_app = None
    if data.get("app") is not None:
        h_app = torch.empty(data["app"].shape, dtype=torch.int16, pin_memory=True).copy_(data["app"])
    ev.step_host(h_logits, h_off, h_lab, host_out, h_app=h_app, global_rows=global_rows)  # warm-up
    torch.cuda.synchronize(dev)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        ev.step_host(h_logits, h_off, h_lab, host_out, h_app=h_app, global_rows=global_rows)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    if dist_on(world):
        import torch.distributed as dist
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t[0])
    h2d = h_logits.numel() * h_logits.element_size() + h_off.numel() * 8 + h_lab.numel() * 4 + \
        (h_app.numel() * 2 if h_app is not None else 0)
    d2h = sum(t.numel() * t.element_size() for t in host_out.values())
    del h_logits
    return {"value": global_rows * args.e2e_steps / dt, "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
            "h2d_gbs_per_gpu": round(h2d * args.e2e_steps / dt / 1e9, 2),  # PCIe-bound: the step moves 4.2 GB host->device
            "bound": "pcie (host->device transfer of the step's logits)",
            "host_mode": {0: "auto", 1: "copy", 2: "zero_copy"}.get(getattr(ev, "host_mode_used", None)),
            "api": "Evaluator.step_host: GT host->device, sc_decision_hist + sc_weights_from_hist, then "
                   "sc_loss_fwd_bwd_host (C ABI, pinned host logits: chunked double-buffered H2D inside libsc, "
                   "or zero copy for sparse contexts), results device->host"}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args):
    """--gpus N: the run must have exactly N ranks.  Under torchrun WORLD_SIZE must equal N;
    without it, N > 1 re-executes this command under torch.distributed.run (one process per
    GPU, 127.0.0.1 rendezvous) and returns its exit code.  None = carry on in this process."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if args.gpus is not None and args.gpus != world:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), file=sys.stderr, flush=True)
            return 2
        args.gpus = world
        return None
    if args.gpus is None:
        args.gpus = 1
    if args.gpus <= 1 or args.impl == "reference":
        return None  # the reference arm runs on rank 0 only: no ranks to launch
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    rc = launch_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

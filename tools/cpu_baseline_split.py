"""The oracle timed on this host's cores per BASELINE config (SURVEY.md §8(d) oracle timing):
(a) one thread over config 1 in full and a row prefix of configs 2-5; (b) the same plain code
fanned out over all cores.  Rows are generated on the host chunk by chunk (not timed); each
timed pass = GT pre-pass + weights + full oracle pass, like one bench step.

usage: python tools/cpu_baseline_split.py OUT.json [PREFIX_ROWS] [CFG3_PREFIX_ROWS]
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import Oracle  # noqa: E402

CHUNK = 512


def batches(cfg, rows):
    spec = synth.config_context(cfg)
    wl = synth.Workload(spec, seed=cfg, layout=0, rows_per_app=1 << 18)
    ch = max(32, CHUNK * 1000 // max(spec.C, 1000))  # ~2 MB of logits per task (cfg3: 25 rows of 80 KB)
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        bs = list(ex.map(lambda lo: wl.host_batch(lo, min(ch, rows - lo)), range(0, rows, ch)))
    return spec, bs


def timed_pass(spec, bs, threads):
    orc = Oracle.from_spec(spec)
    multi = spec.n_apps > 1
    rows = sum(len(b["gt_off"]) - 1 for b in bs)

    def hist(b):
        return orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=b["app"] if multi else None,
                        want_loss=False)["hist_gt"]

    def full(args):
        b, w = args
        return orc.eval(b["logits"], b["gt_off"], b["gt_lab"], app=b["app"] if multi else None, w=w,
                        grad_scale=1.0 / rows)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        H = sum(ex.map(hist, bs))
        w = Oracle.weights_by_mask(H)
        list(ex.map(full, [(b, w) for b in bs]))
    return rows, time.perf_counter() - t0


def main():
    out = sys.argv[1]
    prefix = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
    prefix3 = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 12
    cores = os.cpu_count() or 1
    model = "unknown"
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            model = line.split(":", 1)[1].strip()
            break
    res = {"cpu_model": model, "cores": cores, "kind": "oracle (oracle/sc_oracle.c as it stands)",
           "unit": "samples/s", "configs": {}}
    for cfg in (1, 2, 3, 4, 5):
        rows = 4096 if cfg == 1 else (prefix3 if cfg == 3 else prefix)
        spec, bs = batches(cfg, rows)
        timed_pass(spec, bs, cores)  # warm-up: first touch of the generated rows
        r1, t1 = timed_pass(spec, bs, 1)
        rn, tn = timed_pass(spec, bs, cores)
        res["configs"][f"cfg{cfg}"] = {
            "rows": rows, "sample": "config 1 in full" if cfg == 1 else f"first {rows} rows of the config",
            "single_thread": {"value": r1 / t1, "seconds": t1},
            "all_cores": {"value": rn / tn, "seconds": tn, "threads": cores}}
        print(cfg, res["configs"][f"cfg{cfg}"], flush=True)
        del bs
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()

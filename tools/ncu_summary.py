"""Summarise an ncu report (raw page) and a launch list into profiles/ (run here, no GPU).

usage: python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT.json OUT.txt ROWS [KERNEL_SUBSTRING]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_bytes.sum", "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


def to_bytes(s):
    parts = s.split()
    v, u = parts[0], parts[1] if len(parts) > 1 else "byte"
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
    return float(v.replace(",", "")) * mult


def launches(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    agg = defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            agg[r["Kernel Name"][:100]].append(float(r["Metric Value"]) / 1e3)
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v)} for k, v in agg.items()}


if __name__ == "__main__":
    rep, launch_csv, out_json, out_txt, rows = sys.argv[1:6]
    rows = int(rows)
    want = sys.argv[6] if len(sys.argv) > 6 else ""
    r = [k for k in raw(rep) if want in k["kernel"]][0]
    traffic = to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"])
    summ = {"report": rep, "metrics": r, "dram_bytes_per_launch": traffic, "dram_bytes_per_row": traffic / rows,
            "launch_list": launches(launch_csv)}
    json.dump(summ, open(out_json, "w"), indent=1)
    with open(out_txt, "w") as f:
        f.write(f"# ncu --set full summary of {r['kernel']}\n")
        for k, v in r.items():
            f.write(f"{k:70s} {v}\n")
        f.write(f"\ntraffic (read+write) per launch: {traffic/1e9:.4f} GB = {traffic/rows:.1f} B/row over {rows} rows\n")
        f.write("\n# launch list (ncu gpu__time_duration, cold/serialised)\n")
        for k, v in summ["launch_list"].items():
            f.write(f"{v['launches']:4d} x {v['mean_us']:10.2f} us  {k}\n")
    print(open(out_txt).read())

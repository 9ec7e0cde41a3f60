#!/usr/bin/env python3
"""Turn the raw ncu outputs of a GPU run into the committed profiles/ summaries.

  python tools/summarize_ncu.py --rep gpurun_out/prof_final.ncu-rep \
      --launches gpurun_out/launches.csv --tag r1 --windows 8760000000

Writes profiles/<tag>_sweep_fast_metrics.csv (key counters of the dominant
kernel), profiles/<tag>_sweep_fast_details.txt (ncu --page details),
profiles/<tag>_launches.csv (per-launch durations of one bench step, with each
kernel's share), and updates profiles/ncu_traffic.json (DRAM bytes per planned
window: bench.py's roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "Gbyte"),
    ("dram__bytes_write.sum", "Gbyte"),
    ("smsp__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", ""),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", ""),
    ("launch__registers_per_thread", "register/thread"),
    ("launch__grid_size", ""),
    ("launch__block_size", ""),
    ("launch__shared_mem_per_block_dynamic", "Kbyte/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--windows", type=float, default=8.76e9)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--kernel", default="sweep_fast", help="file-name stem of the captured kernel")
    ap.add_argument("--no-traffic", action="store_true", help="do not update ncu_traffic.json (ALU-bound kernels)")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")

    m = raw_metrics(a.rep)
    with open(os.path.join(prof, f"{a.tag}_{a.kernel}_metrics.csv"), "w") as f:
        f.write("metric,unit,value\n")
        for k, _ in KEYS:
            if k in m:
                f.write(f"{k},{m[k][0]},{m[k][1]}\n")
        stalls = sorted(((k, float(v[1] or 0)) for k, v in m.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")),
                        key=lambda kv: -kv[1])[:8]
        for k, v in stalls:
            f.write(f"{k},ratio,{v:.4f}\n")
    with open(os.path.join(prof, f"{a.tag}_{a.kernel}_details.txt"), "w") as f:
        f.write(ncu("-i", a.rep, "--page", "details"))

    def gb(k):
        u, v = m[k]
        return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1.0}.get(u, 1.0)

    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    path = os.path.join(prof, "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    entry = {"dram_bytes_per_window": (rd + wr) / a.windows, "dram_read_bytes": rd, "dram_write_bytes": wr,
                   "windows": a.windows,
                   "source": f"ncu --set full --clock-control none, sweep_fast_kernel "
                             f"(profiles/{a.tag}_{a.kernel}_metrics.csv)"}
    if not a.no_traffic:
        d[a.config] = entry
        json.dump(d, open(path, "w"), indent=1)

    # launch list: keep the CSV rows, add per-kernel totals of the last bench step
    text = open(a.launches).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = os.path.join(prof, f"{a.tag}_launches.csv")
    tot = defaultdict(float)
    with open(out, "w") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "duration_us"])
        for r in rows[1:]:
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
            us = float(r[vi]) * scale
            name = r[ki].split("(")[0]
            w.writerow([r[0], name, f"{us:.3f}"])
            tot[name] += us
        w.writerow([])
        # shares among the planner's own kernels (input generation and torch copies are setup)
        w.writerow(["kernel", "total_us_all_launches", "share_of_planner_kernels"])
        s = sum(v for k, v in tot.items() if "chase::" in k and "chasegen" not in k)
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            share = f"{v / s:.4f}" if "chase::" in k and "chasegen" not in k else "setup"
            w.writerow([k, f"{v:.1f}", share])
    print(json.dumps(entry))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Summarise an ncu report (or launch-list CSV) into a short text file for
profiles/. Usage:
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
            "Scheduler Statistics", "Warp State Statistics", "Occupancy", "Launch Statistics")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__pipe_tensor_cycles_active",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
       "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
       "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
       "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_no_instructions",
       "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected")


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def report(path):
    rows = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "details", "--csv"))))
    h = rows[0]
    kernel = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Kernel Name") != kernel:
            kernel = d.get("Kernel Name")
            print(f"== {kernel}  grid={d.get('Grid Size')} block={d.get('Block Size')}")
        if d.get("Section Name") in SECTIONS and d.get("Metric Name"):
            print(f"  {d['Section Name'][:28]:28s} {d['Metric Name'][:52]:52s} "
                  f"{d.get('Metric Unit', ''):>12s} {d.get('Metric Value', '')}")
    raw = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "raw", "--csv"))))
    if len(raw) >= 3:
        print("  -- raw")
        hdr, unit = raw[0], raw[1]
        for row in raw[2:]:
            for i, n in enumerate(hdr):
                if n in RAW or any(n.endswith("." + r) for r in RAW):
                    print(f"  {n:60s} {unit[i]:>10s} {row[i]}")


def launches(path):
    per = defaultdict(list)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for d in csv.DictReader(io.StringIO("".join(lines))):
        if d.get("Metric Name") == "gpu__time_duration.sum":
            per[d["Kernel Name"]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in per.values())
    print(f"{'kernel':90s} {'n':>4s} {'avg_us':>10s} {'share':>7s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:90]:90s} {len(v):4d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / tot:7.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])

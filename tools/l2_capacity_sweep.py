#!/usr/bin/env python
"""Effective L2 capacity for random 64-B row gathers on this B200: K5 gather
probe (uniform random rows, 60M gathers) over tables of 8..256 MB.
usage: tools/l2_capacity_sweep.py [--sizes 8,16,...] [--once MB]   (--once: one size, for ncu)"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06800_b200 import probes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="8,16,24,32,40,48,56,64,80,96,112,128,160,256")
ap.add_argument("--once", type=int, default=0)
ap.add_argument("--n", type=int, default=60_000_000)
a = ap.parse_args()
for mb in ([a.once] if a.once else [int(s) for s in a.sizes.split(",")]):
    rows = mb * (1 << 20) // 64
    g = probes.gather_gbps(rows, 16, a.n, reps=1 if a.once else 5)
    print(json.dumps({"table_MB": mb, "rows": rows, "gathers": a.n, "gbps_rows_only": round(g, 1)}),
          flush=True)

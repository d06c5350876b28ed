#!/usr/bin/env python
"""Device event trace of K1: the reference's multi-GPU
trace CSV (R:proj/tools/cli.cpp:144-155, stages LR/LL/AC of
R:proj/src/sim.cpp:102-125) recorded by the real pipelined kernel, plus a
summary of how much of each remote get (LR) overlaps its warp's local work
(LL) — the paper's Fig. 6b interleave, measured.

    python tools/trace_b200.py --workload config1 --warps 64 --out profiles/r01_trace_config1.csv
"""
import argparse
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2209_06800_b200 as mgg  # noqa: E402


def summarize(csv: str) -> dict:
    spans = defaultdict(list)  # (gpu, warp, stage) -> [(b, e)]
    open_ = {}
    for ln in csv.strip().split("\n")[2:]:
        gpu, cyc, _sm, warp, stage, ev = ln.split(",")
        key = (gpu, warp, stage)
        if ev == "begin":
            open_.setdefault(key, []).append(int(cyc))
        elif open_.get(key):
            spans[key].append((open_[key].pop(0), int(cyc)))
    out = {}
    for stage in ("LR", "LL", "AC"):
        d = [e - b for (g, w, s), v in spans.items() if s == stage for b, e in v]
        out[stage] = {"spans": len(d), "mean_cycles": round(sum(d) / len(d), 1) if d else 0}
    # fraction of LR cycles covered by the same warp's LL spans
    cov = tot = 0
    for (g, w, s), lr in spans.items():
        if s != "LR":
            continue
        ll = spans.get((g, w, "LL"), [])
        for b, e in lr:
            tot += e - b
            cov += sum(max(0, min(e, e2) - max(b, b2)) for b2, e2 in ll)
    out["lr_cycles_under_ll"] = round(cov / tot, 4) if tot else None
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config1", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--parts", type=int, default=2)
    ap.add_argument("--warps", type=int, default=64, help="logical warps traced per part")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    label, g, model, _ = bench.build(mgg, args.workload)
    ps, dist, wpb = bench.WORKLOADS[args.workload][3][:3]
    dim = bench.agg_widths(model)[0]
    eng = mgg.Engine(g, args.parts, [0] * args.parts, model, ps, dist, wpb)
    eng.set_remote_fetch("fine")
    csv = eng.trace_csv(dim, capacity=1 << 22, warp_limit=args.warps)
    eng.close()
    if args.out:
        with open(args.out, "w") as f:
            f.write(csv)
    print(json.dumps({"workload": args.workload, "parts": args.parts, "dim": dim,
                      "config": [ps, dist, wpb], "traced_warps_per_part": args.warps,
                      "events": csv.count("\n") - 2, "summary": summarize(csv)}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-GPU K1 time of an N-GPU run, measured with N logical parts on one B200
(each part timed alone: its own local + remote partitions, remote rows from
same-device "peers" — no NVLink cost), for both remote-fetch modes.

    python tools/project_multi_gpu.py --workload reddit-gcn --parts 2,4,8
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2209_06800_b200 as mgg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="reddit-gcn", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--parts", default="1,2,4,8")
    args = ap.parse_args()
    label, g, model, _ = bench.build(mgg, args.workload)
    ps, dist, wpb = bench.WORKLOADS[args.workload][3][:3]
    dim = bench.agg_widths(model)[0]
    for n in (int(p) for p in args.parts.split(",")):
        eng = mgg.Engine(g, n, [0] * n, model, ps, dist, wpb)
        row = {"workload": args.workload, "parts": n, "dim": dim}
        for fetch in (("fine",) if n == 1 else ("fine", "halo")):
            eng.set_remote_fetch(fetch)
            row[f"k1_per_part_ms_{fetch}"] = round(eng.time_aggregate(dim, 5) / 1e6, 4)
        st = eng.stats()
        row["halo_rows_per_part"] = st["halo_rows"] // max(n, 1)
        row["remote_edge_fraction"] = round(
            st["remote_edges"] / max(1, st["remote_edges"] + st["local_edges"]), 4)
        eng.close()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()

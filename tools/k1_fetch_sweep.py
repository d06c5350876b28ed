#!/usr/bin/env python
"""K1 L2 fetch size x rows in flight on the HBM-resident narrow-row shapes
(Orkut's agg_group_hint read ~1.16x its algorithmic
bytes from DRAM). One process per variant (the knobs are read once):
MGG_AGG_L2FETCH = 0 (line fetch) | 64 (L2::64B), MGG_AGG_HINT_UNR = 8 | 16.

  tools/k1_fetch_sweep.py                 time every variant (CUDA events)
  tools/k1_fetch_sweep.py --child W --once   one K1 launch (for ncu)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = [("0", "8"), ("64", "8"), ("0", "16"), ("64", "16")]


def child(workload, once, reps):
    import bench
    import paper_2209_06800_b200 as mgg
    _, g, model, _ = bench.build(mgg, workload)
    ps, dist, wpb = bench.WORKLOADS[workload][3][:3]
    eng = mgg.Engine(g, 1, [0], model, ps=ps, dist=dist, wpb=wpb)
    w = bench.agg_widths(model)[0]
    if once:
        x = mgg.random_features(g.num_nodes, w, seed=1)
        eng.aggregate(x, 1.0)
        print(json.dumps({"workload": workload, "kernels": eng.k1_kernels(0)}))
        return
    ns = eng.time_aggregate(w, reps, 0)
    st = eng.stats()
    algo = bench.agg_bytes(st["local_edges"], st["local_parts"], g.num_nodes, w)
    print(json.dumps({"workload": workload, "l2fetch": os.environ.get("MGG_AGG_L2FETCH"),
                      "unr": os.environ.get("MGG_AGG_HINT_UNR"), "kernels": eng.k1_kernels(0),
                      "k1_ms": ns / 1e6, "algorithmic_bytes": algo,
                      "algo_tbs": round(algo / ns / 1e3, 3)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--child", default=None)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--workloads", default="products-gcn,orkut-gcn")
    args = ap.parse_args()
    if args.child:
        child(args.child, args.once, args.reps)
        return
    for wl in args.workloads.split(","):
        for fetch, unr in VARIANTS:
            env = {**os.environ, "MGG_AGG_L2FETCH": fetch, "MGG_AGG_HINT_UNR": unr}
            r = subprocess.run([sys.executable, __file__, "--child", wl, "--reps",
                                str(args.reps)], env=env, capture_output=True, text=True)
            sys.stdout.write(r.stdout)
            sys.stderr.write(r.stderr[-2000:])
            sys.stdout.flush()


if __name__ == "__main__":
    main()

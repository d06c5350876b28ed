#!/usr/bin/env python
"""Runs the paper's heuristic tuner (mgg::optimize, identical to the
reference's, R:proj/src/tuner.cpp:129) with the MEASURED K1 latency as its
SimulateFn on the bench workload, and (optionally) the exhaustive sweep it is
judged against (acceptance criterion 7's shape). Writes JSON to stdout.

    python tools/tune_b200.py [--parts N] [--exhaustive] [--graph reddit|products]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2209_06800_b200 as mgg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=1)
    ap.add_argument("--exhaustive", action="store_true")
    ap.add_argument("--graph", default="reddit")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    if args.graph == "reddit":
        g = mgg.gen_synthetic(mgg.POWERLAW, 232_965, 492, 0)
        model, dim = mgg.make_gcn(602, 16, 41), 16
    else:  # products-shaped GIN (configs[2]): aggregation width 64
        g = mgg.gen_synthetic(mgg.POWERLAW, 2_449_029, 25.26, 0)
        model, dim = mgg.make_gin(100, 64, 47, layers=5), 64
    eng = mgg.Engine(g, args.parts, [0] * args.parts, model, ps=1, dist=1, wpb=1)
    hw = mgg.resolve_profile("b200")
    calls = []

    def measure(c):
        t0 = time.perf_counter()
        eng.set_config(*c)
        ns = eng.time_aggregate(dim, reps=args.reps)
        calls.append({"cfg": list(c), "ns": ns, "wall_s": round(time.perf_counter() - t0, 3)})
        return ns

    t0 = time.perf_counter()
    trace, best = mgg.optimize(measure, hw, dim)
    out = {"graph": args.graph, "nodes": g.num_nodes, "edges": g.num_edges, "parts": args.parts,
           "dim": dim, "tuner": {"trace": trace, "best": best, "evaluations": len(trace),
                                 "seconds": round(time.perf_counter() - t0, 2)}}
    if args.exhaustive:
        calls.clear()
        t0 = time.perf_counter()
        table = mgg.exhaustive(measure, hw, dim)
        out["exhaustive"] = {"best": table[0], "top5": table[:5], "points": len(table),
                             "seconds": round(time.perf_counter() - t0, 2),
                             "tuner_rank": 1 + [t[3] for t in table].index(
                                 min(t[3] for t in table if t[3] >= best[3]))
                             if any(t[3] >= best[3] for t in table) else 1,
                             "table": table}
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()

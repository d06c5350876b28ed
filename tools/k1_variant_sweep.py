#!/usr/bin/env python
"""K1 time per local-kernel variant (MGG_AGG_LEAN) and config, 1 part.
The variant numbers 20-29 of profiles/r01_k1_variants/*.jsonl refer to the
experiment build at commit d90d2b5 (aggregate.cu pick()); since ad84700 only
1 (auto), 2 (warp-window), 3, 10 and 20 (group) remain."""
import json, os, sys
sys.path.insert(0, '.')
import bench
import paper_2209_06800_b200 as mgg
mode = os.environ.get("MGG_AGG_LEAN", "1")
for w in sys.argv[1:]:
    label, g, model, _ = bench.build(mgg, w)
    dim = bench.agg_widths(model)[0]
    tuned = tuple(bench.WORKLOADS[w][3][:3])
    for cfg in (tuned, (16, 16, 2), (16, 8, 8), (16, 16, 8), (8, 16, 8)):
        eng = mgg.Engine(g, 1, [0], model, *cfg)
        t = eng.time_aggregate(dim, 7) / 1e6
        eng.close()
        print(json.dumps({"mode": mode, "workload": w, "cfg": cfg, "k1_ms": round(t, 4)}), flush=True)

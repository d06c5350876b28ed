#!/usr/bin/env python
"""Fine-fetch (paired) K1 time per pair-kernel variant (MGG_AGG_PAIR) at 2 and 8
logical parts. Variants 2-6 of profiles/r01_k1_variants/pair_variants.jsonl are
from the experiment build at commit d90d2b5; now 0 = warp-window, 1 = agg_gpair."""
import json, os, sys
sys.path.insert(0, '.')
import bench
import paper_2209_06800_b200 as mgg
mode = os.environ.get("MGG_AGG_PAIR", "1")
for w in sys.argv[1:]:
    label, g, model, _ = bench.build(mgg, w)
    dim = bench.agg_widths(model)[0]
    for cfg in (tuple(bench.WORKLOADS[w][3][:3]), (32, 16, 2)):
        for n in (2, 8):
            eng = mgg.Engine(g, n, [0] * n, model, *cfg)
            eng.set_remote_fetch("fine")
            t = eng.time_aggregate(dim, 5) / 1e6
            eng.close()
            print(json.dumps({"mode": mode, "workload": w, "cfg": cfg, "parts": n, "k1_ms": round(t, 4)}), flush=True)

#!/usr/bin/env python
"""agg_group rows-in-flight per group (MGG_AGG_GROUP_UNR=4|8) per workload/config:
profiles/r01_k1_variants/group_unr4_vs_8.jsonl."""
import json, os, sys
sys.path.insert(0, '.')
import bench, paper_2209_06800_b200 as mgg
u = os.environ.get("MGG_AGG_GROUP_UNR", "0") + "/h" + os.environ.get("MGG_AGG_L2HINT", "0")
for w in ("products-gcn", "orkut-gcn", "orkut-rmat-gcn", "products-gin", "products-rmat-gin"):
    label, g, model, _ = bench.build(mgg, w)
    dim = bench.agg_widths(model)[0]
    for cfg in (tuple(bench.WORKLOADS[w][3][:3]), (16, 16, 2), (16, 16, 4)):
        eng = mgg.Engine(g, 1, [0], model, *cfg)
        t = eng.time_aggregate(dim, 7) / 1e6
        eng.close()
        print(json.dumps({"unr": u, "workload": w, "cfg": cfg, "k1_ms": round(t, 4)}), flush=True)

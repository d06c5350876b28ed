#!/usr/bin/env python
"""K1 time vs gather-table size at ~61M edges, width 16 (node count swept):
profiles/r01_k1_table_size.jsonl."""
import json, sys
sys.path.insert(0, '.')
import paper_2209_06800_b200 as mgg
E = 62_000_000
for n in (233_000, 600_000, 1_000_000, 1_500_000, 2_449_029):
    g = mgg.gen_synthetic(mgg.POWERLAW, n, E / n, 0)
    m = mgg.make_gcn(16, 16, 16, seed=2)
    for cfg in ((32, 16, 2),):
        eng = mgg.Engine(g, 1, [0], m, *cfg)
        t = eng.time_aggregate(16, 5) / 1e6
        print(json.dumps({"nodes": n, "edges": g.num_edges if hasattr(g,'num_edges') else None, "table_MB": round(n*64/1e6,1), "k1_ms": round(t,4), "ns_per_edge": round(t*1e6/E,3)}), flush=True)
        eng.close()

#!/usr/bin/env python
"""Column-blocked K1 probe (not adopted): split the columns into B ranges, one K1
pass per range over the same output; sums the per-pass times.
profiles/r01_k1_column_blocking.jsonl."""
import json, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2209_06800_b200 as mgg
m = mgg.make_gcn(16, 16, 16, seed=2)
for name, n, avg in (("products", 2_449_029, 25.259), ("orkut", 3_072_441, 38.141)):
    g = mgg.gen_synthetic(mgg.POWERLAW, n, avg, 0)
    rp = g.row_ptr.astype(np.int64); ci = g.col_idx.astype(np.int64)
    row = np.repeat(np.arange(n), np.diff(rp))
    for B in (1, 2, 3, 4, 6):
        for cfg in ((32, 16, 2), (16, 16, 2), (32, 8, 2)):
            tot = 0.0
            for b in range(B):
                lo, hi = n * b // B, n * (b + 1) // B
                sel = (ci >= lo) & (ci < hi)
                r = row[sel]; c = ci[sel]
                cnt = np.bincount(r, minlength=n)
                srp = np.zeros(n + 1, np.int64); np.cumsum(cnt, out=srp[1:])
                sg = mgg.CsrGraph.from_csr(srp, c)
                eng = mgg.Engine(sg, 1, [0], m, *cfg)
                tot += eng.time_aggregate(16, 5) / 1e6
                eng.close()
            print(json.dumps({"graph": name, "blocks": B, "cfg": cfg, "k1_ms_sum": round(tot, 4)}), flush=True)

"""Small fine-fetch aggregations for compute-sanitizer over the smem-staged
pair kernels (MGG_AGG_PAIR=2 agg_pipe / 3 agg_pipe_bulk):
`MGG_AGG_PAIR=3 compute-sanitizer --tool {memcheck,racecheck,synccheck} python
tools/sanitize_pipe.py` — widths 3-64, 2-3 parts, device and host-mapped
peers, checked against the oracle. MGG_SAN_FETCH=halo: the halo path (the
host-mapped case takes the pull fused into the local pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2209_06800_b200 as mgg  # noqa: E402

g = mgg.gen_rmat(1500, 15000, seed=4)
worst = 0.0
for dim in (3, 16, 64):
    x = mgg.random_features(g.num_nodes, dim, seed=dim)
    ref = oracle.aggregate(g.row_ptr, g.col_idx, x)
    for parts, cfg, host in ((2, (16, 4, 4), False), (3, (8, 2, 2), True), (2, (32, 16, 8), False)):
        eng = mgg.Engine(g, parts, [0] * parts, mgg.make_gcn(dim, 8, 4), *cfg)
        eng.set_remote_fetch(os.environ.get("MGG_SAN_FETCH", "fine"))
        if host:
            eng.set_shard_memory(parts - 1, mgg.MEM_HOST_MAPPED)
        out = eng.aggregate(x, 1.0)
        err = float((np.abs(out - ref) / np.maximum(np.abs(ref).max(1, keepdims=True), 1e-6)).max())
        worst = max(worst, err)
        eng.close()
print("kernels", os.environ.get("MGG_AGG_PAIR"), "max row-relative error", worst)
assert worst <= 1e-4

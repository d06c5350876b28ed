"""Small forwards (GCN/GIN, 1-2 parts, fine/halo, chained GEMMs, streamed I/O) for
compute-sanitizer: `compute-sanitizer --tool {memcheck,racecheck,synccheck} python
tools/sanitize_forward.py`. Round 1: 0 errors / 0 hazards on all three tools."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2209_06800_b200 as mgg  # noqa: E402

g = mgg.gen_rmat(2000, 20000, seed=3)
for model, parts, fetch in [(mgg.make_gcn(100, 16, 41, seed=1), 1, "auto"),
                            (mgg.make_gcn(20, 16, 8, seed=2), 2, "fine"),
                            (mgg.make_gin(64, 64, 47, layers=3, seed=3), 1, "auto"),
                            (mgg.make_gin(40, 32, 11, layers=3, seed=4), 2, "halo")]:
    x = mgg.random_features(g.num_nodes, model.in_dim, seed=5)
    eng = mgg.Engine(g, parts, [0] * parts, model, ps=16, dist=2, wpb=4)
    eng.set_remote_fetch(fetch)
    eng.set_graphs(False)
    z = np.zeros((g.num_nodes, model.out_dim), np.float32)
    eng.forward_host(x, z)
    eng.close()
# K1 variants: group / group-per-pair at several widths, phases, whole-list,
# and the traced pair kernel
for dim in (3, 16, 64, 200):
    x = mgg.random_features(g.num_nodes, dim, seed=dim)
    for ps, parts, fetch in ((32, 1, "auto"), (8, 1, "auto"), (16, 3, "fine"), (16, 3, "halo")):
        eng = mgg.Engine(g, parts, [0] * parts, mgg.make_gcn(dim, 8, 4), ps=ps, dist=4, wpb=2)
        eng.set_remote_fetch(fetch)
        for phase in (0, 1, 2):
            eng.aggregate(x, 1.0, relu_in=True, phase=phase)
        if parts > 1 and fetch == "fine" and dim <= 128:
            eng.trace_csv(dim, capacity=1 << 12)
        eng.set_mapping(0, 1)
        eng.aggregate(x, 1.0)
        eng.close()
print("sanitize run ok")

#!/usr/bin/env python
"""for each BASELINE graph shape, the id-random variant (the
reference's powerlaw generator) and a locality-bearing one (RMAT, ids not
shuffled), the remote-edge fraction of the Alg. 1 split
(R:proj/src/placement.cpp:44-71) at 2/4/8 partitions, and the distinct
remote rows the halo mode pulls. Host-only (no GPU).

    python tools/remote_fraction.py > profiles/r01_remote_fraction.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2209_06800_b200 as mgg  # noqa: E402

SHAPES = [("config1", 100_000, 1_600_000), ("reddit", 232_965, 114_615_892),
          ("products", 2_449_029, 61_859_140), ("orkut", 3_072_441, 117_185_083),
          ("proteins", 132_534, 79_000_000)]


def main():
    for name, n, e in SHAPES:
        for kind in ("powerlaw", "rmat"):
            t0 = time.perf_counter()
            g = (mgg.gen_rmat(n, e, 0) if kind == "rmat"
                 else mgg.gen_synthetic(mgg.POWERLAW, n, e / n, 0))
            gen_s = time.perf_counter() - t0
            row = {"graph": name, "kind": kind, "nodes": g.num_nodes, "edges": g.num_edges,
                   "gen_s": round(gen_s, 2), "parts": {}}
            for parts in (2, 4, 8):
                loc = rem = halo = 0
                for p in range(parts):
                    fp = mgg.build_flat_plan(g, parts, p, 32, 16, 2, 16)
                    loc += fp.local_cols_len
                    rem += fp.remote_cols_len
                    halo += len(np.unique(fp.cols(1)))
                row["parts"][parts] = {"remote_edge_fraction": round(rem / max(1, loc + rem), 4),
                                       "remote_edges": rem, "distinct_remote_rows": halo,
                                       "halo_dedup_ratio": round(rem / max(1, halo), 2)}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()

"""Regenerates tests/golden/*.json from the UNMODIFIED reference library
(oracle/_ref/libpipeshard_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run in the CPU container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the oracle restatement (oracle/oracle.c) and the product's
builder even where oracle/_ref cannot be built (e.g. the GPU box).
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def random_graph(rng, max_nodes=200, max_avg=8.0):
    n = 1 + int(rng.integers(0, max_nodes))
    m = int(rng.integers(0, max(1, int(n * max_avg)) + 1))
    return n, rng.integers(0, n, size=(m, 2), dtype=np.uint64)


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    rng = np.random.default_rng(424242)
    splits = []
    for _ in range(200):
        n, e = random_graph(rng)
        gpus = 1 + int(rng.integers(0, 8))
        r = oracle.RefGraph.from_edges(n, e)
        rp, cl = r.csr()
        splits.append({"row_ptr": rp.tolist(), "gpus": gpus, "split": r.split(gpus).tolist(),
                       "equal_nodes": r.placement(gpus, 0).tolist()})
    plans = []
    cfgs = [(1, 1, 1), (2, 1, 2), (16, 1, 2), (3, 5, 7), (32, 16, 16)]
    for i in range(25):
        n, e = random_graph(rng, 40, 5)
        gpus = 1 + int(rng.integers(0, 4))
        gpu = int(rng.integers(0, gpus))
        mode = int(rng.integers(0, 2))
        ps, dist, wpb = cfgs[i % len(cfgs)]
        mapping, gran = i % 2, (i // 2) % 2
        r = oracle.RefGraph.from_edges(n, e)
        rp, cl = r.csr()
        plans.append({"n": n, "row_ptr": rp.tolist(), "col_idx": cl.tolist(), "gpus": gpus,
                      "gpu": gpu, "mode": mode, "ps": ps, "dist": dist, "wpb": wpb,
                      "dim": 8, "mapping": mapping, "granularity": gran,
                      "plan_json": r.plan(gpus, mode, gpu, ps, dist, wpb, 8, mapping,
                                          gran).json()})

    def convex(c):
        ps, dist, wpb = c
        return 1000 + int(round(30.0 * (math.log2(ps) - 2) ** 2 + 20.0 * (math.log2(dist) - 1)
                                ** 2 + 10.0 * (math.log2(wpb) - 1) ** 2))
    tuner = {"convex": oracle.ref_optimize(convex, 108, 64, 164 * 1024, 16),
             "convex_capped": oracle.ref_optimize(convex, 108, 64, 1000, 16)}
    gens = []
    for kind, n, avg, seed in [(0, 50, 3.5, 1), (1, 60, 4, 2), (1, 7, 2.2, 3)]:
        rp, cl = oracle.RefGraph.gen(kind, n, avg, seed).csr()
        gens.append({"kind": kind, "n": n, "avg": avg, "seed": seed, "row_ptr": rp.tolist(),
                     "col_idx": cl.tolist()})
    out = {"generated_by": "tests/golden/make_golden.py from oracle/_ref (pipeshard)",
           "splits": splits, "plans": plans, "tuner": tuner, "generators": gens}
    with open(os.path.join(HERE, "reference_metadata.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "reference_metadata.json"))


if __name__ == "__main__":
    main()

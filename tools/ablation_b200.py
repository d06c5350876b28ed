#!/usr/bin/env python
"""K4 ablations on B200: the reference's `compare` table
(R:proj/tools/cli.cpp:254-289 — mode, time, ratioVsMgg) measured with the real
kernel instead of the DES. Logical partitions on one GPU exercise the remote
path through the peer-pointer table (same-device "peers").

  mgg            interleaved, ps-partitioned (the plan under test)
  no_interleave  segregated mapping (R:proj/src/workload.cpp:126-146)
  no_np          whole-list tasks (R:proj/src/workload.cpp:187-203)
  phase_separated all remote partitions (one launch), then all local ones —
                 communication before compute (R:proj/src/sim.cpp:530-569)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_06800_b200 as mgg  # noqa: E402


def run(g, parts, dim, cfg, reps=5, fetch="auto"):
    eng = mgg.Engine(g, parts, [0] * parts, mgg.make_gcn(dim, 8, 4), *cfg)
    eng.set_remote_fetch(fetch)
    out = {}
    eng.set_mapping(0, 0)
    out["mgg"] = eng.time_aggregate(dim, reps)
    out["phase_separated"] = eng.time_aggregate(dim, reps, 2) + eng.time_aggregate(dim, reps, 1)
    eng.set_mapping(1, 0)
    out["no_interleave"] = eng.time_aggregate(dim, reps)
    eng.set_mapping(0, 1)
    out["no_np"] = eng.time_aggregate(dim, reps)
    eng.close()
    return {k: {"ns": v, "ratioVsMgg": round(v / out["mgg"], 3)} for k, v in out.items()}


def main():
    res = []
    for name, g, dim in [
            ("powerlaw-10K-avg16 (acceptance crit. 6 graph)",
             mgg.gen_synthetic(mgg.POWERLAW, 10_000, 16, 0), 16),
            ("reddit-shaped", mgg.gen_synthetic(mgg.POWERLAW, 232_965, 492, 0), 16),
            ("products-shaped", mgg.gen_synthetic(mgg.POWERLAW, 2_449_029, 25.259, 0), 64)]:
        for parts in (2, 4):
            for cfg in [(16, 1, 2), (32, 16, 2)]:
                # fine: the paper's per-edge remote reads inside the pair loop;
                # halo: deduplicated pull overlapped with the local pass
                for fetch in ("fine", "halo"):
                    r = run(g, parts, dim, cfg, fetch=fetch)
                    res.append({"graph": name, "edges": g.num_edges, "parts": parts,
                                "dim": dim, "cfg": cfg, "fetch": fetch, "modes": r})
                    print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()

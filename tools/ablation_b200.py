#!/usr/bin/env python
"""K4 ablations on B200: the reference's `compare` table
(R:proj/tools/cli.cpp:254-289 — mode,cycles,occupancy,smUtilization,
remoteBytes,ratioVsMgg) measured with the real kernels instead of the DES,
through the measured MultiGpuReport (Engine.measure_multi_gpu: every part's
K1 concurrently, total = max over parts + barrier). Logical partitions on one
GPU exercise the remote path through the peer-pointer table.

  mgg             interleaved, ps-partitioned, fine-grained remote reads
  no_np           whole-list tasks (R:proj/src/workload.cpp:187-203)
  no_interleave   segregated mapping (R:proj/src/workload.cpp:126-146)
  phase_separated every part: all remote partitions (one launch), then all
                  local ones — communication before compute (sim.cpp:530-569)
  paged_remote    the remote rows are fetched by page faults
                  (R:proj/src/sim.cpp:503-518, 571-595): part 0 measured with
                  every other part's shards in managed memory homed on the
                  host (MGG_MEM_MANAGED_HOST), re-homed before each rep;
                  ratio against part 0's own mgg time. remoteBytes = the
                  reference's paged formula (rows x ceil(4D/page) x page).
  mgg_halo        (B200 addition) deduplicated remote pull overlapped with the
                  local pass

Output: one JSON object per (graph, parts, cfg) with a `csv` member in the
reference's schema (time in ns instead of cycles). usage:
  tools/ablation_b200.py [--out profiles/r02_ablation.jsonl] [--quick]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_06800_b200 as mgg  # noqa: E402

PAGE = 4096


def row(name, ns, occ, util, rbytes, base):
    return {"mode": name, "ns": int(ns), "occupancy": round(occ, 6),
            "smUtilization": round(util, 6), "remoteBytes": int(rbytes),
            "ratioVsMgg": round(ns / max(base, 1), 6)}


def run(g, parts, dim, cfg, reps=5):
    """Every mode's time = the per-GPU time of the measured MultiGpuReport
    (logical parts on one device: the max over parts of each part alone)."""
    eng = mgg.Engine(g, parts, [0] * parts, mgg.make_gcn(dim, 8, 4), *cfg)
    eng.set_remote_fetch("fine")
    rows = []
    eng.set_mapping(0, 0)
    m = eng.measure_multi_gpu(dim, reps)
    base = m["per_gpu_ns"]
    rows.append(row("mgg", base, m["mean_occupancy"], m["mean_utilization"],
                    m["remote_bytes"], base))
    part0_mgg = m["per_gpu"][0]["alone_ns"]
    eng.set_mapping(0, 1)
    r = eng.measure_multi_gpu(dim, reps)
    rows.append(row("no_np", r["per_gpu_ns"], r["mean_occupancy"], r["mean_utilization"],
                    r["remote_bytes"], base))
    eng.set_mapping(1, 0)
    r = eng.measure_multi_gpu(dim, reps)
    rows.append(row("no_interleave", r["per_gpu_ns"], r["mean_occupancy"],
                    r["mean_utilization"], r["remote_bytes"], base))
    eng.set_mapping(0, 0)
    rem = eng.time_aggregate_each(dim, reps, 2)
    loc = eng.time_aggregate_each(dim, reps, 1)
    rows.append(row("phase_separated", max(a + b for a, b in zip(rem, loc)),
                    m["mean_occupancy"], m["mean_utilization"], m["remote_bytes"], base))
    # paged: part 0 gathers its peers' rows through page faults
    for q in range(1, parts):
        eng.set_shard_memory(q, mgg.MEM_MANAGED_HOST)
    paged0 = eng.time_aggregate_each(dim, max(2, reps // 2), 0)[0]
    pages = (4 * dim + PAGE - 1) // PAGE
    paged_bytes = sum(mgg.build_flat_plan(g, parts, p, cfg[0], cfg[1], cfg[2], dim)
                      .remote_cols_len for p in range(parts)) * pages * PAGE
    r0 = rows[0]
    rows.append(row("paged_remote", paged0, r0["occupancy"], r0["smUtilization"],
                    paged_bytes, part0_mgg)
                | {"measured_part": 0, "mgg_part0_ns": int(part0_mgg)})
    for q in range(1, parts):
        eng.set_shard_memory(q, mgg.MEM_DEVICE)
    eng.set_remote_fetch("halo")
    r = eng.measure_multi_gpu(dim, reps)
    rows.append(row("mgg_halo", r["per_gpu_ns"], r["mean_occupancy"], r["mean_utilization"],
                    r["remote_bytes"], base))
    kern = eng.k1_kernels(0)
    eng.close()
    csv = "mode,ns,occupancy,smUtilization,remoteBytes,ratioVsMgg\n" + "".join(
        f"{x['mode']},{x['ns']},{x['occupancy']:.6f},{x['smUtilization']:.6f},"
        f"{x['remoteBytes']},{x['ratioVsMgg']:.6f}\n" for x in rows)
    return rows, csv, kern


def run_slow_peer(g, parts, dim, cfg, reps=5):
    """The same modes timed on part 0 with every other part's shards in pinned
    host memory mapped into the device (MGG_MEM_HOST_MAPPED): remote rows cross
    PCIe with microsecond latency, so interleaving / phase separation measure
    latency hiding (same-device peers have local latency). Part 0 alone."""
    eng = mgg.Engine(g, parts, [0] * parts, mgg.make_gcn(dim, 8, 4), *cfg)
    eng.set_remote_fetch("fine")
    for q in range(1, parts):
        eng.set_shard_memory(q, mgg.MEM_HOST_MAPPED)
    t = {}
    eng.set_mapping(0, 0)
    t["mgg"] = eng.time_aggregate_each(dim, reps, 0)[0]
    t["local_only"] = eng.time_aggregate_each(dim, reps, 3)[0]
    t["remote_only"] = eng.time_aggregate_each(dim, reps, 2)[0]
    t["phase_separated"] = t["remote_only"] + eng.time_aggregate_each(dim, reps, 1)[0]
    eng.set_mapping(1, 0)
    t["no_interleave"] = eng.time_aggregate_each(dim, reps, 0)[0]
    eng.set_mapping(0, 1)
    t["no_np"] = eng.time_aggregate_each(dim, max(2, reps // 2), 0)[0]
    eng.set_mapping(0, 0)
    eng.set_remote_fetch("halo")
    t["mgg_halo"] = eng.time_aggregate_each(dim, reps, 0)[0]
    kern = eng.k1_kernels(0)
    eng.close()
    base = t["mgg"]
    hid = max(0, t["remote_only"] + t["local_only"] - base)
    return {"times_ns": t, "ratio_vs_mgg": {k: round(v / max(base, 1), 4) for k, v in t.items()},
            "hidden_remote_fraction": round(hid / max(t["remote_only"], 1), 4),
            "pair_kernel": kern}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--slow-peer", action="store_true",
                    help="part 0 timed with host-mapped peers (run_slow_peer)")
    args = ap.parse_args()
    graphs = [("powerlaw-10K-avg16 (acceptance crit. 6 graph)",
               lambda: mgg.gen_synthetic(mgg.POWERLAW, 10_000, 16, 0), 16)]
    if args.slow_peer:  # PCIe-bandwidth-bound at the big graphs' remote shares
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from hiding_b200 import locality_graph

        def loc(far):
            rp, cl = locality_graph(2_000_000, 25.0, 64, far)
            return mgg.CsrGraph.from_csr(rp, cl)
        graphs += [(f"locality 2M/50M far={far}", (lambda f=far: loc(f)), 16)
                   for far in (0.002, 0.01)]
    elif not args.quick:
        graphs += [("reddit-shaped", lambda: mgg.gen_synthetic(mgg.POWERLAW, 232_965, 492, 0), 16),
                   ("products-shaped",
                    lambda: mgg.gen_synthetic(mgg.POWERLAW, 2_449_029, 25.259, 0), 16)]
    res = []
    for name, mk, dim in graphs:
        g = mk()
        for parts in (2, 4):
            for cfg in [(16, 8, 8), (32, 16, 2)]:
                if args.slow_peer:
                    res.append({"graph": name, "edges": g.num_edges, "parts": parts,
                                "dim": dim, "cfg": cfg, "remote_shards": "host-mapped (PCIe)",
                                **run_slow_peer(g, parts, dim, cfg)})
                    print(json.dumps(res[-1]), flush=True)
                    continue
                rows, csv, kern = run(g, parts, dim, cfg)
                res.append({"graph": name, "edges": g.num_edges, "parts": parts, "dim": dim,
                            "cfg": cfg, "pair_kernel": kern, "rows": rows, "csv": csv})
                print(json.dumps(res[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for r in res:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Remote-latency hiding of the fine-grained pipelined K1 on ONE B200
(SURVEY §8d hidden fraction; R:PAPER.md:405-419).

Two logical parts on device 0; part 1's shards live in pinned host memory
mapped into the device (MGG_MEM_HOST_MAPPED), so every remote row part 0
gathers crosses PCIe with microsecond latency — a slow "peer". Part 0's K1
is timed local-only (phase 3: the local partitions through the same pair
kernel), remote-only (phase 2) and pipelined (phase 0);
hidden = (T_rem + T_loc - T_pipe) / T_rem, and
overlap_of_shorter = the same numerator over min(T_rem, T_loc) (how much of
the shorter leg disappears; 1.0 = T_pipe == max(T_loc, T_rem)).

The graphs carry tunable locality: every neighbor is drawn from a window
around its target with probability 1 - far, uniformly otherwise (ids not
shuffled), so the remote-edge fraction of the 1D split sweeps from ~0 to
~far/2. Each K1 pair form runs in its own process (MGG_AGG_PAIR is read once).

usage: tools/hiding_b200.py [--out profiles/r02_hiding.jsonl] [--forms 1,0,2]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def locality_graph(n, avg, window, far, seed=0):
    """CSR (row = target) with neighbors near the target except a `far`
    fraction drawn uniformly; rows sorted, duplicates kept."""
    rng = np.random.default_rng(seed)
    deg = rng.poisson(avg, n).astype(np.int64)
    deg = np.maximum(deg, 1)
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(deg)
    e = int(rp[-1])
    tgt = np.repeat(np.arange(n, dtype=np.int64), deg)
    near = tgt + rng.integers(-window, window + 1, e)
    near = np.clip(near, 0, n - 1)
    uni = rng.integers(0, n, e)
    col = np.where(rng.random(e) < far, uni, near)
    key = np.sort(tgt * n + col)  # rows are contiguous already: sort within rows
    return rp, (key % n).astype(np.uint64)


def graphs(args):
    """(far, graph) pairs: the locality sweep, or one bench workload's graph."""
    import paper_2209_06800_b200 as mgg
    if args.graph:
        import bench
        _, g, _, _ = bench.build(mgg, args.graph)
        yield None, g
        return
    for far in [float(x) for x in args.far.split(",")]:
        rp, cl = locality_graph(args.nodes, args.avg, args.window, far)
        yield far, mgg.CsrGraph.from_csr(rp, cl)


def run_one(args):
    import paper_2209_06800_b200 as mgg
    out = []
    for far, g in graphs(args):
        model = mgg.make_gcn(args.dim, 16, 8)
        n = args.parts
        eng = mgg.Engine(g, n, [0] * n, model, ps=args.ps, dist=args.dist, wpb=args.wpb)
        eng.set_remote_fetch(args.fetch)
        eng.set_mapping(args.mapping, 0)
        if args.host:
            for q in range(1, n):
                eng.set_shard_memory(q, mgg.MEM_HOST_MAPPED)
        # phase 3 = the local partitions through the pipelined kernel itself;
        # phase 1 = the lean local-only kernel (reported beside it)
        t = {}
        for ph in (1, 3, 2, 0):  # the pipelined launch last: k1_kernels names it
            t[ph] = eng.time_aggregate_each(args.dim, args.reps, ph)[0]
        kern = eng.k1_kernels(0)
        st = eng.stats()
        eng.close()
        pipe, loc, rem = t[0], t[3], t[2]
        hid = max(0.0, rem + loc - pipe)
        fp = mgg.build_flat_plan(g, n, 0, args.ps, args.dist, args.wpb, args.dim)
        out.append({
            "pair_form": os.environ.get("MGG_AGG_PAIR", "default"),
            "pipe_depth": os.environ.get("MGG_AGG_PIPE_DEPTH", "8"),
            "sched": os.environ.get("MGG_AGG_SCHED", "4 (default)"),
            "dyn": os.environ.get("MGG_AGG_DYN", "default"), "kernels": kern,
            "graph": args.graph or "locality", "far": far, "mapping": args.mapping,
            "fetch": args.fetch, "parts": args.parts,
            "nodes": int(g.num_nodes), "edges": int(g.num_edges), "dim": args.dim,
            "config": [args.ps, args.dist, args.wpb],
            "remote_shard": "host-mapped (PCIe)" if args.host else "device (same GPU)",
            "part0_local_edges": fp.local_cols_len, "part0_remote_edges": fp.remote_cols_len,
            "remote_edge_fraction": round(fp.remote_cols_len / max(
                fp.local_cols_len + fp.remote_cols_len, 1), 4),
            "t_pipelined_ns": pipe, "t_local_only_ns": loc, "t_remote_only_ns": rem,
            "t_local_only_lean_kernel_ns": t[1],
            "hidden_remote_fraction": round(hid / max(rem, 1), 4),
            "overlap_of_shorter": round(hid / max(min(rem, loc), 1), 4),
            "pipe_vs_max": round(pipe / max(loc, rem, 1), 4),
            "remote_parts_total": st["remote_parts"]})
        print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=2_000_000)
    ap.add_argument("--avg", type=float, default=25.0)
    ap.add_argument("--window", type=int, default=64)
    ap.add_argument("--far", default="0.0005,0.001,0.002,0.004,0.01,0.05")
    ap.add_argument("--dim", type=int, default=16)
    ap.add_argument("--ps", type=int, default=16)
    ap.add_argument("--dist", type=int, default=8)
    ap.add_argument("--wpb", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mapping", type=int, default=0, help="0 interleaved, 1 segregated")
    ap.add_argument("--graph", default=None, help="a bench workload's graph instead of the sweep")
    ap.add_argument("--parts", type=int, default=2,
                    help="logical parts; every part but 0 is the (host-mapped) peer")
    ap.add_argument("--fetch", default="fine", choices=["fine", "halo"],
                    help="halo: deduplicated pull on the aux stream || local pass, then the "
                         "remote pass (phase 2 = pull + remote pass)")
    ap.add_argument("--device-peer", dest="host", action="store_false",
                    help="keep part 1's shard in device memory (same-GPU peer)")
    ap.add_argument("--forms", default="1,2,3,3:16",
                    help="MGG_AGG_PAIR[:MGG_AGG_PIPE_DEPTH] values, one process each")
    ap.add_argument("--probe", action="store_true", help="host-mapped gather/latency probes")
    ap.add_argument("--out", default=None)
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        run_one(args)
        return
    rows = []
    if args.probe:
        from paper_2209_06800_b200 import probes
        pr = {"probe": "host-mapped vs device, 16-float rows (64 B), 2M random rows",
              "host_gather_gbps": round(probes.host_gather_gbps(1_000_000, 16, 2_000_000), 2),
              "device_gather_gbps": round(probes.gather_gbps(1_000_000, 16, 2_000_000), 1),
              "host_chase_ns": round(probes.host_chase_ns(64 << 20), 1),
              "device_chase_ns": round(probes.chase_ns(1 << 30), 1)}
        print(json.dumps(pr), flush=True)
        rows.append(pr)
    for form in args.forms.split(","):
        pair, _, rest = form.partition(":")
        depth, _, rest = rest.partition(":")
        sched = rest
        cmd = [sys.executable, os.path.abspath(__file__), "--child"] + [
            a for a in sys.argv[1:] if not a.startswith("--out") and a != args.out
            and a != "--probe"]
        env = {**os.environ, "MGG_AGG_PAIR": pair, "MGG_AGG_PIPE_DEPTH": depth or "8"}
        if sched:  # else the library default (chunks of 4)
            env["MGG_AGG_SCHED"] = sched
        r = subprocess.run(cmd, capture_output=True, text=True, env=env)
        sys.stderr.write(r.stderr[-3000:])
        rows += [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
        for l in r.stdout.splitlines():
            print(l, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()

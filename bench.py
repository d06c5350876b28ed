#!/usr/bin/env python
"""Benchmark of the MGG hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], fits one GPU): 2-layer GCN (hidden 16,
41 classes) on a synthetic Reddit-shaped graph — 232,965 nodes, reference
`powerlaw` generator (SplitMix64 seed 0, avg degree 492 -> ~113.6M edges),
input dim 602, X ~ U[-1,1) (seed 1), Glorot weights (seed 2).

A step = one full GCN forward (both layers: Update GEMM X·W1, K1 layer-1
aggregation, ReLU-on-load K1 layer-2 aggregation, GEMM·W2 + softmax) over
the whole graph. metric = aggregation GEdges/s = layers x E / step time
(and ms_per_step = forward ms). Inputs (X 561 MB + CSR 455 MB) are larger
than the 126 MB L2, so no flush between steps.

  value   : device-resident X, CUDA events on the engine's stream bracketing
            exactly K steps (barrier + synchronize both sides), max over ranks.
  e2e     : the same metric through the C-ABI `mgg_engine_forward_host`
            with pinned HOST X in / Z out (H2D + D2H inside the timed region).
  roofline: dominant kernel (K1 aggregation), algorithmic bytes per launch
            (E·(4D + 4) + 8·P + 8·rows·D) / its average event-timed
            duration inside the timed region vs MEASURED_PEAKS hbm_gbs.
  cpu_baseline: the oracle port (oracle/oracle.c, fp32 accumulate, all host
            threads) of the same forward on the same graph, rank 0 only.

--impl reference: the reference's CPU implementation of the path. The
reference (pipeshard) has no layer arithmetic, so this arm times the oracle
port of the forward (same graph/config) on all host cores, and reports the
reference library's own metadata-build time beside it when oracle/_ref exists.

Multi-GPU: launched by torchrun, one process per GPU; part r = rank r's
edge-balanced node range (Alg. 1), remote rows read over NVLink from peer
shards imported through CUDA IPC; no NCCL on the data path ("scaling":
"strong" — the graph is fixed as N grows).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_NODES = 232_965
AVG_DEG = 492
IN_DIM, HIDDEN, CLASSES = 602, 16, 41
PS, DIST, WPB = 16, 1, 4
WORKLOAD = "GCN-2L Reddit-shaped (BASELINE configs[1])"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mgg", choices=["mgg", "reference"])
    ap.add_argument("--ps", type=int, default=PS)
    ap.add_argument("--dist", type=int, default=DIST)
    ap.add_argument("--wpb", type=int, default=WPB)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def build_graph(mgg):
    t0 = time.perf_counter()
    g = mgg.gen_synthetic(mgg.POWERLAW, N_NODES, AVG_DEG, 0)
    return g, time.perf_counter() - t0


def agg_bytes(edges: int, parts: int, rows: int, dim: int) -> int:
    """Algorithmic bytes of one K1 launch at width dim: gathered
    rows + 4-B column ids + 8-B partition records + accumulator read/write."""
    pitch = (dim + 3) // 4 * 4
    return edges * (4 * pitch + 4) + 8 * parts + 2 * rows * 4 * pitch


def _traffic(args):
    """DRAM bytes per K1 launch from the committed ncu capture of this config."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            t = json.load(f)
        if t.get("config") == [args.ps, args.dist, args.wpb]:
            return t["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        pass
    return None


def cpu_forward_time(g, x, model, threads=0):
    import oracle
    rp, cl = g.row_ptr, g.col_idx
    t0 = time.perf_counter()
    oracle.gcn2_forward(rp, cl, x, model, acc64=False, threads=threads)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: CPU implementation of the path on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import paper_2209_06800_b200 as mgg
    g, _ = build_graph(mgg)
    e = g.num_edges
    model = mgg.make_gcn(IN_DIM, HIDDEN, CLASSES, seed=2)
    x = mgg.random_features(N_NODES, IN_DIM, seed=1)
    cores = os.cpu_count() or 1
    for _ in range(max(args.warmup, 0)):
        cpu_forward_time(g, x, model)
    times = [cpu_forward_time(g, x, model) for _ in range(max(args.steps, 1))]
    t = sum(times) / len(times)
    value = 2 * e / t / 1e9
    meta = None
    if oracle.ref_available():
        r = oracle.RefGraph.from_csr(g.row_ptr, g.col_idx)
        secs, nparts = r.time_metadata(args.gpus, args.ps, args.dist, args.wpb, IN_DIM)
        meta = {"ref_metadata_build_s": round(secs, 4), "partitions": nparts}
    line = {
        "impl": "reference", "metric": "aggregation GEdges/s (GCN-2L forward)",
        "value": round(value, 4), "unit": "GEdges/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": N_NODES, "edges": e, "dim": IN_DIM,
                   "hidden": HIDDEN, "classes": CLASSES, "graph": "powerlaw seed 0"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GEdges/s", "cores": cores,
                         "kind": "port",
                         "sample": "full GCN-2L forward of the workload per step "
                                   "(oracle.c fp32, OpenMP all host threads); the reference "
                                   "library has no layer arithmetic",
                         "reference_metadata": meta},
        "e2e": {"value": round(value, 4), "unit": "GEdges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
        return

    import paper_2209_06800_b200 as mgg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(args.gpus, world)
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group(backend="cpu:gloo,cuda:nccl")
    if not mgg.cuda_available():
        raise SystemExit("bench.py: no CUDA device visible (the product has no CPU path)")

    g, gen_s = build_graph(mgg)
    E = g.num_edges
    model = mgg.make_gcn(IN_DIM, HIDDEN, CLASSES, seed=2)
    x = mgg.host_alloc((N_NODES, IN_DIM))
    x[:] = mgg.random_features(N_NODES, IN_DIM, seed=1)
    z = mgg.host_alloc((N_NODES, CLASSES))

    from paper_2209_06800_b200 import dist as mdist
    if world > 1:
        part_device = mdist.part_devices(world, rank, local_rank)
    else:
        part_device = [0] * n  # N logical partitions on one GPU if --gpus > 1
    gather_peak = None
    if rank == 0:  # K5 probe: the gather ceiling of this table shape, live
        from paper_2209_06800_b200 import probes
        gather_peak = probes.gather_gbps(N_NODES, HIDDEN, E, device=local_rank)
    t0 = time.perf_counter()
    eng = mgg.Engine(g, n, part_device, model, ps=args.ps, dist=args.dist, wpb=args.wpb)
    setup_s = time.perf_counter() - t0
    if world > 1:
        mdist.exchange_ipc(eng, rank, world)
        dist.barrier()
    eng.set_input(x)
    eng.synchronize()

    from paper_2209_06800_b200._lib import lib
    ctx = eng.ctx()
    my_part = rank if world > 1 else 0

    for _ in range(max(args.warmup, 3)):
        eng.forward()
    eng.synchronize()
    if world > 1:
        dist.barrier()

    eng.set_profiling(True)
    launches0 = eng.stats()["launches"]
    with ClockSampler(local_rank) as clk:
        eng.synchronize()
        if world > 1:
            dist.barrier()
        lib.mgg_event_record(ctx, my_part, 1000)
        for _ in range(args.steps):
            eng.forward()
        lib.mgg_event_record(ctx, my_part, 1001)
        eng.synchronize()
        if world > 1:
            dist.barrier()
    import ctypes
    ms = ctypes.c_float()
    lib.mgg_event_elapsed(ctx, my_part, 1000, 1001, ctypes.byref(ms))
    total_ms = ms.value
    launches = eng.stats()["launches"] - launches0
    ops, nfw = eng.profile()
    eng.set_profiling(False)
    if world > 1:
        total_ms = mdist.max_over_ranks(total_ms)
    ms_step = total_ms / args.steps
    value = 2 * E / (ms_step * 1e-3) / 1e9

    # dominant kernel: aggregation (K1) launches inside the timed region
    st = eng.stats()
    agg = [(w, t) for k, w, t in ops if k == "aggregate"]
    agg_ms_per_launch = sum(t for _, t in agg) / (len(agg) * nfw)
    my_edges = st["local_edges"] + st["remote_edges"]
    my_parts = st["local_parts"] + st["remote_parts"]
    rows = N_NODES if world == 1 else N_NODES // world
    algo = agg_bytes(my_edges, my_parts, rows, HIDDEN)
    peak, peak_kind = _peaks()
    achieved = algo / (agg_ms_per_launch * 1e-3) / 1e9
    share = sum(t for _, t in agg) / max(sum(t for _, _, t in ops), 1e-9)

    # end to end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        eng.forward_host(x, z)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        k2 = max(3, args.steps // 2)
        for _ in range(k2):
            eng.forward_host(x, z)
        e2e_s = (time.perf_counter() - t0) / k2
        if world > 1:
            e2e_s = mdist.max_over_ranks(e2e_s)
        e2e = {"value": round(2 * E / e2e_s / 1e9, 4), "unit": "GEdges/s",
               "ms_per_step": round(e2e_s * 1e3, 3),
               "h2d_bytes_per_step": int(N_NODES * IN_DIM * 4 // (world if world > 1 else 1)),
               "d2h_bytes_per_step": int(N_NODES * CLASSES * 4 // (world if world > 1 else 1)),
               "api": "mgg_engine_forward_host (pinned host X in, Z out)"}

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu:
        try:
            xs = np.asarray(x)
            tc = cpu_forward_time(g, xs, model)
            cpu = {"value": round(2 * E / tc / 1e9, 4), "unit": "GEdges/s",
                   "cores": os.cpu_count(), "kind": "port",
                   "sample": "one full GCN-2L forward of the same workload "
                             "(oracle.c, fp32 accumulate, OpenMP all host threads)",
                   "seconds": round(tc, 3)}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "error": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": "aggregation GEdges/s (GCN-2L forward)",
            "value": round(value, 4), "unit": "GEdges/s", "n_gpus": n,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "graph": "powerlaw (reference generator) seed 0",
                       "nodes": N_NODES, "edges": E, "dim": IN_DIM, "hidden": HIDDEN,
                       "classes": CLASSES, "ps": args.ps, "dist": args.dist, "wpb": args.wpb,
                       "parts": n, "l2": "inputs larger than L2 (X 561 MB + CSR), no flush",
                       "layer_forward_ms": round(ms_step, 4)},
            "roofline": {"bound": "hbm", "kernel": "K1 aggregation (agg_kernel<4>)",
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": _traffic(args),
                         "algorithmic_bytes_per_launch": algo,
                         "avg_launch_ms": round(agg_ms_per_launch, 4),
                         "share_of_step": round(share, 4), "peak_source": peak_kind,
                         "l2_gather": None if not gather_peak else {
                             "peak": round(gather_peak, 1), "unit": "GB/s",
                             "frac": round(achieved / gather_peak, 4),
                             "source": "K5 probe (paper_2209_06800_b200/probes.py), this run"},
                         "note": "the gathered rows (16-wide, 15 MB table) are L2-resident, so "
                                 "the binding ceiling is the L2->SM gather rate (l2_gather); "
                                 "algorithmic bytes count every gathered row as in SURVEY 8d; "
                                 "traffic = ncu DRAM bytes per launch (profiles/)"},
            "ops": [{"kind": k, "width": w, "ms": round(t / nfw, 4)} for k, w, t in ops],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
            "setup": {"graph_gen_s": round(gen_s, 2), "engine_setup_s": round(setup_s, 2),
                      "plan_build_ms": round(st["plan_build_ns"] / 1e6, 1),
                      "remote_edge_fraction": round(st["remote_edges"] / max(my_edges, 1), 4)},
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

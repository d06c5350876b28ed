#!/usr/bin/env python
"""Benchmark of the MGG hot path on B200 (contract: one JSON line on rank 0).

Default workload: north_star's target shape — 2-layer GCN (hidden 16, 47
classes) on a synthetic ogbn-products-shaped graph: 2,449,029 nodes, the
reference's `powerlaw` generator (SplitMix64 seed 0, avg degree 25.259 ->
60.8M edges), input dim 100, X ~ U[-1,1) (seed 1), Glorot weights (seed 2).
BASELINE configs[1] (GCN-2L, Reddit-shaped, dim 602) is measured in the same
run and reported under "secondary" (device value + K1 roofline).
Other configs (--workload): config1 (RMAT 100K/1.6M, dim 16, 2 logical
partitions), reddit-gcn (configs[1]), products-gin (configs[2]), orkut-gcn
(configs[3]), RMAT variants.

A step = one full forward (every layer: Update GEMM(s), K1 aggregation(s),
head) over the whole graph. metric = aggregation GEdges/s = layers x E / step
time; ms_per_step = forward ms. Inputs (X + CSR, >= 1 GB) exceed the 126 MB
L2, so no flush between steps.

  value   : device-resident X, CUDA events on the engine's stream bracketing
            exactly K steps (barrier + synchronize both sides), max over ranks.
  e2e     : the same metric through the C-ABI `mgg_engine_forward_host`
            with pinned HOST X in / Z out (H2D + D2H inside the timed region).
  roofline: dominant kernel (K1 aggregation, the kernel names the library
            reports for the launch), bound by what binds it: "hbm" when the
            gathered table exceeds half the L2 — algorithmic bytes per launch
            (E·(4·pitch + 4) + 8·P + 8·rows·pitch) / its average
            event-timed duration vs MEASURED_PEAKS hbm_gbs; "l2" when it fits —
            gathered-row bytes only (E·4·pitch) / duration vs the live K5
            gather probe (uniform random rows, rows-only bytes: like for
            like). `dram` = the committed ncu DRAM bytes of that launch.
  cpu_baseline: the oracle port (oracle/oracle.c, fp32 accumulate, all host
            threads) of the same forward on the same graph, rank 0, N=1.

--impl reference: the reference's CPU implementation of the path. The
reference (pipeshard) has no layer arithmetic, so this arm times the oracle
port of the forward (same workload) on all host cores, and reports the
reference library's own metadata-build time beside it when oracle/_ref exists.
It never loads the product: the graph comes from the reference library's own
generator (oracle/_ref) or the oracle's C restatement of it, X and W from the
numpy generators below (identical arrays, tests/test_bench.py).

hiding  : (N=1) remote-latency hiding of the pipelined K1 against a slow peer
            (host-mapped shard of a second logical part; slow_peer_hiding).

Multi-GPU: torchrun, one process per GPU; part r = rank r's edge-balanced
node range (Alg. 1); remote rows read in-kernel over NVLink from peer shards
imported through CUDA IPC; no NCCL on the data path ("scaling": "strong").
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

# name: (label, graph (kind, nodes, avg_degree | edges), model (kind, in, hidden, out, layers),
#        tuned (ps, dist, wpb) — profiles/r01_tune2_*.json: the exhaustive optimum of the
#        150-point grid with the measured K1 where swept (the tuner lands within 1.2% of it
#        in <= 15 evaluations), the tuner's pick elsewhere)
WORKLOADS = {
    "reddit-gcn": ("GCN-2L Reddit-shaped (BASELINE configs[1])",
                   ("powerlaw", 232_965, 492), ("gcn", 602, 16, 41, 2), (32, 16, 2)),
    "config1": ("GCN-2L RMAT 100K/1.6M dim 16, 2 logical partitions (BASELINE configs[0])",
                ("rmat", 100_000, 1_600_000), ("gcn", 16, 16, 16, 2), (8, 8, 2)),
    "products-gcn": ("GCN-2L ogbn-products-shaped (north_star target shape)",
                     ("powerlaw", 2_449_029, 25.259), ("gcn", 100, 16, 47, 2), (16, 8, 8)),
    "products-gin": ("GIN-5L hidden 64 ogbn-products-shaped (BASELINE configs[2])",
                     ("powerlaw", 2_449_029, 25.259), ("gin", 100, 64, 47, 5), (16, 2, 8)),
    "orkut-gcn": ("GCN-2L com-Orkut-shaped (BASELINE configs[3])",
                  ("powerlaw", 3_072_441, 38.141), ("gcn", 128, 16, 32, 2), (8, 16, 8)),
    # the symmetric-normalised GCN (D^-1/2 (A+I) D^-1/2) on the configs[1] graph
    "reddit-gcn-norm": ("GCN-2L normalised, Reddit-shaped (configs[1] graph)",
                        ("powerlaw", 232_965, 492), ("gcn-norm", 602, 16, 41, 2), (32, 16, 2)),
    # locality-bearing (skewed, ids not shuffled) variants of the same shapes
    # (report both an id-random and an RMAT variant per graph)
    "reddit-rmat-gcn": ("GCN-2L Reddit-shaped RMAT variant",
                        ("rmat", 232_965, 114_615_892), ("gcn", 602, 16, 41, 2), (32, 16, 2)),
    "products-rmat-gin": ("GIN-5L hidden 64 ogbn-products-shaped RMAT variant",
                          ("rmat", 2_449_029, 61_859_140), ("gin", 100, 64, 47, 5), (16, 16, 2)),
    "orkut-rmat-gcn": ("GCN-2L com-Orkut-shaped RMAT variant",
                       ("rmat", 3_072_441, 117_185_083), ("gcn", 128, 16, 32, 2), (16, 16, 2, 3)),
}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mgg", choices=["mgg", "reference"])
    ap.add_argument("--workload", default="products-gcn", choices=sorted(WORKLOADS))
    ap.add_argument("--secondary", default="reddit-gcn",
                    help="comma-separated workloads also measured at N=1 (device value + "
                         "roofline only); 'none' to skip")
    ap.add_argument("--ps", type=int, default=None)
    ap.add_argument("--dist", type=int, default=None)
    ap.add_argument("--wpb", type=int, default=None)
    ap.add_argument("--parts", type=int, default=None,
                    help="logical partitions on one GPU (single process)")
    ap.add_argument("--fetch", default="auto", choices=["auto", "fine", "halo"],
                    help="remote rows: per-edge peer reads in K1 (fine, the paper's design) or "
                         "one deduplicated pull per layer (halo); auto picks by bytes moved")
    ap.add_argument("--k1-form", type=int, default=None, choices=[0, 1, 2, 3],
                    help="local-only K1 form (0 by shape, 1 warp-window, 2/3 group with 8/4 "
                         "rows in flight); default: the workload's tuned form")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-hiding", action="store_true",
                    help="skip the slow-peer remote-latency hiding measurement (N=1)")
    a = ap.parse_args()
    tuned = WORKLOADS[a.workload][3]
    a.ps = a.ps or tuned[0]
    a.dist = a.dist or tuned[1]
    a.wpb = a.wpb or tuned[2]
    if a.k1_form is None:  # the tuner post-pass's K1 form, 0 (by shape) if none
        a.k1_form = tuned[3] if len(tuned) > 3 and (a.ps, a.dist, a.wpb) == tuned[:3] else 0
    return a


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML every
    ~1 ms (the timed region of a default run is only ~10-20 ms), nvidia-smi
    (~5 Hz) as the fallback when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.source = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
            self.source = "nvml"
        except Exception:  # noqa: BLE001
            self.source = "nvidia-smi"

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        if not hasattr(self, "_max"):
            self._max = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        mx = self._max
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        rs = get(h)
        self.samples.append((float(sm), float(mx), int(rs)))

    def _sample_smi(self):
        out = subprocess.run(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits"], capture_output=True, text=True,
            timeout=5).stdout.strip()
        if not out:
            return
        f = [x.strip() for x in out.split(",")]
        mask = 0
        for k, (_, bit) in enumerate(self.REASONS):
            if len(f) > 3 + k and f[3 + k].lower().startswith("active"):
                mask |= bit
        num = [float(x) if x.replace(".", "").isdigit() else float("nan") for x in f[:2]]
        self.samples.append((num[0], num[1], mask))

    def sample_now(self):
        """One sample from the calling thread (used right after the timed work
        is queued, while the device is still executing it)."""
        try:
            if self._nvml:
                self._sample_nvml()
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.001 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [x[0] for x in self.samples if x[0] == x[0]]
        mx = [x[1] for x in self.samples if x[1] == x[1]]
        reasons = sorted({name for _, _, m in self.samples for name, bit in self.REASONS
                          if m & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


L2_BYTES = 126 * 2**20  # B200 L2


def build(mgg, name):
    label, gspec, mspec, _ = WORKLOADS[name]
    t0 = time.perf_counter()
    kind, n, avg = gspec
    if kind == "rmat":
        g = mgg.gen_rmat(n, int(avg), 0)
    else:
        g = mgg.gen_synthetic(mgg.POWERLAW, n, avg, 0)
    gen_s = time.perf_counter() - t0
    mk, din, hid, out, layers = mspec
    if mk in ("gcn", "gcn-norm"):
        model = mgg.make_gcn(din, hid, out, seed=2, norm=mk == "gcn-norm")
    else:
        model = mgg.make_gin(din, hid, out, layers=layers, seed=2)
    return label, g, model, gen_s


# ---- numpy input generators of the reference arm (no product code): the same
# arrays as paper_2209_06800_b200.api.make_gcn / make_gin / random_features
class NpModel:
    def __init__(self, kind, layers, in_dim, hidden, out_dim, w1, b1=None, w2=None, b2=None,
                 eps=0.0, norm=0):
        self.kind, self.layers, self.in_dim, self.hidden, self.out_dim = (
            kind, layers, in_dim, hidden, out_dim)
        self.w1, self.b1, self.w2, self.b2, self.eps, self.norm = w1, b1, w2, b2, eps, norm

    def gin_dims(self):
        return [self.in_dim] + [self.hidden] * (self.layers - 1) + [self.out_dim]


def np_model(mspec, seed=2):
    mk, din, hid, out, layers = mspec
    rng = np.random.default_rng(seed)

    def glorot(fi, fo):
        lim = np.sqrt(6.0 / (fi + fo))
        return rng.uniform(-lim, lim, size=(fi, fo)).astype(np.float32)
    if mk in ("gcn", "gcn-norm"):
        w = np.concatenate([glorot(din, hid).ravel(), glorot(hid, out).ravel()])
        return NpModel(0, 2, din, hid, out, w.astype(np.float32), norm=int(mk == "gcn-norm"))
    dims = [din] + [hid] * (layers - 1) + [out]
    w1, b1, w2, b2 = [], [], [], []
    for l in range(layers):
        w1.append(glorot(dims[l], hid).ravel())
        b1.append(rng.uniform(-0.1, 0.1, hid).astype(np.float32))
        w2.append(glorot(hid, dims[l + 1]).ravel())
        b2.append(rng.uniform(-0.1, 0.1, dims[l + 1]).astype(np.float32))
    cat = lambda xs: np.ascontiguousarray(np.concatenate(xs), np.float32)  # noqa: E731
    return NpModel(1, layers, din, hid, out, cat(w1), cat(b1), cat(w2), cat(b2), 0.0)


def np_features(n, d, seed=1):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, d)).astype(np.float32)


def ref_graph(name):
    """CSR of the workload's graph without the product: the reference
    library's own generator (oracle/_ref) for powerlaw graphs, else the
    oracle's C restatement (bit-identical; tests/test_bench.py)."""
    import oracle
    kind, n, avg = WORKLOADS[name][1]
    t0 = time.perf_counter()
    if kind == "rmat":
        rp, cl = oracle.gen_rmat(n, int(avg), 0)
        src = "oracle.c RMAT restatement"
    elif oracle.ref_available():
        rp, cl = oracle.RefGraph.gen(1, n, avg, 0).csr()
        src = "reference gen_synthetic (oracle/_ref)"
    else:
        rp, cl = oracle.gen_synthetic(1, n, avg, 0)
        src = "oracle.c gen_synthetic restatement"
    return rp, cl, src, time.perf_counter() - t0


def agg_widths(model):
    """Aggregation width of each layer (aggregate at min(in, out) width)."""
    if model.kind == 0:
        return [min(model.in_dim, model.hidden), min(model.hidden, model.out_dim)]
    dims = model.gin_dims()
    return [min(dims[l], model.hidden) for l in range(model.layers)]


def workload_config(name, args, nodes, edges, model, parts):
    """The `config` object both arms print (identical for the same flags)."""
    label, gspec = WORKLOADS[name][0], WORKLOADS[name][1]
    return {"workload": label, "name": name,
            "graph": f"{gspec[0]} (reference generator / RMAT) seed 0",
            "nodes": int(nodes), "edges": int(edges), "dim": model.in_dim,
            "hidden": model.hidden, "classes": model.out_dim, "layers": model.layers,
            "agg_widths": agg_widths(model), "ps": args.ps, "dist": args.dist,
            "wpb": args.wpb, "k1_form": args.k1_form, "parts": parts,
            "remote_fetch": args.fetch,
            "l2": "inputs larger than L2 (X + CSR >= 250 MB), no flush"}


def k1_form(row_ptr, ps: int, parts: int, width: int = 16, form: int = 0) -> str:
    """Which local K1 a single-device launch runs (the launcher's rule,
    csrc/cuda/aggregate.cu pick_lean) — a host-side prediction, checked in
    tests against the names the library reports (mgg_engine_k1_kernels)."""
    if parts > 1:
        return "agg_gpair (group per pair) / agg_group halo passes"
    pitch = (width + 3) // 4 * 4
    if form == 1:
        return "agg_local (warp window)"
    if form == 3:
        return "agg_group (group per partition, 4 rows in flight)"
    if form == 2:
        return ("agg_group_hint (group per partition, L2 hints)" if 8 < pitch <= 16
                else "agg_group (group per partition)")
    deg = np.diff(np.asarray(row_ptr, dtype=np.int64))
    nparts = int(((deg + ps - 1) // ps).sum())
    short = ps <= 16 or 3 * int(deg.sum()) < 2 * ps * nparts
    if not short:
        return "agg_local (warp window)"
    return ("agg_group_hint (group per partition, L2 hints)" if 8 < pitch <= 16
            else "agg_group (group per partition)")


def agg_bytes(edges: int, parts: int, rows: int, dim: int) -> int:
    """Algorithmic bytes of one K1 launch at width dim: gathered
    rows + 4-B column ids + 8-B partition records + accumulator read/write."""
    pitch = (dim + 3) // 4 * 4
    return edges * (4 * pitch + 4) + 8 * parts + 2 * rows * 4 * pitch


def roofline(nodes, edges, parts, rows, dim, launch_ms, gather_peak, traffic, kernels):
    """Roofline of one K1 launch against the resource that binds it (see the
    module docstring). Returns the JSON object."""
    pitch = (dim + 3) // 4 * 4
    table = nodes * pitch * 4
    algo = agg_bytes(edges, parts, rows, dim)
    t = launch_ms * 1e-3
    hbm_peak, hbm_src = _peaks()
    r = {"kernel": f"K1 aggregation, width {dim}: " + " + ".join(kernels),
         "avg_launch_ms": round(launch_ms, 4), "algorithmic_bytes_per_launch": algo,
         "gather_table_bytes": table, "unit": "GB/s"}
    if table <= L2_BYTES // 2 and gather_peak:
        rows_bytes = edges * 4 * pitch
        achieved = rows_bytes / t / 1e9
        r.update(bound="l2", achieved=round(achieved, 1), peak=round(gather_peak, 1),
                 frac=round(achieved / gather_peak, 4),
                 peak_source="K5 gather probe, this run: uniform random rows of the same "
                             "table shape, rows-only bytes (like for like: numerator = "
                             "E*4*pitch gathered-row bytes)")
    else:
        achieved = algo / t / 1e9
        r.update(bound="hbm", achieved=round(achieved, 1), peak=hbm_peak,
                 frac=round(achieved / hbm_peak, 4), peak_source=hbm_src)
    r["traffic"] = traffic
    if traffic:
        r["dram"] = {"bytes_per_launch": traffic, "achieved": round(traffic / t / 1e9, 1),
                     "frac": round(traffic / t / 1e9 / hbm_peak, 4),
                     "vs_algorithmic": round(traffic / algo, 4),
                     "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum of this "
                               "launch (profiles/k1_traffic.json)"}
    return r


def link_roofline(roof, nvl_bytes, launch_ms, hbm_peak_gbs, nvl_peak_gbs=900.0):
    """SURVEY §8d for one GPU of an N-GPU run: T_roof = max(HBM_g / HBM peak,
    NVL_g / NVLink peak). Adds the link term (the peer rows the rank's K1
    pulls: halo = each distinct row once, fine = one row per remote edge) to
    `roof` and makes it the reported bound when it is the larger one."""
    t = launch_ms * 1e-3
    gbs = nvl_bytes / t / 1e9
    hbm_t = roof["algorithmic_bytes_per_launch"] / (hbm_peak_gbs * 1e9)
    roof["nvlink"] = {"bytes_per_launch": int(nvl_bytes), "achieved": round(gbs, 1),
                      "peak": nvl_peak_gbs, "frac": round(gbs / nvl_peak_gbs, 4),
                      "peak_source": "NVLink 5 per direction (datasheet)"}
    if nvl_bytes / (nvl_peak_gbs * 1e9) > hbm_t:
        roof["hbm_bound"] = {k: roof[k] for k in ("achieved", "peak", "frac") if k in roof}
        roof.update(bound="nvlink", achieved=round(gbs, 1), peak=nvl_peak_gbs,
                    frac=round(gbs / nvl_peak_gbs, 4),
                    peak_source="NVLink 5 per direction (datasheet); the HBM term is "
                                "'hbm_bound'")
    return roof


def _traffic(args, parts, name=None):
    """DRAM bytes per K1 launch from the committed ncu capture of this config."""
    name = name or args.workload
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            for t in json.load(f):
                if t.get("workload") == name and t.get("config") == [
                        args.ps, args.dist, args.wpb] and t.get("parts", 1) == parts:
                    return t["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        pass
    return None


def host_threads() -> int:
    """All host threads of the box (torchrun exports OMP_NUM_THREADS=1 to every
    rank; the CPU baseline must not inherit that)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def cpu_forward_time(row_ptr, col, x, model, threads=None):
    threads = host_threads() if threads is None else threads
    import oracle
    t0 = time.perf_counter()
    if model.kind == 0:
        oracle.gcn2_forward(row_ptr, col, x, model, norm=model.norm, acc64=False,
                            threads=threads)
    else:
        oracle.gin_forward(row_ptr, col, x, model, acc64=False, threads=threads)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: CPU implementation of the path on the host cores
    (oracle/ only — the product library is never loaded on this arm)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import oracle
    name = args.workload
    label, _, mspec, _ = WORKLOADS[name]
    row_ptr, col, gsrc, gen_s = ref_graph(name)
    n, e = len(row_ptr) - 1, len(col)
    model = np_model(mspec)
    layers = model.layers
    x = np_features(n, model.in_dim, seed=1)
    cores = host_threads()
    for _ in range(max(args.warmup, 0)):
        cpu_forward_time(row_ptr, col, x, model)
    times = [cpu_forward_time(row_ptr, col, x, model) for _ in range(max(args.steps, 1))]
    t = sum(times) / len(times)
    value = layers * e / t / 1e9
    meta = None
    if oracle.ref_available():
        r = oracle.RefGraph.from_csr(row_ptr, col)
        secs, nparts = r.time_metadata(max(args.gpus, 1), args.ps, args.dist, args.wpb,
                                       model.in_dim)
        meta = {"ref_metadata_build_s": round(secs, 4), "partitions": nparts,
                "what": "the reference library's split + local/remote split + ps-partitions "
                        "+ warp/block mapping of every part, 1 host thread"}
    parts = args.parts or (2 if name == "config1" else max(args.gpus, 1))
    line = {
        "impl": "reference", "metric": f"aggregation GEdges/s ({label.split()[0]} forward)",
        "value": round(value, 4), "unit": "GEdges/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": workload_config(name, args, n, e, model, parts),
        "cpu_baseline": {"value": round(value, 4), "unit": "GEdges/s", "cores": cores,
                         "kind": "port",
                         "sample": "full forward of the workload per step (oracle.c fp32, "
                                   "OpenMP all host threads); the reference library has no "
                                   "layer arithmetic",
                         "graph_source": gsrc, "graph_gen_s": round(gen_s, 2),
                         "reference_metadata": meta},
        "e2e": {"value": round(value, 4), "unit": "GEdges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _reexec_under_torchrun(args):
    """`--gpus N` outside torchrun: one process per GPU via torch.distributed.run."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but {have} CUDA device(s) visible "
                         "(--parts N runs N logical partitions on one GPU)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.run(cmd).returncode)


def measure(name, args, mgg, lib, mdist, world, rank, local_rank, dist, full=True):
    """One workload through the product: device value (+ e2e, cpu, overlap
    when `full`). Returns the JSON fields (rank 0) or None."""
    import ctypes
    label, g, model, gen_s = build(mgg, name)
    N, E = g.num_nodes, g.num_edges
    layers = model.layers
    x = mgg.host_alloc((N, model.in_dim))
    x[:] = mgg.random_features(N, model.in_dim, seed=1)
    z = mgg.host_alloc((N, model.out_dim))

    if world > 1:
        n = world
        part_device = mdist.part_devices(world, rank, local_rank)
    else:
        n = args.parts or (2 if name == "config1" else 1)
        part_device = [0] * n  # logical partitions on one GPU
    widths = agg_widths(model)
    w0 = widths[0]
    gather_peak = None
    if rank == 0:  # K5 probe: the gather ceiling for this table shape, live
        from paper_2209_06800_b200 import probes
        gather_peak = probes.gather_gbps(N, w0, min(E, 200_000_000), device=local_rank)
    t0 = time.perf_counter()
    eng = mgg.Engine(g, n, part_device, model, ps=args.ps, dist=args.dist, wpb=args.wpb)
    setup_s = time.perf_counter() - t0
    if args.fetch != "auto":
        eng.set_remote_fetch(args.fetch)
    if args.k1_form:
        eng.set_k1_form(args.k1_form)
    if world > 1:
        mdist.exchange_ipc(eng, rank, world)
        dist.barrier()
    eng.set_input(x)
    eng.synchronize()
    ctx = eng.ctx()
    my_part = rank if world > 1 else 0

    for _ in range(max(args.warmup, 3)):
        eng.forward()
    eng.synchronize()
    if world > 1:
        dist.barrier()

    launches0 = eng.stats()["launches"]
    with ClockSampler(local_rank) as clk:
        eng.synchronize()
        if world > 1:
            dist.barrier()
        lib.mgg_event_record(ctx, my_part, 100000)
        for _ in range(args.steps):
            eng.forward()  # CUDA-graph replay on a single-device context
        lib.mgg_event_record(ctx, my_part, 100001)
        clk.sample_now()  # the queued steps are still running
        eng.synchronize()
        if world > 1:
            dist.barrier()
    ms = ctypes.c_float()
    lib.mgg_event_elapsed(ctx, my_part, 100000, 100001, ctypes.byref(ms))
    total_ms = ms.value
    launches = eng.stats()["launches"] - launches0
    # per-op breakdown from a separate profiled pass (events around every op;
    # not a graph replay, not part of the timed region)
    eng.set_profiling(True)
    for _ in range(args.steps):
        eng.forward()
    eng.synchronize()
    ops, nfw = eng.profile()
    eng.set_profiling(False)
    # the first layer's K1 (the roofline's kernel): one launch on its stores,
    # then the library names the kernels it ran (the profiled pass ended on
    # the last layer's, which may differ — e.g. ReLU applied on load)
    eng.time_aggregate(w0, 1, 0)
    kernels = eng.k1_kernels(my_part)
    if world > 1:
        dist.barrier()
        total_ms = mdist.max_over_ranks(total_ms)
    ms_step = total_ms / args.steps
    value = layers * E / (ms_step * 1e-3) / 1e9

    # dominant kernel: the first layer's K1 launch(es)
    st = eng.stats()
    agg = [t for k, w, t in ops if k == "aggregate" and w == w0]
    agg_ms_per_launch = agg[0] / nfw if agg else float("nan")
    my_edges = st["local_edges"] + st["remote_edges"]
    my_parts = st["local_parts"] + st["remote_parts"]
    rows = N if world == 1 else N // world
    total_op_ms = max(sum(t for _, _, t in ops), 1e-9)
    share = sum(t for k, _, t in ops if k == "aggregate") / total_op_ms
    roof = roofline(N, my_edges, my_parts, rows, w0, agg_ms_per_launch, gather_peak,
                    _traffic(args, n, name), kernels)
    roof["share_of_step"] = round(share, 4)
    if world > 1 and st["remote_parts"] > 0:
        pitch0 = (w0 + 3) // 4 * 4
        nvl = (st["halo_rows"] if st.get("halo_rows", 0) else st["remote_edges"]) * pitch0 * 4
        link_roofline(roof, nvl, agg_ms_per_launch, _peaks()[0])

    # remote-access hiding (mirrors the phase-separated
    # decomposition R:proj/src/sim.cpp:127-142, 530-569): K1 of the first
    # aggregation width with only remote partitions (comm), only local ones
    # (compute) and both pipelined in one launch; max over parts
    overlap = None
    if full and st["remote_parts"] > 0:
        fine = not st.get("halo_rows", 0)
        t_pipe = eng.time_aggregate(w0, 5, 0)
        # fine fetch: the local leg of the pipelined kernel itself (phase 3)
        t_loc = eng.time_aggregate(w0, 5, 3 if fine else 1)
        t_rem = eng.time_aggregate(w0, 5, 2)
        if world > 1:
            t_pipe, t_loc, t_rem = (mdist.max_over_ranks(float(t)) for t in
                                    (t_pipe, t_loc, t_rem))
        hidden = max(0.0, t_rem + t_loc - t_pipe)
        overlap = {"k1_pipelined_ns": int(t_pipe), "k1_local_only_ns": int(t_loc),
                   "k1_remote_only_ns": int(t_rem),
                   "hidden_remote_fraction": round(hidden / max(t_rem, 1), 4),
                   "overlap_of_shorter_phase": round(hidden / max(min(t_rem, t_loc), 1), 4),
                   "remote_fetch": "halo" if st.get("halo_rows", 0) else "fine"}

    # peer (NVLink) bytes this rank's aggregations pull per step: fine = one
    # row per remote edge, halo = each distinct remote row once per layer
    link = None
    if st["remote_parts"] > 0:
        halo = st.get("halo_rows", 0) > 0
        rows_pulled = st["halo_rows"] if halo else st["remote_edges"]
        by = sum(rows_pulled * ((w + 3) // 4 * 4) * 4 for w in widths)
        agg_ms = sum(t for k, _, t in ops if k == "aggregate") / max(nfw, 1)
        link = {"remote_bytes_per_step": int(by), "mode": "halo" if halo else "fine",
                "rows_per_layer": int(rows_pulled),
                "achieved_gbs_over_k1_time": round(by / max(agg_ms, 1e-9) / 1e6, 1),
                "peak_gbs": 900.0, "peak_source": "NVLink 5 per direction (north_star)",
                "note": "logical parts on one GPU: the 'peer' is the same HBM"
                        if world == 1 else "per rank; max over ranks of the time"}
        if world > 1:
            link["remote_bytes_per_step_all_ranks"] = int(mdist.sum_over_ranks(float(by)))

    e2e = None
    if full and not args.no_e2e:
        # two pinned input/output buffer pairs, alternated: every step copies
        # its own X in and its own Z out
        xs = [x, mgg.host_alloc((N, model.in_dim))]
        xs[1][:] = x
        zs = [z, mgg.host_alloc((N, model.out_dim))]
        eng.forward_host(x, z)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        eng.forward_host(x, z)
        sync_s = time.perf_counter() - t0
        if world > 1:
            dist.barrier()
        k2 = int(os.environ.get("MGG_E2E_STEPS", max(5, args.steps)))
        t0 = time.perf_counter()
        tickets = [eng.submit_host(xs[i % 2], zs[i % 2]) for i in range(k2)]
        eng.wait(tickets[-1])
        e2e_s = (time.perf_counter() - t0) / k2
        if world > 1:
            e2e_s = mdist.max_over_ranks(e2e_s)
            sync_s = mdist.max_over_ranks(sync_s)
        shard = world if world > 1 else 1
        e2e = {"value": round(layers * E / e2e_s / 1e9, 4), "unit": "GEdges/s",
               "ms_per_step": round(e2e_s * 1e3, 3),
               "h2d_bytes_per_step": int(N * model.in_dim * 4 // shard),
               "d2h_bytes_per_step": int(N * model.out_dim * 4 // shard),
               "steps": k2, "single_forward_ms": round(sync_s * 1e3, 3),
               "api": "mgg_engine_submit_host x K + mgg_engine_wait (pinned host X in, "
                      "Z out per step; H2D/D2H on copy lanes overlap the previous "
                      "step's kernels), host wall clock"}

    cpu = None
    if full and rank == 0 and world == 1 and not args.no_cpu:
        try:
            tc = cpu_forward_time(g.row_ptr, g.col_idx, np.asarray(x), model)
            cpu = {"value": round(layers * E / tc / 1e9, 4), "unit": "GEdges/s",
                   "cores": host_threads(), "kind": "port",
                   "sample": "one full forward of the same workload (oracle.c, fp32 "
                             "accumulate, OpenMP all host threads)",
                   "seconds": round(tc, 3)}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "error": str(ex)[:200]}
    eng.close()
    if rank != 0:
        return None
    return {
        "metric": f"aggregation GEdges/s ({label.split()[0]} forward)",
        "value": round(value, 4), "ms_per_step": round(ms_step, 4),
        "config": workload_config(name, args, N, E, model, n),
        "roofline": roof,
        "ops": [{"kind": k, "width": w, "ms": round(t / nfw, 4)} for k, w, t in ops],
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "overlap": overlap,
        "link": link,
        "clocks": clk.summary(),
        "setup": {"graph_gen_s": round(gen_s, 2), "engine_setup_s": round(setup_s, 2),
                  "plan_build_ms": round(st["plan_build_ns"] / 1e6, 1),
                  "remote_edge_fraction": round(st["remote_edges"] / max(my_edges, 1), 4)},
    }


def locality_csr(n, avg, window, far, seed=0):
    """CSR (row = target) whose neighbours lie within +-window of the target
    except a `far` fraction drawn uniformly — tunes the remote-edge share of
    the 1D split (tools/hiding_b200.py uses the same generator)."""
    rng = np.random.default_rng(seed)
    deg = np.maximum(rng.poisson(avg, n), 1).astype(np.int64)
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(deg)
    e = int(rp[-1])
    tgt = np.repeat(np.arange(n, dtype=np.int64), deg)
    near = np.clip(tgt + rng.integers(-window, window + 1, e), 0, n - 1)
    col = np.where(rng.random(e) < far, rng.integers(0, n, e), near)
    return rp, (np.sort(tgt * n + col) % n).astype(np.uint64)


def slow_peer_hiding(mgg, far=0.002, n=2_000_000, dim=16, reps=5):
    """Remote-latency hiding of the fine-grained pipelined K1 (SURVEY §8d,
    R:PAPER.md:405-419) on one GPU: two logical parts, part 1's shards in
    pinned host memory mapped into the device, so part 0's remote rows cross
    PCIe with microsecond latency (a slower stand-in for an NVLink peer).
    Part 0's K1 timed local-only (its local partitions through the same pair
    kernel), remote-only and pipelined; hidden = (T_rem + T_loc - T_pipe) /
    T_rem. tools/hiding_b200.py sweeps the remote share."""
    rp, cl = locality_csr(n, 25.0, 64, far)
    g = mgg.CsrGraph.from_csr(rp, cl)
    eng = mgg.Engine(g, 2, [0, 0], mgg.make_gcn(dim, 16, 8), ps=16, dist=8, wpb=8)
    try:
        eng.set_remote_fetch("fine")
        eng.set_shard_memory(1, mgg.MEM_HOST_MAPPED)
        t = {ph: eng.time_aggregate_each(dim, reps, ph)[0] for ph in (3, 2, 0)}
        kernels = eng.k1_kernels(0)
        st = eng.stats()
    finally:
        eng.close()
    loc, rem, pipe = t[3], t[2], t[0]
    hid = max(0, rem + loc - pipe)
    fp = mgg.build_flat_plan(g, 2, 0, 16, 8, 8, dim)
    return {"method": "2 logical parts on this GPU, part 1 host-mapped (PCIe peer); part 0's K1 "
                      "local-only / remote-only / pipelined, CUDA events, median of 5",
            "graph": f"locality CSR {n} nodes, avg degree 25, far fraction {far}",
            "remote_edge_fraction": round(fp.remote_cols_len / max(
                fp.local_cols_len + fp.remote_cols_len, 1), 5),
            "k1_local_only_ns": int(loc), "k1_remote_only_ns": int(rem),
            "k1_pipelined_ns": int(pipe),
            "hidden_remote_fraction": round(hid / max(rem, 1), 4),
            "pipelined_vs_max_leg": round(pipe / max(loc, rem, 1), 4),
            "kernel": ";".join(kernels), "remote_parts": int(st["remote_parts"])}


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _reexec_under_torchrun(args)

    import paper_2209_06800_b200 as mgg
    from paper_2209_06800_b200 import dist as mdist
    from paper_2209_06800_b200._lib import lib

    world, rank, local_rank = mdist.env_world()
    # MGG_BENCH_DEVICE pins every rank to one device: validates the multi-rank
    # path (IPC + K3 across processes) on a one-GPU box; never set for numbers
    local_rank = int(os.environ.get("MGG_BENCH_DEVICE", local_rank))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group(backend="cpu:gloo,cuda:nccl")
    if not mgg.cuda_available():
        raise SystemExit("bench.py: no CUDA device visible (the product has no CPU path)")

    main_line = measure(args.workload, args, mgg, lib, mdist, world, rank, local_rank, dist)
    secondary = []
    names = [] if args.secondary in ("", "none") else args.secondary.split(",")
    for name in names:
        if name == args.workload or world > 1:
            continue
        sargs = argparse.Namespace(**vars(args))
        tuned = WORKLOADS[name][3]
        sargs.ps, sargs.dist, sargs.wpb = tuned[:3]
        sargs.k1_form = tuned[3] if len(tuned) > 3 else 0
        sargs.parts = None
        r = measure(name, sargs, mgg, lib, mdist, world, rank, local_rank, dist, full=False)
        if r:
            secondary.append({k: r[k] for k in ("metric", "value", "ms_per_step", "config",
                                                 "roofline", "ops", "gpu_launches", "clocks")}
                             | {"unit": "GEdges/s", "steps": args.steps})
    hiding = None
    if rank == 0 and world == 1 and not args.no_hiding:
        try:
            hiding = slow_peer_hiding(mgg)
        except Exception as ex:  # noqa: BLE001  (a box without mapped host memory)
            hiding = {"error": str(ex)[:200]}
    if rank == 0:
        m = main_line
        line = {
            "metric": m["metric"], "value": m["value"], "unit": "GEdges/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": m["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": m["config"], "roofline": m["roofline"], "ops": m["ops"],
            "cpu_baseline": m["cpu_baseline"], "e2e": m["e2e"],
            "gpu_launches": m["gpu_launches"], "overlap": m["overlap"], "link": m["link"],
            "clocks": m["clocks"],
            "setup": m["setup"], "secondary": secondary, "hiding": hiding,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

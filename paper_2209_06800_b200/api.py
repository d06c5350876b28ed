"""Python mirror of the reference's hot-path API over the C-ABI (libmgg.so).

Names, argument meaning and error behaviour follow the reference library
(R:proj/include/pipeshard/*.hpp): CsrGraph / gen_synthetic / from_edges /
load_edge_list / load_csr, split_by_edges, plan_ne_placement, translate,
memory_footprint, build_launch_plan (device form: build_flat_plan), wpw /
smem / launch_geometry / validate, optimize / exhaustive, and the GCN/GIN
engine that replaces the reference's simulated execution. Errors raise the
same taxonomy (InputError, ParseError, ConfigError, IntegrityError) plus
CudaError.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from ._lib import (AggOpts, ConfigError, CudaError, InputError, IntegrityError,  # noqa: F401
                   MEASURE_FN, ModelDesc, MggError, ParseError, check, lib)

UNIFORM, POWERLAW, RMAT = 0, 1, 2
MEM_DEVICE, MEM_HOST_MAPPED, MEM_MANAGED, MEM_MANAGED_HOST = 0, 1, 2, 3
EQUAL_NODES, FOLLOW_SPLIT = 0, 1
INTERLEAVED, SEGREGATED = 0, 1
PARTITIONED, WHOLE_LIST = 0, 1


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def cuda_available() -> bool:
    return bool(lib.mgg_cuda_available())


# --------------------------------------------------------------------------
# graph (R:proj/include/pipeshard/graph.hpp)


class CsrGraph:
    """Directed CSR owned by the library (row v = target, cols = neighbors)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib.mgg_graph_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _dims(self):
        n, m = C.c_uint64(), C.c_uint64()
        check(lib.mgg_graph_dims(self._h, C.byref(n), C.byref(m)))
        return n.value, m.value

    @property
    def num_nodes(self) -> int:
        return self._dims()[0]

    @property
    def num_edges(self) -> int:
        return self._dims()[1]

    @property
    def row_ptr(self) -> np.ndarray:
        n, _ = self._dims()
        return np.ctypeslib.as_array(lib.mgg_graph_row_ptr(self._h), (n + 1,)).copy()

    @property
    def col_idx(self) -> np.ndarray:
        _, m = self._dims()
        if m == 0:
            return np.zeros(0, np.uint64)
        return np.ctypeslib.as_array(lib.mgg_graph_col_idx(self._h), (m,)).copy()

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def save_csr(self, path: str) -> None:
        check(lib.mgg_graph_save_csr(self._h, path.encode()))

    @staticmethod
    def from_csr(row_ptr, col_idx) -> "CsrGraph":
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        ci = np.ascontiguousarray(col_idx, dtype=np.uint64)
        h = C.c_void_p()
        check(lib.mgg_graph_from_csr(len(rp) - 1, len(ci), _p(rp, C.c_uint64),
                                     _p(ci, C.c_uint64), C.byref(h)))
        return CsrGraph(h)


def from_edges(num_nodes: int, edges) -> CsrGraph:
    e = np.asarray(edges, dtype=np.uint64).reshape(-1, 2)
    src = np.ascontiguousarray(e[:, 0])
    dst = np.ascontiguousarray(e[:, 1])
    h = C.c_void_p()
    check(lib.mgg_graph_from_edges(num_nodes, len(src), _p(src, C.c_uint64),
                                   _p(dst, C.c_uint64), C.byref(h)))
    return CsrGraph(h)


def gen_synthetic(kind: int, num_nodes: int, avg_degree: float, seed: int) -> CsrGraph:
    """kind UNIFORM / POWERLAW: bit-identical to the reference generator."""
    h = C.c_void_p()
    check(lib.mgg_graph_generate(kind, num_nodes, float(avg_degree), seed, C.byref(h)))
    return CsrGraph(h)


def gen_rmat(num_nodes: int, num_edges: int, seed: int) -> CsrGraph:
    h = C.c_void_p()
    check(lib.mgg_graph_generate(RMAT, num_nodes, float(num_edges), seed, C.byref(h)))
    return CsrGraph(h)


def load_edge_list(path: str) -> CsrGraph:
    h = C.c_void_p()
    check(lib.mgg_graph_load_edge_list(path.encode(), C.byref(h)))
    return CsrGraph(h)


def load_csr(path: str) -> CsrGraph:
    h = C.c_void_p()
    check(lib.mgg_graph_load_csr(path.encode(), C.byref(h)))
    return CsrGraph(h)


# --------------------------------------------------------------------------
# placement (R:proj/include/pipeshard/placement.hpp)


def split_by_edges(g: CsrGraph, num_gpus: int) -> np.ndarray:
    out = np.zeros(max(num_gpus - 1, 1), np.uint64)
    check(lib.mgg_split_by_edges(g.handle, num_gpus, _p(out, C.c_uint64)))
    return out[: num_gpus - 1]


def chunk_ranges(g: CsrGraph, num_gpus: int) -> np.ndarray:
    pts = [0] + [int(x) for x in split_by_edges(g, num_gpus)] + [g.num_nodes]
    return np.array([[pts[i], pts[i + 1]] for i in range(num_gpus)], np.uint64)


def plan_ne_placement(g: CsrGraph, num_gpus: int, mode: int, dim: int) -> np.ndarray:
    out = np.zeros(2 * num_gpus, np.uint64)
    check(lib.mgg_plan_ne_placement(g.handle, num_gpus, mode, dim, _p(out, C.c_uint64)))
    return out.reshape(num_gpus, 2)


def translate(g: CsrGraph, num_gpus: int, mode: int, ids) -> tuple[np.ndarray, np.ndarray]:
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    gpu = np.zeros(len(ids), np.uint32)
    off = np.zeros(len(ids), np.uint64)
    check(lib.mgg_translate(g.handle, num_gpus, mode, len(ids), _p(ids, C.c_uint64),
                            _p(gpu, C.c_uint32), _p(off, C.c_uint64)))
    return gpu, off


def memory_footprint(g: CsrGraph, num_gpus: int, mode: int, dim: int,
                     device_mem_bytes: int) -> tuple[np.ndarray, bool]:
    per = np.zeros(2 * num_gpus, np.uint64)
    fits = C.c_int()
    check(lib.mgg_memory_footprint(g.handle, num_gpus, mode, dim, device_mem_bytes,
                                   _p(per, C.c_uint64), C.byref(fits)))
    return per.reshape(num_gpus, 2), bool(fits.value)


# --------------------------------------------------------------------------
# neighbor-partition builder (R:proj/include/pipeshard/workload.hpp)


class FlatPlan:
    """Device-form launch plan of one gpu (see include/mgg/workload.hpp)."""

    def __init__(self, handle):
        self._h = handle
        info = np.zeros(10, np.uint64)
        check(lib.mgg_flat_plan_info(self._h, _p(info, C.c_uint64)))
        (self.n_local, self.n_remote, self.local_cols_len, self.remote_cols_len,
         self.num_warps, self.num_blocks, self.first_target, self.rows,
         self.smem_bytes_per_block, self.launch_smem_bytes) = (int(x) for x in info)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.mgg_flat_plan_destroy(self._h)
            self._h = None

    def meta(self, kind: int) -> np.ndarray:
        n = self.n_local if kind == 0 else self.n_remote
        return np.ctypeslib.as_array(lib.mgg_flat_plan_meta(self._h, kind),
                                     (2 * (n + 1),)).copy().reshape(-1, 2)

    def cols(self, kind: int) -> np.ndarray:
        n = self.local_cols_len if kind == 0 else self.remote_cols_len
        if n == 0:
            return np.zeros(0, np.uint32)
        return np.ctypeslib.as_array(lib.mgg_flat_plan_cols(self._h, kind), (n,)).copy()

    def to_json(self) -> str:
        p = C.c_void_p()
        check(lib.mgg_flat_plan_json(self._h, C.byref(p)))
        try:
            return C.string_at(p).decode()
        finally:
            lib.mgg_free(p)

    def tasks(self):
        total = self.n_local + self.n_remote
        off = np.zeros(self.num_warps + 1, np.uint64)
        kind = np.zeros(max(total, 1), np.uint8)
        idx = np.zeros(max(total, 1), np.uint32)
        check(lib.mgg_flat_plan_tasks(self._h, _p(off, C.c_uint64), _p(kind, C.c_uint8),
                                      _p(idx, C.c_uint32)))
        return off, kind[:total], idx[:total]


def build_flat_plan(g: CsrGraph, num_gpus: int, gpu: int, ps: int, dist: int, wpb: int,
                    dim: int, placement_mode: int = FOLLOW_SPLIT,
                    mapping: int = INTERLEAVED, granularity: int = PARTITIONED) -> FlatPlan:
    h = C.c_void_p()
    check(lib.mgg_flat_plan_build(g.handle, num_gpus, placement_mode, gpu, ps, dist, wpb,
                                  dim, mapping, granularity, C.byref(h)))
    return FlatPlan(h)


# --------------------------------------------------------------------------
# cost model + tuner (R:proj/include/pipeshard/costmodel.hpp, tuner.hpp)


def wpw(ps: int, dist: int, wpb: int, dim: int) -> int:
    return int(lib.mgg_wpw(ps, dist, wpb, dim))


def remote_partition_bytes(part_size: int, dim: int, paged: bool = False,
                           page_bytes: int = 4096) -> int:
    return int(lib.mgg_remote_partition_bytes(part_size, dim, int(paged), page_bytes))


def smem(ps: int, dist: int, wpb: int, dim: int) -> int:
    return int(lib.mgg_smem(ps, dist, wpb, dim))


def launch_geometry(n_local: int, n_remote: int, ps: int, dist: int, wpb: int,
                    profile: str = "a100"):
    wb = np.zeros(2, np.uint64)
    bps = C.c_double()
    check(lib.mgg_launch_geometry(n_local, n_remote, ps, dist, wpb, profile.encode(),
                                  _p(wb, C.c_uint64), C.byref(bps)))
    return int(wb[0]), int(wb[1]), bps.value


@dataclass
class HardwareProfile:
    name: str = "a100"
    num_sms: int = 108
    max_warps_per_sm: int = 64
    smem_per_sm_bytes: int = 164 * 1024
    device_mem_bytes: int = 40 << 30
    page_bytes: int = 4096
    barrier_cycles: int = 64
    latencies: dict = field(default_factory=dict)


def resolve_profile(name_or_path: str) -> HardwareProfile:
    p = C.c_void_p()
    check(lib.mgg_profile_json(name_or_path.encode(), C.byref(p)))
    try:
        j = json.loads(C.string_at(p).decode())
    finally:
        lib.mgg_free(p)
    return HardwareProfile(j["name"], j["numSMs"], j["maxWarpsPerSM"], j["smemPerSMBytes"],
                           j["deviceMemBytes"], j.get("pageBytes", 4096),
                           j.get("barrierCycles", 64), j.get("latencies", {}))


def validate(ps: int, dist: int, wpb: int, dim: int, hw: HardwareProfile) -> list[str]:
    buf = C.create_string_buffer(256)
    n = lib.mgg_validate(ps, dist, wpb, dim, hw.num_sms, hw.max_warps_per_sm,
                         hw.smem_per_sm_bytes, buf, 256)
    return [x for x in buf.value.decode().split(";") if x][:n]


def _measure_cb(fn):
    err_box = {}

    def cb(ps, dist, wpb, _user, err):
        try:
            return int(fn((ps, dist, wpb)))
        except Exception as e:  # noqa: BLE001 - surfaced through the ABI
            err_box["e"] = e
            err[0] = 1
            return 0
    return MEASURE_FN(cb), err_box


def optimize(fn: Callable[[tuple], int], hw: HardwareProfile, dim: int,
             retreat_value_rank: bool = False, max_evaluations: int = 15):
    """Returns (trace [(ps,dist,wpb,cycles)...], best (ps,dist,wpb,cycles))."""
    cb, box = _measure_cb(fn)
    cap = 4096
    trace = np.zeros(4 * cap, np.uint64)
    best = np.zeros(4, np.uint64)
    n = C.c_size_t()
    st = lib.mgg_optimize(cb, None, hw.num_sms, hw.max_warps_per_sm, hw.smem_per_sm_bytes,
                          dim, int(retreat_value_rank), max_evaluations,
                          _p(trace, C.c_uint64), cap, C.byref(n), _p(best, C.c_uint64))
    if st and "e" in box:
        raise RuntimeError(lib.mgg_last_error().decode()) from box["e"]
    check(st)
    t = trace[: 4 * n.value].reshape(-1, 4)
    return [tuple(int(x) for x in r) for r in t], tuple(int(x) for x in best)


def exhaustive(fn: Callable[[tuple], int], hw: HardwareProfile, dim: int):
    cb, box = _measure_cb(fn)
    cap = 1024
    table = np.zeros(4 * cap, np.uint64)
    n = C.c_size_t()
    st = lib.mgg_exhaustive(cb, None, hw.num_sms, hw.max_warps_per_sm, hw.smem_per_sm_bytes,
                            dim, _p(table, C.c_uint64), cap, C.byref(n))
    if st and "e" in box:
        raise RuntimeError(lib.mgg_last_error().decode()) from box["e"]
    check(st)
    return [tuple(int(x) for x in r) for r in table[: 4 * n.value].reshape(-1, 4)]


# --------------------------------------------------------------------------
# models


@dataclass
class Model:
    """GCN (R:PAPER.md:504-508) or GIN (R:PAPER.md:511-517) with packed weights."""
    kind: int  # 0 GCN, 1 GIN
    layers: int
    in_dim: int
    hidden: int
    out_dim: int
    w1: np.ndarray
    b1: np.ndarray | None = None
    w2: np.ndarray | None = None
    b2: np.ndarray | None = None
    eps: float = 0.0
    norm: int = 0  # GCN: 1 = D^-1/2 (A+I) D^-1/2 (oracle norm=1), 0 = the paper's plain sum

    def gin_dims(self) -> list[int]:
        return [self.in_dim] + [self.hidden] * (self.layers - 1) + [self.out_dim]


def _glorot(rng: np.random.Generator, fan_in: int, fan_out: int) -> np.ndarray:
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, size=(fan_in, fan_out)).astype(np.float32)


def make_gcn(in_dim: int, hidden: int, classes: int, seed: int = 2, norm: bool = False) -> Model:
    rng = np.random.default_rng(seed)
    w = np.concatenate([_glorot(rng, in_dim, hidden).ravel(),
                        _glorot(rng, hidden, classes).ravel()])
    return Model(0, 2, in_dim, hidden, classes, w.astype(np.float32), norm=int(norm))


def make_gin(in_dim: int, hidden: int, classes: int, layers: int = 5, seed: int = 2,
             eps: float = 0.0) -> Model:
    rng = np.random.default_rng(seed)
    dims = [in_dim] + [hidden] * (layers - 1) + [classes]
    w1, b1, w2, b2 = [], [], [], []
    for l in range(layers):
        w1.append(_glorot(rng, dims[l], hidden).ravel())
        b1.append(rng.uniform(-0.1, 0.1, hidden).astype(np.float32))
        w2.append(_glorot(rng, hidden, dims[l + 1]).ravel())
        b2.append(rng.uniform(-0.1, 0.1, dims[l + 1]).astype(np.float32))
    cat = lambda xs: np.ascontiguousarray(np.concatenate(xs), np.float32)  # noqa: E731
    return Model(1, layers, in_dim, hidden, classes, cat(w1), cat(b1), cat(w2), cat(b2), eps)


def random_features(n: int, d: int, seed: int = 1) -> np.ndarray:
    """X ~ U[-1, 1) fp32 (SURVEY §8d synthetic inputs)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, d)).astype(np.float32)


class Engine:
    """The multi-GPU forward driver (include/mgg/engine.hpp) over the C-ABI."""

    def __init__(self, g: CsrGraph, num_parts: int, part_device: Sequence[int],
                 model: Model, ps: int = 16, dist: int = 1, wpb: int = 4):
        self.graph = g  # keep alive: the engine reads it when re-planning
        self.model = model
        self.num_parts = num_parts
        self._keep = [np.ascontiguousarray(x, np.float32) if x is not None else None
                      for x in (model.w1, model.b1, model.w2, model.b2)]
        f = C.POINTER(C.c_float)
        arg = [x.ctypes.data_as(f) if x is not None else None for x in self._keep]
        desc = ModelDesc(model.kind, model.layers, model.in_dim, model.hidden,
                         model.out_dim, model.eps, *arg, getattr(model, "norm", 0))
        dev = np.ascontiguousarray(part_device, np.int32)
        self._h = C.c_void_p()
        check(lib.mgg_engine_create(g.handle, num_parts, _p(dev, C.c_int32), ps, dist, wpb,
                                    C.byref(desc), C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib.mgg_engine_destroy(self._h)
            self._h = None

    __del__ = close

    def ipc_export(self, part: int) -> bytes:
        n = C.c_size_t(0)
        check(lib.mgg_engine_ipc_export(self._h, part, None, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(lib.mgg_engine_ipc_export(self._h, part, buf, C.byref(n)))
        return bytes(buf)

    def ipc_import(self, part: int, blob: bytes) -> None:
        b = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(lib.mgg_engine_ipc_import(self._h, part, b, len(blob)))

    def vmm_ipc(self) -> bool:
        """True when the stores are cross-process symmetric VMM ranges (MGG_VMM_IPC=1)."""
        on = C.c_int(0)
        check(lib.mgg_engine_vmm_ipc(self._h, C.byref(on)))
        return bool(on.value)

    def vmm_export(self, part: int) -> list[int]:
        """One POSIX fd per store of local part `part` (caller closes them)."""
        n = C.c_size_t(0)
        check(lib.mgg_engine_vmm_export(self._h, part, None, C.byref(n)))
        buf = (C.c_int * n.value)()
        check(lib.mgg_engine_vmm_export(self._h, part, buf, C.byref(n)))
        return list(buf)

    def vmm_import(self, part: int, fds: list[int]) -> None:
        buf = (C.c_int * len(fds))(*fds)
        check(lib.mgg_engine_vmm_import(self._h, part, buf, len(fds)))

    def set_config(self, ps: int, dist: int, wpb: int) -> None:
        check(lib.mgg_engine_set_config(self._h, ps, dist, wpb))

    FETCH = {"auto": 0, "fine": 1, "halo": 2}

    def set_remote_fetch(self, mode: str = "auto") -> None:
        check(lib.mgg_engine_set_remote_fetch(self._h, self.FETCH[mode]))

    def set_mapping(self, mapping: int = INTERLEAVED, granularity: int = PARTITIONED) -> None:
        check(lib.mgg_engine_set_mapping(self._h, mapping, granularity))

    def set_input(self, x: np.ndarray) -> None:
        assert x.dtype == np.float32 and x.flags.c_contiguous
        check(lib.mgg_engine_set_input(self._h, _p(x, C.c_float)))

    def forward(self) -> None:
        check(lib.mgg_engine_forward(self._h))

    def set_k1_form(self, form: int) -> None:
        """Local-only K1 form: 0 by the plan's shape, 1 warp-window, 2 group (8 rows
        in flight per group), 3 group (4) — mgg_engine_set_k1_form."""
        check(lib.mgg_engine_set_k1_form(self._h, form))

    def set_graphs(self, on: bool) -> None:
        """CUDA-graph replay of forward() on single-device contexts (default on)."""
        check(lib.mgg_engine_set_graphs(self._h, int(on)))

    def synchronize(self) -> None:
        check(lib.mgg_ctx_synchronize(lib.mgg_engine_ctx(self._h)))

    def get_output(self, z: np.ndarray | None = None) -> np.ndarray:
        if z is None:
            z = np.zeros((self.graph.num_nodes, self.model.out_dim), np.float32)
        check(lib.mgg_engine_get_output(self._h, _p(z, C.c_float)))
        return z

    def forward_host(self, x: np.ndarray, z: np.ndarray) -> np.ndarray:
        check(lib.mgg_engine_forward_host(self._h, _p(x, C.c_float), _p(z, C.c_float)))
        return z

    def submit_host(self, x: np.ndarray, z: np.ndarray) -> int:
        """Streamed forward (mgg_engine_submit_host): returns a ticket at once;
        keep x alive and z untouched until wait(ticket)."""
        assert x.dtype == np.float32 and x.flags.c_contiguous
        assert z.dtype == np.float32 and z.flags.c_contiguous
        t = C.c_uint64()
        check(lib.mgg_engine_submit_host(self._h, _p(x, C.c_float), _p(z, C.c_float),
                                         C.byref(t)))
        return t.value

    def wait(self, ticket: int) -> None:
        check(lib.mgg_engine_wait(self._h, ticket))

    def get_hidden(self, which: int) -> np.ndarray:
        w = C.c_uint32()
        check(lib.mgg_engine_get_hidden(self._h, which, None, C.byref(w)))
        out = np.zeros((self.graph.num_nodes, w.value), np.float32)
        check(lib.mgg_engine_get_hidden(self._h, which, _p(out, C.c_float), C.byref(w)))
        return out

    def aggregate(self, x: np.ndarray, self_scale: float = 1.0, relu_in: bool = False,
                  phase: int = 0):
        """out = self_scale*f(x) + sum of f(x_u); phase 1/2 = local/remote partitions only."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        if phase:
            check(lib.mgg_engine_aggregate_phase_host(self._h, _p(x, C.c_float), x.shape[1],
                                                      self_scale, int(relu_in), phase,
                                                      _p(out, C.c_float)))
        else:
            check(lib.mgg_engine_aggregate_host(self._h, _p(x, C.c_float), x.shape[1],
                                                self_scale, int(relu_in), _p(out, C.c_float)))
        return out

    def time_aggregate(self, dim: int, reps: int = 5, phase: int = 0) -> int:
        ns = C.c_uint64()
        check(lib.mgg_engine_time_aggregate(self._h, dim, reps, phase, C.byref(ns)))
        return ns.value

    def get_logits(self) -> np.ndarray:
        """Pre-softmax logits of the last forward (the engine's head K2, no
        softmax epilogue), N x out_dim."""
        z = np.zeros((self.graph.num_nodes, self.model.out_dim), np.float32)
        check(lib.mgg_engine_get_logits(self._h, _p(z, C.c_float)))
        return z

    def time_aggregate_each(self, dim: int, reps: int = 5, phase: int = 0) -> list[int]:
        """Median K1 ns per part, each part alone (0 for remote parts)."""
        ns = np.zeros(self.num_parts, np.uint64)
        check(lib.mgg_engine_time_aggregate_each(self._h, dim, reps, phase, _p(ns, C.c_uint64)))
        return [int(v) for v in ns]

    def measure_multi_gpu(self, dim: int, reps: int = 5) -> dict:
        """Measured MultiGpuReport (R:proj/include/pipeshard/sim.hpp:115-123):
        every local part's K1 concurrently; see mgg_engine_measure_multi_gpu."""
        n = self.num_parts
        summ = np.zeros(6, np.uint64)
        pp = np.zeros(9 * n, np.uint64)
        pf = np.zeros(2 * n, np.float64)
        check(lib.mgg_engine_measure_multi_gpu(self._h, dim, reps, _p(summ, C.c_uint64),
                                               _p(pp, C.c_uint64),
                                               pf.ctypes.data_as(C.POINTER(C.c_double))))
        keys = ["local", "total_ns", "alone_ns", "remote_bytes", "local_bytes", "num_warps",
                "num_blocks", "active_sms", "part"]
        per = []
        for p in range(n):
            row = {k: int(v) for k, v in zip(keys, pp[9 * p: 9 * p + 9])}
            if not row.pop("local"):
                continue
            row["achieved_occupancy"] = float(pf[2 * p])
            row["sm_utilization"] = float(pf[2 * p + 1])
            per.append(row)
        return {"per_gpu": per, "max_gpu_ns": int(summ[0]), "barrier_ns": int(summ[1]),
                "total_ns": int(summ[2]), "remote_bytes": int(summ[3]),
                "max_alone_ns": int(summ[4]), "devices": int(summ[5]),
                # the per-GPU time: logical parts sharing one device are timed
                # alone (their concurrent run is contention no 8-GPU box has)
                "per_gpu_ns": int(summ[4]) if int(summ[5]) == 1 and len(per) > 1
                else int(summ[2]),
                "mean_occupancy": float(np.mean([r["achieved_occupancy"] for r in per])),
                "mean_utilization": float(np.mean([r["sm_utilization"] for r in per]))}

    def set_shard_memory(self, part: int, kind: int) -> None:
        """MEM_DEVICE / MEM_HOST_MAPPED / MEM_MANAGED / MEM_MANAGED_HOST for part
        `part`'s shards (re-creates the stores: set_input again)."""
        check(lib.mgg_engine_set_shard_memory(self._h, part, kind))

    def trace_csv(self, dim: int, capacity: int = 1 << 20, warp_limit: int = 0xFFFFFFFF) -> str:
        """Device event trace of one K1 at width `dim` (mgg_engine_trace_csv):
        the reference's "gpu,cycle,sm,warp,stage,event" CSV."""
        out = C.c_void_p()
        check(lib.mgg_engine_trace_csv(self._h, dim, capacity, warp_limit, C.byref(out)))
        try:
            return C.string_at(out.value).decode()
        finally:
            lib.mgg_free(out)

    def set_profiling(self, on: bool) -> None:
        check(lib.mgg_engine_set_profiling(self._h, int(on)))

    OP_KINDS = ("dense", "init", "aggregate", "barrier", "softmax", "dense_chain")

    def profile(self):
        """[(kind, width, accumulated ms)] per program op, and #forwards."""
        cap = 256
        ms = np.zeros(cap, np.float64)
        kind = np.zeros(cap, np.uint32)
        width = np.zeros(cap, np.uint32)
        n = C.c_size_t()
        fw = C.c_uint64()
        check(lib.mgg_engine_profile(self._h, _p(ms, C.c_double), _p(kind, C.c_uint32),
                                     _p(width, C.c_uint32), cap, C.byref(n), C.byref(fw)))
        ops = [(self.OP_KINDS[int(kind[i])], int(width[i]), float(ms[i]))
               for i in range(n.value)]
        return ops, fw.value

    def ctx(self):
        return lib.mgg_engine_ctx(self._h)

    def stats(self) -> dict:
        s = np.zeros(10, np.uint64)
        check(lib.mgg_engine_stats(self._h, _p(s, C.c_uint64)))
        keys = ["local_parts", "remote_parts", "local_edges", "remote_edges", "warps",
                "blocks", "launches", "plan_build_ns", "halo_rows", "halo_parts"]
        return {k: int(v) for k, v in zip(keys, s)}

    def k1_kernels(self, part: int = 0) -> list[str]:
        """Kernels the latest K1 of local part `part` launched (demangled)."""
        buf = C.create_string_buffer(1024)
        check(lib.mgg_engine_k1_kernels(self._h, part, buf, len(buf)))
        return [k for k in buf.value.decode().split(";") if k]


def host_alloc(shape, dtype=np.float32) -> np.ndarray:
    """Pinned host array (cudaHostAlloc) for full-speed H2D/D2H. The block is
    kept for the life of the process (bench/e2e buffers are few and large)."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = C.c_void_p()
    check(lib.mgg_host_alloc(nbytes, C.byref(p)))
    _PINNED.append(p)
    buf = (C.c_uint8 * nbytes).from_address(p.value)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


_PINNED: list = []

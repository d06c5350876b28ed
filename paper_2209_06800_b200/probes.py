"""K5 hardware probes (include/mgg.h mgg_probe_*): the measured ceilings the
aggregation kernel is judged against and the b200 cost-model profile is
re-fitted from."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib


class _Ctx:
    """Probe context: part i on devices[i] (peer access enabled between them)."""

    def __init__(self, device: int = 0, devices=None):
        self.h = C.c_void_p()
        devs = list(devices) if devices is not None else [device]
        dev = np.array(devs, np.int32)
        check(lib.mgg_ctx_create(len(devs), dev.ctypes.data_as(C.POINTER(C.c_int32)),
                                 C.byref(self.h)))
        self.bufs = []

    def buf(self, arr: np.ndarray, part: int = 0):
        b = C.c_void_p()
        arr = np.ascontiguousarray(arr)
        check(lib.mgg_dbuf_create(self.h, part, arr.ctypes.data, arr.nbytes, C.byref(b)))
        self.bufs.append(b)
        return lib.mgg_dbuf_ptr(b)

    def close(self):
        for b in self.bufs:
            lib.mgg_dbuf_destroy(b)
        lib.mgg_ctx_destroy(self.h)


def gather_gbps(rows: int, dim: int, n_idx: int, device: int = 0, reps: int = 5,
                seed: int = 0) -> float:
    """Sustained GB/s of gathering n_idx uniformly random rows (dim fp32,
    pitch rounded to 4) from a rows x dim table — the K1 gather ceiling."""
    pitch = (dim + 3) // 4 * 4
    rng = np.random.default_rng(seed)
    ctx = _Ctx(device)
    try:
        table = ctx.buf(rng.uniform(-1, 1, (rows, pitch)).astype(np.float32))
        idx = ctx.buf(rng.integers(0, rows, n_idx, dtype=np.uint32))
        g = C.c_double()
        check(lib.mgg_probe_gather(ctx.h, 0, table, pitch, idx, n_idx, reps, C.byref(g)))
        return g.value
    finally:
        ctx.close()


def chase_ns(nbytes: int, device: int = 0, steps: int = 20000, seed: int = 0) -> float:
    """Dependent-load latency (ns) over a random cycle spanning nbytes."""
    n = max(nbytes // 128, 2)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n).astype(np.uint64)
    nxt = np.zeros(n * 32, np.uint32)  # one pointer per 128-B line
    order = perm * 32
    nxt[order] = np.roll(order, -1)
    ctx = _Ctx(device)
    try:
        p = ctx.buf(nxt)
        ns = C.c_double()
        check(lib.mgg_probe_chase(ctx.h, 0, p, steps, C.byref(ns)))
        return ns.value
    finally:
        ctx.close()


def host_gather_gbps(rows: int, dim: int, n_idx: int, device: int = 0, reps: int = 3,
                     seed: int = 0) -> float:
    """gather_gbps with the table in pinned host memory read in place over
    PCIe (MGG_MEM_HOST_MAPPED shards): the ceiling of a host-mapped "peer"."""
    from .api import host_alloc
    pitch = (dim + 3) // 4 * 4
    rng = np.random.default_rng(seed)
    table = host_alloc((rows, pitch))
    table[:] = rng.uniform(-1, 1, (rows, pitch)).astype(np.float32)
    ctx = _Ctx(device)
    try:
        idx = ctx.buf(rng.integers(0, rows, n_idx, dtype=np.uint32))
        g = C.c_double()
        check(lib.mgg_probe_gather(ctx.h, 0, table.ctypes.data, pitch, idx, n_idx, reps,
                                   C.byref(g)))
        return g.value
    finally:
        ctx.close()


def host_chase_ns(nbytes: int, device: int = 0, steps: int = 2000, seed: int = 0) -> float:
    """chase_ns over pinned host memory: the dependent-load latency of a
    host-mapped "peer" row (one PCIe round trip per load)."""
    from .api import host_alloc
    n = max(nbytes // 128, 2)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n).astype(np.uint64)
    nxt = host_alloc((n * 32,), np.uint32)
    nxt[:] = 0
    order = perm * 32
    nxt[order] = np.roll(order, -1)
    ctx = _Ctx(device)
    try:
        ns = C.c_double()
        check(lib.mgg_probe_chase(ctx.h, 0, nxt.ctypes.data, steps, C.byref(ns)))
        return ns.value
    finally:
        ctx.close()


def device_count() -> int:
    return int(lib.mgg_device_count())


def peer_gather_gbps(reader: int, owner: int, rows: int, dim: int, n_idx: int, reps: int = 3,
                     seed: int = 0) -> float:
    """Rows gathered by device `reader` from a table in device `owner`'s HBM
    over NVLink (peer access; the K1 fine-fetch path)."""
    pitch = (dim + 3) // 4 * 4
    rng = np.random.default_rng(seed)
    ctx = _Ctx(devices=[reader, owner])
    try:
        table = ctx.buf(rng.uniform(-1, 1, (rows, pitch)).astype(np.float32), part=1)
        idx = ctx.buf(rng.integers(0, rows, n_idx, dtype=np.uint32), part=0)
        g = C.c_double()
        check(lib.mgg_probe_gather(ctx.h, 0, table, pitch, idx, n_idx, reps, C.byref(g)))
        return g.value
    finally:
        ctx.close()


def peer_chase_ns(reader: int, owner: int, nbytes: int = 256 << 20, steps: int = 5000,
                  seed: int = 0) -> float:
    """Dependent-load latency of device `reader` reading `owner`'s HBM."""
    n = max(nbytes // 128, 2)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n).astype(np.uint64)
    nxt = np.zeros(n * 32, np.uint32)
    order = perm * 32
    nxt[order] = np.roll(order, -1)
    ctx = _Ctx(devices=[reader, owner])
    try:
        p = ctx.buf(nxt, part=1)
        ns = C.c_double()
        check(lib.mgg_probe_chase(ctx.h, 0, p, steps, C.byref(ns)))
        return ns.value
    finally:
        ctx.close()


def refit_latencies(m: dict, sm_ghz: float, num_sms: int) -> dict:
    """The b200 LatencyModel (R:proj/include/pipeshard/costmodel.hpp:32-49)
    from measured numbers: bases = dependent-load latency x SM clock; the
    per-element costs = SM cycles per fp32 element at the measured per-SM
    share of the gather bandwidth (the schema stores integers: >= 1).
    m: local_chase_ns, local_gather_gbps, and (>= 2 GPUs) peer_chase_ns,
    peer_gather_gbps. Returns {latencies, source}."""
    def per_elem(gbps):
        bytes_per_cycle = gbps / num_sms / sm_ghz  # per SM
        return max(1, int(round(4.0 / bytes_per_cycle)))
    lat = {"localLoadBase": int(round(m["local_chase_ns"] * sm_ghz)),
           "perElemLocal": per_elem(m["local_gather_gbps"]), "perElemCompute": 1}
    src = {"localLoadBase": f"K5 chase probe: {m['local_chase_ns']:.1f} ns dependent HBM load "
                            f"x {sm_ghz:.3f} GHz",
           "perElemLocal": f"K5 gather probe {m['local_gather_gbps']:.0f} GB/s over {num_sms} SMs"}
    if "peer_chase_ns" in m:
        lat["remoteGetBase"] = int(round(m["peer_chase_ns"] * sm_ghz))
        lat["perElemRemote"] = per_elem(m["peer_gather_gbps"])
        src["remoteGetBase"] = (f"K5 peer chase probe: {m['peer_chase_ns']:.1f} ns dependent "
                                f"NVLink load x {sm_ghz:.3f} GHz")
        src["perElemRemote"] = f"K5 peer gather probe {m['peer_gather_gbps']:.0f} GB/s"
    return {"latencies": lat, "source": src}

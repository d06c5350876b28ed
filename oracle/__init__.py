"""TEST INFRASTRUCTURE ONLY — the parity oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package, and only as the checker or
the timed CPU baseline; the product (paper_2209_06800_b200/) never does.

* `ref`    — the UNMODIFIED reference library (pipeshard) compiled from
             /root/reference/proj/src into oracle/_ref/libpipeshard_ref.so by
             oracle/Makefile, behind the flat C shim oracle/ref_shim.cpp.
             Pins partition metadata bit-for-bit.
* `orc`    — oracle.c: a plain-C restatement of the metadata rules (pinned
             against `ref` and the reference's own known-answer tests) and of
             the GCN/GIN layer forward from the paper's equations
             (PARITY UNPINNED by reference code — the reference stores no
             embedding values; see oracle.h).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpipeshard_ref.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _load(path):
    if not os.path.exists(path):
        raise ImportError(f"{path} missing — run `make -C oracle` (build() does it)")
    return C.CDLL(path)


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


# ----------------------------------------------------------------------------
# oracle.c

_orc = None


def orc():
    global _orc
    if _orc is None:
        L = _load(ORACLE_SO)
        U32, U64, I, D = C.c_uint32, C.c_uint64, C.c_int, C.c_double
        _sig(L, "orc_split_points", None, U64, u64p, U32, u64p)
        _sig(L, "orc_placement", None, U64, u64p, U32, I, u64p)
        _sig(L, "orc_translate", None, U32, u64p, U64, u32p, u64p)
        _sig(L, "orc_partition_counts", None, U64, u64p, u64p, U32, u64p, u64p, U32, U32, u64p)
        _sig(L, "orc_warp_tasks", U32, U64, U64, U32, U64, u8p, u32p)
        _sig(L, "orc_aggregate", None, I, I, U64, u64p, u64p, f32p, U32, D, I, I, U64, U64, f32p)
        _sig(L, "orc_dense", None, I, I, U64, f32p, U32, f32p, f32p, U32, I, f32p)
        _sig(L, "orc_gcn2_forward", None, I, I, U64, u64p, u64p, f32p, U32, f32p, U32, f32p,
             U32, I, f32p, f32p, f32p)
        _sig(L, "orc_gin_forward", None, I, I, U64, u64p, u64p, f32p, U32, u32p, U32, f32p,
             f32p, f32p, f32p, D, f32p, f32p)
        _sig(L, "orc_gen_synthetic", U64, I, U64, D, U64, u64p, u64p)
        _sig(L, "orc_gen_rmat", None, U64, U64, U64, D, D, D, u64p, u64p)
        _orc = L
    return _orc


def split_points(row_ptr: np.ndarray, num_gpus: int) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    out = np.zeros(max(num_gpus - 1, 1), np.uint64)
    orc().orc_split_points(len(rp) - 1, _p(rp, C.c_uint64), num_gpus, _p(out, C.c_uint64))
    return out[: num_gpus - 1]


def placement(row_ptr, num_gpus: int, mode: int) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    out = np.zeros(2 * num_gpus, np.uint64)
    orc().orc_placement(len(rp) - 1, _p(rp, C.c_uint64), num_gpus, mode, _p(out, C.c_uint64))
    return out.reshape(-1, 2)


def partition_counts(row_ptr, col, num_gpus, ranges, chunk, gpu, ps):
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    cl = np.ascontiguousarray(col, np.uint64)
    rg = np.ascontiguousarray(ranges, np.uint64).ravel()
    ch = np.ascontiguousarray(chunk, np.uint64)
    out = np.zeros(4, np.uint64)
    orc().orc_partition_counts(len(rp) - 1, _p(rp, C.c_uint64), _p(cl, C.c_uint64), num_gpus,
                               _p(rg, C.c_uint64), _p(ch, C.c_uint64), gpu, ps,
                               _p(out, C.c_uint64))
    return [int(x) for x in out]


def warp_tasks(n_local, n_remote, dist, w):
    k = np.zeros(2 * dist, np.uint8)
    i = np.zeros(2 * dist, np.uint32)
    n = orc().orc_warp_tasks(n_local, n_remote, dist, w, _p(k, C.c_uint8), _p(i, C.c_uint32))
    return list(zip(k[:n].tolist(), i[:n].tolist()))


def aggregate(row_ptr, col, x, self_scale=1.0, norm=0, relu_in=False, acc64=True,
              threads=0, rows=None):
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    cl = np.ascontiguousarray(col, np.uint64)
    x = np.ascontiguousarray(x, np.float32)
    n = len(rp) - 1
    lo, hi = rows if rows is not None else (0, n)
    out = np.zeros((hi - lo, x.shape[1]), np.float32)
    orc().orc_aggregate(int(acc64), threads, n, _p(rp, C.c_uint64), _p(cl, C.c_uint64),
                        _p(x, C.c_float), x.shape[1], self_scale, norm, int(relu_in), lo, hi,
                        _p(out, C.c_float))
    return out


def dense(x, w, b=None, act=0, acc64=True, threads=0):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    y = np.zeros((x.shape[0], w.shape[1]), np.float32)
    bb = np.ascontiguousarray(b, np.float32) if b is not None else None
    orc().orc_dense(int(acc64), threads, x.shape[0], _p(x, C.c_float), x.shape[1],
                    _p(w, C.c_float), _p(bb, C.c_float) if bb is not None else None,
                    w.shape[1], act, _p(y, C.c_float))
    return y


def gcn2_forward(row_ptr, col, x, model, norm=0, acc64=True, threads=0):
    """Returns (h1 post-ReLU, logits, z)."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    cl = np.ascontiguousarray(col, np.uint64)
    x = np.ascontiguousarray(x, np.float32)
    n, d = x.shape
    h, c = model.hidden, model.out_dim
    w1 = np.ascontiguousarray(model.w1[: d * h], np.float32)
    w2 = np.ascontiguousarray(model.w1[d * h: d * h + h * c], np.float32)
    h1 = np.zeros((n, h), np.float32)
    lg = np.zeros((n, c), np.float32)
    z = np.zeros((n, c), np.float32)
    orc().orc_gcn2_forward(int(acc64), threads, n, _p(rp, C.c_uint64), _p(cl, C.c_uint64),
                           _p(x, C.c_float), d, _p(w1, C.c_float), h, _p(w2, C.c_float), c,
                           norm, _p(h1, C.c_float), _p(lg, C.c_float), _p(z, C.c_float))
    return h1, lg, z


def gin_forward(row_ptr, col, x, model, acc64=True, threads=0):
    """Returns (logits, z)."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    cl = np.ascontiguousarray(col, np.uint64)
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    dims = np.ascontiguousarray(model.gin_dims(), np.uint32)
    c = model.out_dim
    lg = np.zeros((n, c), np.float32)
    z = np.zeros((n, c), np.float32)
    arrs = [np.ascontiguousarray(a, np.float32) for a in (model.w1, model.b1, model.w2, model.b2)]
    orc().orc_gin_forward(int(acc64), threads, n, _p(rp, C.c_uint64), _p(cl, C.c_uint64),
                          _p(x, C.c_float), model.layers, _p(dims, C.c_uint32), model.hidden,
                          *[_p(a, C.c_float) for a in arrs], model.eps, _p(lg, C.c_float),
                          _p(z, C.c_float))
    return lg, z


def gen_synthetic(kind, n, avg, seed):
    """R:proj/src/graph.cpp:139-176 restated (kind 0 uniform, 1 powerlaw):
    (row_ptr u64[n+1], col u64[E]) — bench.py's reference arm builds its
    input with this (or the reference library itself), never the product."""
    L = orc()
    e = L.orc_gen_synthetic(kind, n, float(avg), seed, None, None)
    rp = np.zeros(n + 1, np.uint64)
    cl = np.zeros(max(e, 1), np.uint64)
    L.orc_gen_synthetic(kind, n, float(avg), seed, _p(rp, C.c_uint64), _p(cl, C.c_uint64))
    return rp, cl[:e]


def gen_rmat(n, m, seed, a=0.57, b=0.19, c=0.19):
    """The RMAT input of bench/tests as plain C (see oracle.c): CSR arrays."""
    rp = np.zeros(n + 1, np.uint64)
    cl = np.zeros(max(m, 1), np.uint64)
    orc().orc_gen_rmat(n, m, seed, a, b, c, _p(rp, C.c_uint64), _p(cl, C.c_uint64))
    return rp, cl[:m]


# ----------------------------------------------------------------------------
# reference library (oracle/_ref)

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = _load(REF_SO)
        U32, U64, I, D, SZ = C.c_uint32, C.c_uint64, C.c_int, C.c_double, C.c_size_t
        PP = C.POINTER(C.c_void_p)
        _sig(L, "ref_last_error", C.c_char_p)
        _sig(L, "ref_graph_free", None, C.c_void_p)
        _sig(L, "ref_graph_gen", I, I, U64, D, U64, PP)
        _sig(L, "ref_graph_from_edges", I, U64, U64, u64p, u64p, PP)
        _sig(L, "ref_graph_from_csr", I, U64, U64, u64p, u64p, PP)
        _sig(L, "ref_graph_dims", None, C.c_void_p, u64p, u64p)
        _sig(L, "ref_graph_copy", None, C.c_void_p, u64p, u64p)
        _sig(L, "ref_split", I, C.c_void_p, U32, u64p)
        _sig(L, "ref_placement", I, C.c_void_p, U32, I, U64, u64p)
        _sig(L, "ref_translate", I, C.c_void_p, U32, I, U64, u64p, u32p, u64p)
        _sig(L, "ref_footprint", I, C.c_void_p, U32, I, U64, U64, u64p, C.POINTER(I))
        _sig(L, "ref_lr_split", I, C.c_void_p, U32, I, U32, u64p, u64p, u64p, u64p, u64p)
        _sig(L, "ref_plan_build", I, C.c_void_p, U32, I, U32, U32, U32, U32, U64, I, I, PP)
        _sig(L, "ref_plan_free", None, C.c_void_p)
        _sig(L, "ref_plan_counts", None, C.c_void_p, u64p)
        _sig(L, "ref_plan_parts", None, C.c_void_p, I, u64p, u64p, u64p)
        _sig(L, "ref_plan_warps", None, C.c_void_p, u64p, u32p, u8p, u32p, u32p, u32p)
        _sig(L, "ref_plan_json", C.c_char_p, C.c_void_p)
        _sig(L, "ref_wpw", U64, U32, U32, U32, U64)
        _sig(L, "ref_smem", U64, U32, U32, U32, U64)
        _sig(L, "ref_launch_geometry", I, U64, U64, U32, U32, U32, C.c_char_p, u64p,
             C.POINTER(D))
        _sig(L, "ref_validate", I, U32, U32, U32, U64, U32, U32, U64, C.c_char_p, SZ)
        MF = C.CFUNCTYPE(U64, U32, U32, U32, C.c_void_p)
        L.MEASURE = MF
        _sig(L, "ref_optimize", I, MF, C.c_void_p, U32, U32, U64, U64, I, U64, u64p, SZ,
             C.POINTER(SZ), u64p)
        _sig(L, "ref_exhaustive", I, MF, C.c_void_p, U32, U32, U64, U64, u64p, SZ,
             C.POINTER(SZ))
        _sig(L, "ref_multi_gpu_cycles", I, C.c_void_p, U32, U32, U32, U32, U64, C.c_char_p,
             u64p)
        _sig(L, "ref_time_metadata", I, C.c_void_p, U32, U32, U32, U32, U64, C.POINTER(D),
             u64p)
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _rchk(st):
    if st:
        raise RefError(st, ref().ref_last_error().decode())


class RefGraph:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_graph_free(self.h)
            self.h = None

    @staticmethod
    def gen(kind, n, avg, seed):
        h = C.c_void_p()
        _rchk(ref().ref_graph_gen(kind, n, float(avg), seed, C.byref(h)))
        return RefGraph(h)

    @staticmethod
    def from_edges(n, edges):
        e = np.asarray(edges, np.uint64).reshape(-1, 2)
        s, d = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
        h = C.c_void_p()
        _rchk(ref().ref_graph_from_edges(n, len(s), _p(s, C.c_uint64), _p(d, C.c_uint64),
                                         C.byref(h)))
        return RefGraph(h)

    @staticmethod
    def from_csr(row_ptr, col):
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        cl = np.ascontiguousarray(col, np.uint64)
        h = C.c_void_p()
        _rchk(ref().ref_graph_from_csr(len(rp) - 1, len(cl), _p(rp, C.c_uint64),
                                       _p(cl, C.c_uint64), C.byref(h)))
        return RefGraph(h)

    def csr(self):
        n, m = C.c_uint64(), C.c_uint64()
        ref().ref_graph_dims(self.h, C.byref(n), C.byref(m))
        rp = np.zeros(n.value + 1, np.uint64)
        cl = np.zeros(max(m.value, 1), np.uint64)
        ref().ref_graph_copy(self.h, _p(rp, C.c_uint64), _p(cl, C.c_uint64))
        return rp, cl[: m.value]

    def split(self, num_gpus):
        out = np.zeros(max(num_gpus - 1, 1), np.uint64)
        _rchk(ref().ref_split(self.h, num_gpus, _p(out, C.c_uint64)))
        return out[: num_gpus - 1]

    def placement(self, num_gpus, mode, dim=4):
        out = np.zeros(2 * num_gpus, np.uint64)
        _rchk(ref().ref_placement(self.h, num_gpus, mode, dim, _p(out, C.c_uint64)))
        return out.reshape(-1, 2)

    def translate(self, num_gpus, mode, ids):
        ids = np.ascontiguousarray(ids, np.uint64)
        g = np.zeros(len(ids), np.uint32)
        o = np.zeros(len(ids), np.uint64)
        _rchk(ref().ref_translate(self.h, num_gpus, mode, len(ids), _p(ids, C.c_uint64),
                                  _p(g, C.c_uint32), _p(o, C.c_uint64)))
        return g, o

    def footprint(self, num_gpus, mode, dim, device_mem):
        per = np.zeros(2 * num_gpus, np.uint64)
        fits = C.c_int()
        _rchk(ref().ref_footprint(self.h, num_gpus, mode, dim, device_mem,
                                  _p(per, C.c_uint64), C.byref(fits)))
        return per.reshape(-1, 2), bool(fits.value)

    def lr_split(self, num_gpus, mode, gpu):
        sz = np.zeros(4, np.uint64)
        _rchk(ref().ref_lr_split(self.h, num_gpus, mode, gpu, _p(sz, C.c_uint64), None, None,
                                 None, None))
        rows, le, re_, first = (int(x) for x in sz)
        lr = np.zeros(rows + 1, np.uint64)
        lc = np.zeros(max(le, 1), np.uint64)
        rr = np.zeros(rows + 1, np.uint64)
        rc = np.zeros(max(re_, 1), np.uint64)
        _rchk(ref().ref_lr_split(self.h, num_gpus, mode, gpu, _p(sz, C.c_uint64),
                                 _p(lr, C.c_uint64), _p(lc, C.c_uint64), _p(rr, C.c_uint64),
                                 _p(rc, C.c_uint64)))
        return first, (lr, lc[:le]), (rr, rc[:re_])

    def plan(self, num_gpus, mode, gpu, ps, dist, wpb, dim, mapping=0, granularity=0):
        h = C.c_void_p()
        _rchk(ref().ref_plan_build(self.h, num_gpus, mode, gpu, ps, dist, wpb, dim, mapping,
                                   granularity, C.byref(h)))
        return RefPlan(h)

    def multi_gpu_cycles(self, num_gpus, ps, dist, wpb, dim, profile="a100"):
        c = C.c_uint64()
        _rchk(ref().ref_multi_gpu_cycles(self.h, num_gpus, ps, dist, wpb, dim,
                                         profile.encode(), C.byref(c)))
        return c.value

    def time_metadata(self, num_gpus, ps, dist, wpb, dim):
        s = C.c_double()
        n = C.c_uint64()
        _rchk(ref().ref_time_metadata(self.h, num_gpus, ps, dist, wpb, dim, C.byref(s),
                                      C.byref(n)))
        return s.value, n.value


class RefPlan:
    def __init__(self, h):
        self.h = h
        c = np.zeros(8, np.uint64)
        ref().ref_plan_counts(h, _p(c, C.c_uint64))
        (self.n_local, self.n_remote, self.local_nbrs, self.remote_nbrs, self.n_warps,
         self.n_tasks, self.n_blocks, self.smem) = (int(x) for x in c)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_plan_free(self.h)
            self.h = None

    def parts(self, kind):
        n = self.n_local if kind == 0 else self.n_remote
        tot = self.local_nbrs if kind == 0 else self.remote_nbrs
        t = np.zeros(max(n, 1), np.uint64)
        s = np.zeros(max(n, 1), np.uint64)
        nb = np.zeros(max(tot, 1), np.uint64)
        ref().ref_plan_parts(self.h, kind, _p(t, C.c_uint64), _p(s, C.c_uint64),
                             _p(nb, C.c_uint64))
        return t[:n], s[:n], nb[:tot]

    def warps(self):
        off = np.zeros(self.n_warps + 1, np.uint64)
        wid = np.zeros(max(self.n_warps, 1), np.uint32)
        kind = np.zeros(max(self.n_tasks, 1), np.uint8)
        idx = np.zeros(max(self.n_tasks, 1), np.uint32)
        bf = np.zeros(max(self.n_blocks, 1), np.uint32)
        bc = np.zeros(max(self.n_blocks, 1), np.uint32)
        ref().ref_plan_warps(self.h, _p(off, C.c_uint64), _p(wid, C.c_uint32),
                             _p(kind, C.c_uint8), _p(idx, C.c_uint32), _p(bf, C.c_uint32),
                             _p(bc, C.c_uint32))
        return (off, wid[: self.n_warps], kind[: self.n_tasks], idx[: self.n_tasks],
                bf[: self.n_blocks], bc[: self.n_blocks])

    def json(self):
        return ref().ref_plan_json(self.h).decode()


def ref_wpw(ps, dist, wpb, dim):
    return int(ref().ref_wpw(ps, dist, wpb, dim))


def ref_smem(ps, dist, wpb, dim):
    return int(ref().ref_smem(ps, dist, wpb, dim))


def ref_validate(ps, dist, wpb, dim, num_sms, max_warps, smem_per_sm):
    buf = C.create_string_buffer(256)
    n = ref().ref_validate(ps, dist, wpb, dim, num_sms, max_warps, smem_per_sm, buf, 256)
    return [x for x in buf.value.decode().split(";") if x][:n]


def ref_optimize(fn, num_sms, max_warps, smem_per_sm, dim, retreat_value_rank=False,
                 max_evaluations=15):
    L = ref()
    cb = L.MEASURE(lambda ps, dist, wpb, _u: int(fn((ps, dist, wpb))))
    cap = 4096
    trace = np.zeros(4 * cap, np.uint64)
    best = np.zeros(4, np.uint64)
    n = C.c_size_t()
    _rchk(L.ref_optimize(cb, None, num_sms, max_warps, smem_per_sm, dim,
                         int(retreat_value_rank), max_evaluations, _p(trace, C.c_uint64), cap,
                         C.byref(n), _p(best, C.c_uint64)))
    t = trace[: 4 * n.value].reshape(-1, 4)
    return [tuple(int(x) for x in r) for r in t], tuple(int(x) for x in best)


def ref_exhaustive(fn, num_sms, max_warps, smem_per_sm, dim):
    L = ref()
    cb = L.MEASURE(lambda ps, dist, wpb, _u: int(fn((ps, dist, wpb))))
    cap = 1024
    table = np.zeros(4 * cap, np.uint64)
    n = C.c_size_t()
    _rchk(L.ref_exhaustive(cb, None, num_sms, max_warps, smem_per_sm, dim,
                           _p(table, C.c_uint64), cap, C.byref(n)))
    return [tuple(int(x) for x in r) for r in table[: 4 * n.value].reshape(-1, 4)]

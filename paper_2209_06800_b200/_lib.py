"""ctypes binding of libmgg.so (include/mgg.h).

The product path has no fallback: if the in-tree library is missing or does
not load, importing this module raises. Nothing here imports oracle/.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MGG_LIB selects an alternative in-tree build (A/B experiments); default libmgg.so
LIB_PATH = os.path.join(_HERE, os.environ.get("MGG_LIB", "libmgg.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or make -C paper_2209_06800_b200). There is no CPU fallback.")

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p

MEASURE_FN = C.CFUNCTYPE(C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, vp,
                         C.POINTER(C.c_int))


class ModelDesc(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("layers", C.c_uint32), ("in_dim", C.c_uint32),
                ("hidden", C.c_uint32), ("out_dim", C.c_uint32), ("eps", C.c_float),
                ("w1", f32p), ("b1", f32p), ("w2", f32p), ("b2", f32p), ("norm", C.c_uint32)]


class PlanDesc(C.Structure):
    _fields_ = [("part", C.c_uint32), ("ps", C.c_uint32), ("dist", C.c_uint32),
                ("wpb", C.c_uint32), ("mapping", C.c_uint32), ("granularity", C.c_uint32),
                ("rows", C.c_uint64), ("n_local", C.c_uint64), ("n_remote", C.c_uint64),
                ("local_meta", i32p), ("local_cols", u32p), ("local_cols_len", C.c_uint64),
                ("remote_meta", i32p), ("remote_cols", u32p), ("remote_cols_len", C.c_uint64),
                ("halo_rows", u32p), ("halo_len", C.c_uint64), ("remote_halo_cols", u32p)]


class AggOpts(C.Structure):
    _fields_ = [("relu_in", C.c_int), ("phase", C.c_int), ("halo", vp), ("halo_pull", C.c_int)]


class DenseDesc(C.Structure):
    _fields_ = [("w", vp), ("bias", vp), ("pre_bias", vp), ("pre", C.c_uint32),
                ("act", C.c_uint32), ("out2_scale", C.c_float), ("row_scale", vp)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


I = C.c_int
U32 = C.c_uint32
U64 = C.c_uint64
SZ = C.c_size_t
PP = C.POINTER(vp)

# --- common
_sig("mgg_last_error", C.c_char_p)
_sig("mgg_version", C.c_char_p)
_sig("mgg_cuda_available", I)
_sig("mgg_free", None, vp)
# --- layer A
_sig("mgg_ctx_create", I, U32, i32p, PP)
_sig("mgg_ctx_destroy", I, vp)
_sig("mgg_ctx_synchronize", I, vp)
_sig("mgg_ctx_launch_count", U64, vp)
_sig("mgg_store_create", I, vp, u64p, U32, PP)
_sig("mgg_store_destroy", I, vp)
_sig("mgg_store_info", I, vp, u32p, u32p)
_sig("mgg_store_layout", I, vp, C.POINTER(C.c_int), u64p)
_sig("mgg_store_vmm_export", I, vp, U32, C.POINTER(C.c_int))
_sig("mgg_store_vmm_import", I, vp, U32, C.c_int)
_sig("mgg_store_ipc_export", I, vp, U32, vp)
_sig("mgg_store_ipc_import", I, vp, U32, vp)
_sig("mgg_store_upload", I, vp, f32p, U64, U64, U32)
_sig("mgg_store_download", I, vp, f32p, U64, U64, U32)
_sig("mgg_store_shard", I, vp, U32, PP)
_sig("mgg_dbuf_create", I, vp, U32, vp, SZ, PP)
_sig("mgg_dbuf_destroy", I, vp)
_sig("mgg_dbuf_ptr", vp, vp)
_sig("mgg_probe_gather", I, vp, U32, vp, U32, vp, U64, U32, C.POINTER(C.c_double))
_sig("mgg_probe_chase", I, vp, U32, vp, U32, C.POINTER(C.c_double))
_sig("mgg_host_alloc", I, SZ, PP)
_sig("mgg_host_free", I, vp)
_sig("mgg_dplan_upload", I, vp, C.POINTER(PlanDesc), PP)
_sig("mgg_dplan_destroy", I, vp)
_sig("mgg_aggregate", I, vp, vp, vp, vp, C.POINTER(AggOpts))
_sig("mgg_rows_init", I, vp, U32, vp, vp, C.c_float, I)
_sig("mgg_rows_init_copy", I, vp, U32, vp, vp, C.c_float, I, vp)
_sig("mgg_rows_softmax", I, vp, U32, vp, vp)
_sig("mgg_rows_softmax_rs", I, vp, U32, vp, vp, vp)
_sig("mgg_rows_init_rs", I, vp, U32, vp, vp, C.c_float, I, vp, vp)
_sig("mgg_dense", I, vp, U32, vp, C.POINTER(DenseDesc), vp, vp)
_sig("mgg_dense_chain", I, vp, U32, vp, C.POINTER(DenseDesc), U32, C.POINTER(DenseDesc), vp, vp)
_sig("mgg_dense_chain_supported", I, U32, U32, U32)
_sig("mgg_barrier", I, vp, vp)
_sig("mgg_time_aggregate", I, vp, vp, vp, vp, C.POINTER(AggOpts), U32, u64p)
# --- layer B
_sig("mgg_graph_from_csr", I, U64, U64, u64p, u64p, PP)
_sig("mgg_graph_from_edges", I, U64, U64, u64p, u64p, PP)
_sig("mgg_graph_generate", I, I, U64, C.c_double, U64, PP)
_sig("mgg_graph_load_edge_list", I, C.c_char_p, PP)
_sig("mgg_graph_load_csr", I, C.c_char_p, PP)
_sig("mgg_graph_save_csr", I, vp, C.c_char_p)
_sig("mgg_graph_dims", I, vp, u64p, u64p)
_sig("mgg_graph_row_ptr", u64p, vp)
_sig("mgg_graph_col_idx", u64p, vp)
_sig("mgg_graph_destroy", I, vp)
_sig("mgg_split_by_edges", I, vp, U32, u64p)
_sig("mgg_plan_ne_placement", I, vp, U32, I, U64, u64p)
_sig("mgg_translate", I, vp, U32, I, U64, u64p, u32p, u64p)
_sig("mgg_memory_footprint", I, vp, U32, I, U64, U64, u64p, C.POINTER(I))
_sig("mgg_flat_plan_build", I, vp, U32, I, U32, U32, U32, U32, U64, I, I, PP)
_sig("mgg_flat_plan_info", I, vp, u64p)
_sig("mgg_flat_plan_meta", i32p, vp, I)
_sig("mgg_flat_plan_cols", u32p, vp, I)
_sig("mgg_flat_plan_json", I, vp, C.POINTER(C.c_void_p))
_sig("mgg_flat_plan_tasks", I, vp, u64p, u8p, u32p)
_sig("mgg_flat_plan_destroy", I, vp)
_sig("mgg_wpw", U64, U32, U32, U32, U64)
_sig("mgg_smem", U64, U32, U32, U32, U64)
_sig("mgg_launch_geometry", I, U64, U64, U32, U32, U32, C.c_char_p, u64p,
     C.POINTER(C.c_double))
_sig("mgg_validate", I, U32, U32, U32, U64, U32, U32, U64, C.c_char_p, SZ)
_sig("mgg_profile_json", I, C.c_char_p, C.POINTER(C.c_void_p))
_sig("mgg_optimize", I, MEASURE_FN, vp, U32, U32, U64, U64, I, U64, u64p, SZ,
     C.POINTER(SZ), u64p)
_sig("mgg_exhaustive", I, MEASURE_FN, vp, U32, U32, U64, U64, u64p, SZ, C.POINTER(SZ))
_sig("mgg_engine_create", I, vp, U32, i32p, U32, U32, U32, C.POINTER(ModelDesc), PP)
_sig("mgg_engine_destroy", I, vp)
_sig("mgg_engine_ipc_export", I, vp, U32, vp, C.POINTER(SZ))
_sig("mgg_engine_ipc_import", I, vp, U32, vp, SZ)
_sig("mgg_engine_vmm_ipc", I, vp, C.POINTER(C.c_int))
_sig("mgg_engine_vmm_export", I, vp, U32, C.POINTER(C.c_int), C.POINTER(SZ))
_sig("mgg_engine_vmm_import", I, vp, U32, C.POINTER(C.c_int), SZ)
_sig("mgg_engine_set_config", I, vp, U32, U32, U32)
_sig("mgg_engine_set_mapping", I, vp, I, I)
_sig("mgg_engine_set_remote_fetch", I, vp, I)
_sig("mgg_halo_pull", I, vp, vp, vp, vp)
_sig("mgg_dplan_halo_len", I, vp, u64p)
_sig("mgg_dplan_k1_kernels", I, vp, C.c_char_p, C.c_size_t)
_sig("mgg_remote_partition_bytes", U64, U64, U64, I, U64)
_sig("mgg_engine_set_input", I, vp, f32p)
_sig("mgg_engine_forward", I, vp)
_sig("mgg_engine_set_graphs", I, vp, I)
_sig("mgg_engine_set_k1_form", I, vp, U32)
_sig("mgg_engine_get_output", I, vp, f32p)
_sig("mgg_engine_forward_host", I, vp, f32p, f32p)
_sig("mgg_engine_submit_host", I, vp, f32p, f32p, u64p)
_sig("mgg_engine_wait", I, vp, U64)
_sig("mgg_store_upload_on", I, vp, f32p, U64, U64, U32, I)
_sig("mgg_store_download_on", I, vp, f32p, U64, U64, U32, I)
_sig("mgg_lane_fence", I, vp, U32, I, I)
_sig("mgg_lane_mark", I, vp, U32, I, U32)
_sig("mgg_lane_wait_host", I, vp, U32, U32)
_sig("mgg_lane_wait_mark", I, vp, U32, I, U32)
_sig("mgg_engine_get_hidden", I, vp, U32, f32p, u32p)
_sig("mgg_engine_aggregate_host", I, vp, f32p, U32, C.c_float, I, f32p)
_sig("mgg_engine_aggregate_phase_host", I, vp, f32p, U32, C.c_float, I, I, f32p)
_sig("mgg_engine_time_aggregate", I, vp, U32, U32, I, u64p)
_sig("mgg_engine_stats", I, vp, u64p)
_sig("mgg_engine_k1_kernels", I, vp, U32, C.c_char_p, C.c_size_t)
_sig("mgg_engine_time_aggregate_each", I, vp, U32, U32, I, u64p)
_sig("mgg_engine_measure_multi_gpu", I, vp, U32, U32, u64p, u64p, C.POINTER(C.c_double))
_sig("mgg_engine_set_shard_memory", I, vp, U32, I)
_sig("mgg_engine_get_logits", I, vp, C.POINTER(C.c_float))
_sig("mgg_device_count", I)
_sig("mgg_ctx_set_shard_memory", I, vp, U32, I)
_sig("mgg_store_rehome", I, vp)
_sig("mgg_dplan_k1_launch_info", I, vp, C.POINTER(C.c_uint32))
_sig("mgg_event_elapsed_between", I, vp, U32, U32, U32, U32, C.POINTER(C.c_float))
_sig("mgg_engine_trace_csv", I, vp, U32, U64, U32, C.POINTER(C.c_void_p))
_sig("mgg_trace_create", I, vp, U32, U64, U32, PP)
_sig("mgg_trace_destroy", I, vp)
_sig("mgg_aggregate_traced", I, vp, vp, vp, vp, C.POINTER(AggOpts), vp)
_sig("mgg_trace_read", I, vp, u64p, U64, u64p, u64p)
_sig("mgg_engine_ctx", vp, vp)
_sig("mgg_engine_set_profiling", I, vp, I)
_sig("mgg_engine_profile", I, vp, C.POINTER(C.c_double), u32p, u32p, SZ, C.POINTER(SZ), u64p)
_sig("mgg_event_record", I, vp, U32, U32)
_sig("mgg_ctx_join", I, vp)
_sig("mgg_capture_begin", I, vp)
_sig("mgg_capture_end", I, vp, PP)
_sig("mgg_exec_launch", I, vp, vp)
_sig("mgg_exec_destroy", I, vp)
_sig("mgg_event_elapsed", I, vp, U32, U32, U32, f32p)

# every exported symbol the header declares (checked by the CPU test suite)
HEADER = os.path.join(os.path.dirname(_HERE), "include", "mgg.h")


class MggError(RuntimeError):
    """Base of the Python mirror of the reference exception taxonomy."""
    code = 0


class InputError(MggError):
    code = 1


class ParseError(InputError):
    code = 2


class ConfigError(MggError):
    code = 3


class IntegrityError(MggError):
    code = 4


class CudaError(MggError):
    code = 5


_ERRORS = {1: InputError, 2: ParseError, 3: ConfigError, 4: IntegrityError, 5: CudaError}


def check(status: int) -> None:
    if status != 0:
        msg = lib.mgg_last_error().decode(errors="replace")
        raise _ERRORS.get(status, MggError)(msg)

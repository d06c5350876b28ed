"""B200-native MGG hot path: graph partition, neighbor-partition builder,
pipelined multi-GPU aggregation (sm_100a), Update GEMM, runtime tuner.

Host logic is C++ (libmgg.so, include/mgg/*.hpp) behind the C-ABI in
include/mgg.h; this package is the Python binding used by tests and bench.py.
Importing it fails loudly when libmgg.so is missing — there is no CPU path.
"""
from .api import *  # noqa: F401,F403
from .api import (CsrGraph, Engine, FlatPlan, HardwareProfile, Model,  # noqa: F401
                  build_flat_plan, chunk_ranges, cuda_available, exhaustive, from_edges,
                  gen_rmat, gen_synthetic, host_alloc, launch_geometry, load_csr,
                  load_edge_list, make_gcn, make_gin, memory_footprint, optimize,
                  plan_ne_placement, random_features, resolve_profile, smem,
                  split_by_edges, translate, validate, wpw)
from ._lib import (ConfigError, CudaError, InputError, IntegrityError, MggError,  # noqa: F401
                   ParseError, LIB_PATH)

__all__ = [n for n in dir() if not n.startswith("_")]

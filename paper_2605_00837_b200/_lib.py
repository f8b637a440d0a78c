"""ctypes binding of liblsk.so (the C ABI declared in include/lsk.h).

There is deliberately no fallback: if the library is missing or no CUDA
device is visible, every compute entry point raises ``BackendError``.
"""

import ctypes
import os

from .errors import BackendError, DimensionMismatch

_HERE = os.path.dirname(os.path.abspath(__file__))
# LSK_LIB overrides the library path (experiments with alternative builds)
LIB_PATH = os.environ.get("LSK_LIB") or os.path.join(_HERE, "liblsk.so")

LSK_OK = 0
LSK_EINVAL = -1
LSK_ECUDA = -2
LSK_EUNSUPPORTED = -3
LSK_FLAG_STALE_SHIFT = 1
LSK_FLAG_COST = 2
LSK_FLAG_EXPANSION = 8
LSK_FLAG_UNIFORM_NU = 16
LSK_FLAG_MULT = 32
LSK_FLAG_STD_MULTIKERNEL = 64
LSK_FLAG_SHARD_PARTIALS = 128
LSK_FLAG_SHARD_ALLREDUCE = 256
LSK_FLAG_NO_CLUSTER = 512
LSK_FLAG_NO_GRAPH = 1024
LSK_FLAG_GRAPH_NCCL = 2048
LSK_SHARD_NONE = 0
LSK_SHARD_OWNER = 1
LSK_SHARD_PARTIALS = 2
LSK_SHARD_ALLREDUCE = 3
LSK_EMU_MAX_RANKS = 16

_c_i32, _c_i64, _c_sz, _c_dbl, _c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double, ctypes.c_void_p

# name -> (restype, argtypes), mirrors include/lsk.h
SIGNATURES = {
    "lsk_last_error": (ctypes.c_char_p, []),
    "lsk_version": (_c_i32, []),
    "lsk_solve_dense_max_cols": (_c_i32, []),
    "lsk_trace_capacity": (_c_i32, [_c_i32, _c_i32]),
    "lsk_solve_dense_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "lsk_solve_dense_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_dbl, _c_dbl, _c_i32,
                                     _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_debug_arg3_f32": (_c_i32, [_c_p, _c_p, _c_dbl, _c_p, _c_p, _c_i32, _c_p]),
    "lsk_update_alpha_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_p, _c_p]),
    "lsk_update_beta_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "lsk_update_beta_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_marginal_error_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_dbl,
                                        _c_p, _c_p, _c_sz, _c_p]),
    "lsk_transport_cost_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl, _c_p,
                                        _c_p, _c_sz, _c_p]),
    "lsk_materialize_plan_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl, _c_p,
                                          _c_i64, _c_p, _c_p]),
    "lsk_build_cost_workspace_bytes": (_c_sz, []),
    "lsk_build_cost_f32": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_i64, _c_p, _c_p,
                                    _c_sz, _c_p]),
    "lsk_h2d_cost_f32": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_i32, _c_p]),
    "lsk_cost_range_f64": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_build_cost_div_f32": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_dbl, _c_p, _c_i64, _c_p]),
    "lsk_cast_cost_f32": (_c_i32, [_c_p, _c_i32, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_p]),
    "lsk_solve_dense_f64_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "lsk_solve_dense_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_dbl, _c_dbl, _c_i32, _c_i32,
                                     _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_update_alpha_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_p, _c_p]),
    "lsk_update_beta_f64_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "lsk_update_beta_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_marginal_error_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_dbl, _c_p,
                                        _c_p, _c_sz, _c_p]),
    "lsk_transport_cost_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl, _c_p, _c_p,
                                        _c_sz, _c_p]),
    "lsk_materialize_plan_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl, _c_p,
                                          _c_i64, _c_p, _c_p]),
    "lsk_solve_points_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32]),
    "lsk_solve_points_f32": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl,
                                      _c_dbl, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                      _c_sz, _c_p, _c_p]),
    "lsk_solve_points_sharded_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32, _c_i32]),
    "lsk_solve_points_emulated_f32": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl,
                                               _c_dbl, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p,
                                               _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_points_consume_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32]),
    "lsk_points_consume_f32": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p,
                                        _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_points_cost_range_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32]),
    "lsk_points_cost_range": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_points_cost_max_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32]),
    "lsk_points_cost_max": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_build_cost_f64": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_i64, _c_p, _c_p, _c_sz,
                                    _c_p]),
    "lsk_barycentric_points_f64": (_c_i32, [_c_p, _c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_dbl, _c_p, _c_p,
                                            _c_p, _c_p, _c_dbl, _c_p, _c_p, _c_p]),
    "lsk_recolor_nearest_f64": (_c_i32, [_c_p, _c_i64, _c_p, _c_i32, _c_p, _c_p, _c_p, _c_p]),
    "lsk_barycentric_plan_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i32, _c_p, _c_p, _c_p]),
    "lsk_nearest_map_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_p, _c_i32, _c_p, _c_i32, _c_i32, _c_p, _c_p, _c_p]),
    "lsk_kkt_residual": (_c_i32, [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_dbl, _c_i32, _c_p,
                                  _c_p, _c_p, _c_sz, _c_p]),
    "lsk_regularized_objective_f64": (_c_i32, [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_p, _c_p,
                                               _c_sz, _c_p]),
    "lsk_reduce_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "lsk_reduce_rows": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_reduce_cols": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_solve_standard_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32]),
    "lsk_solve_standard_f32": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_dbl, _c_i32, _c_i32,
                                        _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_solve_standard_f64": (_c_i32, [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl, _c_dbl, _c_i32, _c_i32,
                                        _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "lsk_nccl_unique_id_bytes": (_c_i32, []),
    "lsk_nccl_unique_id": (_c_i32, [_c_p]),
    "lsk_comm_create": (_c_i32, [_c_p, _c_i32, _c_i32, _c_p]),
    "lsk_comm_destroy": (_c_i32, [_c_p]),
}

_lib = None


def load():
    """Load liblsk.so and declare its signatures (no GPU needed)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BackendError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2605_00837_b200._build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def call(name, *args):
    """Call an lsk_* entry point and map its return code to an exception."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != LSK_OK:
        msg = (lib.lsk_last_error() or b"").decode(errors="replace")
        if rc == LSK_EINVAL:
            raise DimensionMismatch(f"{name}: {msg}")
        raise BackendError(f"{name} failed ({rc}): {msg}")
    return rc


def loaded_path():
    return LIB_PATH if _lib is not None else None

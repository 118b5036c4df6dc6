"""ctypes binding of include/octgpu.h (libocgpu.so, built in-tree).

The product path has no fallback: if the shared library is missing this
module raises at import time.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libocgpu.so"

OCG_OK = 0
OCG_EVAL_DOMAIN = 1
OCG_BUF_JAC, OCG_BUF_HESS, OCG_BUF_GRAD, OCG_BUF_ROWSCALE, OCG_BUF_OBJV = range(5)
OCG_LDL_BAND, OCG_LDL_REFERENCE = 0, 1

# every symbol include/octgpu.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "ocg_last_error", "ocg_free", "ocg_version", "ocg_release_cached_memory",
    "ocg_model_create", "ocg_model_create_from_nlp", "ocg_model_destroy", "ocg_model_nvar", "ocg_model_mcon", "ocg_model_grid",
    "ocg_model_arrays", "ocg_model_structure_json", "ocg_model_synth_acceptance", "ocg_synth_uniform",
    "ocg_eval_default_options", "ocg_eval_create", "ocg_eval_destroy", "ocg_eval_sizes", "ocg_eval_structure",
    "ocg_eval_buffer", "ocg_eval_bind_buffer", "ocg_eval_set_scaling", "ocg_eval_get_scaling", "ocg_eval_compute_scaling",
    "ocg_eval_constraints", "ocg_eval_constraints_jacobian", "ocg_eval_objective", "ocg_eval_gradient",
    "ocg_eval_hessian", "ocg_eval_jac_hess", "ocg_eval_jac_hess_host", "ocg_eval_max_abs_hessian", "ocg_eval_status", "ocg_eval_status_async",
    "ocg_eval_objective_chunks", "ocg_eval_objective_partials", "ocg_eval_objective_combine",
    "ocg_eval_launch_count",
    "ocg_debug_generated_source", "ocg_debug_generated_source_ex", "ocg_debug_compile", "ocg_debug_compile_log",
    "ocg_kkt_create", "ocg_kkt_destroy", "ocg_kkt_dims", "ocg_kkt_pattern", "ocg_kkt_maps", "ocg_kkt_values",
    "ocg_kkt_assemble", "ocg_kkt_matvec", "ocg_kkt_jt_lambda",
    "ocg_ldl_create", "ocg_ldl_destroy", "ocg_ldl_info", "ocg_ldl_factor", "ocg_ldl_solve",
    "ocg_ldl_create_ex", "ocg_ldl_factor_many", "ocg_ldl_select", "ocg_ldl_order", "ocg_ldl_factor_nnz", "ocg_ldl_factors", "ocg_ldl_ref_symbolic",
    "ocg_comm_nccl_unique_id", "ocg_comm_create_nccl", "ocg_comm_create_host", "ocg_comm_destroy",
    "ocg_eval_create_sharded", "ocg_eval_shard", "ocg_eval_scatter_x", "ocg_eval_halo_exchange",
    "ocg_eval_scatter_rows", "ocg_eval_status_all", "ocg_eval_objective_all", "ocg_shard_plan_json",
    "ocg_kkt_norm_inf", "ocg_ipm_default_options", "ocg_ipm_solve",
    "ocg_ipm_ctx_create", "ocg_ipm_ctx_destroy", "ocg_ipm_ctx_solve", "ocg_ipm_batch_solve",
]


class EvalOptions(C.Structure):
    _fields_ = [("device", C.c_int), ("fma", C.c_int), ("block", C.c_int), ("idx_lo", C.c_int64),
                ("idx_hi", C.c_int64), ("specials", C.c_int), ("min_blocks", C.c_int),
                ("split_kinds", C.c_int), ("input_staging", C.c_int)]


class IpmOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("mu_init", C.c_double), ("tau_min", C.c_double),
                ("reg_initial_scale", C.c_double), ("reg_grow", C.c_double), ("reg_shrink", C.c_double),
                ("reg_dual_scale", C.c_double), ("reg_dual_power", C.c_double), ("reg_max_delta", C.c_double),
                ("scale", C.c_int), ("bound_relax_factor", C.c_double), ("refine_rounds", C.c_int),
                ("refine_trigger", C.c_double), ("verbose", C.c_int), ("kkt_order", C.c_int)]


# ocg_comm_host_fns callbacks
ALLREDUCE_F64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
ALLREDUCE_I32 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32), C.c_int64)
SENDRECV_F64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_int, C.POINTER(C.c_double),
                           C.c_int64, C.c_int)


class CommHostFns(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allreduce_sum_f64", ALLREDUCE_F64), ("allreduce_max_i32", ALLREDUCE_I32),
                ("sendrecv_f64", SENDRECV_F64)]


class IpmResult(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("objective", C.c_double), ("theta", C.c_double),
                ("stationarity", C.c_double), ("complementarity", C.c_double), ("factorizations", C.c_int),
                ("time_total", C.c_double), ("time_derivatives", C.c_double), ("time_factorize", C.c_double),
                ("time_solve", C.c_double), ("kkt_dim", C.c_int64), ("kkt_nnz", C.c_int64),
                ("bandwidth", C.c_int64), ("time_plan_eval", C.c_double), ("time_plan_kkt", C.c_double),
                ("time_plan_ldl", C.c_double), ("time_setup", C.c_double)]


class OcgError(RuntimeError):
    pass


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                          "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(str(LIB_PATH))
    vp, i64, i32, dp, ip = C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.POINTER(C.c_int64)
    sig = {
        "ocg_last_error": (C.c_char_p, []),
        "ocg_free": (None, [vp]),
        "ocg_version": (C.c_char_p, []),
        "ocg_release_cached_memory": (C.c_int, [C.c_int]),
        "ocg_model_create": (i32, [C.c_char_p, i32, i64, i32, C.POINTER(vp)]),
        "ocg_model_create_from_nlp": (i32, [vp, C.POINTER(vp)]),
        "ocg_model_destroy": (None, [vp]),
        "ocg_model_nvar": (i64, [vp]),
        "ocg_model_mcon": (i64, [vp]),
        "ocg_model_grid": (i64, [vp]),
        "ocg_model_arrays": (i32, [vp] + [dp] * 7),
        "ocg_model_structure_json": (vp, [vp]),
        "ocg_model_synth_acceptance": (i32, [vp, C.c_uint32, dp, dp]),
        "ocg_synth_uniform": (i32, [C.c_uint32, C.c_double, C.c_double, i64, dp]),
        "ocg_eval_default_options": (None, [C.POINTER(EvalOptions)]),
        "ocg_eval_create": (i32, [vp, C.POINTER(EvalOptions), C.POINTER(vp)]),
        "ocg_eval_destroy": (None, [vp]),
        "ocg_eval_sizes": (i32, [vp, ip, ip, ip]),
        "ocg_eval_structure": (i32, [vp] + [dp] * 5),
        "ocg_eval_buffer": (vp, [vp, i32]),
        "ocg_eval_bind_buffer": (i32, [vp, i32, dp]),
        "ocg_eval_set_scaling": (i32, [vp, C.c_double, dp]),
        "ocg_eval_get_scaling": (i32, [vp, C.POINTER(C.c_double), dp]),
        "ocg_eval_compute_scaling": (i32, [vp, dp, i32, vp]),
        "ocg_eval_constraints": (i32, [vp, dp, dp, vp]),
        "ocg_eval_constraints_jacobian": (i32, [vp, dp, dp, vp]),
        "ocg_eval_objective": (i32, [vp, dp, dp, vp]),
        "ocg_eval_gradient": (i32, [vp, dp, dp, vp]),
        "ocg_eval_hessian": (i32, [vp, dp, dp, vp]),
        "ocg_eval_jac_hess": (i32, [vp, dp, dp, dp, vp]),
        "ocg_eval_jac_hess_host": (i32, [vp, dp, dp, dp, dp, dp, i32, ip, vp]),
        "ocg_eval_max_abs_hessian": (i32, [vp, dp, vp]),
        "ocg_eval_status": (i32, [vp, vp]),
        "ocg_eval_status_async": (i32, [vp, dp, vp]),
        "ocg_eval_objective_chunks": (i64, [vp]),
        "ocg_eval_objective_partials": (i32, [vp, dp, dp, vp]),
        "ocg_eval_objective_combine": (i32, [vp, dp, dp, vp]),
        "ocg_eval_launch_count": (i64, [vp]),
        "ocg_debug_generated_source": (vp, [vp, i32, i32]),
        "ocg_debug_generated_source_ex": (vp, [vp, i32, i32, i32]),
        "ocg_debug_compile": (i32, [vp, i32, i32]),
        "ocg_debug_compile_log": (vp, [vp, C.POINTER(EvalOptions)]),
        "ocg_kkt_create": (i32, [vp, vp, C.POINTER(vp)]),
        "ocg_kkt_destroy": (None, [vp]),
        "ocg_kkt_dims": (i32, [vp, dp]),
        "ocg_kkt_pattern": (i32, [vp, dp, dp]),
        "ocg_kkt_maps": (i32, [vp] + [dp] * 6),
        "ocg_kkt_values": (vp, [vp]),
        "ocg_kkt_assemble": (i32, [vp, dp, vp]),
        "ocg_kkt_matvec": (i32, [vp, dp, dp, vp]),
        "ocg_kkt_jt_lambda": (i32, [vp, dp, dp, vp]),
        "ocg_kkt_norm_inf": (i32, [vp, dp, vp]),
        "ocg_ipm_default_options": (None, [C.POINTER(IpmOptions)]),
        "ocg_ipm_solve": (i32, [vp, C.POINTER(IpmOptions), i32, C.POINTER(IpmResult), dp]),
        "ocg_ipm_ctx_create": (i32, [vp, i32, C.POINTER(vp)]),
        "ocg_ipm_ctx_destroy": (None, [vp]),
        "ocg_ipm_ctx_solve": (i32, [vp, C.POINTER(IpmOptions), dp, dp, dp, dp, dp, C.POINTER(IpmResult), dp]),
        "ocg_ipm_batch_solve": (i32, [vp, C.POINTER(IpmOptions), i32, i32, dp, dp, dp, dp, dp, C.POINTER(IpmResult),
                                      dp]),
        "ocg_ldl_create": (i32, [vp, C.POINTER(vp)]),
        "ocg_ldl_destroy": (None, [vp]),
        "ocg_ldl_info": (i32, [vp, dp]),
        "ocg_ldl_factor": (i32, [vp, C.c_double, C.c_double, dp, vp]),
        "ocg_ldl_solve": (i32, [vp, dp, dp, vp]),
        "ocg_ldl_create_ex": (i32, [vp, i32, C.POINTER(vp)]),
        "ocg_ldl_factor_many": (i32, [vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64), vp]),
        "ocg_ldl_select": (i32, [vp, i32]),
        "ocg_ldl_order": (i32, [vp]),
        "ocg_ldl_factor_nnz": (i64, [vp]),
        "ocg_ldl_factors": (i32, [vp, dp, dp, dp, dp, dp]),
        "ocg_ldl_ref_symbolic": (i32, [i64, dp, dp, i64, i64, dp, dp, dp, dp, dp]),
        "ocg_comm_nccl_unique_id": (i32, [dp]),
        "ocg_comm_create_nccl": (i32, [dp, i32, i32, i32, C.POINTER(vp)]),
        "ocg_comm_create_host": (i32, [C.POINTER(CommHostFns), i32, i32, i32, C.POINTER(vp)]),
        "ocg_comm_destroy": (None, [vp]),
        "ocg_eval_create_sharded": (i32, [vp, C.POINTER(EvalOptions), vp, C.POINTER(vp)]),
        "ocg_eval_shard": (i32, [vp, dp]),
        "ocg_eval_scatter_x": (i32, [vp, dp, dp, dp, vp]),
        "ocg_eval_halo_exchange": (i32, [vp, dp, vp]),
        "ocg_eval_scatter_rows": (i32, [vp, dp, dp, dp, vp]),
        "ocg_eval_status_all": (i32, [vp, vp]),
        "ocg_eval_objective_all": (i32, [vp, dp, dp, vp]),
        "ocg_shard_plan_json": (vp, [vp, i32, i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def check(rc: int, what: str = "") -> int:
    """Raise on negative (API/CUDA) codes; pass OCG_OK / OCG_EVAL_DOMAIN through."""
    if rc < 0:
        msg = LIB.ocg_last_error().decode(errors="replace")
        raise OcgError(f"{what}: {msg} (code {rc})")
    return rc


def take_string(ptr: int) -> str:
    s = C.cast(ptr, C.c_char_p).value.decode()
    LIB.ocg_free(ptr)
    return s

"""ctypes binding of the C-ABI in include/stratcox_b200.h.

This is the only module that touches the shared library. It loads the in-tree
``libstratcox_b200.so`` (built by ``make lib`` / ``__graft_entry__.build()``)
and fails loudly when it is missing: there is no CPU fallback for the product
path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCX_LIB selects another build of the same library (the profiling build
# libstratcox_b200_trace.so: make trace); default: the shipped one
LIB_PATH = os.environ.get("SCX_LIB") or os.path.join(_HERE, "libstratcox_b200.so")

_i8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p

SCX_OK, SCX_ERR_VALIDATION, SCX_ERR_NUMERIC, SCX_ERR_INTERNAL, SCX_ERR_CUDA = range(5)


class FitOptions(C.Structure):
    _fields_ = [("max_cycles", C.c_int32), ("tolerance", C.c_double), ("initial_trust", C.c_double)]


class FitResultC(C.Structure):
    _fields_ = [
        ("beta", _dp),
        ("trust", _dp),
        ("objective_trace", _dp),
        ("trace_len", C.c_int32),
        ("cycles_used", C.c_int32),
        ("converged", C.c_int32),
        ("n_warnings", C.c_int32),
        ("warning_coords", _i64p),
        ("warning_cap", C.c_int32),
        ("updates_since_refresh", C.c_uint32),
        ("n_evaluations", C.c_int64),
    ]


# name -> (restype, argtypes); every symbol declared in include/stratcox_b200.h
SIGNATURES = {
    "scx_version": (C.c_char_p, []),
    "scx_device_count": (C.c_int, []),
    "scx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "scx_destroy": (None, [_vp]),
    "scx_last_error": (C.c_char_p, [_vp]),
    "scx_upload_design": (C.c_int, [_vp, C.c_int64, C.c_int32, _i64p, _i8p, _i64p, C.c_int64,
                                    _i64p, _i64p, _dp]),
    "scx_upload_design_i32": (C.c_int, [_vp, C.c_int64, C.c_int32, _i64p, _i8p, _i64p,
                                        C.c_int64, _i64p, _i32p, _dp]),
    "scx_design_info": (C.c_int, [_vp, _i64p, _i32p, _i64p, _i64p, _i32p, _i64p, _i64p]),
    "scx_make_state": (C.c_int, [_vp, _dp]),
    "scx_set_state": (C.c_int, [_vp, _dp, _dp, _dp, C.c_uint32]),
    "scx_get_state": (C.c_int, [_vp, _dp, _dp, _dp, _u32p]),
    "scx_refresh_xbeta": (C.c_int, [_vp]),
    "scx_update_xbeta": (C.c_int, [_vp, C.c_int64, C.c_double]),
    "scx_gradient_hessian": (C.c_int, [_vp, C.c_int64, _dp, _dp]),
    "scx_gradient_hessian_rs": (C.c_int, [_vp, C.c_int64, _dp, _dp]),
    "scx_risk_prefix": (C.c_int, [_vp]),
    "scx_risk_prefix_n": (C.c_int, [_vp, C.c_int]),
    "scx_set_fit_path": (C.c_int, [_vp, C.c_int, _ip]),
    "scx_fit_path_stats": (C.c_int, [_vp, _i64p]),
    "scx_log_partial_likelihood": (C.c_int, [_vp, _dp]),
    "scx_naive_gradient_hessian": (C.c_int, [_vp, C.c_int64, _dp, _dp]),
    "scx_naive_log_partial_likelihood": (C.c_int, [_vp, _dp]),
    "scx_segmented_inclusive_scan": (C.c_int, [_vp, C.c_int64, _dp, _i8p, _dp]),
    "scx_newton_step": (C.c_int, [C.c_double, C.c_double, _dp, _ip]),
    "scx_apply_trust_region": (C.c_int, [C.c_double, C.c_double, _dp, _dp]),
    "scx_l1_coordinate_update": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, _dp,
                                           _ip, _ip]),
    "scx_coordinate_update": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_double, _dp, _ip, _ip]),
    "scx_rule_error": (C.c_char_p, []),
    "scx_ccd_fit": (C.c_int, [_vp, _dp, C.POINTER(FitOptions), _dp, C.POINTER(FitResultC)]),
    "scx_ccd_fit_prior": (C.c_int, [_vp, _dp, _dp, C.POINTER(FitOptions), _dp,
                                    C.POINTER(FitResultC)]),
    "scx_gamma_max": (C.c_int, [_vp, _dp, _dp]),
    "scx_design_export": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_uint8),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64), _dp]),
    "scx_timing_enable": (C.c_int, [_vp, C.c_int]),
    "scx_timing_reset": (C.c_int, [_vp]),
    "scx_timing_get": (C.c_int, [_vp, C.c_int, _dp, _i64p]),
    "scx_stream": (_vp, [_vp]),
    "scx_launch_count": (C.c_int64, [_vp]),
    "scx_debug_k1_trace": (C.c_int, [_i64p]),
    "scx_set_k1_mode": (C.c_int, [_vp, C.c_int, _ip]),
    "scx_debug_risk_arrays": (C.c_int, [_vp, _dp, _dp, _dp, _dp, C.POINTER(C.c_int32)]),
    "scx_set_sm_budget": (C.c_int, [_vp, C.c_int]),
    "scx_xchg_slots": (C.c_int, [_vp, C.POINTER(C.c_void_p)]),
    "scx_xchg_ipc_handle": (C.c_int, [_vp, C.c_char_p]),
    "scx_xchg_connect": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "scx_xchg_connect_ipc": (C.c_int, [_vp, C.c_int, C.c_int, C.c_char_p]),
    "scx_shard_local_columns": (C.c_int, [_vp, _i8p, _dp, _dp, C.POINTER(C.c_int)]),
    "scx_shard_set_columns": (C.c_int, [_vp, _i8p, _dp, _dp, C.c_int]),
}

class DatasetC(C.Structure):
    """scx_dataset"""
    _fields_ = [("n_rows", C.c_int64), ("time", C.POINTER(C.c_double)),
                ("event", C.POINTER(C.c_uint8)), ("stratum", C.POINTER(C.c_int32)),
                ("subject", C.POINTER(C.c_int64)), ("n_covariates", C.c_int64),
                ("col_ptr", C.POINTER(C.c_int64)), ("row_idx", C.POINTER(C.c_int64)),
                ("values", C.POINTER(C.c_double))]


class CvConfigC(C.Structure):
    """scx_cv_config"""
    _fields_ = [("folds", C.c_int), ("gamma_grid", C.POINTER(C.c_double)),
                ("grid_size", C.c_int64), ("seed", C.c_uint64)]


class CvResultC(C.Structure):
    """scx_cv_result"""
    _fields_ = [("gamma_star", C.c_double), ("fold_scores", C.POINTER(C.c_double)),
                ("mean_scores", C.POINTER(C.c_double)), ("n_warnings", C.c_int32)]


SIGNATURES.update({
    "scx_build_design": (C.c_int, [_vp, C.POINTER(DatasetC), _i64p]),
    "scx_default_gamma_grid": (C.c_int, [C.c_double, C.c_int64, _dp]),
    "scx_build_lowered_design": (C.c_int, [_vp, C.POINTER(DatasetC), _dp, C.c_int64, _i64p, _i64p,
                                           _dp, C.c_int64, _i64p, _i64p, C.POINTER(C.c_int32),
                                           _dp, _dp]),
    "scx_fold_assignment": (C.c_int, [C.POINTER(DatasetC), C.c_int, C.c_uint64,
                                      C.POINTER(C.c_int32)]),
    "scx_lower_time_varying": (C.c_int, [C.POINTER(DatasetC), _dp, C.c_int64, _i64p, _i64p, _dp,
                                         C.c_int64, C.POINTER(_vp), C.c_char_p, C.c_int]),
    "scx_lowered_sizes": (C.c_int, [_vp, _i64p, _i64p, _i64p]),
    "scx_lowered_dataset": (C.c_int, [_vp, C.POINTER(DatasetC)]),
    "scx_lowered_column_map": (C.c_int, [_vp, _i64p, C.POINTER(C.c_int32), _dp, _dp]),
    "scx_lowered_free": (None, [_vp]),
    "scx_read_wide_csv": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]),
    "scx_table_dataset": (C.c_int, [_vp, C.POINTER(DatasetC)]),
    "scx_table_covariate_name": (C.c_char_p, [_vp, C.c_int64]),
    "scx_table_n_strata": (C.c_int32, [_vp]),
    "scx_table_stratum_label": (C.c_char_p, [_vp, C.c_int32]),
    "scx_table_free": (None, [_vp]),
    "scx_write_wide_csv": (C.c_int, [C.c_char_p, C.POINTER(DatasetC), C.POINTER(C.c_char_p),
                                     C.POINTER(C.c_char_p), C.c_char_p, C.c_int]),
    "scx_read_long_csv": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]),
    "scx_long_sizes": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64), _dp]),
    "scx_long_covariate_name": (C.c_char_p, [_vp, C.c_int64]),
    "scx_write_long_csv": (C.c_int, [C.c_char_p, _vp, C.c_char_p, C.c_int]),
    "scx_long_lower": (C.c_int, [_vp, _dp, C.c_int64, _i64p, _i64p, _dp, C.c_int64,
                                 C.POINTER(C.c_void_p), C.c_char_p, C.c_int]),
    "scx_long_free": (None, [_vp]),
    "scx_lowered_covariate_name": (C.c_char_p, [_vp, C.c_int64]),
    "scx_config_from_string": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p),
                                         C.c_char_p, C.c_int]),
    "scx_config_from_file": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]),
    "scx_config_has": (C.c_int, [_vp, C.c_char_p]),
    "scx_config_get_string": (C.c_char_p, [_vp, C.c_char_p, C.c_char_p]),
    "scx_config_get_double": (C.c_int, [_vp, C.c_char_p, C.c_double, _dp, C.c_char_p, C.c_int]),
    "scx_config_get_int": (C.c_int, [_vp, C.c_char_p, C.c_int64, C.POINTER(C.c_int64),
                                     C.c_char_p, C.c_int]),
    "scx_config_get_double_list": (C.c_int, [_vp, C.c_char_p, _dp, C.c_int64,
                                             C.POINTER(C.c_int64), C.c_char_p, C.c_int]),
    "scx_config_get_string_list": (C.c_char_p, [_vp, C.c_char_p, C.POINTER(C.c_int64)]),
    "scx_config_finish": (C.c_int, [_vp, C.c_char_p, C.c_int]),
    "scx_config_free": (None, [_vp]),
    "scx_kfold_select_gamma": (C.c_int, [C.POINTER(DatasetC), _dp, C.POINTER(CvConfigC),
                                         C.POINTER(FitOptions), C.POINTER(C.c_int), C.c_int,
                                         C.POINTER(CvResultC), C.c_char_p, C.c_int]),
})

_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library (idempotent). Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the sm_100a library first (make lib or "
            "__graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("SCX_LIB") and not hasattr(lib, name):
            continue  # an older profiling build (A/B): entry points it lacks stay unbound
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a, ctype):
    """Pointer to a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))

"""ctypes declarations of include/hc.h (argument marshalling only).

Loads the in-tree paper_2112_03444_b200/lib/libhc.so and fails loudly when it is missing:
there is no CPU or PyTorch fallback for any step of the path.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HC_LIB_PATH") or os.path.join(_PKG, "lib", "libhc.so")

HC_OK, HC_E_INVALID_ARG, HC_E_TOO_LARGE, HC_E_CUDA, HC_E_OOM, HC_E_INTERNAL = range(6)
HC_CONVERGED, HC_DIVERGED, HC_STEP_UNDERFLOW, HC_MAX_STEPS, HC_SINGULAR, HC_NONFINITE, HC_AT_INFINITY = range(7)
STATUS_NAMES = ["CONVERGED", "DIVERGED", "STEP_UNDERFLOW", "MAX_STEPS", "SINGULAR", "NONFINITE", "AT_INFINITY"]
HC_RK4, HC_EULER = 0, 1
HC_MEM_DEVICE, HC_MEM_HOST = 0, 1
HC_LAYOUT_AUTO, HC_LAYOUT_THROUGHPUT, HC_LAYOUT_WIDE = 0, 1, 2

EXPORTED = [
    "hc_system_create", "hc_system_create_total_degree", "hc_total_degree_params", "hc_total_degree_count",
    "hc_total_degree_start", "hc_system_info_get", "hc_system_destroy", "hc_system_compile_info",
    "hc_system_compile_tables", "hc_tracker_settings_default", "hc_track_batch", "hc_result_wait",
    "hc_result_elapsed_ms", "hc_result_launch", "hc_result_get", "hc_result_destroy", "hc_batched_zgesv", "hc_fp64_peak_probe", "hc_solutions",
    "hc_last_error", "hc_version", "hc_debug_phase_cycles",
]


class hc_complex(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class hc_system_desc(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("n_params", C.c_int32), ("n_terms", C.c_int32),
                ("term_eq", C.c_void_p), ("term_xexp", C.c_void_p), ("term_coef", C.c_void_p),
                ("n_coefs", C.c_int32), ("coef_ptr", C.c_void_p), ("coef_w", C.c_void_p),
                ("coef_pexp", C.c_void_p)]


class hc_system_info(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("n_params", C.c_int32), ("n_coefs", C.c_int32),
                ("coef_degree_t", C.c_int32), ("lanes_per_track", C.c_int32), ("tracks_per_warp", C.c_int32),
                ("op_steps", C.c_int32), ("max_factors", C.c_int32), ("n_ops_J", C.c_int32),
                ("n_ops_rhs", C.c_int32), ("n_terms", C.c_int32), ("flops_coef", C.c_int64),
                ("flops_eval", C.c_int64), ("flops_lu", C.c_int64), ("flops_solve", C.c_int64),
                ("smem_per_track", C.c_int64), ("n_coef_slots", C.c_int32), ("n_monos", C.c_int32),
                ("mono_levels", C.c_int32), ("flops_eval_kernel", C.c_int64), ("flops_solve_kernel", C.c_int64)]

    def as_dict(self):
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


class hc_tracker_settings(C.Structure):
    _fields_ = [("predictor", C.c_int32), ("dt_init", C.c_double), ("dt_min", C.c_double),
                ("dt_max", C.c_double), ("grow_after", C.c_int32), ("grow", C.c_double),
                ("shrink", C.c_double), ("max_newton", C.c_int32), ("newton_tol", C.c_double),
                ("max_steps", C.c_int32), ("inf_norm", C.c_double), ("end_newton", C.c_int32),
                ("end_tol", C.c_double), ("res_abs", C.c_double), ("res_rel", C.c_double),
                ("pivot_rel", C.c_double), ("eg_start", C.c_double), ("eg_inf_mu", C.c_double),
                ("eg_sing_mu", C.c_double), ("eg_stab", C.c_double), ("eg_inf_s", C.c_double),
                ("eg_inf_norm", C.c_double), ("eg_samples", C.c_int32), ("eg_max_winding", C.c_int32),
                ("eg_max_radii", C.c_int32), ("eg_tol", C.c_double),
                ("lane_layout", C.c_int32)]


class hc_batch(C.Structure):
    _fields_ = [("n_instances", C.c_int64), ("n_start", C.c_int64), ("start_x", C.c_void_p),
                ("p_start", C.c_void_p), ("p_target", C.c_void_p), ("x_out", C.c_void_p),
                ("status_out", C.c_void_p), ("counters_out", C.c_void_p), ("resid_out", C.c_void_p),
                ("memory", C.c_int32), ("stream", C.c_void_p), ("winding_out", C.c_void_p)]


class hc_track_info(C.Structure):
    _fields_ = [("status", C.c_int32), ("steps", C.c_int32), ("rejections", C.c_int32),
                ("newton_iters", C.c_int32), ("solves", C.c_int32), ("resid_abs", C.c_double),
                ("resid_rel", C.c_double)]


class HCError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where} failed with status {code}: {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """The loaded libhc.so (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.hc_system_create.argtypes = [P(hc_system_desc), C.c_int, P(C.c_void_p)]
    L.hc_system_create_total_degree.argtypes = [P(hc_system_desc), C.c_int, P(C.c_void_p)]
    L.hc_total_degree_params.argtypes = [C.c_void_p, hc_complex, C.c_void_p, C.c_void_p]
    L.hc_total_degree_count.argtypes = [C.c_void_p]
    L.hc_total_degree_count.restype = C.c_int64
    L.hc_total_degree_start.argtypes = [C.c_void_p, C.c_void_p]
    L.hc_system_info_get.argtypes = [C.c_void_p, P(hc_system_info)]
    L.hc_system_destroy.argtypes = [C.c_void_p]
    L.hc_system_compile_info.argtypes = [P(hc_system_desc), P(hc_system_info)]
    L.hc_system_compile_tables.argtypes = [P(hc_system_desc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hc_tracker_settings_default.argtypes = [P(hc_tracker_settings)]
    L.hc_track_batch.argtypes = [C.c_void_p, P(hc_tracker_settings), P(hc_batch), P(C.c_void_p)]
    L.hc_result_wait.argtypes = [C.c_void_p]
    L.hc_result_elapsed_ms.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float), P(C.c_float)]
    L.hc_result_launch.argtypes = [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int64)]
    L.hc_result_get.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, P(hc_track_info)]
    L.hc_result_destroy.argtypes = [C.c_void_p]
    L.hc_batched_zgesv.argtypes = [C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_double, C.c_void_p]
    L.hc_fp64_peak_probe.argtypes = [C.c_int, P(C.c_double)]
    L.hc_solutions.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_void_p,
                               C.c_void_p, P(C.c_int64)]
    L.hc_debug_phase_cycles.argtypes = [C.c_void_p, C.c_void_p]
    L.hc_last_error.restype = C.c_char_p
    L.hc_version.restype = C.c_char_p
    for name in EXPORTED:
        fn = getattr(L, name)
        if fn.restype is C.c_int:   # ctypes default
            fn.restype = C.c_int
    _lib = L
    return L


def check(code: int, where: str) -> None:
    if code != HC_OK:
        raise HCError(code, where, lib().hc_last_error().decode(errors="replace"))

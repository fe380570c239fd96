"""ctypes binding of the C ABI in include/rfk.h (librfk.so, built in-tree).

The shared library is the product: every call below lands in a CUDA kernel
(no host fallback).  If librfk.so is missing, importing the compute API
raises immediately — build it with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2603_00035_b200``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RFK_LIBRARY: an alternative build of the same C ABI (diagnostic variants from
# scripts/build_variant.sh, e.g. the protocol-checked sweep)
LIB_PATH = os.environ.get("RFK_LIBRARY") or os.path.join(HERE, "librfk.so")

RFK_OK = 0
RFK_ERR_DIMENSION_MISMATCH = 1
RFK_ERR_ZERO_DIMENSION = 2
RFK_ERR_INVALID_ARGUMENT = 3
RFK_ERR_INCONSISTENT_FIXED_POINT = 4
RFK_ERR_CUDA = 5
RFK_ERR_NO_DEVICE = 6
RFK_ERR_ALLOC = 7
RFK_ERR_NOT_CONVERGED = 8
RFK_ERR_NON_SPD_INPUT = 9
RFK_ERR_DIVERGED_LOSS = 10

RFK_MEM_HOST = 0
RFK_MEM_DEVICE = 1

# Every exported entry point of include/rfk.h (checked by tests/test_capi.py).
EXPORTS = (
    "rfk_create", "rfk_destroy", "rfk_set_stream", "rfk_last_error", "rfk_status_string",
    "rfk_version", "rfk_launch_count", "rfk_solve", "rfk_solve_jacobi", "rfk_best_candidate",
    "rfk_two_point_update", "rfk_identify", "rfk_jacobian_entries", "rfk_solve_adjoint",
    "rfk_param_gradients", "rfk_loss_grad_mse", "rfk_backward", "rfk_project_spd",
    "rfk_project_drift", "rfk_drift_norm_sq", "rfk_debug_trace", "rfk_project_spd_vjp",
    "rfk_project_drift_vjp", "rfk_project_vjp", "rfk_objective_and_grad",
    "rfk_tv_value_grad", "rfk_tikhonov_value_grad", "rfk_clip_global_norm", "rfk_adam_step",
    "rfk_gd_step", "rfk_relative_error", "rfk_inverse_config_default", "rfk_objective",
    "rfk_recover", "rfk_generate_observations", "rfk_multi_source_recover", "rfk_workspace_bytes",
    "rfk_release_workspace", "rfk_solve_f32", "rfk_backward_f32", "rfk_solve_projected", "rfk_backward_projected",
)


class rfk_fields(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("rows", C.c_int32), ("cols", C.c_int32), ("h", C.c_double),
        ("g11", C.c_void_p), ("g12", C.c_void_p), ("g22", C.c_void_p),
        ("b1", C.c_void_p), ("b2", C.c_void_p), ("param_stride", C.c_int64),
        ("src", C.c_void_p), ("src_stride", C.c_int64), ("fixed_values", C.c_void_p),
    ]


class rfk_projection(C.Structure):
    _fields_ = [("mode", C.c_int32), ("eps_min", C.c_double), ("lambda_max", C.c_double),
                ("tau", C.c_double), ("euclid_cap", C.c_double)]


class rfk_fields_f32(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("rows", C.c_int32), ("cols", C.c_int32), ("h", C.c_double),
        ("g11", C.c_void_p), ("g12", C.c_void_p), ("g22", C.c_void_p),
        ("b1", C.c_void_p), ("b2", C.c_void_p), ("param_stride", C.c_int64),
        ("src", C.c_void_p), ("src_stride", C.c_int64),
    ]


class rfk_solve_options(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int32), ("sweep_order", C.c_int32 * 4)]


class rfk_records(C.Structure):
    _fields_ = [("type", C.c_void_p), ("stencil", C.c_void_p), ("donor1", C.c_void_p),
                ("donor2", C.c_void_p), ("c", C.c_void_p * 5)]


class rfk_observations(C.Structure):
    _fields_ = [("count", C.c_int32), ("sources", C.c_void_p), ("observed", C.c_void_p),
                ("values", C.c_void_p)]


class rfk_objective_options(C.Structure):
    _fields_ = [("solve_tol", C.c_double), ("solve_max_iters", C.c_int32),
                ("unreached_penalty_cap", C.c_double), ("exact_sum", C.c_int32)]


class rfk_inverse_config(C.Structure):
    """InverseConfig (inversion.hpp:15-45) + ProjectionConfig (feasibility.hpp:9-21)."""
    _fields_ = [
        ("param", C.c_int), ("optimizer", C.c_int), ("step_g", C.c_double), ("step_b", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("adam_eps", C.c_double),
        ("grad_clip_norm", C.c_double), ("lambda_g", C.c_double), ("lambda_b", C.c_double),
        ("tv_variant", C.c_int), ("iters", C.c_int32), ("eps_min", C.c_double),
        ("lambda_max", C.c_double), ("tau", C.c_double), ("euclid_cap", C.c_double),
        ("solve_tol", C.c_double), ("solve_max_iters", C.c_int32), ("plateau_window", C.c_int32),
        ("plateau_factor", C.c_double), ("unreached_penalty_cap", C.c_double), ("exact_sum", C.c_int32),
    ]


class rfk_objective_value(C.Structure):
    _fields_ = [("loss", C.c_double), ("data_loss", C.c_double), ("reg_loss", C.c_double),
                ("unreached_observed", C.c_int32)]


class rfk_multi_source_row(C.Structure):
    _fields_ = [("k", C.c_int32), ("total_observations", C.c_int32), ("error", C.c_double)]


class rfk_recovery(C.Structure):
    _fields_ = [("g11", C.c_void_p), ("g12", C.c_void_p), ("g22", C.c_void_p), ("b1", C.c_void_p),
                ("b2", C.c_void_p), ("iso_g", C.c_void_p), ("loss_history", C.c_void_p),
                ("error_history", C.c_void_p), ("iterations", C.c_int32), ("final_error", C.c_double),
                ("unreached_observed_total", C.c_int32)]


_VP, _I32, _I64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_CTX = C.c_void_p

_SIGS = {
    "rfk_create": ([C.POINTER(C.c_void_p), C.c_int], C.c_int),
    "rfk_destroy": ([_CTX], None),
    "rfk_set_stream": ([_CTX, _VP], C.c_int),
    "rfk_last_error": ([_CTX], C.c_char_p),
    "rfk_status_string": ([C.c_int], C.c_char_p),
    "rfk_version": ([], C.c_int),
    "rfk_launch_count": ([_CTX], C.c_int64),
    "rfk_workspace_bytes": ([_CTX], C.c_int64),
    "rfk_release_workspace": ([_CTX], C.c_int),
    "rfk_debug_trace": ([_CTX, _VP, C.c_int64], C.c_int64),
    "rfk_solve": ([_CTX, C.c_int, C.POINTER(rfk_fields), C.POINTER(rfk_solve_options),
                   _VP, _VP, _VP, _VP], C.c_int),
    "rfk_solve_f32": ([_CTX, C.c_int, C.POINTER(rfk_fields_f32), C.POINTER(rfk_solve_options),
                       _VP, _VP, _VP, _VP], C.c_int),
    "rfk_backward_f32": ([_CTX, C.c_int, C.POINTER(rfk_fields_f32), _VP, _D, _VP] + [_VP] * 5
                         + [_I32, _VP, _VP], C.c_int),
    "rfk_solve_jacobi": ([_CTX, C.c_int, C.POINTER(rfk_fields), C.POINTER(rfk_solve_options),
                          _VP, _VP, _VP, _VP], C.c_int),
    "rfk_best_candidate": ([_CTX, C.c_int, C.POINTER(rfk_fields), _VP, _I64, _VP, _I32]
                           + [_VP] * 8, C.c_int),
    "rfk_two_point_update": ([_CTX, C.c_int, _I64] + [_VP] * 15, C.c_int),
    "rfk_identify": ([_CTX, C.c_int, C.POINTER(rfk_fields), _VP, _D, C.POINTER(rfk_records),
                      _VP, _VP, _VP], C.c_int),
    "rfk_jacobian_entries": ([_CTX, C.c_int, _I64] + [_VP] * 10, C.c_int),
    "rfk_solve_adjoint": ([_CTX, C.c_int, _I32, _I32, _I32, _VP, C.POINTER(rfk_records), _VP,
                           _VP, _VP], C.c_int),
    "rfk_param_gradients": ([_CTX, C.c_int, _I32, _I32, _I32, _D, C.POINTER(rfk_records), _VP]
                            + [_VP] * 5, C.c_int),
    "rfk_loss_grad_mse": ([_CTX, C.c_int, _I32, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _I32],
                          C.c_int),
    "rfk_backward": ([_CTX, C.c_int, C.POINTER(rfk_fields), _VP, _D, _VP, _VP] + [_VP] * 5
                     + [_I32, _VP, _VP], C.c_int),
    "rfk_solve_projected": ([_CTX, C.c_int, C.POINTER(rfk_fields), C.POINTER(rfk_projection),
                             C.POINTER(rfk_solve_options), _VP, _VP, _VP, _VP, C.POINTER(_VP)], C.c_int),
    "rfk_backward_projected": ([_CTX, C.c_int, C.POINTER(rfk_fields), C.POINTER(rfk_projection), C.POINTER(_VP),
                                _VP, _D, _VP, _VP] + [_VP] * 5 + [_I32, _VP, _VP], C.c_int),
    "rfk_project_spd": ([_CTX, C.c_int, _I64, _VP, _VP, _VP, _D, _D], C.c_int),
    "rfk_project_drift": ([_CTX, C.c_int, _I64, _VP, _VP, _VP, _VP, _VP, _D, _D], C.c_int),
    "rfk_drift_norm_sq": ([_CTX, C.c_int, _I64] + [_VP] * 6, C.c_int),
    "rfk_project_spd_vjp": ([_CTX, C.c_int, _I64, _VP, _VP, _VP, _D, _D, _VP, _VP, _VP], C.c_int),
    "rfk_project_drift_vjp": ([_CTX, C.c_int, _I64] + [_VP] * 5 + [_D, _D] + [_VP] * 5, C.c_int),
    "rfk_project_vjp": ([_CTX, C.c_int, _I64] + [_VP] * 5 + [_D] * 4 + [_VP] * 5, C.c_int),
    "rfk_objective_and_grad": ([_CTX, C.c_int, C.POINTER(rfk_fields), C.POINTER(rfk_observations),
                                C.POINTER(rfk_objective_options), _VP, _VP] + [_VP] * 5, C.c_int),
    "rfk_tv_value_grad": ([_CTX, C.c_int, _I32, _I32, _I32, C.c_int, _D, _VP, _VP, _VP, _I32], C.c_int),
    "rfk_tikhonov_value_grad": ([_CTX, C.c_int, _I64, _I32, _D, _VP, _VP, _VP, _I32], C.c_int),
    "rfk_clip_global_norm": ([_CTX, C.c_int, _I64, _I32, _VP, _D, _VP, _I32], C.c_int),
    "rfk_adam_step": ([_CTX, C.c_int, _I64, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _D, _D, _D, _D, _I32],
                      C.c_int),
    "rfk_gd_step": ([_CTX, C.c_int, _I64, _I32, _VP, _VP, _VP, _D, _I32], C.c_int),
    "rfk_relative_error": ([_CTX, C.c_int, _I64, _I32, _VP, _VP, _VP, _I32], C.c_int),
    "rfk_inverse_config_default": ([C.POINTER(rfk_inverse_config)], None),
    "rfk_objective": ([_CTX, C.c_int, C.POINTER(rfk_fields), C.POINTER(rfk_observations),
                       C.POINTER(rfk_inverse_config), C.POINTER(rfk_objective_value)] + [_VP] * 5, C.c_int),
    "rfk_recover": ([_CTX, C.c_int, _I32, _I32, _D, C.POINTER(rfk_observations),
                     C.POINTER(rfk_inverse_config), _VP, _VP, _VP, _VP, C.POINTER(rfk_recovery)], C.c_int),
    "rfk_multi_source_recover": ([_CTX, _VP, _I32, _D, C.POINTER(rfk_inverse_config), _I32, C.c_uint64,
                                  _VP], C.c_int),
    "rfk_generate_observations": ([_CTX, C.c_int, C.POINTER(rfk_fields), _I32, _VP, _D, _D, C.c_uint64,
                                   _VP, _VP], C.c_int),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load librfk.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: the CUDA library was not built "
                          "(run __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib

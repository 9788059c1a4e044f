"""ctypes binding of the C ABI in include/ksvm_nfft.h (libksvm_nfft.so).

The library is built in-tree (``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_2312_00538_b200/csrc``). There is no fallback: if the
shared library is missing, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libksvm_nfft.so")

OK, ERR_DATA, ERR_CONFIG, ERR_INTERNAL = 0, 2, 4, 5
ROW_MAJOR, COL_MAJOR = 0, 1
HOST, DEVICE = 0, 1
FP64 = 0
FP32 = 1  # optional fp32 mode (include/ksvm_nfft.h)
PREDICT_EXACT, PREDICT_FAST = 0, 1


class GmresStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("relative_residual", C.c_double),
                ("converged", C.c_int), ("breakdown", C.c_int)]


class IpmConfig(C.Structure):
    _fields_ = [("C", C.c_double), ("sigma", C.c_double), ("gamma0", C.c_double), ("tol_ip", C.c_double),
                ("max_ip_iters", C.c_int), ("tol_gmres", C.c_double), ("max_gmres_iters", C.c_int),
                ("mu0", C.c_double)]


class IpmResult(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("mu_final", C.c_double), ("xi_alpha_rel", C.c_double),
                ("xi_lambda_rel", C.c_double), ("status", C.c_int), ("iterations", C.c_int),
                ("mean_gmres_iters", C.c_double)]


class IpmLog(C.Structure):
    _fields_ = [("it", C.c_int), ("mu", C.c_double), ("xi_alpha_rel", C.c_double), ("xi_lambda_rel", C.c_double),
                ("step_alpha", C.c_double), ("gmres_iterations", C.c_int), ("gmres_relative_residual", C.c_double),
                ("gmres_converged", C.c_int), ("gmres_breakdown", C.c_int)]


class Config(C.Structure):
    _fields_ = [("bandwidth", C.c_int), ("window_cutoff", C.c_int),
                ("oversampling", C.c_int), ("torus_radius", C.c_double)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_int64)
_vp = C.c_void_p

_SIGS = {
    "ksvm_nfft_last_error": (C.c_char_p, []),
    "ksvm_nfft_version": (C.c_char_p, []),
    "ksvm_nfft_launch_count": (C.c_int64, []),
    "ksvm_nfft_config_default": (None, [C.POINTER(Config)]),
    "ksvm_nfft_config_validate": (C.c_int, [C.POINTER(Config)]),
    "ksvm_nfft_plan_create": (C.c_int, [_vp, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_double,
                                        C.POINTER(Config), C.c_double, C.c_int, C.POINTER(_vp)]),
    "ksvm_nfft_plan_apply": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_plan_apply_cross": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.c_int, _vp, _vp,
                                             C.c_int, _vp]),
    "ksvm_nfft_plan_num_sources": (C.c_int64, [_vp]),
    "ksvm_nfft_plan_dim": (C.c_int, [_vp]),
    "ksvm_nfft_plan_scaled_length": (C.c_double, [_vp]),
    "ksvm_nfft_plan_coefficient_sum": (C.c_double, [_vp]),
    "ksvm_nfft_plan_scale_points": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.c_int, _vp]),
    "ksvm_nfft_plan_free": (None, [_vp]),
    "ksvm_nfft_op_create": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int, _ip, _ip,
                                      C.c_int, _dp, _dp, C.POINTER(Config), C.c_double, _ip,
                                      C.c_int, C.c_int, C.POINTER(_vp)]),
    "ksvm_nfft_op_size": (C.c_int64, [_vp]),
    "ksvm_nfft_op_num_windows": (C.c_int, [_vp]),
    "ksvm_nfft_op_window_points": (C.c_int64, [_vp, C.c_int]),
    "ksvm_nfft_op_apply": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_op_apply_batch": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int64, C.c_int, _vp]),
    "ksvm_nfft_op_entry": (C.c_double, [_vp, C.c_int64, C.c_int64]),
    "ksvm_nfft_kernel_rows": (C.c_int, [_vp, C.c_int, _lp, C.c_int, _vp, C.c_int, _vp]),
    "ksvm_nfft_kernel_diag": (C.c_int, [_vp, C.c_int, _vp, C.c_int, _vp]),
    "ksvm_nfft_op_set_stage_timing": (C.c_int, [_vp, C.c_int]),
    "ksvm_nfft_op_last_stage_ms": (C.c_int, [_vp, C.POINTER(C.c_float), C.c_int]),
    "ksvm_nfft_op_stage_name": (C.c_char_p, [_vp, C.c_int]),
    "ksvm_nfft_op_free": (None, [_vp]),
    "ksvm_nfft_op_create_sharded": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int, _ip, _ip, C.c_int, _dp,
                                              _dp, C.POINTER(Config), C.c_double, _vp, C.c_int64, C.c_int, C.c_int,
                                              C.POINTER(_vp)]),
    "ksvm_nfft_op_apply_spread": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_op_grids": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "ksvm_nfft_op_apply_finish": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_op_grid_pool": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(C.c_int64)]),
    "ksvm_nfft_op_apply_windows": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_op_combine_range": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.c_int, _vp]),
    "ksvm_nfft_op_device": (C.c_int, [_vp]),
    # Newton saddle system
    "ksvm_nfft_saddle_create": (C.c_int, [_vp, _vp, _vp, C.POINTER(_vp)]),
    "ksvm_nfft_saddle_set_theta": (C.c_int, [_vp, _vp]),
    "ksvm_nfft_saddle_apply": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_saddle_free": (None, [_vp]),
    "ksvm_nfft_precond_create": (C.c_int, [_vp, C.c_int, C.c_int64, _vp, C.c_int, C.POINTER(_vp)]),
    "ksvm_nfft_precond_create_ex": (C.c_int, [_vp, C.c_int, C.c_int64, _vp, C.c_int, C.c_int, _vp,
                                              C.POINTER(_vp)]),
    "ksvm_nfft_precond_refresh": (C.c_int, [_vp, _vp]),
    "ksvm_nfft_precond_apply": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_precond_identity": (C.c_int, [_vp]),
    "ksvm_nfft_precond_diagonal_fallback": (C.c_int, [_vp]),
    "ksvm_nfft_precond_free": (None, [_vp]),
    "ksvm_nfft_gmres_solve": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int, _vp, _vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_saddle_set_theta_ex": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    "ksvm_nfft_precond_refresh_ex": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    # interior point trainer
    "ksvm_nfft_ipm_config_default": (None, [C.POINTER(IpmConfig)]),
    "ksvm_nfft_ipm_train": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(IpmConfig), _vp,
                                      C.POINTER(IpmResult),
                                      C.POINTER(IpmLog)]),
    "ksvm_nfft_compute_bias": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_double, _dp, _lp]),
    "ksvm_nfft_nystrom": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, _vp, C.c_int, _vp]),
    "ksvm_nfft_balance_and_split": (C.c_int, [_vp, C.c_int64, C.c_double, C.c_uint64, _vp, _lp, _vp, _lp]),
    # prediction
    "ksvm_nfft_decision_values": (C.c_int, [_vp, C.c_int64, C.c_int, C.c_int64, C.c_int, _vp, _vp, C.c_int, _vp,
                                            _vp, C.POINTER(Config), _vp, C.c_double, _vp, C.c_int64, C.c_int64,
                                            C.c_int, C.c_int, _vp, _vp]),
    # greedy pivoted Cholesky
    "ksvm_nfft_pivoted_cholesky": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, _vp, _ip, _dp, _vp, C.c_int,
                                             _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load libksvm_nfft.so (raises if it was not built — no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                              "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return load().ksvm_nfft_last_error().decode()


def launch_count() -> int:
    return int(load().ksvm_nfft_launch_count())

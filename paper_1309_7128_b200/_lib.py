"""Loader for the in-tree sm_100a library (libismg_b200.so) with argtypes.

Fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from ._abi import (CCycleConfig, CGridSpec, CReport, CSolveStats, CStepMetrics, DP, I32P)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISMG_LIB") or os.path.join(HERE, "libismg_b200.so")  # ISMG_LIB: experiment builds

_lib = None


class IsmgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("ismg_b200 error %d: %s" % (code, msg))
        self.code = code


class InvalidArgument(IsmgError, ValueError):
    """std::invalid_argument"""


class DomainError(IsmgError, ArithmeticError):
    """std::domain_error"""


class LogicError(IsmgError):
    """std::logic_error"""


_EXC = {1: InvalidArgument, 2: DomainError, 3: LogicError}

VP = C.c_void_p
G = C.POINTER(CGridSpec)
CF = C.POINTER(CCycleConfig)
R = C.POINTER(CReport)
M = C.POINTER(CStepMetrics)
PP = C.POINTER(C.c_void_p)

# name -> argtypes (restype int unless noted)
SIGNATURES = {
    "ismg_abi_version": [],
    "ismg_device_count": [C.POINTER(C.c_int)],
    "ismg_ctx_create": [C.c_int, VP, PP],
    "ismg_ctx_destroy": [VP],
    "ismg_ctx_synchronize": [VP],
    "ismg_ctx_attach_comm": [VP, VP, C.c_int, C.c_int],
    "ismg_nccl_unique_id": [VP, C.c_size_t],
    "ismg_strip_rows": [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "ismg_grid_validate": [G],
    "ismg_cycle_validate": [CF],
    "ismg_pressure_bc": [G, I32P, I32P],
    "ismg_build_fine_diag": [G, DP, C.c_size_t],
    "ismg_build_ismg_operator": [G, I32P, I32P, DP, C.c_size_t],
    "ismg_build_gmg_operator": [G, I32P, I32P, DP, C.c_size_t],
    "ismg_field_create": [VP, C.c_int, C.c_int, PP],
    "ismg_field_destroy": [VP],
    "ismg_field_dims": [VP, I32P, I32P],
    "ismg_field_upload": [VP, DP, C.c_size_t],
    "ismg_field_download": [VP, DP, C.c_size_t],
    "ismg_field_fill": [VP, C.c_double],
    "ismg_velocity_create": [VP, C.c_int, C.c_int, PP],
    "ismg_velocity_destroy": [VP],
    "ismg_velocity_upload": [VP, DP, C.c_size_t, DP, C.c_size_t],
    "ismg_velocity_download": [VP, DP, C.c_size_t, DP, C.c_size_t],
    "ismg_solver_create": [VP, G, CF, PP],
    "ismg_solver_destroy": [VP],
    "ismg_solver_info": [VP, G, I32P, I32P, I32P],
    "ismg_rbgs_sweep": [VP, VP, VP],
    "ismg_fine_residual": [VP, VP, VP, VP, DP],
    "ismg_anchor_mean": [VP, VP],
    "ismg_zero_ghosts": [VP, VP],
    "ismg_restrict_sum": [VP, VP, VP],
    "ismg_prolongate_bilinear": [VP, VP, VP],
    "ismg_coarse_residual": [VP, VP, VP, VP, DP],
    "ismg_gs_sweep_lex": [VP, VP, VP],
    "ismg_coarse_anchor_mean": [VP, VP],
    "ismg_solve": [VP, VP, VP, R, M, C.c_int64],
    "ismg_solve_host": [VP, DP, DP, C.c_size_t, R, M, C.c_int64],
    "ismg_solver_last_stats": [VP, C.POINTER(CSolveStats)],
    "ismg_solver_visit_log": [VP, I32P, C.c_size_t, C.POINTER(C.c_size_t)],
    "ismg_bench_fine_pass": [VP, VP, VP, C.c_int, DP],
    "ismg_bench_coarse_visit": [VP, VP, VP, C.c_int64, C.c_int, C.POINTER(C.c_int64), DP, DP],
    "ismg_ctx_launch_count": [VP, C.POINTER(C.c_int64)],
    "ismg_apply_scalar_bc": [VP, G, VP],
    "ismg_apply_velocity_bc": [VP, G, VP],
    "ismg_divergence": [VP, G, VP, VP, C.c_double],
    "ismg_correct": [VP, G, VP, VP, C.c_double],
    "ismg_predictor": [VP, G, VP, VP, C.c_double, C.c_double, VP],
    "ismg_state_create": [VP, G, PP],
    "ismg_state_destroy": [VP],
    "ismg_state_set_scalars": [VP, C.c_double, C.c_double, C.c_double, C.c_int64],
    "ismg_state_get_scalars": [VP, DP, DP, DP, C.POINTER(C.c_int64)],
    "ismg_state_upload": [VP, DP, C.c_size_t, DP, C.c_size_t, DP, C.c_size_t],
    "ismg_state_download": [VP, DP, C.c_size_t, DP, C.c_size_t, DP, C.c_size_t],
    "ismg_step": [VP, VP, R, M, C.c_int64],
}


def header_symbols() -> list:
    """Every function declared in include/ismg_b200.h."""
    import re
    path = os.path.join(os.path.dirname(HERE), "include", "ismg_b200.h")
    src = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ismg_\w+)\s*\(", src, re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libismg_b200.so not built (python -m paper_1309_7128_b200.build); "
                              "there is no CPU fallback for the ISM pressure path")
        L = C.CDLL(LIB_PATH)
        L.ismg_last_error.restype = C.c_char_p
        L.ismg_last_error.argtypes = []
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().ismg_last_error().decode()
        raise _EXC.get(rc, IsmgError)(rc, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))

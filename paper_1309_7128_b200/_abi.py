"""ctypes mirrors of the value types in include/ismg_b200.h.

Shared by the product bindings (`_lib.py`) and the test-only oracle loader,
so both sides of every parity test are driven by the same struct layout.
"""
from __future__ import annotations

import ctypes as C

ISMG_OK = 0
ISMG_ERR_INVALID_ARGUMENT = 1
ISMG_ERR_DOMAIN = 2
ISMG_ERR_LOGIC = 3
ISMG_ERR_CUDA = 4
ISMG_ERR_NCCL = 5
ISMG_ERR_NO_DEVICE = 6
ISMG_ERR_INTERNAL = 7


class CBc(C.Structure):
    """BoundaryCondition — grid.hpp:30-65."""

    _fields_ = [
        ("kind", C.c_int32),
        ("inlet_start", C.c_int32),
        ("inlet_width", C.c_int32),
        ("reserved", C.c_int32),
        ("u_wall", C.c_double),
        ("v_wall", C.c_double),
        ("p_wall", C.c_double),
        ("v_inflow", C.c_double),
    ]


class CGridSpec(C.Structure):
    """GridSpec — grid.hpp:67-97."""

    _fields_ = [
        ("nx", C.c_int32),
        ("ny", C.c_int32),
        ("h", C.c_double),
        ("tile", C.c_int32),
        ("reserved", C.c_int32),
        ("bc", CBc * 4),
    ]


class CCycleConfig(C.Structure):
    """CycleConfig — cycles.hpp:20-45."""

    _fields_ = [
        ("scheme", C.c_int32),
        ("tile", C.c_int32),
        ("depth", C.c_int32),
        ("acm_pre_smooth", C.c_int32),
        ("acm_post_smooth", C.c_int32),
        ("reserved", C.c_int32),
        ("tol_fine", C.c_double),
        ("tol_coarse", C.c_double),
        ("max_total_sweeps", C.c_int64),
        ("stall_factor", C.c_double),
    ]


class CReport(C.Structure):
    """ConvergenceReport — cycles.hpp:47-52 (+ NaN side channel)."""

    _fields_ = [
        ("converged", C.c_int32),
        ("nan_seen", C.c_int32),
        ("fine_sweeps", C.c_int64),
        ("coarse_sweeps", C.c_int64),
        ("residual", C.c_double),
    ]


class CStepMetrics(C.Structure):
    """StepMetrics — metrics.hpp:22-35."""

    _fields_ = [
        ("step", C.c_int64),
        ("fine_sweeps", C.c_int64),
        ("coarse_sweeps", C.c_int64),
        ("sync_fine", C.c_int64),
        ("sync_coarse", C.c_int64),
        ("lap_equiv", C.c_double),
        ("restrictions", C.c_int64),
        ("prolongations", C.c_int64),
        ("residual_final", C.c_double),
        ("converged", C.c_int32),
        ("reserved", C.c_int32),
    ]


class CSolveStats(C.Structure):
    _fields_ = [
        ("fine_passes", C.c_int64),
        ("prolong_passes", C.c_int64),
        ("coarse_visits", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("host_syncs", C.c_int64),
        ("collectives", C.c_int64),
        ("fine_pass_ms", C.c_double),
        ("coarse_ms", C.c_double),
        ("solve_ms", C.c_double),
        ("coarse_steps", C.c_int64),
        ("coarse_engine", C.c_int64),
    ]


assert C.sizeof(CBc) == 48
assert C.sizeof(CGridSpec) == 24 + 4 * 48
assert C.sizeof(CCycleConfig) == 56
assert C.sizeof(CStepMetrics) == 80

DP = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)


def dptr(a):
    """double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    assert a.dtype.name == "float64" and a.flags["C_CONTIGUOUS"], "need contiguous float64"
    return a.ctypes.data_as(DP)

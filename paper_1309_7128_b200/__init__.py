"""B200-native ISM pressure solve (arXiv 1309.7128) behind the reference's operator API.

Host value types mirror the reference (`api`); the compute runs in the in-tree
sm_100a library libismg_b200.so through its C-ABI (`solver`).
"""
from .api import *  # noqa: F401,F403
from .solver import (  # noqa: F401
    CaseResult, Context, DeviceField, DeviceState, DeviceVelocity, PressureSolver, apply_scalar_bc,
    apply_velocity_bc, build_gmg_operator, build_ismg_operator, correct, device_count, divergence, nccl_unique_id,
    predictor, run_case, step, strip_rows)

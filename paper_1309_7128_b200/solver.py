"""Device-side API mirroring the reference's PressureSolver / step / run_case.

    solver = PressureSolver(grid, cfg)                     # cycles.hpp:289-308
    rep = solver.solve(x, b, metrics)                      # cycles.hpp:310-321
    rep = step(state, grid, solver, metrics)               # projection.hpp:139-190
    res = run_case(case, cfg)                              # bench.hpp:127-158

`x`, `b` may be host ScalarFields (copied in and out) or DeviceFields (stay in
HBM). Every call goes through the C-ABI of libismg_b200.so (sm_100a); there is
no CPU path.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._abi import CGridSpec, CReport, CSolveStats, CStepMetrics, dptr
from .api import (BenchmarkCase, ConvergenceReport, CycleConfig, FluidState, GridSpec, MacVelocity, RunMetrics,
                  ScalarField, Scheme)


class Context:
    """One device + stream (ismg_ctx)."""

    _default = {}

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        _lib.call("ismg_ctx_create", device, C.c_void_p(stream) if stream else None, C.byref(h))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def synchronize(self) -> None:
        _lib.call("ismg_ctx_synchronize", self.h)

    def launch_count(self) -> int:
        n = C.c_int64()
        _lib.call("ismg_ctx_launch_count", self.h, C.byref(n))
        return n.value

    def attach_comm(self, unique_id: bytes, rank: int, nranks: int) -> None:
        """Join the NCCL strip decomposition (before creating solvers on this context)."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _lib.call("ismg_ctx_attach_comm", self.h, buf, int(rank), int(nranks))

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib.lib().ismg_ctx_destroy(self.h)
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 makes it; the caller shares it)."""
    buf = C.create_string_buffer(128)
    _lib.call("ismg_nccl_unique_id", buf, 128)
    return buf.raw


def strip_rows(ny: int, tile: int, nranks: int, rank: int) -> tuple:
    """Fine rows [r0, r1) owned by `rank` in the strip decomposition (whole tiles)."""
    a, b = C.c_int32(), C.c_int32()
    _lib.call("ismg_strip_rows", int(ny), int(tile), int(nranks), int(rank), C.byref(a), C.byref(b))
    return a.value, b.value


def device_count() -> int:
    n = C.c_int()
    _lib.call("ismg_device_count", C.byref(n))
    return n.value


class DeviceField:
    """ScalarField<double> resident in HBM (ismg_field)."""

    def __init__(self, nx: int, ny: int, ctx: Optional[Context] = None, host: Optional[ScalarField] = None):
        self.ctx = ctx or Context.default()
        self.nx, self.ny = int(nx), int(ny)
        h = C.c_void_p()
        _lib.call("ismg_field_create", self.ctx.h, self.nx, self.ny, C.byref(h))
        self.h = h
        if host is not None:
            self.upload(host)

    @classmethod
    def from_host(cls, f: ScalarField, ctx: Optional[Context] = None) -> "DeviceField":
        return cls(f.nx, f.ny, ctx, f)

    def upload(self, f: ScalarField) -> None:
        assert (f.nx, f.ny) == (self.nx, self.ny)
        _lib.call("ismg_field_upload", self.h, dptr(f.data), f.data.size)

    def download(self, f: Optional[ScalarField] = None) -> ScalarField:
        f = f or ScalarField(self.nx, self.ny)
        _lib.call("ismg_field_download", self.h, dptr(f.data), f.data.size)
        return f

    def fill(self, v: float) -> None:
        _lib.call("ismg_field_fill", self.h, float(v))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().ismg_field_destroy(self.h)
        except Exception:
            pass


class DeviceVelocity:
    """MacVelocity<double> resident in HBM (ismg_velocity)."""

    def __init__(self, nx: int, ny: int, ctx: Optional[Context] = None, host: Optional[MacVelocity] = None):
        self.ctx = ctx or Context.default()
        self.nx, self.ny = int(nx), int(ny)
        h = C.c_void_p()
        _lib.call("ismg_velocity_create", self.ctx.h, self.nx, self.ny, C.byref(h))
        self.h = h
        if host is not None:
            self.upload(host)

    def upload(self, v: MacVelocity) -> None:
        _lib.call("ismg_velocity_upload", self.h, dptr(v.u_data), v.u_data.size, dptr(v.v_data), v.v_data.size)

    def download(self, v: Optional[MacVelocity] = None) -> MacVelocity:
        v = v or MacVelocity(self.nx, self.ny)
        _lib.call("ismg_velocity_download", self.h, dptr(v.u_data), v.u_data.size, dptr(v.v_data), v.v_data.size)
        return v

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().ismg_velocity_destroy(self.h)
        except Exception:
            pass


def _report(c: CReport) -> ConvergenceReport:
    return ConvergenceReport(bool(c.converged), int(c.fine_sweeps), int(c.coarse_sweeps), float(c.residual),
                             bool(c.nan_seen))


class PressureSolver:
    """cycles.hpp:286-333 on the B200."""

    def __init__(self, grid: GridSpec, cfg: CycleConfig, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self._g, self._cfg = grid.copy(), cfg
        self._gc, self._cc = grid.to_c(), cfg.to_c()
        h = C.c_void_p()
        _lib.call("ismg_solver_create", self.ctx.h, C.byref(self._gc), C.byref(self._cc), C.byref(h))
        self.h = h
        eff = CGridSpec()
        ncx, ncy, sing = C.c_int32(), C.c_int32(), C.c_int32()
        _lib.call("ismg_solver_info", self.h, C.byref(eff), C.byref(ncx), C.byref(ncy), C.byref(sing))
        self._g.tile = eff.tile
        self.ncx, self.ncy, self.singular = ncx.value, ncy.value, bool(sing.value)

    def grid(self) -> GridSpec:
        return self._g

    def config(self) -> CycleConfig:
        return self._cfg

    # -- the solve ----------------------------------------------------------
    def solve(self, x, b, m: Optional[RunMetrics] = None) -> ConvergenceReport:
        rep = CReport()
        cur = m.current.to_c() if m is not None else CStepMetrics()
        fc = m.fine_cells if m is not None else self._g.nx * self._g.ny
        if isinstance(x, DeviceField):
            _lib.call("ismg_solve", self.h, x.h, b.h, C.byref(rep), C.byref(cur), C.c_int64(fc))
        else:
            assert x.data.size == b.data.size == (self._g.nx + 2) * (self._g.ny + 2)
            _lib.call("ismg_solve_host", self.h, dptr(x.data), dptr(b.data), x.data.size, C.byref(rep),
                      C.byref(cur), C.c_int64(fc))
        if m is not None:
            m.current.load_c(cur)
        return _report(rep)

    def last_stats(self) -> dict:
        s = CSolveStats()
        _lib.call("ismg_solver_last_stats", self.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in CSolveStats._fields_}

    def bench_fine_pass(self, x: DeviceField, b: DeviceField, iters: int) -> float:
        """Mean CUDA-event time (ms) of one fused fine pass on (x, b)."""
        ms = C.c_double()
        _lib.call("ismg_bench_fine_pass", self.h, x.h, b.h, int(iters), C.byref(ms))
        return ms.value

    def bench_coarse_visit(self, cb: DeviceField, ce: DeviceField, budget: int, first_group: int = 1):
        """One coarse visit of the fused engine on rhs cb from ce = 0 (coarse extent);
        returns (sweeps, final coarse residual max, kernel ms)."""
        n, rc, ms = C.c_int64(), C.c_double(), C.c_double()
        _lib.call("ismg_bench_coarse_visit", self.h, cb.h, ce.h, int(budget), int(first_group), C.byref(n),
                  C.byref(rc), C.byref(ms))
        return n.value, rc.value, ms.value

    def visit_log(self):
        """[(coarse sweeps, fine sweeps)] per outer iteration of the last fused solve."""
        n = C.c_size_t()
        _lib.call("ismg_solver_visit_log", self.h, None, 0, C.byref(n))
        buf = (C.c_int32 * (2 * max(n.value, 1)))()
        _lib.call("ismg_solver_visit_log", self.h, buf, n.value, C.byref(n))
        return [(buf[2 * k], buf[2 * k + 1]) for k in range(n.value)]

    # -- op-level reference calls (device fields) ---------------------------
    def rbgs_sweep(self, x: DeviceField, b: DeviceField) -> None:
        _lib.call("ismg_rbgs_sweep", self.h, x.h, b.h)

    def fine_residual(self, x: DeviceField, b: DeviceField, out: Optional[DeviceField] = None) -> float:
        r = C.c_double()
        _lib.call("ismg_fine_residual", self.h, x.h, b.h, out.h if out else None, C.byref(r))
        return r.value

    def anchor_mean(self, x: DeviceField) -> None:
        _lib.call("ismg_anchor_mean", self.h, x.h)

    def zero_ghosts(self, x: DeviceField) -> None:
        _lib.call("ismg_zero_ghosts", self.h, x.h)

    def restrict_sum(self, fine: DeviceField, coarse: DeviceField) -> None:
        _lib.call("ismg_restrict_sum", self.h, fine.h, coarse.h)

    def prolongate_bilinear(self, coarse: DeviceField, fine: DeviceField) -> None:
        _lib.call("ismg_prolongate_bilinear", self.h, coarse.h, fine.h)

    def coarse_residual(self, x: DeviceField, b: DeviceField, out: Optional[DeviceField] = None) -> float:
        r = C.c_double()
        _lib.call("ismg_coarse_residual", self.h, x.h, b.h, out.h if out else None, C.byref(r))
        return r.value

    def gs_sweep_lex(self, x: DeviceField, b: DeviceField) -> None:
        _lib.call("ismg_gs_sweep_lex", self.h, x.h, b.h)

    def coarse_anchor_mean(self, x: DeviceField) -> None:
        _lib.call("ismg_coarse_anchor_mean", self.h, x.h)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().ismg_solver_destroy(self.h)
        except Exception:
            pass


# ---- host-side geometry through the library (no device needed) -------------
def build_ismg_operator(g: GridSpec):
    """coarsening.hpp:196-305 -> (ncx, ncy, w[9, ncy, ncx])."""
    return _build("ismg_build_ismg_operator", g)


def build_gmg_operator(g: GridSpec):
    return _build("ismg_build_gmg_operator", g)


def _build(fn, g):
    gc = g.to_c()
    ncx, ncy = C.c_int32(), C.c_int32()
    _lib.call(fn, C.byref(gc), C.byref(ncx), C.byref(ncy), None, 0)
    w = np.zeros(9 * ncx.value * ncy.value)
    _lib.call(fn, C.byref(gc), C.byref(ncx), C.byref(ncy), dptr(w), w.size)
    return ncx.value, ncy.value, w.reshape(9, ncy.value, ncx.value)


# ---- projection ----------------------------------------------------------------
class DeviceState:
    """FluidState<double> resident in HBM (ismg_state)."""

    def __init__(self, g: GridSpec, ctx: Optional[Context] = None, host: Optional[FluidState] = None):
        self.ctx = ctx or Context.default()
        self.g = g.copy()
        self._gc = g.to_c()
        h = C.c_void_p()
        _lib.call("ismg_state_create", self.ctx.h, C.byref(self._gc), C.byref(h))
        self.h = h
        if host is not None:
            self.upload(host)

    def upload(self, st: FluidState) -> None:
        _lib.call("ismg_state_upload", self.h, dptr(st.vel.u_data), st.vel.u_data.size, dptr(st.vel.v_data),
                  st.vel.v_data.size, dptr(st.p.data), st.p.data.size)
        _lib.call("ismg_state_set_scalars", self.h, st.t, st.dt, st.nu, st.step_count)

    def download(self, st: Optional[FluidState] = None) -> FluidState:
        st = st or FluidState(self.g)
        _lib.call("ismg_state_download", self.h, dptr(st.vel.u_data), st.vel.u_data.size, dptr(st.vel.v_data),
                  st.vel.v_data.size, dptr(st.p.data), st.p.data.size)
        t, dt, nu, sc = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        _lib.call("ismg_state_get_scalars", self.h, C.byref(t), C.byref(dt), C.byref(nu), C.byref(sc))
        st.t, st.dt, st.nu, st.step_count = t.value, dt.value, nu.value, sc.value
        return st

    def scalars(self):
        t, dt, nu, sc = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        _lib.call("ismg_state_get_scalars", self.h, C.byref(t), C.byref(dt), C.byref(nu), C.byref(sc))
        return t.value, dt.value, nu.value, sc.value

    def step(self, solver: PressureSolver, m: RunMetrics) -> ConvergenceReport:
        rep = CReport()
        cur = m.current.to_c()
        _lib.call("ismg_step", self.h, solver.h, C.byref(rep), C.byref(cur), C.c_int64(m.fine_cells))
        m.current.load_c(cur)
        r = _report(rep)
        _, dt, _, sc = self.scalars()
        # metrics.hpp:61-67 via projection.hpp:164 / :188
        m.close_timestep(sc, 0.0 if dt == 0.0 else r.residual, True if dt == 0.0 else r.converged)
        return r

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().ismg_state_destroy(self.h)
        except Exception:
            pass


def step(st, g: GridSpec, solver: PressureSolver, m: RunMetrics) -> ConvergenceReport:
    """projection.hpp:139-190. `st` is a DeviceState (stays in HBM) or a host
    FluidState (uploaded, stepped on the device, downloaded)."""
    if isinstance(st, DeviceState):
        return st.step(solver, m)
    ds = DeviceState(g, solver.ctx, st)
    rep = ds.step(solver, m)
    ds.download(st)
    return rep


def apply_scalar_bc(f: DeviceField, g: GridSpec) -> None:
    gc = g.to_c()
    _lib.call("ismg_apply_scalar_bc", f.ctx.h, C.byref(gc), f.h)


def apply_velocity_bc(v: DeviceVelocity, g: GridSpec) -> None:
    gc = g.to_c()
    _lib.call("ismg_apply_velocity_bc", v.ctx.h, C.byref(gc), v.h)


def divergence(v: DeviceVelocity, g: GridSpec, out: DeviceField, scale: float = 1.0) -> None:
    gc = g.to_c()
    _lib.call("ismg_divergence", v.ctx.h, C.byref(gc), v.h, out.h, float(scale))


def correct(v: DeviceVelocity, dp: DeviceField, dt: float, g: GridSpec) -> None:
    gc = g.to_c()
    _lib.call("ismg_correct", v.ctx.h, C.byref(gc), v.h, dp.h, float(dt))


def predictor(v: DeviceVelocity, p: DeviceField, dt: float, nu: float, g: GridSpec, out: DeviceVelocity) -> None:
    gc = g.to_c()
    _lib.call("ismg_predictor", v.ctx.h, C.byref(gc), v.h, p.h, float(dt), float(nu), out.h)


class CaseResult:
    def __init__(self, g: GridSpec):
        self.metrics = RunMetrics(1)
        self.state = FluidState(g)
        self.all_converged = True
        self.steps_run = 0


def run_case(bc: BenchmarkCase, cfg: CycleConfig, hook: Optional[Callable] = None,
             ctx: Optional[Context] = None) -> CaseResult:
    """bench.hpp:127-158 with the state resident in HBM between steps."""
    bc.grid.validate()
    solver = PressureSolver(bc.grid, cfg, ctx)
    out = CaseResult(bc.grid)
    out.state.dt, out.state.nu = bc.dt, bc.nu
    out.metrics = RunMetrics(bc.grid.nx * bc.grid.ny)
    if bc.seed != 0:
        raise NotImplementedError("seeded perturbation (std::mt19937_64) is not reproduced; use seed = 0")
    ds = DeviceState(bc.grid, solver.ctx, out.state)
    prev = None
    for _ in range(bc.steps):
        t, _, _, _ = ds.scalars()
        if bc.t_max > 0.0 and t >= bc.t_max:
            break
        if bc.steady_tol > 0.0:
            prev = ds.download().vel
        rep = ds.step(solver, out.metrics)
        out.all_converged = out.all_converged and rep.converged
        out.steps_run += 1
        if hook is not None or bc.steady_tol > 0.0:
            ds.download(out.state)
        if hook is not None:
            hook(out.state, rep)
        if bc.steady_tol > 0.0 and out.state.vel.max_change(prev) < bc.steady_tol:
            break
    ds.download(out.state)
    return out

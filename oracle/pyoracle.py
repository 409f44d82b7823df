"""ctypes loader for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two interchangeable back ends with one Python surface:
  * `Oracle("port")`      -> oracle/libismg_oracle.so, the plain-C restatement;
  * `Oracle("reference")` -> oracle/_ref/libismg_ref.so, the unmodified reference
                              compiled from its own headers (oracle/build.sh).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may use this module — as the checker, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))

from paper_1309_7128_b200._abi import (  # noqa: E402
    CCycleConfig, CGridSpec, CReport, CStepMetrics, DP, dptr)
from paper_1309_7128_b200.api import (  # noqa: E402
    ConvergenceReport, CycleConfig, GridSpec, MacVelocity, ScalarField, StepMetrics)

PORT_PATH = os.path.join(_HERE, "libismg_oracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libismg_ref.so")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("oracle error %d: %s" % (code, msg))
        self.code = code


def available(kind: str) -> bool:
    return os.path.exists(PORT_PATH if kind == "port" else REF_PATH)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_PATH if kind == "port" else REF_PATH
        if not os.path.exists(path):
            raise FileNotFoundError("oracle library missing: %s (run oracle/build.sh)" % path)
        self.lib = C.CDLL(path)
        self.p = "orc_" if kind == "port" else "ref_"
        L, p = self.lib, self.p
        G, CF = C.POINTER(CGridSpec), C.POINTER(CCycleConfig)
        getattr(L, p + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc: int):
        if rc != 0:
            msg = self._fn("last_error")().decode()
            raise OracleError(rc, msg)

    # -- fine level ----------------------------------------------------------
    def rbgs_sweep(self, g: GridSpec, x: ScalarField, b: ScalarField) -> None:
        gc = g.to_c()
        self._check(self._fn("rbgs_sweep")(C.byref(gc), dptr(x.data), dptr(b.data)))

    def fine_residual(self, g: GridSpec, x: ScalarField, b: ScalarField, out: ScalarField | None = None) -> float:
        gc = g.to_c()
        o = dptr(out.data) if out is not None else None
        if self.kind == "port":
            f = self._fn("fine_residual")
            f.restype = C.c_double
            return float(f(C.byref(gc), dptr(x.data), dptr(b.data), o))
        r = C.c_double()
        self._check(self._fn("fine_residual")(C.byref(gc), dptr(x.data), dptr(b.data), o, C.byref(r)))
        return r.value

    def anchor_mean(self, g: GridSpec, x: ScalarField) -> None:
        gc = g.to_c()
        self._fn("anchor_mean")(C.byref(gc), dptr(x.data))

    def build_fine_diag(self, g: GridSpec) -> ScalarField:
        gc = g.to_c()
        d = ScalarField(g.nx, g.ny)
        self._check(self._fn("build_fine_diag")(C.byref(gc), dptr(d.data)))
        return d

    # -- coarse operators ------------------------------------------------------
    def _build(self, which: str, g: GridSpec):
        gc = g.to_c()
        ncx, ncy = C.c_int32(), C.c_int32()
        if self.kind == "port":
            self._check(self._fn("ismg_dims")(C.byref(gc), C.byref(ncx), C.byref(ncy)))
            w = np.zeros(9 * ncx.value * ncy.value)
            self._check(self._fn("build_%s_operator" % which)(C.byref(gc), dptr(w)))
        else:
            self._check(self._fn("build_%s_operator" % which)(C.byref(gc), C.byref(ncx), C.byref(ncy), None))
            w = np.zeros(9 * ncx.value * ncy.value)
            self._check(self._fn("build_%s_operator" % which)(C.byref(gc), C.byref(ncx), C.byref(ncy), dptr(w)))
        return ncx.value, ncy.value, w.reshape(9, ncy.value, ncx.value)

    def build_ismg_operator(self, g: GridSpec):
        return self._build("ismg", g)

    def build_gmg_operator(self, g: GridSpec):
        return self._build("gmg", g)

    def restrict_sum(self, g: GridSpec, fine: ScalarField, coarse: ScalarField) -> None:
        gc = g.to_c()
        self._fn("restrict_sum")(C.byref(gc), dptr(fine.data), dptr(coarse.data))

    def prolongate_bilinear(self, g: GridSpec, coarse: ScalarField, fine: ScalarField) -> None:
        gc = g.to_c()
        self._fn("prolongate_bilinear")(C.byref(gc), dptr(coarse.data), dptr(fine.data))

    def coarse_residual(self, w, px, py, five, x: ScalarField, b: ScalarField, out: ScalarField | None = None) -> float:
        w = np.ascontiguousarray(w, dtype=np.float64)
        o = dptr(out.data) if out is not None else None
        if self.kind == "port":
            f = self._fn("coarse_residual")
            f.restype = C.c_double
            return float(f(x.nx, x.ny, int(px), int(py), int(five), dptr(w), dptr(x.data), dptr(b.data), o))
        r = C.c_double()
        self._check(self._fn("coarse_residual")(x.nx, x.ny, int(px), int(py), int(five), dptr(w), dptr(x.data),
                                                dptr(b.data), o, C.byref(r)))
        return r.value

    def gs_sweep_lex(self, w, px, py, five, x: ScalarField, b: ScalarField) -> None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        self._check(self._fn("gs_sweep_lex")(x.nx, x.ny, int(px), int(py), int(five), dptr(w), dptr(x.data),
                                             dptr(b.data)))

    # -- solves ---------------------------------------------------------------
    def solve(self, g: GridSpec, cfg: CycleConfig, x: ScalarField, b: ScalarField,
              current: StepMetrics | None = None, fine_cells: int | None = None):
        """PressureSolver(g, cfg).solve(x, b, m); returns (report, current, seconds|None)."""
        gc, cc = g.to_c(), cfg.to_c()
        rep = CReport()
        cur = (current or StepMetrics()).to_c()
        fc = fine_cells if fine_cells is not None else g.nx * g.ny
        secs = C.c_double(-1.0)
        if self.kind == "port":
            self._check(self._fn("solve")(C.byref(gc), C.byref(cc), dptr(x.data), dptr(b.data), C.byref(rep),
                                          C.byref(cur), C.c_int64(fc)))
        else:
            self._check(self._fn("solve")(C.byref(gc), C.byref(cc), dptr(x.data), dptr(b.data), C.byref(rep),
                                          C.byref(cur), C.c_int64(fc), C.byref(secs)))
        out = StepMetrics()
        out.load_c(cur)
        r = ConvergenceReport(bool(rep.converged), rep.fine_sweeps, rep.coarse_sweeps, rep.residual)
        return r, out, (secs.value if secs.value >= 0 else None)

    # -- projection -------------------------------------------------------------
    def apply_scalar_bc(self, g: GridSpec, f: ScalarField) -> None:
        gc = g.to_c()
        self._fn("apply_scalar_bc")(C.byref(gc), dptr(f.data))

    def apply_velocity_bc(self, g: GridSpec, vel: MacVelocity) -> None:
        gc = g.to_c()
        self._fn("apply_velocity_bc")(C.byref(gc), dptr(vel.u_data), dptr(vel.v_data))

    def divergence(self, g: GridSpec, vel: MacVelocity, out: ScalarField) -> None:
        gc = g.to_c()
        self._fn("divergence")(C.byref(gc), dptr(vel.u_data), dptr(vel.v_data), dptr(out.data))

    def correct(self, g: GridSpec, vel: MacVelocity, dp: ScalarField, dt: float) -> None:
        gc = g.to_c()
        self._fn("correct")(C.byref(gc), dptr(vel.u_data), dptr(vel.v_data), dptr(dp.data), C.c_double(dt))

    def predictor(self, g: GridSpec, vel: MacVelocity, p: ScalarField, dt: float, nu: float, out: MacVelocity):
        gc = g.to_c()
        self._fn("predictor")(C.byref(gc), dptr(vel.u_data), dptr(vel.v_data), dptr(p.data), C.c_double(dt),
                              C.c_double(nu), dptr(out.u_data), dptr(out.v_data))

    def op_costs(self, g: GridSpec, cfg: CycleConfig, dt: float, nu: float, reps: int = 1):
        """Reference only (ref_op_costs, oracle/ref_shim.cpp): seconds per call of
        rbgs_sweep, fine_residual(+store), anchor_mean, restrict_sum,
        prolongate_bilinear, gs_sweep_lex, coarse_residual, coarse anchor_mean,
        and one step() from rest with a 1-sweep budget (the per-step fixed cost)."""
        if self.kind == "port":
            raise OracleError(-1, "op_costs: reference library only")
        gc, cc = g.to_c(), cfg.to_c()
        out = np.zeros(9)
        self._check(self._fn("op_costs")(C.byref(gc), C.byref(cc), C.c_double(dt), C.c_double(nu), C.c_int(reps),
                                         dptr(out)))
        return out

    def run_steps(self, g: GridSpec, cfg: CycleConfig, state, nsteps: int):
        """run_case with seed 0 / no steady exit: returns (rows, seconds|None); state updated in place."""
        gc, cc = g.to_c(), cfg.to_c()
        scal = np.array([state.t, state.dt, state.nu, float(state.step_count)])
        rows = (CStepMetrics * max(nsteps, 1))()
        secs = C.c_double(-1.0)
        args = [C.byref(gc), C.byref(cc), dptr(state.vel.u_data), dptr(state.vel.v_data), dptr(state.p.data),
                dptr(scal), C.c_long(nsteps), rows]
        if self.kind != "port":
            args.append(C.byref(secs))
        self._check(self._fn("run_steps")(*args))
        state.t, state.step_count = float(scal[0]), int(scal[3])
        out = []
        for k in range(nsteps):
            s = StepMetrics()
            s.load_c(rows[k])
            out.append(s)
        return out, (secs.value if secs.value >= 0 else None)

"""Host-side value types mirroring the reference's C++ API (namespace ismg).

Same names, fields, defaults and validation errors as the reference headers so
that callers (and the parity tests) read like the reference's own code:

  Side, BcKind, BoundaryCondition, GridSpec, padded_dims   grid.hpp:18-117
  PressureBcKind, pressure_bc, pressure_singular           grid.hpp:119-149
  ScalarField, MacVelocity                                  field.hpp:18-137
  Scheme, CycleConfig, ConvergenceReport, NonConvergence   coarsening.hpp:27, cycles.hpp:20-69
  StepMetrics, RunMetrics, write_metrics_csv, write_summary metrics.hpp:22-139
  FluidState                                                projection.hpp:26-36
  BenchmarkCase, setup_*                                    bench.hpp:22-109

Fields are host numpy arrays with the reference's ghosted row-major layout;
the compute lives behind the C-ABI (see solver.py).
"""
from __future__ import annotations

import copy
import enum
import io
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._abi import CBc, CCycleConfig, CGridSpec


class Side(enum.IntEnum):
    west = 0
    east = 1
    south = 2
    north = 3


all_sides = (Side.west, Side.east, Side.south, Side.north)


class BcKind(enum.IntEnum):
    dirichlet_velocity = 0
    symmetry_fixed_pressure = 1
    periodic = 2
    inlet = 3


class PressureBcKind(enum.IntEnum):
    neumann = 0
    dirichlet_zero = 1
    periodic = 2


class Scheme(enum.IntEnum):
    plain_gs = 0
    ismg = 1
    gmg = 2
    acm = 3


def scheme_name(s: Scheme) -> str:
    """coarsening.hpp:29-37"""
    return {Scheme.plain_gs: "plain", Scheme.ismg: "ismg", Scheme.gmg: "gmg", Scheme.acm: "acm"}[Scheme(s)]


@dataclass
class BoundaryCondition:
    """grid.hpp:30-65"""

    kind: BcKind = BcKind.dirichlet_velocity
    u_wall: float = 0.0
    v_wall: float = 0.0
    p_wall: float = 0.0
    v_inflow: float = 0.0
    inlet_start: int = 0
    inlet_width: int = 0

    @staticmethod
    def no_slip() -> "BoundaryCondition":
        return BoundaryCondition()

    @staticmethod
    def moving_wall(u: float, v: float) -> "BoundaryCondition":
        return BoundaryCondition(u_wall=u, v_wall=v)

    @staticmethod
    def symmetry(p: float = 0.0) -> "BoundaryCondition":
        return BoundaryCondition(kind=BcKind.symmetry_fixed_pressure, p_wall=p)

    @staticmethod
    def wrap() -> "BoundaryCondition":
        return BoundaryCondition(kind=BcKind.periodic)

    @staticmethod
    def inflow(v: float, start: int, width: int) -> "BoundaryCondition":
        return BoundaryCondition(kind=BcKind.inlet, v_inflow=v, inlet_start=start, inlet_width=width)

    def to_c(self) -> CBc:
        return CBc(int(self.kind), int(self.inlet_start), int(self.inlet_width), 0,
                   float(self.u_wall), float(self.v_wall), float(self.p_wall), float(self.v_inflow))


@dataclass
class GridSpec:
    """grid.hpp:67-97"""

    nx: int = 0
    ny: int = 0
    h: float = 1.0
    tile: int = 16
    bc: List[BoundaryCondition] = field(default_factory=lambda: [BoundaryCondition() for _ in range(4)])

    def side(self, s: Side) -> BoundaryCondition:
        return self.bc[int(s)]

    def set_side(self, s: Side, b: BoundaryCondition) -> "GridSpec":
        self.bc[int(s)] = b
        return self

    def validate(self) -> None:
        """grid.hpp:79-96 (raises ValueError where the reference throws invalid_argument)."""
        if self.nx < 1 or self.ny < 1:
            raise ValueError("grid: nx, ny must be >= 1")
        if self.h <= 0.0:
            raise ValueError("grid: h must be positive")
        if self.tile < 2:
            raise ValueError("grid: tile must be >= 2")
        per = lambda s: self.side(s).kind == BcKind.periodic  # noqa: E731
        if per(Side.west) != per(Side.east):
            raise ValueError("grid: periodic west/east must pair")
        if per(Side.south) != per(Side.north):
            raise ValueError("grid: periodic south/north must pair")
        for s in all_sides:
            b = self.side(s)
            if b.kind != BcKind.inlet:
                continue
            extent = self.nx if s in (Side.south, Side.north) else self.ny
            if b.inlet_width < 1 or b.inlet_start < 0 or b.inlet_start + b.inlet_width > extent:
                raise ValueError("grid: inlet span out of range")

    def to_c(self) -> CGridSpec:
        g = CGridSpec()
        g.nx, g.ny, g.h, g.tile = int(self.nx), int(self.ny), float(self.h), int(self.tile)
        for k in range(4):
            g.bc[k] = self.bc[k].to_c()
        return g

    def copy(self) -> "GridSpec":
        return copy.deepcopy(self)


@dataclass
class PaddedDims:
    padded_nx: int = 0
    padded_ny: int = 0
    last_tile_w: int = 0
    last_tile_h: int = 0


def padded_dims(g: GridSpec) -> PaddedDims:
    """grid.hpp:108-117"""
    tcx = (g.nx + g.tile - 1) // g.tile
    tcy = (g.ny + g.tile - 1) // g.tile
    return PaddedDims(tcx * g.tile, tcy * g.tile, g.nx - (tcx - 1) * g.tile, g.ny - (tcy - 1) * g.tile)


def pressure_bc(g: GridSpec) -> List[PressureBcKind]:
    """grid.hpp:124-141"""
    out = []
    for s in all_sides:
        k = g.side(s).kind
        if k in (BcKind.dirichlet_velocity, BcKind.inlet):
            out.append(PressureBcKind.neumann)
        elif k == BcKind.symmetry_fixed_pressure:
            out.append(PressureBcKind.dirichlet_zero)
        else:
            out.append(PressureBcKind.periodic)
    return out


def pressure_singular(bc: List[PressureBcKind]) -> bool:
    """grid.hpp:145-149"""
    return all(k != PressureBcKind.dirichlet_zero for k in bc)


# --------------------------------------------------------------------------
# fields (field.hpp)


class ScalarField:
    """Cell-centred scalar with a one-cell ghost ring (field.hpp:18-71).

    `data` is the flat (nx+2)*(ny+2) float64 array in the reference layout;
    `grid` is a (ny+2, nx+2) view so that grid[j+1, i+1] == f(i, j).
    """

    def __init__(self, nx: int = 0, ny: int = 0, data: np.ndarray | None = None):
        self.nx, self.ny = int(nx), int(ny)
        if data is None:
            self.data = np.zeros((self.nx + 2) * (self.ny + 2), dtype=np.float64)
        else:
            self.data = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
            assert self.data.size == (self.nx + 2) * (self.ny + 2)

    @property
    def grid(self) -> np.ndarray:
        return self.data.reshape(self.ny + 2, self.nx + 2)

    def interior(self) -> np.ndarray:
        """(ny, nx) view of the interior, indexed [j, i]."""
        return self.grid[1:-1, 1:-1]

    def __call__(self, i: int, j: int) -> float:
        return float(self.grid[j + 1, i + 1])

    def set(self, i: int, j: int, v: float) -> None:
        self.grid[j + 1, i + 1] = v

    def stride(self) -> int:
        return self.nx + 2

    def fill(self, v: float) -> None:
        self.data[:] = v

    def fill_interior(self, v: float) -> None:
        self.interior()[:] = v

    def interior_sum(self) -> float:
        """Serial row-major sum (field.hpp:41-48)."""
        s = 0.0
        for v in self.interior().reshape(-1).tolist():
            s += v
        return s

    def interior_mean(self) -> float:
        return self.interior_sum() / float(self.nx * self.ny)

    def interior_max_abs(self) -> float:
        return float(np.max(np.abs(self.interior()))) if self.nx * self.ny else 0.0

    def shift_interior(self, c: float) -> None:
        self.interior()[:] += c

    def add_interior(self, o: "ScalarField") -> None:
        self.interior()[:] += o.interior()

    def copy(self) -> "ScalarField":
        return ScalarField(self.nx, self.ny, self.data.copy())


class MacVelocity:
    """Staggered velocity (field.hpp:102-137): u (nx+3)*(ny+2), v (nx+2)*(ny+3)."""

    def __init__(self, nx: int = 0, ny: int = 0):
        self.nx, self.ny = int(nx), int(ny)
        self.u_data = np.zeros((self.nx + 3) * (self.ny + 2), dtype=np.float64)
        self.v_data = np.zeros((self.nx + 2) * (self.ny + 3), dtype=np.float64)

    @property
    def u_grid(self) -> np.ndarray:
        return self.u_data.reshape(self.ny + 2, self.nx + 3)

    @property
    def v_grid(self) -> np.ndarray:
        return self.v_data.reshape(self.ny + 3, self.nx + 2)

    def u(self, i: int, j: int) -> float:
        return float(self.u_grid[j + 1, i + 1])

    def v(self, i: int, j: int) -> float:
        return float(self.v_grid[j + 1, i + 1])

    def max_abs(self) -> float:
        """field.hpp:180-187 (faces the time step owns, ghosts excluded)."""
        ug = np.abs(self.u_grid[1:self.ny + 1, 1:self.nx + 2])
        vg = np.abs(self.v_grid[1:self.ny + 2, 1:self.nx + 1])
        return float(max(ug.max(initial=0.0), vg.max(initial=0.0)))

    def max_change(self, o: "MacVelocity") -> float:
        du = np.abs(self.u_grid[1:self.ny + 1, 1:self.nx + 2] - o.u_grid[1:self.ny + 1, 1:self.nx + 2])
        dv = np.abs(self.v_grid[1:self.ny + 2, 1:self.nx + 1] - o.v_grid[1:self.ny + 2, 1:self.nx + 1])
        return float(max(du.max(initial=0.0), dv.max(initial=0.0)))

    def copy(self) -> "MacVelocity":
        m = MacVelocity(self.nx, self.ny)
        m.u_data[:] = self.u_data
        m.v_data[:] = self.v_data
        return m


# --------------------------------------------------------------------------
# cycles.hpp


@dataclass
class CycleConfig:
    """cycles.hpp:20-45"""

    scheme: Scheme = Scheme.ismg
    tile: int = 16
    depth: int = 4
    tol_fine: float = 1e-6
    tol_coarse: float = 1e-5
    max_total_sweeps: int = 20000
    acm_pre_smooth: int = 0
    acm_post_smooth: int = 1
    stall_factor: float = 0.9

    def validate(self) -> None:
        if not (self.tol_fine > 0) or not (self.tol_coarse > 0):
            raise ValueError("cycle: tolerances must be positive")
        if self.tol_coarse < self.tol_fine:
            raise ValueError("cycle: tol_coarse must be >= tol_fine")
        if self.max_total_sweeps < 1:
            raise ValueError("cycle: max_total_sweeps must be positive")
        if not (0.0 < self.stall_factor < 1.0):
            raise ValueError("cycle: stall_factor must lie in (0,1)")
        if self.acm_pre_smooth < 0 or self.acm_post_smooth < 0:
            raise ValueError("cycle: smoothing counts must be non-negative")
        if self.depth < 2:
            raise ValueError("cycle: depth must be >= 2")
        if self.tile < 2:
            raise ValueError("cycle: tile must be >= 2")

    def to_c(self) -> CCycleConfig:
        c = CCycleConfig()
        c.scheme, c.tile, c.depth = int(self.scheme), int(self.tile), int(self.depth)
        c.acm_pre_smooth, c.acm_post_smooth = int(self.acm_pre_smooth), int(self.acm_post_smooth)
        c.tol_fine, c.tol_coarse = float(self.tol_fine), float(self.tol_coarse)
        c.max_total_sweeps, c.stall_factor = int(self.max_total_sweeps), float(self.stall_factor)
        return c


@dataclass
class ConvergenceReport:
    """cycles.hpp:47-52"""

    converged: bool = True
    fine_sweeps: int = 0
    coarse_sweeps: int = 0
    residual: float = 0.0
    nan_seen: bool = False


class NonConvergence(RuntimeError):
    """cycles.hpp:56-69"""

    def __init__(self, iterations: int, final_residual: float):
        super().__init__(
            "pressure solve not converged after %d sweeps (residual %.3e)" % (iterations, final_residual))
        self.iterations = iterations
        self.final_residual = final_residual


# --------------------------------------------------------------------------
# metrics.hpp


class LevelKind(enum.IntEnum):
    fine = 0
    coarse = 1


@dataclass
class StepMetrics:
    """metrics.hpp:22-35"""

    step: int = 0
    fine_sweeps: int = 0
    coarse_sweeps: int = 0
    sync_fine: int = 0
    sync_coarse: int = 0
    lap_equiv: float = 0.0
    restrictions: int = 0
    prolongations: int = 0
    residual_final: float = 0.0
    converged: bool = True

    def sync_total(self) -> int:
        return self.sync_fine + self.sync_coarse

    _FIELDS = ("step", "fine_sweeps", "coarse_sweeps", "sync_fine", "sync_coarse", "lap_equiv",
               "restrictions", "prolongations", "residual_final")

    def to_c(self):
        from ._abi import CStepMetrics
        c = CStepMetrics()
        for f in self._FIELDS:
            setattr(c, f, getattr(self, f))
        c.converged = 1 if self.converged else 0
        return c

    def load_c(self, c) -> None:
        for f in self._FIELDS:
            setattr(self, f, getattr(c, f))
        self.converged = bool(c.converged)


@dataclass
class Means:
    fine_sweeps: float = 0.0
    coarse_sweeps: float = 0.0
    sync_fine: float = 0.0
    sync_coarse: float = 0.0
    sync_total: float = 0.0
    lap_equiv: float = 0.0
    all_converged: bool = True


class RunMetrics:
    """metrics.hpp:39-100: per-sweep cost accounting closed into per-step rows."""

    def __init__(self, fine_cells_total: int = 1):
        self.fine_cells = int(fine_cells_total)
        self.current = StepMetrics()
        self.rows: List[StepMetrics] = []

    def record_sweep(self, kind: LevelKind, stencil_points: int, cells: int) -> None:
        if kind == LevelKind.fine:
            self.current.fine_sweeps += 1
            self.current.sync_fine += 2
        else:
            self.current.coarse_sweeps += 1
            self.current.sync_coarse += 1
        self.current.lap_equiv += (float(cells) / float(self.fine_cells)) * (float(stencil_points) / 5.0)

    def record_restriction(self) -> None:
        self.current.restrictions += 1

    def record_prolongation(self) -> None:
        self.current.prolongations += 1

    def close_timestep(self, step: int, residual_final: float, converged: bool) -> None:
        self.current.step = step
        self.current.residual_final = residual_final
        self.current.converged = converged
        self.rows.append(self.current)
        self.current = StepMetrics()

    def window_means(self, window: int) -> Means:
        m = Means()
        if not self.rows or window == 0:
            return m
        window = min(window, len(self.rows))
        for r in self.rows[len(self.rows) - window:]:
            m.fine_sweeps += float(r.fine_sweeps)
            m.coarse_sweeps += float(r.coarse_sweeps)
            m.sync_fine += float(r.sync_fine)
            m.sync_coarse += float(r.sync_coarse)
            m.lap_equiv += r.lap_equiv
            m.all_converged = m.all_converged and r.converged
        inv = 1.0 / float(window)
        m.fine_sweeps *= inv
        m.coarse_sweeps *= inv
        m.sync_fine *= inv
        m.sync_coarse *= inv
        m.lap_equiv *= inv
        m.sync_total = m.sync_fine + m.sync_coarse
        return m


def _g10(v: float) -> str:
    return "%.10g" % v


def write_metrics_csv(m: RunMetrics, os: io.TextIOBase | None = None) -> str:
    """metrics.hpp:102-113 (same header and number formats)."""
    out = ["step,I_f,I_c,NCC_f,NCC_c,NCC_t,N_Lap,restrictions,prolongations,residual_final\n"]
    for r in m.rows:
        out.append("%d,%d,%d,%d,%d,%d,%s,%d,%d,%s\n" % (
            r.step, r.fine_sweeps, r.coarse_sweeps, r.sync_fine, r.sync_coarse, r.sync_total(),
            _g10(r.lap_equiv), r.restrictions, r.prolongations, _g10(r.residual_final)))
    s = "".join(out)
    if os is not None:
        os.write(s)
    return s


def write_summary(m: RunMetrics, window: int, os: io.TextIOBase | None = None) -> str:
    """metrics.hpp:123-139"""
    w = m.window_means(window)
    lines = ["steps = %d\n" % len(m.rows), "window = %d\n" % window]
    for key, v in (("mean_I_f", w.fine_sweeps), ("mean_I_c", w.coarse_sweeps), ("mean_NCC_f", w.sync_fine),
                   ("mean_NCC_c", w.sync_coarse), ("mean_NCC_t", w.sync_total), ("mean_N_Lap", w.lap_equiv)):
        lines.append("%s = %s\n" % (key, _g10(v)))
    lines.append("all_converged = %s\n" % ("true" if w.all_converged else "false"))
    s = "".join(lines)
    if os is not None:
        os.write(s)
    return s


# --------------------------------------------------------------------------
# io.hpp: snapshot and diagnostic output (same formats as the reference)


def _open(path):
    try:
        return open(path, "w", newline="\n")
    except OSError as e:
        raise RuntimeError("io: cannot open '%s' for writing" % path) from e


def write_field_csv(f: "ScalarField", g: "GridSpec", path: str) -> None:
    """io.hpp:35-50: header `nx,ny,h`, its values, then one row of interior
    values per grid row (south to north), `%.10g`."""
    with _open(path) as os_:
        os_.write("nx,ny,h\n%d,%d,%s\n" % (g.nx, g.ny, _g10(g.h)))
        a = f.interior()
        for j in range(g.ny):
            os_.write(",".join(_g10(float(v)) for v in a[j]) + "\n")


def write_vtk(p: "ScalarField", vel: "MacVelocity", g: "GridSpec", path: str) -> None:
    """io.hpp:54-94: legacy ASCII VTK structured points over cell centres, the
    pressure and the face-averaged velocity."""
    with _open(path) as os_:
        w = os_.write
        w("# vtk DataFile Version 3.0\nismg snapshot\nASCII\nDATASET STRUCTURED_POINTS\n")
        w("DIMENSIONS %d %d 1\n" % (g.nx, g.ny))
        w("ORIGIN %s %s 0\n" % (_g10(0.5 * g.h), _g10(0.5 * g.h)))
        w("SPACING %s %s 1\n" % (_g10(g.h), _g10(g.h)))
        w("POINT_DATA %d\nSCALARS pressure double 1\nLOOKUP_TABLE default\n" % (g.nx * g.ny))
        a = p.interior()
        for j in range(g.ny):
            w("".join(_g10(float(v)) + "\n" for v in a[j]))
        w("VECTORS velocity double\n")
        U, V = vel.u_grid, vel.v_grid
        for j in range(g.ny):
            for i in range(g.nx):
                uc = 0.5 * (float(U[j + 1, i + 1]) + float(U[j + 1, i + 2]))
                vc = 0.5 * (float(V[j + 1, i + 1]) + float(V[j + 2, i + 1]))
                w("%s %s 0\n" % (_g10(uc), _g10(vc)))


def write_operator_csv(ncx: int, ncy: int, w, path_or_stream) -> str:
    """io.hpp:97-117: per-cell stencil rows `ci,cj,C,E,W,N,S,NE,NW,SE,SW`,
    `%.17g` (exact). `w` is the (9, ncy, ncx) plane stack of build_ismg_operator."""
    import numpy as _np
    w = _np.asarray(w).reshape(9, ncy, ncx)
    out = ["ci,cj,C,E,W,N,S,NE,NW,SE,SW\n"]
    for J in range(ncy):
        for I in range(ncx):
            out.append("%d,%d,%s\n" % (I, J, ",".join("%.17g" % float(w[sl, J, I]) for sl in range(9))))
    s = "".join(out)
    if isinstance(path_or_stream, str):
        with _open(path_or_stream) as os_:
            os_.write(s)
    elif path_or_stream is not None:
        path_or_stream.write(s)
    return s


# --------------------------------------------------------------------------
# projection.hpp / bench.hpp


class FluidState:
    """projection.hpp:26-36"""

    def __init__(self, g: GridSpec):
        self.vel = MacVelocity(g.nx, g.ny)
        self.p = ScalarField(g.nx, g.ny)
        self.t = 0.0
        self.dt = 1.0
        self.nu = 0.1
        self.step_count = 0


@dataclass
class BenchmarkCase:
    """bench.hpp:22-32"""

    name: str = ""
    grid: GridSpec = field(default_factory=GridSpec)
    nu: float = 0.1
    dt: float = 1.0
    steps: int = 1000
    window: int = 1000
    steady_tol: float = 0.0
    t_max: float = 0.0
    seed: int = 0


def setup_shear_cavity(n: int = 500, v0: float = 0.1) -> BenchmarkCase:
    """bench.hpp:37-51"""
    c = BenchmarkCase(name="shear_cavity")
    c.grid.nx = c.grid.ny = n
    c.grid.h = 1.0
    c.grid.set_side(Side.west, BoundaryCondition.moving_wall(0.0, v0))
    c.grid.set_side(Side.east, BoundaryCondition.moving_wall(0.0, v0))
    c.grid.set_side(Side.south, BoundaryCondition.moving_wall(v0, 0.0))
    c.grid.set_side(Side.north, BoundaryCondition.moving_wall(-v0, 0.0))
    c.nu, c.dt, c.steps, c.window = 0.1, 1.0, 1000, 1000
    return c


def setup_lid_cavity(n: int = 256, re: float = 1000.0, u_lid: float = 0.1) -> BenchmarkCase:
    """bench.hpp:56-69"""
    c = BenchmarkCase(name="lid_cavity")
    c.grid.nx = c.grid.ny = n
    c.grid.h = 1.0
    c.grid.set_side(Side.north, BoundaryCondition.moving_wall(u_lid, 0.0))
    c.nu = u_lid * n * c.grid.h / re
    c.dt, c.steps, c.t_max, c.steady_tol, c.window = 1.0, 40000, 40000.0, 1e-10, 1
    return c


def setup_jet(nx: int = 250, ny: int = 500, v0: float = 0.1, inlet_width: int = 16) -> BenchmarkCase:
    """bench.hpp:73-88"""
    c = BenchmarkCase(name="jet")
    c.grid.nx, c.grid.ny, c.grid.h = nx, ny, 1.0
    c.grid.set_side(Side.south, BoundaryCondition.inflow(v0, nx // 2 - inlet_width // 2, inlet_width))
    c.grid.set_side(Side.north, BoundaryCondition.symmetry(0.0))
    c.nu, c.dt, c.steps, c.window = 0.01, 1.0, 2000, 2000
    return c


def setup_channel_jets(nx: int = 200, ny: int = 400, v0: float = 0.1, inlet_width: int = 25) -> BenchmarkCase:
    """bench.hpp:92-109"""
    c = BenchmarkCase(name="channel_jets")
    c.grid.nx, c.grid.ny, c.grid.h = nx, ny, 1.0
    c.grid.set_side(Side.west, BoundaryCondition.wrap())
    c.grid.set_side(Side.east, BoundaryCondition.wrap())
    c.grid.set_side(Side.south, BoundaryCondition.inflow(v0, (nx - inlet_width) // 2, inlet_width))
    c.grid.set_side(Side.north, BoundaryCondition.symmetry(0.0))
    c.nu, c.dt, c.steps, c.window = 0.01, 1.0, 1000, 1000
    return c

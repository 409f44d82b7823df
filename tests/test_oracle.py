"""CPU oracle pinning (no GPU).

1. The reference's own known-answer tests, restated against the C port
   (test_smoother.cpp, test_coarsening.cpp, test_cycles.cpp, test_projection.cpp,
   test_metrics.cpp; file:line cited per test).
2. Golden vectors produced by the unmodified reference (tests/golden/golden.npz,
   generator tests/golden/make_golden.py) — bit-exact.
3. Port == reference bit-for-bit on fresh random cases, when oracle/_ref is built.
"""
import os

import numpy as np
import pytest

from cases import a3_rhs, cavity, golden_grids, periodic_flags, random_field, torus, with_side
from paper_1309_7128_b200.api import (
    BcKind, BoundaryCondition, CycleConfig, FluidState, GridSpec, RunMetrics, ScalarField, Scheme, Side,
    StepMetrics, setup_jet, setup_lid_cavity, write_metrics_csv)


# ---------------------------------------------------------------- KATs ------
def test_fine_diag_values(port):
    """test_smoother.cpp:71-93"""
    g = cavity(3, 3)
    d = port.build_fine_diag(g)
    assert d(0, 0) == 2.0 and d(1, 0) == 3.0 and d(1, 1) == 4.0
    g = with_side(g, Side.north, BoundaryCondition.symmetry(0.0))
    d = port.build_fine_diag(g)
    assert d(1, 2) == 5.0 and d(0, 0) == 2.0
    g = with_side(with_side(cavity(4, 3), Side.west, BoundaryCondition.wrap()), Side.east, BoundaryCondition.wrap())
    d = port.build_fine_diag(g)
    assert d(0, 1) == 4.0 and d(0, 0) == 3.0


def test_empty_stencil_is_domain_error(port):
    """test_smoother.cpp:95-98"""
    from pyoracle import OracleError
    with pytest.raises(OracleError) as e:
        port.build_fine_diag(cavity(1, 1))
    assert e.value.code == 2


def test_3x1_chain(port):
    """test_smoother.cpp:100-124: one sweep gives (0, 0.5, 0); 200 give (0.25, 0.75, 0.25)."""
    g = cavity(3, 1)
    g.set_side(Side.west, BoundaryCondition.symmetry(0.0)).set_side(Side.east, BoundaryCondition.symmetry(0.0))
    x, b = ScalarField(3, 1), ScalarField(3, 1)
    b.set(1, 0, -1.0)
    port.rbgs_sweep(g, x, b)
    assert (x(0, 0), x(1, 0), x(2, 0)) == (0.0, 0.5, 0.0)
    for _ in range(200):
        port.rbgs_sweep(g, x, b)
    assert np.allclose([x(0, 0), x(1, 0), x(2, 0)], [0.25, 0.75, 0.25], atol=1e-12)


def test_fine_residual_matches_dense(port):
    """test_smoother.cpp:186-220 (dense b - A x)."""
    rng = np.random.default_rng(13)
    for g in (cavity(6, 5), with_side(with_side(with_side(cavity(4, 6), Side.west, BoundaryCondition.wrap()),
                                                Side.east, BoundaryCondition.wrap()),
                                      Side.north, BoundaryCondition.symmetry(0.0))):
        x, b, r = random_field(g.nx, g.ny, rng), random_field(g.nx, g.ny, rng), ScalarField(g.nx, g.ny)
        rmax = port.fine_residual(g, x, b, r)
        A = dense_fine_matrix(g)
        xv = x.interior().reshape(-1)
        want = b.interior().reshape(-1) - A @ xv
        assert np.allclose(r.interior().reshape(-1), want, atol=1e-13)
        assert abs(rmax - np.abs(want).max()) < 1e-13


def dense_fine_matrix(g: GridSpec) -> np.ndarray:
    """oracles.hpp:43-76 fine_matrix."""
    from paper_1309_7128_b200.api import PressureBcKind, pressure_bc
    pbc = pressure_bc(g)
    nx, ny = g.nx, g.ny
    A = np.zeros((nx * ny, nx * ny))
    sides = [Side.west, Side.east, Side.south, Side.north]
    for j in range(ny):
        for i in range(nx):
            r = j * nx + i
            for d, (di, dj) in enumerate(((-1, 0), (1, 0), (0, -1), (0, 1))):
                ii, jj = i + di, j + dj
                if 0 <= ii < nx and 0 <= jj < ny:
                    A[r, jj * nx + ii] += 1.0
                    A[r, r] -= 1.0
                    continue
                k = pbc[int(sides[d])]
                if k == PressureBcKind.dirichlet_zero:
                    A[r, r] -= 2.0
                elif k == PressureBcKind.periodic:
                    A[r, ((jj + ny) % ny) * nx + (ii + nx) % nx] += 1.0
                    A[r, r] -= 1.0
    return A


def test_interior_ismg_stencil(port):
    """test_coarsening.cpp:136-149: interior rows C=-3, E/W/N/S=0.5, corners 0.25, any tile."""
    for tile in (4, 8, 16):
        g = cavity(8 * tile, 8 * tile, tile)
        ncx, ncy, w = port.build_ismg_operator(g)
        J = I = 4
        assert w[0, J, I] == -3.0
        assert all(w[s, J, I] == 0.5 for s in (1, 2, 3, 4))
        assert all(w[s, J, I] == 0.25 for s in (5, 6, 7, 8))


def test_ismg_equals_galerkin(port):
    """test_coarsening.cpp:151-170 / acceptance A2: ISMG == R A P."""
    from test_oracle import dense_fine_matrix as fm
    for g in [cavity(8, 8, 2), with_side(cavity(16, 16, 4), Side.north, BoundaryCondition.symmetry(0.0)),
              with_side(with_side(cavity(16, 12, 4), Side.west, BoundaryCondition.wrap()), Side.east,
                        BoundaryCondition.wrap()),
              with_side(with_side(cavity(20, 12, 8), Side.south, BoundaryCondition.inflow(0.1, 8, 4)), Side.north,
                        BoundaryCondition.symmetry(0.0))]:
        ncx, ncy, w = port.build_ismg_operator(g)
        A = fm(g)
        Rm, Pm = restriction_prolongation(g)
        G = Rm @ A @ Pm
        D = dense_from_planes(w, *periodic_flags(g))
        scale = max(1.0, np.abs(G).max())
        assert np.abs(D - G).max() / scale < 1e-12


def restriction_prolongation(g):
    """oracles.hpp:81-154 (R = tile sums, P = bilinear quadrant weights)."""
    px, py = periodic_flags(g)

    def axis(n, tile, per):
        nc = (n + tile - 1) // tile
        start = [k * tile for k in range(nc)]
        width = [tile if k < nc - 1 else n - k * tile for k in range(nc)]
        center = [start[k] + width[k] / 2.0 for k in range(nc)]
        W = np.zeros((n, nc))
        for i in range(n):
            c = i + 0.5
            if nc == 1:
                W[i, 0] = 1.0
            elif per and (c < center[0] or c >= center[-1]):
                dk = (width[-1] + width[0]) / 2.0
                t = c - center[-1]
                t = t + n if t < 0 else t
                s = t / dk
                W[i, nc - 1] += 1 - s
                W[i, 0] += s
            elif c <= center[0]:
                W[i, 0] = 1.0
            elif c >= center[-1]:
                W[i, nc - 1] = 1.0
            else:
                k = 0
                while center[k + 1] <= c:
                    k += 1
                s = (c - center[k]) / (center[k + 1] - center[k])
                W[i, k] += 1 - s
                W[i, k + 1] += s
        Rax = np.zeros((nc, n))
        for i in range(n):
            Rax[i // tile, i] = 1.0
        return W, Rax

    Wx, Rx = axis(g.nx, g.tile, px)
    Wy, Ry = axis(g.ny, g.tile, py)
    return np.kron(Ry, Rx), np.kron(Wy, Wx)


def dense_from_planes(w, px, py):
    """oracles.hpp:160-183 dense_from_operator."""
    _, ncy, ncx = w.shape
    di = [0, 1, -1, 0, 0, 1, -1, 1, -1]
    dj = [0, 0, 0, 1, -1, 1, 1, -1, -1]
    D = np.zeros((ncx * ncy, ncx * ncy))
    for J in range(ncy):
        for I in range(ncx):
            for s in range(9):
                if w[s, J, I] == 0.0:
                    continue
                II, JJ = I + di[s], J + dj[s]
                if px:
                    II %= ncx
                if py:
                    JJ %= ncy
                if 0 <= II < ncx and 0 <= JJ < ncy:
                    D[J * ncx + I, JJ * ncx + II] += w[s, J, I]
    return D


def test_restriction_short_tile(port):
    """test_coarsening.cpp:305-329: 36x4 tile 16 -> 64, 64, 16."""
    g = cavity(36, 4, 16)
    f = ScalarField(36, 4)
    f.fill_interior(1.0)
    c = ScalarField(3, 1)
    port.restrict_sum(g, f, c)
    assert (c(0, 0), c(1, 0), c(2, 0)) == (64.0, 64.0, 16.0)


def test_prolongation_partition_of_unity_and_ramp(port):
    """test_coarsening.cpp:331-378"""
    g = cavity(20, 12, 8)
    c = ScalarField(3, 2)
    c.fill_interior(1.0)
    f = ScalarField(20, 12)
    port.prolongate_bilinear(g, c, f)
    assert np.allclose(f.interior(), 1.0)
    g = cavity(16, 8, 4)
    g.tile = 4
    # ramp along x with 4-wide tiles (by has tile 8 in the reference; here one tile column of 2 rows)
    c = ScalarField(4, 2)
    for I in range(4):
        for J in range(2):
            c.set(I, J, 3.0 * (I * 4 + 2.0))
    f = ScalarField(16, 8)
    port.prolongate_bilinear(g, c, f)
    for i in range(2, 14):
        assert abs(f(i, 3) - 3.0 * (i + 0.5)) < 1e-12
    assert abs(f(0, 0) - 6.0) < 1e-12


def test_zero_rhs_no_sweeps(port):
    """test_cycles.cpp:75-93"""
    g = cavity(16, 16)
    for s in Scheme:
        cfg = CycleConfig(scheme=s, tile=4, depth=3)
        x, b = ScalarField(16, 16), ScalarField(16, 16)
        rep, cur, _ = port.solve(g, cfg, x, b)
        assert rep.converged and rep.fine_sweeps == 0 and rep.coarse_sweeps == 0 and rep.residual == 0.0
        assert x.interior_max_abs() == 0.0


def test_sync_counts_follow_tallies(port):
    """test_cycles.cpp:180-212: NCC_f = 2 I_f, NCC_c = I_c."""
    g = cavity(16, 16)
    rng = np.random.default_rng(7)
    b = random_field(16, 16, rng)
    b.shift_interior(-b.interior_mean())
    for s in (Scheme.plain_gs, Scheme.ismg, Scheme.acm):
        cfg = CycleConfig(scheme=s, tile=4, depth=3, tol_fine=1e-8, tol_coarse=1e-7)
        rep, cur, _ = port.solve(g, cfg, ScalarField(16, 16), b)
        assert rep.converged
        assert cur.sync_fine == 2 * cur.fine_sweeps and cur.sync_coarse == cur.coarse_sweeps
        assert (cur.restrictions == 0) == (s == Scheme.plain_gs)


def test_tile_aligned_oscillation(port):
    """test_cycles.cpp:214-234: coarse grid never visited."""
    g = cavity(8, 8)
    x, b = ScalarField(8, 8), ScalarField(8, 8)
    for j in range(8):
        for i in range(8):
            b.set(i, j, 1e-3 if (i + j) % 2 == 0 else -1e-3)
    rep, cur, _ = port.solve(g, CycleConfig(tile=2, tol_fine=1e-8, tol_coarse=1e-7), x, b)
    assert rep.converged and rep.coarse_sweeps == 0 and rep.fine_sweeps > 0
    assert cur.prolongations == 0 and cur.restrictions > 0


def test_budget_exhaustion_reports(port):
    """test_cycles.cpp:268-291"""
    g = cavity(32, 32)
    rng = np.random.default_rng(11)
    b = random_field(32, 32, rng)
    b.shift_interior(-b.interior_mean())
    for s in (Scheme.plain_gs, Scheme.ismg, Scheme.acm):
        cfg = CycleConfig(scheme=s, tile=8, depth=3, tol_fine=1e-12, tol_coarse=1e-12, max_total_sweeps=3)
        rep, cur, _ = port.solve(g, cfg, ScalarField(32, 32), b)
        assert not rep.converged and rep.fine_sweeps + rep.coarse_sweeps <= 3


def test_all_schemes_reach_dense_solution(port):
    """test_cycles.cpp:95-126: all four schemes == singular LU to 1e-7."""
    g = cavity(16, 16)
    rng = np.random.default_rng(97)
    b = random_field(16, 16, rng)
    b.shift_interior(-b.interior_mean())
    A = dense_fine_matrix(g)
    want = np.linalg.lstsq(A, b.interior().reshape(-1), rcond=None)[0]
    want -= want.mean()
    for s in Scheme:
        cfg = CycleConfig(scheme=s, tile=4, depth=3, tol_fine=1e-10, tol_coarse=1e-10)
        x = ScalarField(16, 16)
        rep, _, _ = port.solve(g, cfg, x, b)
        assert rep.converged and rep.residual <= 1e-10
        assert np.abs(x.interior().reshape(-1) - want).max() < 1e-7


def test_metrics_csv_golden():
    """test_metrics.cpp:69-85 header and formats."""
    m = RunMetrics(256)
    m.record_sweep(0, 5, 256)
    m.record_sweep(1, 9, 16)
    m.record_restriction()
    m.close_timestep(1, 2.5e-7, True)
    s = write_metrics_csv(m)
    assert s.splitlines()[0] == "step,I_f,I_c,NCC_f,NCC_c,NCC_t,N_Lap,restrictions,prolongations,residual_final"
    assert s.splitlines()[1] == "1,1,1,2,1,3,1.1125,1,0,2.5e-07"


def test_nlap_coarse_sweep_kat():
    """test_metrics.cpp:11-30: a 9-point 16h coarse sweep adds 0.00703125."""
    m = RunMetrics(256 * 256)
    m.record_sweep(1, 9, 16 * 16)
    assert m.current.lap_equiv == pytest.approx(0.00703125)


def test_a3_rhs_all_schemes_agree(port):
    """acceptance.cpp:173-248 (A3) on the frozen 64^2 instance."""
    b = a3_rhs(64)
    g = cavity(64, 64)
    sols = []
    for s, size in ((Scheme.plain_gs, 0), (Scheme.ismg, 8), (Scheme.gmg, 8), (Scheme.acm, 4)):
        cfg = CycleConfig(scheme=s, tol_fine=1e-7, tol_coarse=1e-7)
        if s == Scheme.acm:
            cfg.depth = size
        elif s != Scheme.plain_gs:
            cfg.tile = size
        x = ScalarField(64, 64)
        rep, _, _ = port.solve(g, cfg, x, b)
        assert rep.converged
        x.shift_interior(-x.interior_mean())
        sols.append(x.interior().copy())
    worst = max(np.abs(sols[a] - sols[c]).max() for a in range(4) for c in range(a + 1, 4))
    assert worst < 1e-5


# ---------------------------------------------------------------- golden ----
@pytest.mark.parametrize("name,g", golden_grids(), ids=[n for n, _ in golden_grids()])
def test_port_matches_golden_ops(port, golden, name, g):
    z = golden
    x = ScalarField(g.nx, g.ny, z[name + "/x0"].copy())
    b = ScalarField(g.nx, g.ny, z[name + "/b"])
    for _ in range(3):
        port.rbgs_sweep(g, x, b)
    assert np.array_equal(x.data, z[name + "/rbgs3"])
    r = ScalarField(g.nx, g.ny)
    assert port.fine_residual(g, x, b, r) == z[name + "/rmax"][0]
    assert np.array_equal(r.data, z[name + "/res"])
    assert np.array_equal(x.data, z[name + "/x_after_res"])
    port.anchor_mean(g, x)
    assert np.array_equal(x.data, z[name + "/anchored"])
    assert np.array_equal(port.build_fine_diag(g).data, z[name + "/diag"])
    ncx, ncy, w = port.build_ismg_operator(g)
    assert np.array_equal(w, z[name + "/ismg_w"])
    assert np.array_equal(port.build_gmg_operator(g)[2], z[name + "/gmg_w"])
    cb = ScalarField(ncx, ncy)
    port.restrict_sum(g, r, cb)
    assert np.array_equal(cb.data, z[name + "/restrict"])
    f = ScalarField(g.nx, g.ny, z[name + "/x0"].copy())
    port.prolongate_bilinear(g, cb, f)
    assert np.array_equal(f.data, z[name + "/prolong"])
    px, py = periodic_flags(g)
    ce = ScalarField(ncx, ncy)
    for _ in range(5):
        port.gs_sweep_lex(w, px, py, 0, ce, cb)
    assert np.array_equal(ce.data, z[name + "/gs5"])
    cr = ScalarField(ncx, ncy)
    assert port.coarse_residual(w, px, py, 0, ce, cb, cr) == z[name + "/crmax"][0]
    assert np.array_equal(cr.data, z[name + "/cres"])


@pytest.mark.parametrize("name,g", golden_grids(), ids=[n for n, _ in golden_grids()])
def test_port_matches_golden_solves(port, golden, name, g):
    from pyoracle import OracleError
    z = golden
    bb = ScalarField(g.nx, g.ny, z[name + "/b"].copy())
    bb.shift_interior(-bb.interior_mean())
    for s in Scheme:
        key = "%s/solve_%d" % (name, int(s))
        if key + "/x" not in z and key + "/error" not in z:
            continue
        cfg = CycleConfig(scheme=s, tile=g.tile, depth=3, tol_fine=1e-9, tol_coarse=1e-8, max_total_sweeps=4000)
        x = ScalarField(g.nx, g.ny)
        if key + "/error" in z:
            with pytest.raises(OracleError) as e:
                port.solve(g, cfg, x, bb)
            assert e.value.code == z[key + "/error"][0]
            continue
        rep, cur, _ = port.solve(g, cfg, x, bb)
        assert np.array_equal(x.data, z[key + "/x"])
        assert [rep.converged, rep.fine_sweeps, rep.coarse_sweeps, cur.restrictions, cur.prolongations] == \
            z[key + "/counts"].tolist()
        assert [rep.residual, cur.lap_equiv] == z[key + "/scalars"].tolist()


def golden_runs():
    c1 = setup_lid_cavity(32, 100.0)
    c1.dt = 100.0 / 32
    from paper_1309_7128_b200.api import setup_channel_jets
    return [("lid32", c1, CycleConfig(tile=8), 25), ("jet32x64", setup_jet(32, 64, 0.1, 8), CycleConfig(tile=8), 12),
            ("chan24x48", setup_channel_jets(24, 48, 0.1, 6), CycleConfig(tile=8), 8)]


@pytest.mark.parametrize("name,case,cfg,nsteps", golden_runs(), ids=[r[0] for r in golden_runs()])
def test_port_matches_golden_runs(port, golden, name, case, cfg, nsteps):
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, _ = port.run_steps(case.grid, cfg, st, nsteps)
    got = [[r.step, r.fine_sweeps, r.coarse_sweeps, r.sync_fine, r.sync_coarse, r.restrictions, r.prolongations,
            int(r.converged)] for r in rows]
    assert got == golden["run/%s/rows" % name].tolist()
    assert [[r.lap_equiv, r.residual_final] for r in rows] == golden["run/%s/rowsf" % name].tolist()
    assert np.array_equal(st.vel.u_data, golden["run/%s/u" % name])
    assert np.array_equal(st.vel.v_data, golden["run/%s/v" % name])
    assert np.array_equal(st.p.data, golden["run/%s/p" % name])


# ------------------------------------------------- port == reference (live) -
def test_port_equals_reference_random(port, ref):
    rng = np.random.default_rng(2024)
    grids = [cavity(33, 17, 8), torus(15, 9, 4),
             with_side(with_side(cavity(31, 40, 8), Side.south, BoundaryCondition.inflow(0.1, 3, 7)), Side.north,
                       BoundaryCondition.symmetry(0.0))]
    for g in grids:
        x = random_field(g.nx, g.ny, rng)
        b = random_field(g.nx, g.ny, rng)
        x1, x2 = x.copy(), x.copy()
        for _ in range(2):
            port.rbgs_sweep(g, x1, b)
            ref.rbgs_sweep(g, x2, b)
        assert np.array_equal(x1.data, x2.data)
        bb = b.copy()
        bb.shift_interior(-bb.interior_mean())
        for s in Scheme:
            cfg = CycleConfig(scheme=s, tile=4, depth=3, tol_fine=1e-8, tol_coarse=1e-7, max_total_sweeps=3000)
            X1, X2 = ScalarField(g.nx, g.ny), ScalarField(g.nx, g.ny)
            r1 = port.solve(g, cfg, X1, bb)
            r2 = ref.solve(g, cfg, X2, bb)
            assert r1[0] == r2[0] and r1[1] == r2[1]
            assert np.array_equal(X1.data, X2.data)


def test_bench_fine_iteration_sample(port, ref):
    """bench.py's bounded CPU sample at 16384^2 (ref_fine_iterations in oracle/ref_shim.cpp)
    runs the outer fine iteration of cycles.hpp:148-161: same x as the port's op loop."""
    import ctypes as C
    import dataclasses
    g = dataclasses.replace(setup_lid_cavity(48, 1000.0).grid, tile=8)
    b = random_field(48, 48, np.random.default_rng(3))
    x_ref, x_port = ScalarField(48, 48), ScalarField(48, 48)
    secs = C.c_double()
    rc = ref._fn("fine_iterations")(C.byref(g.to_c()), C.c_void_p(x_ref.data.ctypes.data),
                                    C.c_void_p(b.data.ctypes.data), C.c_long(3), C.byref(secs))
    assert rc == 0 and secs.value >= 0.0
    res, cb = ScalarField(48, 48), ScalarField(6, 6)
    for _ in range(3):
        port.rbgs_sweep(g, x_port, b)
        port.fine_residual(g, x_port, b, res)
        port.anchor_mean(g, x_port)
        port.restrict_sum(g, res, cb)
    assert np.array_equal(x_ref.data, x_port.data)


def test_bench_workloads():
    """bench.py: the default line is BASELINE config 3 (lid 16384^2, tile 32); --case jet is
    config 4 (setup_jet(8192, 16384, 0.1, 16), bench.hpp:73-88, tile 16, jet.cfg:15); an explicit
    --grid always wins (jet --grid 4096 is 4096 x 8192)."""
    import argparse
    import bench
    ns = lambda **k: argparse.Namespace(**{"case": "lid", "grid": None, **k})  # noqa: E731
    assert bench.grid_side(ns()) == 16384
    assert bench.grid_side(ns(case="jet")) == 8192
    assert bench.grid_side(ns(case="jet", grid=4096)) == 4096
    assert bench.grid_side(ns(grid=4096)) == 4096
    case, cfg = bench.workload(bench.JET_NX, "jet")
    assert (case.grid.nx, case.grid.ny, cfg.tile) == (8192, 16384, 16)
    assert "config 4" in bench.workload_desc(bench.JET_NX, "jet")
    case, cfg = bench.workload(16384, "lid")
    assert (case.grid.nx, cfg.tile, case.dt) == (16384, 32, 1000.0 / 16384)
    assert "config 3" in bench.workload_desc(16384, "lid")


def test_bench_cpu_model_tracks_the_reference(ref):
    """bench.py's same-work CPU baseline: the reference's per-operation costs (ref_op_costs)
    times a run's per-step counts reproduce the reference's own wall time of that run."""
    import bench
    from paper_1309_7128_b200.api import FluidState
    n = 256
    case, cfg = bench.workload(n, "lid")
    o = ref.op_costs(case.grid, cfg, case.dt, case.nu, 3)
    assert o.shape == (9,) and (o > 0).all()
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, secs = ref.run_steps(case.grid, cfg, st, 4)
    counts = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations) for r in rows]
    t = bench.model_seconds(o, counts)
    assert 0.4 * secs <= t <= 1.6 * secs, (t, secs)


def test_bench_reference_counts_are_the_references():
    """The reference arm's per-step counts come from the reference's own fixtures first."""
    import bench
    import numpy as np
    rows, src = bench.reference_counts(4096, "lid", 3)
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale", "c2.npz"))
    assert rows == [(int(r[1]), int(r[2]), int(r[5]), int(r[6])) for r in z["rows"]]
    assert "c2.npz" in src
    rows5, src5 = bench.reference_counts(4096, "lid", 5)
    assert rows5[:3] == rows and len(rows5) == 5


@pytest.mark.parametrize("which", ["lid", "jet"])
def test_writers_match_the_reference_bytes(ref, tmp_path, which):
    """io.hpp:35-117: write_field_csv, write_vtk and write_operator_csv (`%.17g`, the
    exact-coefficient dump) produce the reference's bytes on a stepped state."""
    import ctypes as C
    from paper_1309_7128_b200 import api
    from paper_1309_7128_b200._abi import dptr
    if which == "lid":
        case = api.setup_lid_cavity(24, 100.0)
        case.dt = 100.0 / 24
        tile = 4
    else:
        case = api.setup_jet(20, 40, 0.1, 4)
        tile = 4
    g = case.grid.copy()
    g.tile = tile
    st = api.FluidState(g)
    st.dt, st.nu = case.dt, case.nu
    ref.run_steps(g, api.CycleConfig(tile=tile), st, 3)
    paths = [str(tmp_path / ("ref_" + n)) for n in ("p.csv", "s.vtk", "op.csv")]
    rc = ref._fn("write_outputs")(C.byref(g.to_c()), dptr(st.vel.u_data), dptr(st.vel.v_data), dptr(st.p.data),
                                  *[q.encode() for q in paths])
    assert rc == 0
    mine = [str(tmp_path / ("our_" + n)) for n in ("p.csv", "s.vtk", "op.csv")]
    api.write_field_csv(st.p, g, mine[0])
    api.write_vtk(st.p, st.vel, g, mine[1])
    ncx, ncy, w = ref.build_ismg_operator(g)
    api.write_operator_csv(ncx, ncy, w, mine[2])
    for a, b in zip(paths, mine):
        assert open(a, "rb").read() == open(b, "rb").read(), b


def _fma(a, b, c):
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))  # one rounding (float(Fraction) is RN)


def _div_cr(num, w, y):
    """kernels.cuh div_cr restated: two Markstein corrections with y = RN(1/w)."""
    q0 = num * y
    q1 = _fma(_fma(-q0, w, num), y, q0)
    return _fma(_fma(-q1, w, num), y, q1)


def test_markstein_division_is_correctly_rounded():
    """The coarse engines' division (kernels.cuh div_cr) equals IEEE num / w bit for
    bit on the divisors the ISMG operators produce (-3 in the interior; ring and
    Dirichlet-closure classes) and on random ones, for random numerators across the
    guarded exponent range [2^-900, 2^1000] plus adversarial significands (all-ones,
    powers of two, values next to multiples of w)."""
    import math
    import struct
    rng = np.random.default_rng(1309)
    divisors = [-3.0, -2.25, -2.5, -2.75, -3.5, -4.0, -1.75, -5.0, -6.0, -0.75, 3.0, -2.875, -3.125, -2.375]
    divisors += [float(-rng.uniform(0.5, 8.0)) for _ in range(10)]
    bad = 0
    for w in divisors:
        y = 1.0 / w
        nums = []
        for _ in range(1500):
            m = rng.uniform(1.0, 2.0)
            nums.append(math.ldexp(m, int(rng.integers(-899, 999))) * (1 if rng.random() < 0.5 else -1))
        for e in (-899, -1, 0, 1, 52, 998):
            for mant in (1.0, 2.0 - 2.0 ** -52, 1.0 + 2.0 ** -52, 1.5):
                nums.append(math.ldexp(mant, e))
        for k in range(1, 200):  # next to exact multiples: k*w and its neighbours
            base = k * w * 1.000000001
            nums += [base, math.nextafter(base, math.inf), math.nextafter(base, -math.inf)]
        for n in nums:
            got, want = _div_cr(n, w, y), n / w
            if struct.pack("<d", got) != struct.pack("<d", want):
                bad += 1
    assert bad == 0

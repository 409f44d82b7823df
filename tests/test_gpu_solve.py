"""GPU parity, solve and projection-step level (north star: identical
iteration counts, fields within 1e-10 relative L2 in fp64).

The reference answers come from the committed golden vectors (produced by the
unmodified reference) and from the C oracle run in the same process.
"""
import numpy as np
import pytest

from cases import a3_rhs, cavity, golden_grids, random_field, torus, with_side
from paper_1309_7128_b200.api import (BoundaryCondition, CycleConfig, FluidState, RunMetrics, ScalarField, Scheme,
                                      Side, setup_channel_jets, setup_jet, setup_lid_cavity)

pytestmark = pytest.mark.gpu
REL_L2 = 1e-10  # BASELINE.json north_star tolerance


@pytest.fixture(scope="module")
def dev():
    import paper_1309_7128_b200 as P
    if P.device_count() < 1:
        pytest.skip("no GPU")
    return P


def rel_l2(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


@pytest.mark.parametrize("name,g", golden_grids(), ids=[n for n, _ in golden_grids()])
def test_solves_match_golden(dev, golden, name, g):
    P, z = dev, golden
    bb = ScalarField(g.nx, g.ny, z[name + "/b"].copy())
    bb.shift_interior(-bb.interior_mean())
    for s in Scheme:
        key = "%s/solve_%d" % (name, int(s))
        if key + "/x" not in z and key + "/error" not in z:
            continue
        cfg = CycleConfig(scheme=s, tile=g.tile, depth=3, tol_fine=1e-9, tol_coarse=1e-8, max_total_sweeps=4000)
        if key + "/error" in z:
            from paper_1309_7128_b200._lib import IsmgError
            with pytest.raises(IsmgError) as e:
                solver = P.PressureSolver(g, cfg)
                solver.solve(ScalarField(g.nx, g.ny), bb, RunMetrics(g.nx * g.ny))
            assert e.value.code == z[key + "/error"][0]
            continue
        solver = P.PressureSolver(g, cfg)
        m = RunMetrics(g.nx * g.ny)
        x = ScalarField(g.nx, g.ny)
        rep = solver.solve(x, bb, m)
        counts = [int(rep.converged), rep.fine_sweeps, rep.coarse_sweeps, m.current.restrictions,
                  m.current.prolongations]
        assert counts == z[key + "/counts"].tolist(), (s, counts)
        assert rel_l2(x.interior(), ScalarField(g.nx, g.ny, z[key + "/x"]).interior()) <= REL_L2
        assert m.current.lap_equiv == z[key + "/scalars"][1]


def golden_runs():
    c1 = setup_lid_cavity(32, 100.0)
    c1.dt = 100.0 / 32
    return [("lid32", c1, CycleConfig(tile=8), 25), ("jet32x64", setup_jet(32, 64, 0.1, 8), CycleConfig(tile=8), 12),
            ("chan24x48", setup_channel_jets(24, 48, 0.1, 6), CycleConfig(tile=8), 8)]


@pytest.mark.parametrize("name,case,cfg,nsteps", golden_runs(), ids=[r[0] for r in golden_runs()])
def test_projection_runs_match_golden(dev, golden, name, case, cfg, nsteps):
    P = dev
    case.steps = nsteps
    case.t_max = 0.0
    case.steady_tol = 0.0
    res = P.run_case(case, cfg)
    rows = [[r.step, r.fine_sweeps, r.coarse_sweeps, r.sync_fine, r.sync_coarse, r.restrictions, r.prolongations,
             int(r.converged)] for r in res.metrics.rows]
    assert rows == golden["run/%s/rows" % name].tolist()
    st = res.state
    assert rel_l2(st.vel.u_data, golden["run/%s/u" % name]) <= REL_L2
    assert rel_l2(st.vel.v_data, golden["run/%s/v" % name]) <= REL_L2
    assert rel_l2(st.p.data, golden["run/%s/p" % name]) <= REL_L2


def test_lid256_config1_counts_and_fields(dev, port):
    """BASELINE config 1 (lid 256^2, Re 100, tile 16, dt = Re/n) for 60 steps."""
    P = dev
    case = setup_lid_cavity(256, 100.0)
    case.dt, case.steps, case.t_max, case.steady_tol = 100.0 / 256, 60, 0.0, 0.0
    cfg = CycleConfig(tile=16)
    res = P.run_case(case, cfg)
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, _ = port.run_steps(case.grid, cfg, st, 60)
    got = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in res.metrics.rows]
    want = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in rows]
    assert got == want
    assert rel_l2(res.state.vel.u_data, st.vel.u_data) <= REL_L2
    assert rel_l2(res.state.vel.v_data, st.vel.v_data) <= REL_L2
    assert rel_l2(res.state.p.data, st.p.data) <= REL_L2


def test_a3_four_schemes_agree(dev):
    """acceptance.cpp:173-248 (A3) on the GPU."""
    P = dev
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
        rep = P.PressureSolver(g, cfg).solve(x, b, RunMetrics(64 * 64))
        assert rep.converged
        x.shift_interior(-x.interior_mean())
        sols.append(x.interior().copy())
    worst = max(np.abs(sols[a] - sols[c]).max() for a in range(4) for c in range(a + 1, 4))
    assert worst < 1e-5


def test_zero_rhs_and_budget(dev):
    """test_cycles.cpp:75-93 and :268-291 on the device path."""
    P = dev
    g = cavity(16, 16)
    for s in Scheme:
        rep = P.PressureSolver(g, CycleConfig(scheme=s, tile=4, depth=3)).solve(
            ScalarField(16, 16), ScalarField(16, 16), RunMetrics(256))
        assert rep.converged and rep.fine_sweeps == 0 and rep.coarse_sweeps == 0 and rep.residual == 0.0
    rng = np.random.default_rng(11)
    b = random_field(32, 32, rng)
    b.shift_interior(-b.interior_mean())
    for s in (Scheme.plain_gs, Scheme.ismg, Scheme.acm):
        cfg = CycleConfig(scheme=s, tile=8, depth=3, tol_fine=1e-12, tol_coarse=1e-12, max_total_sweeps=3)
        rep = P.PressureSolver(cavity(32, 32), cfg).solve(ScalarField(32, 32), b, RunMetrics(1024))
        assert not rep.converged and rep.fine_sweeps + rep.coarse_sweeps <= 3


@pytest.mark.parametrize("kernel", ["sp", "cl", "tmem", "smem", "global"])
@pytest.mark.parametrize("which", ["lid96", "jet48x96"])
def test_coarse_visit_kernels_match_oracle(dev, port, monkeypatch, kernel, which):
    """Every coarse-visit kernel of the fused path (TMEM-resident rhs,
    shared-memory iterate, global wavefront) reproduces the reference's
    per-step counts; the jet (non-singular: no anchoring) must be bit-exact
    in the coarse solve, so its fields match to round-off of the tree sums."""
    P = dev
    monkeypatch.setenv("ISMG_COARSE_KERNEL", kernel)
    if which == "lid96":
        case = setup_lid_cavity(96, 100.0)
        case.dt = 100.0 / 96
        cfg, nsteps = CycleConfig(tile=8), 15
    else:
        case = setup_jet(48, 96, 0.1, 8)
        cfg, nsteps = CycleConfig(tile=8), 8
    case.steps, case.t_max, case.steady_tol = nsteps, 0.0, 0.0
    res = P.run_case(case, cfg)
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, _ = port.run_steps(case.grid, cfg, st, nsteps)
    got = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in res.metrics.rows]
    want = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in rows]
    assert got == want
    for a, b in ((res.state.vel.u_data, st.vel.u_data), (res.state.vel.v_data, st.vel.v_data),
                 (res.state.p.data, st.p.data)):
        assert rel_l2(a, b) <= REL_L2


@pytest.mark.parametrize("n,tile,env", [(256, 4, {}), (256, 4, {"ISMG_CL_HYBRID": "0"}),
                                        (256, 4, {"ISMG_CL_HYBRID": "1"}), (256, 4, {"ISMG_CL_BAND": "64"}),
                                        (256, 4, {"ISMG_CL_BAND": "128"}), (400, 4, {}), (520, 4, {}),
                                        (520, 2, {})])
def test_coarse_cluster_plans_match_oracle(dev, port, monkeypatch, n, tile, env):
    """The cluster coarse kernel under every plan: on a 64x64 coarse grid 32-row
    bands on 2 SMs with the one-SM hand-off (default) or without it, 64-row bands
    on one SM, and a forced hybrid; on 100x100 four bands of 32, 32, 32 and 4 rows
    and on 130x130 five bands (barrier every 3 steps); on 260x260 nine bands
    (barrier every 4 steps). Per-step counts equal the reference's."""
    P = dev
    monkeypatch.setenv("ISMG_COARSE_KERNEL", "cl")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    case = setup_lid_cavity(n, 1000.0)
    case.dt = 1000.0 / n
    cfg, nsteps = CycleConfig(tile=tile), 3
    case.steps, case.t_max, case.steady_tol = nsteps, 0.0, 0.0
    res = P.run_case(case, cfg)
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, _ = port.run_steps(case.grid, cfg, st, nsteps)
    got = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in res.metrics.rows]
    want = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in rows]
    assert got == want
    for a, b in ((res.state.vel.u_data, st.vel.u_data), (res.state.vel.v_data, st.vel.v_data),
                 (res.state.p.data, st.p.data)):
        assert rel_l2(a, b) <= REL_L2


@pytest.mark.parametrize("case_name,nsteps", [("lid256t4", 3), ("lid512t4", 2), ("jet256x512t4", 4),
                                              ("lid1024t4", 1)])
def test_coarse_register_wavefront_matches_oracle(dev, port, monkeypatch, case_name, nsteps):
    """The register-wavefront coarse engine (coarse_rw.cu) on coarse grids of
    64^2 (2 lane segments per row, 32 warps), 128^2, a rectangular non-singular
    jet 64x128 with Dirichlet closures on the top rows, and 256^2 (8 segments,
    128 warps over 32 CTAs): per-step counts equal the reference's and fields
    match within the north star's tolerance."""
    P = dev
    monkeypatch.setenv("ISMG_COARSE_KERNEL", "rw")
    if case_name.startswith("lid"):
        n = int(case_name[3:].split("t")[0])
        case = setup_lid_cavity(n, 1000.0)
        case.dt = 1000.0 / n
    else:
        case = setup_jet(256, 512, 0.1, 8)
    cfg = CycleConfig(tile=4)
    case.steps, case.t_max, case.steady_tol = nsteps, 0.0, 0.0
    res = P.run_case(case, cfg)
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, _ = port.run_steps(case.grid, cfg, st, nsteps)
    got = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in res.metrics.rows]
    want = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in rows]
    assert got == want
    for a, b in ((res.state.vel.u_data, st.vel.u_data), (res.state.vel.v_data, st.vel.v_data),
                 (res.state.p.data, st.p.data)):
        assert rel_l2(a, b) <= REL_L2
    # the solve ran on the register-wavefront engine
    solver = P.PressureSolver(case.grid, cfg)
    x = ScalarField(case.grid.nx, case.grid.ny)
    b = random_field(case.grid.nx, case.grid.ny, np.random.default_rng(5))
    b.shift_interior(-b.interior_mean())
    solver.solve(x, b, RunMetrics(case.grid.nx * case.grid.ny))
    assert solver.last_stats()["coarse_engine"] == 4


@pytest.mark.parametrize("case_name,nsteps", [("lid128t16", 6), ("jet64x128t16", 5)])
def test_fused_prolongation_pass_matches_two_passes(dev, port, monkeypatch, case_name, nsteps):
    """The fused prolongation + sweep pass (fine_pass_w.cu fused_w, uniform
    power-of-two tiles) against the two-pass path (ISMG_FUSE=0) and the oracle:
    identical per-step counts; fields equal to round-off (the fused pass takes the
    prolonged field's anchor from a coarse-grid sum)."""
    P = dev

    def make():
        if case_name.startswith("lid"):
            case = setup_lid_cavity(128, 100.0)
            case.dt = 100.0 / 128
        else:
            case = setup_jet(64, 128, 0.1, 16)
        case.steps, case.t_max, case.steady_tol = nsteps, 0.0, 0.0
        return case

    cfg = CycleConfig(tile=16)
    out = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("ISMG_FUSE", fuse)
        res = P.run_case(make(), cfg)
        out[fuse] = res
    case = make()
    st = FluidState(case.grid)
    st.dt, st.nu = case.dt, case.nu
    rows, _ = port.run_steps(case.grid, cfg, st, nsteps)
    want = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged) for r in rows]
    assert sum(r.prolongations for r in rows) > 0  # the fused pass had work
    for fuse, res in out.items():
        got = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, r.converged)
               for r in res.metrics.rows]
        assert got == want, fuse
        for a, b in ((res.state.vel.u_data, st.vel.u_data), (res.state.vel.v_data, st.vel.v_data),
                     (res.state.p.data, st.p.data)):
            assert rel_l2(a, b) <= REL_L2, fuse
    assert rel_l2(out["1"].state.p.data, out["0"].state.p.data) <= 1e-12
    # the fused slot was planned: its graph slot launches two more kernels (anchor sum, fused pass)
    grid = make().grid
    rng = np.random.default_rng(5)
    rhs = random_field(grid.nx, grid.ny, rng)
    rhs.shift_interior(-rhs.interior_mean())
    launches = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("ISMG_FUSE", fuse)
        s = P.PressureSolver(grid, cfg)
        rep = s.solve(ScalarField(grid.nx, grid.ny), rhs, RunMetrics(grid.nx * grid.ny))
        st_ = s.last_stats()
        launches[fuse] = (st_["kernel_launches"], rep.fine_sweeps, rep.coarse_sweeps, st_["prolong_passes"])
    assert launches["1"][1:] == launches["0"][1:] and launches["1"][3] > 0
    assert launches["1"][0] > launches["0"][0]

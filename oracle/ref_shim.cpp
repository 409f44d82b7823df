// ref_shim.cpp — C entry points onto the UNMODIFIED reference library
// (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/build.sh against the reference's own headers where
// they lie (-I $REF/proj/include, never copied into this repo) with the
// reference's flags (proj/CMakeLists.txt:14: -O3, no -march => no FMA), into
// oracle/_ref/libismg_ref.so. Used to pin the C restatement (ismg_oracle.c)
// bit-for-bit and as the CPU baseline (`kind: "reference"`) in bench.py.
// The function set mirrors ismg_oracle.h with a ref_ prefix.
#include <chrono>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "ismg/ismg.hpp"
#include "../include/ismg_b200.h"

using namespace ismg;

namespace {
thread_local std::string g_err;

int on_exception() {
    try {
        throw;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return ISMG_ERR_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return ISMG_ERR_DOMAIN;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return ISMG_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ISMG_ERR_INTERNAL;
    }
}

GridSpec to_grid(const ismg_grid_spec* s) {
    GridSpec g;
    g.nx = s->nx;
    g.ny = s->ny;
    g.h = s->h;
    g.tile = s->tile;
    for (int k = 0; k < 4; ++k) {
        BoundaryCondition& b = g.bc[size_t(k)];
        b.kind = static_cast<BcKind>(s->bc[k].kind);
        b.u_wall = s->bc[k].u_wall;
        b.v_wall = s->bc[k].v_wall;
        b.p_wall = s->bc[k].p_wall;
        b.v_inflow = s->bc[k].v_inflow;
        b.inlet_start = s->bc[k].inlet_start;
        b.inlet_width = s->bc[k].inlet_width;
    }
    return g;
}

CycleConfig to_cfg(const ismg_cycle_config* c) {
    CycleConfig cfg;
    switch (c->scheme) {
        case ISMG_SCHEME_PLAIN_GS: cfg.scheme = Scheme::plain_gs; break;
        case ISMG_SCHEME_ISMG: cfg.scheme = Scheme::ismg; break;
        case ISMG_SCHEME_GMG: cfg.scheme = Scheme::gmg; break;
        default: cfg.scheme = Scheme::acm; break;
    }
    cfg.tile = c->tile;
    cfg.depth = c->depth;
    cfg.tol_fine = c->tol_fine;
    cfg.tol_coarse = c->tol_coarse;
    cfg.max_total_sweeps = long(c->max_total_sweeps);
    cfg.acm_pre_smooth = c->acm_pre_smooth;
    cfg.acm_post_smooth = c->acm_post_smooth;
    cfg.stall_factor = c->stall_factor;
    return cfg;
}

ScalarField<double> load(int nx, int ny, const double* p) {
    ScalarField<double> f(nx, ny);
    std::memcpy(f.data.data(), p, f.data.size() * sizeof(double));
    return f;
}
void store(const ScalarField<double>& f, double* p) {
    std::memcpy(p, f.data.data(), f.data.size() * sizeof(double));
}

StepMetrics to_row(const ismg_step_metrics* m) {
    StepMetrics r;
    if (!m) return r;
    r.step = long(m->step);
    r.fine_sweeps = m->fine_sweeps;
    r.coarse_sweeps = m->coarse_sweeps;
    r.sync_fine = m->sync_fine;
    r.sync_coarse = m->sync_coarse;
    r.lap_equiv = m->lap_equiv;
    r.restrictions = m->restrictions;
    r.prolongations = m->prolongations;
    r.residual_final = m->residual_final;
    r.converged = m->converged != 0;
    return r;
}
void from_row(const StepMetrics& r, ismg_step_metrics* m) {
    if (!m) return;
    std::memset(m, 0, sizeof *m);
    m->step = r.step;
    m->fine_sweeps = r.fine_sweeps;
    m->coarse_sweeps = r.coarse_sweeps;
    m->sync_fine = r.sync_fine;
    m->sync_coarse = r.sync_coarse;
    m->lap_equiv = r.lap_equiv;
    m->restrictions = r.restrictions;
    m->prolongations = r.prolongations;
    m->residual_final = r.residual_final;
    m->converged = r.converged ? 1 : 0;
}

CoarseOperator<double> op_from(int ncx, int ncy, int px, int py, int five, const double* w) {
    CoarseOperator<double> op;
    op.init(TileAxis(ncx, 1, px != 0), TileAxis(ncy, 1, py != 0));
    op.five_point = five != 0;
    size_t n = size_t(ncx) * ncy;
    for (int s = 0; s < 9; ++s) std::memcpy(op.w[size_t(s)].data(), w + s * n, n * sizeof(double));
    return op;
}

void copy_planes(const CoarseOperator<double>& op, double* w) {
    size_t n = size_t(op.ncx) * op.ncy;
    for (int s = 0; s < 9; ++s) std::memcpy(w + s * n, op.w[size_t(s)].data(), n * sizeof(double));
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_rbgs_sweep(const ismg_grid_spec* gs, double* x, const double* b) try {
    GridSpec g = to_grid(gs);
    FineStage<double> st = build_fine_stage<double>(g);
    ScalarField<double> X = load(g.nx, g.ny, x), B = load(g.nx, g.ny, b);
    rbgs_sweep(st, X, B);
    store(X, x);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_fine_residual(const ismg_grid_spec* gs, double* x, const double* b, double* out,
                      double* rmax) try {
    GridSpec g = to_grid(gs);
    FineStage<double> st = build_fine_stage<double>(g);
    ScalarField<double> X = load(g.nx, g.ny, x), B = load(g.nx, g.ny, b), R(g.nx, g.ny);
    if (out) R = load(g.nx, g.ny, out);
    *rmax = fine_residual(st, X, B, out ? &R : nullptr);
    store(X, x);
    if (out) store(R, out);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_anchor_mean(const ismg_grid_spec* gs, double* x) try {
    GridSpec g = to_grid(gs);
    FineStage<double> st = build_fine_stage<double>(g);
    ScalarField<double> X = load(g.nx, g.ny, x);
    anchor_mean(st, X);
    store(X, x);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_build_fine_diag(const ismg_grid_spec* gs, double* diag) try {
    FineStage<double> st = build_fine_stage<double>(to_grid(gs));
    store(st.diag, diag);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_build_ismg_operator(const ismg_grid_spec* gs, int32_t* ncx, int32_t* ncy, double* w) try {
    CoarseOperator<double> op = build_ismg_operator<double>(to_grid(gs));
    *ncx = op.ncx;
    *ncy = op.ncy;
    if (w) copy_planes(op, w);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_build_gmg_operator(const ismg_grid_spec* gs, int32_t* ncx, int32_t* ncy, double* w) try {
    CoarseOperator<double> op = build_gmg_operator<double>(to_grid(gs));
    *ncx = op.ncx;
    *ncy = op.ncy;
    if (w) copy_planes(op, w);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_restrict_sum(const ismg_grid_spec* gs, const double* fine, double* coarse) try {
    GridSpec g = to_grid(gs);
    auto bc = pressure_bc(g);
    TileAxis ax(g.nx, g.tile, bc[0] == PressureBcKind::periodic);
    TileAxis ay(g.ny, g.tile, bc[2] == PressureBcKind::periodic);
    ScalarField<double> F = load(g.nx, g.ny, fine), C = load(ax.nc, ay.nc, coarse);
    restrict_sum(F, ax, ay, C);
    store(C, coarse);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_prolongate_bilinear(const ismg_grid_spec* gs, const double* coarse, double* fine) try {
    GridSpec g = to_grid(gs);
    auto bc = pressure_bc(g);
    TileAxis ax(g.nx, g.tile, bc[0] == PressureBcKind::periodic);
    TileAxis ay(g.ny, g.tile, bc[2] == PressureBcKind::periodic);
    ScalarField<double> F = load(g.nx, g.ny, fine), C = load(ax.nc, ay.nc, coarse);
    prolongate_bilinear(C, ax, ay, F);
    store(F, fine);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_coarse_residual(int ncx, int ncy, int px, int py, int five, const double* w,
                        const double* x, const double* b, double* out, double* rmax) try {
    CoarseOperator<double> op = op_from(ncx, ncy, px, py, five, w);
    ScalarField<double> X = load(ncx, ncy, x), B = load(ncx, ncy, b), R(ncx, ncy);
    if (out) R = load(ncx, ncy, out);
    *rmax = coarse_residual(op, X, B, out ? &R : nullptr);
    if (out) store(R, out);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_gs_sweep_lex(int ncx, int ncy, int px, int py, int five, const double* w, double* x,
                     const double* b) try {
    CoarseOperator<double> op = op_from(ncx, ncy, px, py, five, w);
    ScalarField<double> X = load(ncx, ncy, x), B = load(ncx, ncy, b);
    gs_sweep_lex(op, X, B);
    store(X, x);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_solve(const ismg_grid_spec* gs, const ismg_cycle_config* cs, double* x, const double* b,
              ismg_report* rep, ismg_step_metrics* current, int64_t fine_cells,
              double* seconds) try {
    GridSpec g = to_grid(gs);
    PressureSolver<double> solver(g, to_cfg(cs));
    RunMetrics m(fine_cells);
    m.current = to_row(current);
    ScalarField<double> X = load(g.nx, g.ny, x), B = load(g.nx, g.ny, b);
    auto t0 = std::chrono::steady_clock::now();
    ConvergenceReport r = solver.solve(X, B, m);
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    store(X, x);
    rep->converged = r.converged ? 1 : 0;
    rep->nan_seen = 0;
    rep->fine_sweeps = r.fine_sweeps;
    rep->coarse_sweeps = r.coarse_sweeps;
    rep->residual = r.residual;
    from_row(m.current, current);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_apply_scalar_bc(const ismg_grid_spec* gs, double* f) try {
    GridSpec g = to_grid(gs);
    ScalarField<double> F = load(g.nx, g.ny, f);
    apply_scalar_bc(F, pressure_bc(g));
    store(F, f);
    return 0;
} catch (...) {
    return on_exception();
}

namespace {
MacVelocity<double> load_vel(int nx, int ny, const double* u, const double* v) {
    MacVelocity<double> vel(nx, ny);
    std::memcpy(vel.u_data.data(), u, vel.u_data.size() * sizeof(double));
    std::memcpy(vel.v_data.data(), v, vel.v_data.size() * sizeof(double));
    return vel;
}
void store_vel(const MacVelocity<double>& vel, double* u, double* v) {
    std::memcpy(u, vel.u_data.data(), vel.u_data.size() * sizeof(double));
    std::memcpy(v, vel.v_data.data(), vel.v_data.size() * sizeof(double));
}
}  // namespace

int ref_apply_velocity_bc(const ismg_grid_spec* gs, double* u, double* v) try {
    GridSpec g = to_grid(gs);
    MacVelocity<double> vel = load_vel(g.nx, g.ny, u, v);
    apply_velocity_bc(vel, g);
    store_vel(vel, u, v);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_divergence(const ismg_grid_spec* gs, const double* u, const double* v, double* out) try {
    GridSpec g = to_grid(gs);
    MacVelocity<double> vel = load_vel(g.nx, g.ny, u, v);
    ScalarField<double> D = load(g.nx, g.ny, out);
    divergence(vel, g, D);
    store(D, out);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_correct(const ismg_grid_spec* gs, double* u, double* v, double* dp, double dt) try {
    GridSpec g = to_grid(gs);
    MacVelocity<double> vel = load_vel(g.nx, g.ny, u, v);
    ScalarField<double> DP = load(g.nx, g.ny, dp);
    correct(vel, DP, dt, g);
    store_vel(vel, u, v);
    store(DP, dp);
    return 0;
} catch (...) {
    return on_exception();
}

int ref_predictor(const ismg_grid_spec* gs, const double* u, const double* v, const double* p,
                  double dt, double nu, double* ou, double* ov) try {
    GridSpec g = to_grid(gs);
    FluidState<double> st(g);
    st.vel = load_vel(g.nx, g.ny, u, v);
    st.p = load(g.nx, g.ny, p);
    st.dt = dt;
    st.nu = nu;
    MacVelocity<double> out = load_vel(g.nx, g.ny, ou, ov);
    predictor(st, g, out);
    store_vel(out, ou, ov);
    return 0;
} catch (...) {
    return on_exception();
}

// run_case (bench.hpp:127-158) with seed = 0 and no steady/t_max exits:
// `nsteps` projection steps; rows receives the closed per-step rows;
// solve_seconds (optional) the summed wall time of the steps.
int ref_run_steps(const ismg_grid_spec* gs, const ismg_cycle_config* cs, double* u, double* v,
                  double* p, double* scal, long nsteps, ismg_step_metrics* rows,
                  double* seconds) try {
    GridSpec g = to_grid(gs);
    g.validate();
    PressureSolver<double> solver(g, to_cfg(cs));
    FluidState<double> st(g);
    st.vel = load_vel(g.nx, g.ny, u, v);
    st.p = load(g.nx, g.ny, p);
    st.t = scal[0];
    st.dt = scal[1];
    st.nu = scal[2];
    st.step_count = long(scal[3]);
    RunMetrics m(std::int64_t(g.nx) * g.ny);
    double secs = 0.0;
    for (long s = 0; s < nsteps; ++s) {
        auto t0 = std::chrono::steady_clock::now();
        step(st, g, solver, m);
        secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (seconds) *seconds = secs;
    store_vel(st.vel, u, v);
    store(st.p, p);
    scal[0] = st.t;
    scal[3] = double(st.step_count);
    for (size_t k = 0; k < m.rows.size() && rows; ++k) from_row(m.rows[k], &rows[k]);
    return 0;
} catch (...) {
    return on_exception();
}

// Bounded CPU sample for bench.py at grids whose capped step 1 never reaches a fine
// sweep (16384^2): `iters` outer fine iterations as solve_two_level runs them
// (cycles.hpp:148-161: rbgs_sweep, fine_residual into the residual field,
// anchor_mean when singular, restrict_sum), stage and fields built once, the
// iterations alone timed. x is updated in place.
int ref_fine_iterations(const ismg_grid_spec* gs, double* x, const double* b, long iters,
                        double* seconds) try {
    GridSpec g = to_grid(gs);
    g.validate();
    FineStage<double> st = build_fine_stage<double>(g);
    auto bc = pressure_bc(g);
    TileAxis ax(g.nx, g.tile, bc[0] == PressureBcKind::periodic);
    TileAxis ay(g.ny, g.tile, bc[2] == PressureBcKind::periodic);
    ScalarField<double> X = load(g.nx, g.ny, x), B = load(g.nx, g.ny, b), R(g.nx, g.ny), C(ax.nc, ay.nc);
    auto t0 = std::chrono::steady_clock::now();
    for (long k = 0; k < iters; ++k) {
        rbgs_sweep(st, X, B);
        fine_residual(st, X, B, &R);
        anchor_mean(st, X);
        restrict_sum(R, ax, ay, C);
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    store(X, x);
    return 0;
} catch (...) {
    return on_exception();
}

// The reference's own writers (io.hpp:35-117) on the given state: field CSV of
// p, VTK of (p, velocity), and the ISMG operator dump of grid gs (its tile).
int ref_write_outputs(const ismg_grid_spec* gs, const double* u, const double* v, const double* p,
                      const char* field_csv, const char* vtk, const char* op_csv) try {
    GridSpec g = to_grid(gs);
    g.validate();
    ScalarField<double> P = load(g.nx, g.ny, p);
    MacVelocity<double> vel = load_vel(g.nx, g.ny, u, v);
    write_field_csv(P, g, field_csv);
    write_vtk(P, vel, g, vtk);
    write_operator_csv(build_ismg_operator<double>(g), std::string(op_csv));
    return 0;
} catch (...) {
    return on_exception();
}

// Per-operation wall cost of the reference on grid gs with cycle cs (bench.py's
// CPU arms: the reference's own functions on this host, multiplied by a GPU
// run's exact counts). Seconds per call, the minimum over `reps` calls, on the
// step-1 state from rest (predictor, divergence, rhs scale as step(),
// projection.hpp:166-178):
//   out[0] rbgs_sweep            smoother.hpp:101-117
//   out[1] fine_residual + store  smoother.hpp:121-141
//   out[2] anchor_mean           smoother.hpp:145-148
//   out[3] restrict_sum          coarsening.hpp:471-480
//   out[4] prolongate_bilinear   coarsening.hpp:485-503
//   out[5] gs_sweep_lex          coarsening.hpp:552-567
//   out[6] coarse_residual       coarsening.hpp:531-549
//   out[7] anchor_mean (coarse)  coarsening.hpp:592-595
//   out[8] step() from rest with max_total_sweeps = 1: the per-step fixed
//          cost (BCs, CFL scan, copies, predictor, divergence, solve set-up with
//          its initial residual, one restriction, one coarse sweep, correction)
int ref_op_costs(const ismg_grid_spec* gs, const ismg_cycle_config* cs, double dt, double nu, int reps,
                 double* out) try {
    GridSpec g = to_grid(gs);
    CycleConfig cfg = to_cfg(cs);
    g.tile = cfg.tile;
    g.validate();
    using clk = std::chrono::steady_clock;
    auto timed = [&](auto&& fn) {
        double best = 1e300;
        for (int r = 0; r < std::max(1, reps); ++r) {
            auto t0 = clk::now();
            fn();
            best = std::min(best, std::chrono::duration<double>(clk::now() - t0).count());
        }
        return best;
    };
    {  // out[8]: one projection step from rest, budget 1
        CycleConfig c1 = cfg;
        c1.max_total_sweeps = 1;
        PressureSolver<double> solver(g, c1);
        FluidState<double> st(g);
        st.dt = dt, st.nu = nu;
        RunMetrics m(std::int64_t(g.nx) * g.ny);
        auto t0 = clk::now();
        step(st, g, solver, m);
        out[8] = std::chrono::duration<double>(clk::now() - t0).count();
    }
    FluidState<double> st(g);
    st.dt = dt, st.nu = nu;
    apply_scalar_bc(st.p, pressure_bc(g));
    apply_velocity_bc(st.vel, g);
    MacVelocity<double> vstar = st.vel;
    predictor(st, g, vstar);
    apply_velocity_bc(vstar, g);
    ScalarField<double> b(g.nx, g.ny), x(g.nx, g.ny), res(g.nx, g.ny);
    divergence(vstar, g, b);
    const double scale = g.h * g.h / dt;
    for (int j = 0; j < g.ny; ++j) {
        double* r = b.row(j);
        for (int i = 0; i < g.nx; ++i) r[i] *= scale;
    }
    volatile double sink = 0.0;  // keeps the residual maxima observable
    FineStage<double> stage = build_fine_stage<double>(g);
    CoarseOperator<double> op = build_ismg_operator<double>(g);
    auto bc = pressure_bc(g);
    TileAxis ax(g.nx, g.tile, bc[0] == PressureBcKind::periodic);
    TileAxis ay(g.ny, g.tile, bc[2] == PressureBcKind::periodic);
    ScalarField<double> cb(ax.nc, ay.nc), ce(ax.nc, ay.nc), cr(ax.nc, ay.nc);
    out[0] = timed([&] { rbgs_sweep(stage, x, b); });
    out[1] = timed([&] { sink = sink + fine_residual(stage, x, b, &res); });
    out[2] = timed([&] { anchor_mean(stage, x); });
    out[3] = timed([&] { restrict_sum(res, ax, ay, cb); });
    int creps = std::max(1, reps) * 8;
    double best5 = 1e300, best6 = 1e300, best7 = 1e300;
    for (int r = 0; r < creps; ++r) {
        auto t0 = clk::now();
        gs_sweep_lex(op, ce, cb);
        auto t1 = clk::now();
        sink = sink + coarse_residual(op, ce, cb);
        auto t2 = clk::now();
        anchor_mean(op, ce);
        auto t3 = clk::now();
        best5 = std::min(best5, std::chrono::duration<double>(t1 - t0).count());
        best6 = std::min(best6, std::chrono::duration<double>(t2 - t1).count());
        best7 = std::min(best7, std::chrono::duration<double>(t3 - t2).count());
    }
    out[5] = best5, out[6] = best6, out[7] = best7;
    out[4] = timed([&] { prolongate_bilinear(ce, ax, ay, x); });
    return 0;
} catch (...) {
    return on_exception();
}

}  // extern "C"

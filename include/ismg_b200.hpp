// ismg_b200.hpp — header-only C++17 facade over the C-ABI (ismg_b200.h) with the
// reference's call signatures, so a caller of the reference's `ismg` library
// switches the pressure path by changing a type name:
//
//     ismg::PressureSolver<double> solver(grid, cfg);              // reference, CPU
//     ismg_b200::PressureSolver solver(grid, cfg, ctx);            // this library, B200
//     ConvergenceReport rep = solver.solve(x, b, metrics);         // same call
//     rep = ismg_b200::step(state, grid, solver, metrics);         // projection.hpp:139-190
//
// The facade is generic over the reference's value types (duck-typed by member
// name), so it compiles against the reference's own headers without depending
// on them: GridSpec (grid.hpp:67-97: nx, ny, h, tile, bc[4] with kind, u_wall,
// v_wall, p_wall, v_inflow, inlet_start, inlet_width), CycleConfig
// (cycles.hpp:20-45), ScalarField<double> (field.hpp:18-71: nx, ny, data),
// MacVelocity<double> (field.hpp:102-137: u_data, v_data), FluidState<double>
// (projection.hpp:26-36: vel, p, t, dt, nu, step_count) and RunMetrics
// (metrics.hpp:37-67: fine_cells, current.{fine_sweeps, coarse_sweeps, sync_fine,
// sync_coarse, lap_equiv, restrictions, prolongations}).
//
// Errors are the reference's exception types: std::invalid_argument,
// std::domain_error, std::logic_error; device failures are std::runtime_error.
#ifndef ISMG_B200_HPP
#define ISMG_B200_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "ismg_b200.h"

namespace ismg_b200 {

[[noreturn]] inline void raise(int rc) {
    const std::string msg = ismg_last_error();
    switch (rc) {
        case ISMG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case ISMG_ERR_DOMAIN: throw std::domain_error(msg);
        case ISMG_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error("ismg_b200: " + msg);
    }
}
inline void check(int rc) {
    if (rc != ISMG_OK) raise(rc);
}

// ConvergenceReport — cycles.hpp:47-52 (same member names)
struct ConvergenceReport {
    bool converged = true;
    long fine_sweeps = 0;
    long coarse_sweeps = 0;
    double residual = 0.0;
};

template <class BC>
ismg_bc to_c(const BC& b, int) {
    ismg_bc c{};
    c.kind = static_cast<int32_t>(b.kind);  // BcKind order = ISMG_BC_* order
    c.inlet_start = b.inlet_start;
    c.inlet_width = b.inlet_width;
    c.u_wall = b.u_wall, c.v_wall = b.v_wall, c.p_wall = b.p_wall, c.v_inflow = b.v_inflow;
    return c;
}
template <class Grid>
ismg_grid_spec grid_to_c(const Grid& g) {
    ismg_grid_spec c{};
    c.nx = g.nx, c.ny = g.ny, c.h = g.h, c.tile = g.tile;
    for (int s = 0; s < 4; ++s) c.bc[s] = to_c(g.bc[s], 0);  // Side order = ISMG_SIDE_* order
    return c;
}
template <class Cfg>
ismg_cycle_config cycle_to_c(const Cfg& k) {
    ismg_cycle_config c{};
    c.scheme = static_cast<int32_t>(k.scheme);  // Scheme order = ISMG_SCHEME_* order
    c.tile = k.tile, c.depth = k.depth;
    c.acm_pre_smooth = k.acm_pre_smooth, c.acm_post_smooth = k.acm_post_smooth;
    c.tol_fine = k.tol_fine, c.tol_coarse = k.tol_coarse;
    c.max_total_sweeps = k.max_total_sweeps, c.stall_factor = k.stall_factor;
    return c;
}

template <class Metrics>
ismg_step_metrics metrics_in(const Metrics& m) {
    ismg_step_metrics c{};
    c.fine_sweeps = m.current.fine_sweeps, c.coarse_sweeps = m.current.coarse_sweeps;
    c.sync_fine = m.current.sync_fine, c.sync_coarse = m.current.sync_coarse;
    c.lap_equiv = m.current.lap_equiv;
    c.restrictions = m.current.restrictions, c.prolongations = m.current.prolongations;
    return c;
}
template <class Metrics>
void metrics_out(Metrics& m, const ismg_step_metrics& c) {
    m.current.fine_sweeps = c.fine_sweeps, m.current.coarse_sweeps = c.coarse_sweeps;
    m.current.sync_fine = c.sync_fine, m.current.sync_coarse = c.sync_coarse;
    m.current.lap_equiv = c.lap_equiv;
    m.current.restrictions = c.restrictions, m.current.prolongations = c.prolongations;
}
inline ConvergenceReport report(const ismg_report& r) {
    ConvergenceReport o;
    o.converged = r.converged != 0;
    o.fine_sweeps = long(r.fine_sweeps), o.coarse_sweeps = long(r.coarse_sweeps);
    o.residual = r.residual;
    return o;
}

// One device (and stream) per context; one context per host thread.
class Context {
  public:
    explicit Context(int device = 0, void* stream = nullptr) { check(ismg_ctx_create(device, stream, &h_)); }
    ~Context() {
        if (h_) ismg_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    void synchronize() { check(ismg_ctx_synchronize(h_)); }
    ismg_ctx* get() const { return h_; }

  private:
    ismg_ctx* h_ = nullptr;
};

// PressureSolver — cycles.hpp:286-333. Builds the operator once (host) and
// keeps it on the device; solve() is const like the reference's. The solver
// remembers its context, so step() takes the reference's four arguments.
class PressureSolver {
  public:
    template <class Grid, class Cfg>
    PressureSolver(const Grid& grid, const Cfg& cfg, Context& ctx) : ctx_(&ctx), nx_(grid.nx), ny_(grid.ny) {
        const ismg_grid_spec g = grid_to_c(grid);
        const ismg_cycle_config c = cycle_to_c(cfg);
        check(ismg_solver_create(ctx.get(), &g, &c, &h_));
    }
    ~PressureSolver() {
        if (h_) ismg_solver_destroy(h_);
    }
    PressureSolver(const PressureSolver&) = delete;
    PressureSolver& operator=(const PressureSolver&) = delete;

    // solve(x, b, m) on host ScalarField<double>s (one upload / download per solve)
    template <class Field, class Metrics>
    ConvergenceReport solve(Field& x, const Field& b, Metrics& m) const {
        if (x.nx != nx_ || x.ny != ny_ || b.nx != nx_ || b.ny != ny_)
            throw std::invalid_argument("pressure solver: field dimensions differ from the grid");
        ismg_report r{};
        ismg_step_metrics cur = metrics_in(m);
        check(ismg_solve_host(h_, x.data.data(), b.data.data(), x.data.size(), &r, &cur, m.fine_cells));
        metrics_out(m, cur);
        return report(r);
    }

    ismg_solver* get() const { return h_; }
    Context& context() const { return *ctx_; }
    int nx() const { return nx_; }
    int ny() const { return ny_; }

  private:
    Context* ctx_;
    ismg_solver* h_ = nullptr;
    int nx_, ny_;
};

// FluidState<double> resident in HBM across steps (no per-step upload /
// download): upload once, step many times, download when needed.
class DeviceState {
  public:
    template <class Grid>
    DeviceState(const Grid& grid, Context& ctx) {
        const ismg_grid_spec g = grid_to_c(grid);
        check(ismg_state_create(ctx.get(), &g, &h_));
    }
    ~DeviceState() {
        if (h_) ismg_state_destroy(h_);
    }
    DeviceState(const DeviceState&) = delete;
    DeviceState& operator=(const DeviceState&) = delete;

    template <class State>
    void upload(const State& st) {
        check(ismg_state_set_scalars(h_, st.t, st.dt, st.nu, int64_t(st.step_count)));
        check(ismg_state_upload(h_, st.vel.u_data.data(), st.vel.u_data.size(), st.vel.v_data.data(),
                                st.vel.v_data.size(), st.p.data.data(), st.p.data.size()));
    }
    template <class State>
    void download(State& st) const {
        check(ismg_state_download(h_, st.vel.u_data.data(), st.vel.u_data.size(), st.vel.v_data.data(),
                                  st.vel.v_data.size(), st.p.data.data(), st.p.data.size()));
        int64_t steps = 0;
        check(ismg_state_get_scalars(h_, &st.t, &st.dt, &st.nu, &steps));
        st.step_count = decltype(st.step_count)(steps);
    }
    // projection.hpp:139-190 on the resident state; closes the metrics row like
    // the reference (m.close_timestep, with (0, true) for dt == 0, :163-165)
    template <class Metrics>
    ConvergenceReport step(const PressureSolver& solver, Metrics& m) {
        ismg_report r{};
        ismg_step_metrics cur = metrics_in(m);
        check(ismg_step(h_, solver.get(), &r, &cur, m.fine_cells));
        metrics_out(m, cur);
        double t = 0, dt = 0, nu = 0;
        int64_t steps = 0;
        check(ismg_state_get_scalars(h_, &t, &dt, &nu, &steps));
        const ConvergenceReport rep = report(r);
        m.close_timestep(long(steps), dt == 0.0 ? 0.0 : rep.residual, dt == 0.0 ? true : rep.converged);
        return rep;
    }
    ismg_state* get() const { return h_; }

  private:
    ismg_state* h_ = nullptr;
};

// step — projection.hpp:139-190 with the reference's signature, on a host
// FluidState<double>: the state is uploaded, advanced one projection step on
// the device (the solver's context) and downloaded; the metrics row is closed
// as the reference closes it. For many steps keep a DeviceState instead.
template <class State, class Grid, class Metrics>
ConvergenceReport step(State& st, const Grid& grid, const PressureSolver& solver, Metrics& m) {
    DeviceState ds(grid, solver.context());
    ds.upload(st);
    const ConvergenceReport rep = ds.step(solver, m);
    ds.download(st);
    return rep;
}

}  // namespace ismg_b200

#endif  // ISMG_B200_HPP

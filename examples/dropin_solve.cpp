// examples/dropin_solve.cpp — the reference's own types driving the B200 solver
// through include/ismg_b200.hpp (built by tests/test_capi.py against the
// reference headers when they are present; run it on a GPU box).
//
//   g++ -std=c++20 -O2 -I include -I <reference>/proj/include examples/dropin_solve.cpp \
//       -L paper_1309_7128_b200 -lismg_b200 -Wl,-rpath,$PWD/paper_1309_7128_b200
#include <cmath>
#include <cstdio>

#include <ismg/projection.hpp>  // the reference: GridSpec, CycleConfig, ScalarField, FluidState, RunMetrics

#include "ismg_b200.hpp"

int main() {
    const int n = 64;
    ismg::GridSpec grid;
    grid.nx = grid.ny = n;
    grid.bc[int(ismg::Side::north)] = ismg::BoundaryCondition::moving_wall(0.1, 0.0);  // lid cavity
    ismg::CycleConfig cfg;
    cfg.tile = 8;
    ismg::FluidState<double> st(grid);
    st.dt = 100.0 / n;
    st.nu = 0.1 * n / 100.0;
    ismg::RunMetrics m(int64_t(n) * n);

    ismg::PressureSolver<double> ref_solver(grid, cfg);  // reference (CPU)
    ismg::FluidState<double> ref = st;
    ismg::RunMetrics mr(int64_t(n) * n);

    ismg_b200::Context ctx(0);
    ismg_b200::PressureSolver solver(grid, cfg, ctx);  // B200
    for (int k = 0; k < 5; ++k) {
        const auto rep = ismg_b200::step(st, grid, solver, m);  // same call as the reference's
        const auto rr = ismg::step(ref, grid, ref_solver, mr);
        std::printf("step %d: B200 I_f %ld I_c %ld | reference I_f %ld I_c %ld\n", k + 1, rep.fine_sweeps,
                    rep.coarse_sweeps, rr.fine_sweeps, rr.coarse_sweeps);
    }
    double num = 0, den = 0;
    for (size_t i = 0; i < st.p.data.size(); ++i) {
        const double d = st.p.data[i] - ref.p.data[i];
        num += d * d, den += ref.p.data[i] * ref.p.data[i];
    }
    const double err = den > 0 ? std::sqrt(num / den) : std::sqrt(num);
    bool same = m.rows.size() == mr.rows.size();
    for (size_t k = 0; same && k < m.rows.size(); ++k)
        same = m.rows[k].fine_sweeps == mr.rows[k].fine_sweeps && m.rows[k].coarse_sweeps == mr.rows[k].coarse_sweeps &&
               m.rows[k].restrictions == mr.rows[k].restrictions && m.rows[k].step == mr.rows[k].step;
    std::printf("pressure rel L2 %.3e, metrics rows %s\n", err, same ? "identical" : "DIFFER");
    return (same && err <= 1e-10) ? 0 : 1;
}

// solver.h — PressureSolver (cycles.hpp:286-333) and FluidState (projection.hpp:26-36)
// on the device.
#pragma once

#include <memory>
#include <vector>

#include "engine.h"

namespace ismgb {

// One coarse level resident in HBM: coefficient planes + transfer tables.
struct LevelDev {
    CoarseOpH h;
    double* d_w = nullptr;  // 9 planes
    AxisDev ax{}, ay{};     // TileAxis tables of the parent -> this tiling
    std::unique_ptr<Field> x, b, r;
    void upload(Ctx& c, int parent_nx, int parent_ny);
    void release();
};

struct FusedEngine;  // fused.cu

struct Metrics {  // RunMetrics::record_* (metrics.hpp:46-58) onto a C row
    ismg_step_metrics* m;
    int64_t fine_cells;
    void sweep(bool fine, int stencil, int64_t cells) {
        if (!m) return;
        if (fine) {
            m->fine_sweeps += 1;
            m->sync_fine += 2;
        } else {
            m->coarse_sweeps += 1;
            m->sync_coarse += 1;
        }
        m->lap_equiv += (double(cells) / double(fine_cells)) * (double(stencil) / 5.0);
    }
    void restriction() {
        if (m) m->restrictions += 1;
    }
    void prolongation() {
        if (m) m->prolongations += 1;
    }
};

struct Solver {
    Ctx* ctx;
    ismg_grid_spec g;  // effective grid (tile adopted for two-level schemes)
    ismg_cycle_config cfg;
    PBC bc;
    bool singular = false;
    std::vector<LevelDev> levels;  // ISMG/GMG: one; ACM: depth-1 (finest first)
    std::unique_ptr<Field> res;    // residual scratch of the op-level paths
    FusedEngine* fused = nullptr;
    FusedEngine* acm_coarse = nullptr;  // ACM: coarse-visit engine of the coarsest level (device-resident loop)
    ismg_solve_stats last{};
    std::vector<int> visit_log;  // (coarse sweeps, fine sweeps) per outer iteration of the last solve
    int mode = 0;  // 0 = auto (fused hot path when supported), 1 = op-level reference order

    Solver(Ctx* c, const ismg_grid_spec& g, const ismg_cycle_config& cfg);
    ~Solver();

    // op-level API
    void rbgs_sweep(Field& x, const Field& b);
    double fine_residual(Field& x, const Field& b, Field* out, bool want_max);
    void anchor_mean(Field& x);
    void coarse_anchor(Field& x, bool singular);
    double coarse_residual(const LevelDev& L, const Field& x, const Field& b, Field* out, bool want_max);
    void gs_sweep_lex(const LevelDev& L, Field& x, const Field& b);

    // PressureSolver::solve
    void solve(Field& x, const Field& b, ismg_report& rep, ismg_step_metrics* m, int64_t fine_cells);

  private:
    double fetch(const double* d);
    void solve_plain(Field& x, const Field& b, ismg_report& rep, Metrics& M);
    void solve_two_level_ops(Field& x, const Field& b, ismg_report& rep, Metrics& M);
    void solve_acm(Field& x, const Field& b, ismg_report& rep, Metrics& M);
};

struct State {
    Ctx* ctx;
    ismg_grid_spec g;
    Velocity vel, vstar;
    Field p, rhs, dp;
    double t = 0.0, dt = 1.0, nu = 0.1;
    int64_t step_count = 0;
    State(Ctx* c, const ismg_grid_spec& g);
    void step(Solver& s, ismg_report& rep, ismg_step_metrics* m, int64_t fine_cells);
};

// fused.cu
bool fused_supported(const Solver& s);
FusedEngine* make_fused(Solver& s);
void fused_solve(Solver& s, Field& x, const Field& b, ismg_report& rep, Metrics& M, bool leave_pending_shift,
                 double** pending_shift);
void destroy_fused(FusedEngine* e);
double fused_bench_fine_pass(Solver& s, Field& x, const Field& b, int iters);
FusedEngine* make_coarse_engine(Solver& s, LevelDev& L);
long long coarse_engine_visit(FusedEngine& e, long long total, double rc0, int pred, double* rc);
double fused_bench_coarse_visit(Solver& s, const Field& cb, Field& ce, long long budget, int first,
                                long long* sweeps, double* rc);

}  // namespace ismgb

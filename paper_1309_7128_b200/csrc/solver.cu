// solver.cu — PressureSolver on the device (cycles.hpp:286-333) and the
// projection step (projection.hpp:139-190).
//
// Two execution paths share the same kernels' arithmetic:
//  * the fused hot path (fused.cu) for the interpolated/re-discretised
//    two-level schemes: device-resident control flow, one fused HBM pass per
//    fine iteration, pipelined coarse wavefront;
//  * the op-level path below, which replays cycles.hpp's control flow on the
//    host one reference call at a time (plain GS, the ACM V-cycle, and
//    configurations the fused kernels do not cover).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "solver.h"

namespace ismgb {

static void upload_axis(const TileAxisH& a, AxisDev& d) {
    d.n = a.n, d.tile = a.tile, d.nc = a.nc, d.periodic = a.periodic;
    ISMG_CUDA(cudaMalloc(&d.k0, sizeof(int) * a.n));
    ISMG_CUDA(cudaMalloc(&d.k1, sizeof(int) * a.n));
    ISMG_CUDA(cudaMalloc(&d.t, sizeof(double) * a.n));
    ISMG_CUDA(cudaMalloc(&d.dk, sizeof(double) * a.n));
    ISMG_H2D(d.k0, a.k0.data(), sizeof(int) * a.n);
    ISMG_H2D(d.k1, a.k1.data(), sizeof(int) * a.n);
    ISMG_H2D(d.t, a.t.data(), sizeof(double) * a.n);
    ISMG_H2D(d.dk, a.dk.data(), sizeof(double) * a.n);
}

static void free_axis(AxisDev& d) {
    cudaFree(d.k0), cudaFree(d.k1), cudaFree(d.t), cudaFree(d.dk);
    d = AxisDev{};
}

void LevelDev::upload(Ctx& c, int, int) {
    ISMG_CUDA(cudaMalloc(&d_w, sizeof(double) * h.w.size()));
    ISMG_H2D(d_w, h.w.data(), sizeof(double) * h.w.size());
    upload_axis(h.ax, ax);
    upload_axis(h.ay, ay);
    x = std::make_unique<Field>(&c, h.ncx, h.ncy);
    b = std::make_unique<Field>(&c, h.ncx, h.ncy);
    r = std::make_unique<Field>(&c, h.ncx, h.ncy);
}

void LevelDev::release() {
    if (d_w) cudaFree(d_w);
    d_w = nullptr;
    free_axis(ax);
    free_axis(ay);
    x.reset(), b.reset(), r.reset();
}

Solver::Solver(Ctx* c, const ismg_grid_spec& g0, const ismg_cycle_config& cfg0) : ctx(c), g(g0), cfg(cfg0) {
    cycle_validate(cfg);  // cycles.hpp:290
    if (cfg.scheme == ISMG_SCHEME_ISMG || cfg.scheme == ISMG_SCHEME_GMG) g.tile = cfg.tile;  // :291
    grid_validate(g);                                                                        // :292
    check_fine_stage(g);                                                                     // :293
    bc = pressure_bc(g, &singular);
    ISMG_CUDA(cudaSetDevice(ctx->device));
    if (cfg.scheme == ISMG_SCHEME_ISMG || cfg.scheme == ISMG_SCHEME_GMG) {
        levels.emplace_back();
        levels[0].h = cfg.scheme == ISMG_SCHEME_ISMG ? build_ismg_operator(g) : build_gmg_operator(g);
    } else if (cfg.scheme == ISMG_SCHEME_ACM) {
        for (auto& op : build_acm_hierarchy(g, cfg.depth)) {
            levels.emplace_back();
            levels.back().h = std::move(op);
        }
    }
    for (auto& L : levels) L.upload(*ctx, 0, 0);
    res = std::make_unique<Field>(ctx, g.nx, g.ny);
    if (fused_supported(*this)) fused = make_fused(*this);
    if (cfg.scheme == ISMG_SCHEME_ACM && !levels.empty() && !levels.back().h.px && !levels.back().h.py) {
        bool ok = true;  // a zero diagonal raises on the op-level path (coarsening.hpp:563-564)
        const CoarseOpH& h = levels.back().h;
        for (size_t k = 0; k < size_t(h.ncx) * h.ncy && ok; ++k) ok = h.w[k] != 0.0;
        if (ok) acm_coarse = make_coarse_engine(*this, levels.back());
    }
}

Solver::~Solver() {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);  // no throw from a destructor (the context may be torn down at exit)
    destroy_fused(fused);
    fused = nullptr;
    destroy_fused(acm_coarse);
    acm_coarse = nullptr;
    for (auto& L : levels) L.release();
}

double Solver::fetch(const double* d) {
    ISMG_CUDA(cudaMemcpyAsync(ctx->s.host, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    last.host_syncs += 1;
    return ctx->s.host[0];
}

// ---- op-level calls ---------------------------------------------------------
void Solver::rbgs_sweep(Field& x, const Field& b) {  // smoother.hpp:101-117
    for (int color = 0; color < 2; ++color) {
        k_refresh_periodic(*ctx, x.view(), bc.px(), bc.py());
        k_rbgs_half(*ctx, x.view(), b.view(), bc, color);
    }
    last.kernel_launches += (bc.px() || bc.py()) ? 4 : 2;
}

double Solver::fine_residual(Field& x, const Field& b, Field* out, bool want_max) {  // smoother.hpp:121-141
    k_refresh_periodic(*ctx, x.view(), bc.px(), bc.py());
    View o = out ? out->view() : View{};
    k_fine_residual(*ctx, x.view(), b.view(), o, bc, ctx->s.scal, nullptr);
    last.kernel_launches += 1;
    return want_max ? fetch(ctx->s.scal) : 0.0;
}

void Solver::anchor_mean(Field& x) {  // smoother.hpp:145-148
    if (!singular) return;
    k_mean_shift(*ctx, x.view(), ctx->s.scal + 2);
    k_shift_interior(*ctx, x.view(), ctx->s.scal + 3);
    last.kernel_launches += 3;
}

void Solver::coarse_anchor(Field& x, bool sing) {  // coarsening.hpp:592-595
    if (!sing) return;
    k_mean_shift(*ctx, x.view(), ctx->s.scal + 4);
    k_shift_interior(*ctx, x.view(), ctx->s.scal + 5);
    last.kernel_launches += 3;
}

double Solver::coarse_residual(const LevelDev& L, const Field& x, const Field& b, Field* out, bool want_max) {
    View o = out ? out->view() : View{};
    k_coarse_residual(*ctx, x.view(), b.view(), o, L.d_w, L.h.ncx, L.h.ncy, L.h.px, L.h.py, L.h.stencil_points(),
                      ctx->s.scal + 1);
    last.kernel_launches += 1;
    return want_max ? fetch(ctx->s.scal + 1) : 0.0;
}

void Solver::gs_sweep_lex(const LevelDev& L, Field& x, const Field& b) {  // coarsening.hpp:552-567
    const size_t n = size_t(L.h.ncx) * L.h.ncy;
    for (size_t k = 0; k < n; ++k)
        if (L.h.w[k] == 0.0) fail(ISMG_ERR_DOMAIN, "coarsening: singular stencil row");
    k_gs_lex(*ctx, x.view(), b.view(), L.d_w, L.h.ncx, L.h.ncy, L.h.px, L.h.py, L.h.stencil_points());
    last.kernel_launches += 1;
}

// ---- solves -------------------------------------------------------------------
void Solver::solve(Field& x, const Field& b, ismg_report& rep, ismg_step_metrics* m, int64_t fine_cells) {
    if (x.nx != g.nx || x.ny != g.ny || b.nx != g.nx || b.ny != g.ny)
        fail(ISMG_ERR_INVALID_ARGUMENT, "solve: field extents do not match the grid");
    ISMG_CUDA(cudaSetDevice(ctx->device));
    rep = ismg_report{1, 0, 0, 0, 0.0};
    last = ismg_solve_stats{};
    last.coarse_engine = -1;
    Metrics M{m, fine_cells > 0 ? fine_cells : int64_t(g.nx) * g.ny};
    cudaEvent_t e0, e1;
    ISMG_CUDA(cudaEventCreate(&e0));
    ISMG_CUDA(cudaEventCreate(&e1));
    ISMG_CUDA(cudaEventRecord(e0, ctx->stream));
    if (cfg.scheme == ISMG_SCHEME_PLAIN_GS) {
        solve_plain(x, b, rep, M);
    } else if (cfg.scheme == ISMG_SCHEME_ACM) {
        solve_acm(x, b, rep, M);
    } else if (fused && mode == 0) {
        fused_solve(*this, x, b, rep, M, false, nullptr);
    } else {
        solve_two_level_ops(x, b, rep, M);
    }
    ISMG_CUDA(cudaEventRecord(e1, ctx->stream));
    ISMG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    last.solve_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

// cycles.hpp:71-94
void Solver::solve_plain(Field& x, const Field& b, ismg_report& rep, Metrics& M) {
    const int64_t cells = int64_t(g.nx) * g.ny;
    k_zero_ghosts(*ctx, x.view());
    double r = fine_residual(x, b, nullptr, true);
    anchor_mean(x);
    long total = 0;
    while (r > cfg.tol_fine) {
        if (total >= cfg.max_total_sweeps) {
            rep.converged = 0;
            break;
        }
        rbgs_sweep(x, b);
        M.sweep(true, 5, cells);
        ++rep.fine_sweeps;
        ++total;
        last.fine_passes += 1;
        r = fine_residual(x, b, nullptr, true);
        anchor_mean(x);
    }
    rep.residual = r;
}

// cycles.hpp:101-165 replayed call by call (reference order).
void Solver::solve_two_level_ops(Field& x, const Field& b, ismg_report& rep, Metrics& M) {
    LevelDev& L = levels.front();
    const int64_t cells = int64_t(g.nx) * g.ny, ccells = int64_t(L.h.ncx) * L.h.ncy;
    const int stencil = L.h.stencil_points();
    for (size_t k = 0; k < size_t(ccells); ++k)
        if (L.h.w[k] == 0.0) fail(ISMG_ERR_DOMAIN, "coarsening: singular stencil row");
    k_zero_ghosts(*ctx, x.view());
    long total = 0;
    double r = fine_residual(x, b, res.get(), true);
    anchor_mean(x);
    while (r > cfg.tol_fine) {
        if (total >= cfg.max_total_sweeps) {
            rep.converged = 0;
            break;
        }
        k_restrict_exact(*ctx, res->view(), L.b->view(), g.tile, g.tile, L.h.ncx, L.h.ncy);
        M.restriction();
        k_fill(*ctx, L.x->view(), 0.0);
        double rc = coarse_residual(L, *L.x, *L.b, nullptr, true);
        long visit = 0;
        while (rc > cfg.tol_coarse && total < cfg.max_total_sweeps) {
            gs_sweep_lex(L, *L.x, *L.b);
            M.sweep(false, stencil, ccells);
            ++rep.coarse_sweeps;
            ++total;
            ++visit;
            rc = coarse_residual(L, *L.x, *L.b, nullptr, true);
            coarse_anchor(*L.x, L.h.singular);
        }
        last.coarse_visits += visit > 0;
        if (rc > cfg.tol_coarse) {
            rep.converged = 0;
            break;
        }
        if (visit > 0) {
            k_prolong_bilinear(*ctx, L.x->view(), x.view(), L.ax, L.ay);
            M.prolongation();
            last.prolong_passes += 1;
            r = fine_residual(x, b, res.get(), true);
            anchor_mean(x);
            if (r <= cfg.tol_fine) break;
        }
        double prev = r;
        while (total < cfg.max_total_sweeps) {
            rbgs_sweep(x, b);
            M.sweep(true, 5, cells);
            ++rep.fine_sweeps;
            ++total;
            last.fine_passes += 1;
            r = fine_residual(x, b, res.get(), true);
            anchor_mean(x);
            if (r <= cfg.tol_fine) break;
            if (r > cfg.stall_factor * prev) break;
            prev = r;
        }
        if (r > cfg.tol_fine && total >= cfg.max_total_sweeps) {
            rep.converged = 0;
            break;
        }
    }
    rep.residual = r;
}

// cycles.hpp:172-282 summed-hierarchy V-cycle; levels[k] tiles level k-1 (k=0: fine).
void Solver::solve_acm(Field& x, const Field& b, ismg_report& rep, Metrics& M) {
    const int L = int(levels.size());
    const int64_t cells = int64_t(g.nx) * g.ny;
    k_zero_ghosts(*ctx, x.view());
    long total = 0;
    int acm_pred = 1;  // first sweep group of the next coarsest visit (the last visit's length)
    double r = fine_residual(x, b, res.get(), true);
    anchor_mean(x);
    auto check_diag = [&](const LevelDev& lv) {
        const size_t n = size_t(lv.h.ncx) * lv.h.ncy;
        for (size_t k = 0; k < n; ++k)
            if (lv.h.w[k] == 0.0) fail(ISMG_ERR_DOMAIN, "coarsening: singular stencil row");
    };
    auto rbgs_level = [&](LevelDev& lv) {
        check_diag(lv);
        for (int color = 0; color < 2; ++color)
            k_rbgs_op(*ctx, lv.x->view(), lv.b->view(), lv.d_w, lv.h.ncx, lv.h.ncy, lv.h.px, lv.h.py, color);
        last.kernel_launches += 2;
    };
    while (r > cfg.tol_fine) {
        if (total >= cfg.max_total_sweeps) {
            rep.converged = 0;
            break;
        }
        bool capped = false;
        for (int k = 1; k <= L && !capped; ++k) {  // descend
            LevelDev& lv = levels[k - 1];
            const Field& above = (k == 1) ? *res : *levels[k - 2].r;
            k_restrict_exact(*ctx, above.view(), lv.b->view(), lv.h.ax.tile, lv.h.ay.tile, lv.h.ncx, lv.h.ncy);
            M.restriction();
            k_fill(*ctx, lv.x->view(), 0.0);
            if (k < L) {
                for (int s = 0; s < cfg.acm_pre_smooth; ++s) {
                    if (total >= cfg.max_total_sweeps) {
                        capped = true;
                        break;
                    }
                    rbgs_level(lv);
                    M.sweep(true, 5, int64_t(lv.h.ncx) * lv.h.ncy);
                    ++rep.fine_sweeps;
                    ++total;
                }
                coarse_residual(lv, *lv.x, *lv.b, lv.r.get(), false);
            } else if (acm_coarse && mode == 0) {
                // the coarsest level's GS loop (cycles.hpp:222-235) as ONE device-resident
                // coarse visit (the fused path's coarse kernel): one launch, one wait
                const double rc = coarse_residual(lv, *lv.x, *lv.b, nullptr, true);  // x = 0: max|b|
                if (rc > cfg.tol_coarse) {
                    if (total >= cfg.max_total_sweeps) {
                        capped = true;
                    } else {
                        double rc_end = 0.0;
                        const long long n = coarse_engine_visit(*acm_coarse, total, rc, acm_pred, &rc_end);
                        last.host_syncs += 1;
                        last.coarse_visits += 1;
                        for (long long q = 0; q < n; ++q) M.sweep(false, 5, int64_t(lv.h.ncx) * lv.h.ncy);
                        rep.coarse_sweeps += n;
                        total += long(n);
                        if (n > 0) acm_pred = int(std::min<long long>(n, 1 << 20));
                        if (rc_end > cfg.tol_coarse) capped = true;  // the budget ran out first
                    }
                }
            } else {
                double rc = coarse_residual(lv, *lv.x, *lv.b, nullptr, true);
                while (rc > cfg.tol_coarse) {
                    if (total >= cfg.max_total_sweeps) {
                        capped = true;
                        break;
                    }
                    gs_sweep_lex(lv, *lv.x, *lv.b);
                    M.sweep(false, 5, int64_t(lv.h.ncx) * lv.h.ncy);
                    ++rep.coarse_sweeps;
                    ++total;
                    rc = coarse_residual(lv, *lv.x, *lv.b, nullptr, true);
                    coarse_anchor(*lv.x, lv.h.singular);
                }
            }
        }
        if (capped) {
            rep.converged = 0;
            break;
        }
        for (int k = L - 1; k >= 1 && !capped; --k) {  // ascend
            LevelDev& below = levels[k];
            LevelDev& lv = levels[k - 1];
            k_prolong_constant(*ctx, below.x->view(), lv.x->view(), below.h.ax.tile, below.h.ay.tile);
            M.prolongation();
            for (int s = 0; s < cfg.acm_post_smooth; ++s) {
                if (total >= cfg.max_total_sweeps) {
                    capped = true;
                    break;
                }
                rbgs_level(lv);
                M.sweep(true, 5, int64_t(lv.h.ncx) * lv.h.ncy);
                ++rep.fine_sweeps;
                ++total;
            }
        }
        if (!capped) {
            k_prolong_constant(*ctx, levels[0].x->view(), x.view(), levels[0].h.ax.tile, levels[0].h.ay.tile);
            M.prolongation();
            for (int s = 0; s < cfg.acm_post_smooth; ++s) {
                if (total >= cfg.max_total_sweeps) {
                    capped = true;
                    break;
                }
                rbgs_sweep(x, b);
                M.sweep(true, 5, cells);
                ++rep.fine_sweeps;
                ++total;
                last.fine_passes += 1;
            }
        }
        r = fine_residual(x, b, res.get(), true);
        anchor_mean(x);
        if (capped && r > cfg.tol_fine) {
            rep.converged = 0;
            break;
        }
    }
    rep.residual = r;
}

// ---- FluidState / step ----------------------------------------------------------
State::State(Ctx* c, const ismg_grid_spec& g_)
    : ctx(c), g(g_), vel(c, g_.nx, g_.ny), vstar(c, g_.nx, g_.ny), p(c, g_.nx, g_.ny), rhs(c, g_.nx, g_.ny),
      dp(c, g_.nx, g_.ny) {
    grid_validate(g);
}

// projection.hpp:139-190 with every array resident in HBM.
void State::step(Solver& s, ismg_report& rep, ismg_step_metrics* m, int64_t fine_cells) {
    ISMG_CUDA(cudaSetDevice(ctx->device));
    Ctx& c = *ctx;
    const PBC bc = pressure_bc(g);
    k_scalar_bc(c, p.view(), bc);       // :142
    k_velocity_bc(c, vel, g);           // :143
    rep = ismg_report{1, 0, 0, 0, 0.0};
    if (dt == 0.0) {                    // :162-166
        step_count += 1;
        return;
    }
    // vstar = vel (:168) — full arrays including ghosts
    ISMG_CUDA(cudaMemcpyAsync(vstar.u.base, vel.u.base, vel.u.bytes, cudaMemcpyDeviceToDevice, c.stream));
    ISMG_CUDA(cudaMemcpyAsync(vstar.v.base, vel.v.base, vel.v.bytes, cudaMemcpyDeviceToDevice, c.stream));
    const bool px = g.bc[ISMG_SIDE_WEST].kind == ISMG_BC_PERIODIC;
    const bool py = g.bc[ISMG_SIDE_SOUTH].kind == ISMG_BC_PERIODIC;
    k_predictor(c, vel, p.view(), dt, nu, 1.0 / g.h, 1.0 / (g.h * g.h), px, py, vstar);  // :169
    k_velocity_bc(c, vstar, g);                                                           // :170
    k_fill(c, rhs.view(), 0.0);
    k_divergence(c, vstar, rhs.view(), 1.0 / g.h, g.h * g.h / dt, true);  // :172-178
    k_fill(c, dp.view(), 0.0);                                             // :180
    s.solve(dp, rhs, rep, m, fine_cells);                                  // :181
    k_scalar_bc(c, dp.view(), bc);                                         // :183 correct()
    k_correct(c, vstar, dp.view(), dt / g.h);
    std::swap(vel.u, vstar.u);  // :184 st.vel = vstar
    std::swap(vel.v, vstar.v);
    k_add_interior(c, p.view(), dp.view());  // :185
    t += dt;
    step_count += 1;
}

}  // namespace ismgb

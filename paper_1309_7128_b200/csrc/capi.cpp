// capi.cpp — the extern "C" boundary (include/ismg_b200.h). Every entry point
// catches C++ exceptions and maps them to the status codes that stand for the
// reference's exception types; the message is kept per thread.
#include <cstring>
#include <string>

#include "solver.h"

using namespace ismgb;

struct ismg_ctx {
    Ctx impl;
    ismg_ctx(int d, cudaStream_t s) : impl(d, s) {}
};
struct ismg_field {
    Field impl;
    ismg_field(Ctx* c, int nx, int ny) : impl(c, nx, ny) {}
};
struct ismg_velocity {
    Velocity impl;
    ismg_velocity(Ctx* c, int nx, int ny) : impl(c, nx, ny) {}
};
struct ismg_solver {
    Solver impl;
    ismg_solver(Ctx* c, const ismg_grid_spec& g, const ismg_cycle_config& cf) : impl(c, g, cf) {}
};
struct ismg_state {
    State impl;
    ismg_state(Ctx* c, const ismg_grid_spec& g) : impl(c, g) {}
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return ISMG_OK;
    } catch (const Status& s) {
        g_err = s.what();
        return s.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return ISMG_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ISMG_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return ISMG_ERR_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) fail(ISMG_ERR_INVALID_ARGUMENT, std::string(what) + " is null");
}

// host <-> device copies of a ghosted logical block starting at (-1, -1)
void copy_in(Ctx& c, const DevBuf& d, const double* host, int w, int h, size_t count) {
    if (count != size_t(w) * size_t(h)) fail(ISMG_ERR_INVALID_ARGUMENT, "host array size does not match the field");
    ISMG_CUDA(cudaSetDevice(c.device));
    double* dst = d.origin() - d.pitch - 1;
    ISMG_CUDA(cudaMemcpy2DAsync(dst, d.pitch * sizeof(double), host, w * sizeof(double), w * sizeof(double), h,
                                cudaMemcpyHostToDevice, c.stream));
    c.sync();
}
void copy_out(Ctx& c, const DevBuf& d, double* host, int w, int h, size_t count) {
    if (count != size_t(w) * size_t(h)) fail(ISMG_ERR_INVALID_ARGUMENT, "host array size does not match the field");
    ISMG_CUDA(cudaSetDevice(c.device));
    const double* src = d.origin() - d.pitch - 1;
    ISMG_CUDA(cudaMemcpy2DAsync(host, w * sizeof(double), src, d.pitch * sizeof(double), w * sizeof(double), h,
                                cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

void write_planes(const CoarseOpH& op, int32_t* ncx, int32_t* ncy, double* w, size_t count) {
    need(ncx, "ncx");
    need(ncy, "ncy");
    *ncx = op.ncx;
    *ncy = op.ncy;
    if (!w) return;
    if (count != op.w.size()) fail(ISMG_ERR_INVALID_ARGUMENT, "coefficient buffer size mismatch");
    std::memcpy(w, op.w.data(), op.w.size() * sizeof(double));
}

Solver& S(ismg_solver* s) {
    need(s, "solver");
    return s->impl;
}
Field& F(ismg_field* f) {
    need(f, "field");
    return f->impl;
}
const Field& F(const ismg_field* f) {
    need(f, "field");
    return f->impl;
}
void same_ctx(const Solver& s, const Field& f) {
    if (f.ctx != s.ctx) fail(ISMG_ERR_INVALID_ARGUMENT, "field and solver belong to different contexts");
}
void fine_dims(const Solver& s, const Field& f) {
    same_ctx(s, f);
    if (f.nx != s.g.nx || f.ny != s.g.ny) fail(ISMG_ERR_INVALID_ARGUMENT, "field extents do not match the grid");
}
const LevelDev& coarse_level(const Solver& s, const Field& f) {
    same_ctx(s, f);
    if (s.levels.empty()) fail(ISMG_ERR_INVALID_ARGUMENT, "solver has no coarse level");
    const LevelDev& L = s.levels.front();
    if (f.nx != L.h.ncx || f.ny != L.h.ncy) fail(ISMG_ERR_INVALID_ARGUMENT, "coarse field extents mismatch");
    return L;
}
}  // namespace

extern "C" {

const char* ismg_last_error(void) { return g_err.c_str(); }
int ismg_abi_version(void) { return ISMG_B200_ABI_VERSION; }

int ismg_device_count(int* out) {
    return guard([&] {
        need(out, "out");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *out = n;
    });
}

int ismg_ctx_create(int device, void* stream, ismg_ctx** out) {
    return guard([&] {
        need(out, "out");
        *out = new ismg_ctx(device, static_cast<cudaStream_t>(stream));
    });
}
int ismg_ctx_destroy(ismg_ctx* c) {
    return guard([&] { delete c; });
}
int ismg_ctx_synchronize(ismg_ctx* c) {
    return guard([&] {
        need(c, "ctx");
        c->impl.sync();
    });
}

int ismg_grid_validate(const ismg_grid_spec* g) {
    return guard([&] {
        need(g, "grid");
        grid_validate(*g);
    });
}
int ismg_cycle_validate(const ismg_cycle_config* c) {
    return guard([&] {
        need(c, "config");
        cycle_validate(*c);
    });
}
int ismg_pressure_bc(const ismg_grid_spec* g, int32_t out[4], int32_t* singular) {
    return guard([&] {
        need(g, "grid");
        need(out, "out");
        bool sing = false;
        PBC p = pressure_bc(*g, &sing);
        for (int s = 0; s < 4; ++s) out[s] = p.k[s];
        if (singular) *singular = sing;
    });
}
int ismg_build_fine_diag(const ismg_grid_spec* g, double* diag, size_t count) {
    return guard([&] {
        need(g, "grid");
        need(diag, "diag");
        check_fine_stage(*g);
        if (count != size_t(g->nx + 2) * size_t(g->ny + 2)) fail(ISMG_ERR_INVALID_ARGUMENT, "diag size mismatch");
        PBC p = pressure_bc(*g);
        auto fw = [](int k) { return k == ISMG_PBC_NEUMANN ? 0.0 : k == ISMG_PBC_DIRICHLET_ZERO ? 2.0 : 1.0; };
        std::memset(diag, 0, count * sizeof(double));
        for (int j = 0; j < g->ny; ++j)
            for (int i = 0; i < g->nx; ++i) {
                double d = 0;
                d += (i > 0) ? 1.0 : fw(p.k[0]);
                d += (i < g->nx - 1) ? 1.0 : fw(p.k[1]);
                d += (j > 0) ? 1.0 : fw(p.k[2]);
                d += (j < g->ny - 1) ? 1.0 : fw(p.k[3]);
                diag[size_t(j + 1) * (g->nx + 2) + (i + 1)] = d;
            }
    });
}
int ismg_build_ismg_operator(const ismg_grid_spec* g, int32_t* ncx, int32_t* ncy, double* w, size_t count) {
    return guard([&] {
        need(g, "grid");
        write_planes(build_ismg_operator(*g), ncx, ncy, w, count);
    });
}
int ismg_build_gmg_operator(const ismg_grid_spec* g, int32_t* ncx, int32_t* ncy, double* w, size_t count) {
    return guard([&] {
        need(g, "grid");
        write_planes(build_gmg_operator(*g), ncx, ncy, w, count);
    });
}

int ismg_field_create(ismg_ctx* c, int nx, int ny, ismg_field** out) {
    return guard([&] {
        need(c, "ctx");
        need(out, "out");
        *out = new ismg_field(&c->impl, nx, ny);
    });
}
int ismg_field_destroy(ismg_field* f) {
    return guard([&] { delete f; });
}
int ismg_field_dims(const ismg_field* f, int32_t* nx, int32_t* ny) {
    return guard([&] {
        need(f, "field");
        if (nx) *nx = f->impl.nx;
        if (ny) *ny = f->impl.ny;
    });
}
int ismg_field_upload(ismg_field* f, const double* host, size_t count) {
    return guard([&] {
        Field& x = F(f);
        need(host, "host");
        copy_in(*x.ctx, x.buf, host, x.nx + 2, x.ny + 2, count);
    });
}
int ismg_field_download(const ismg_field* f, double* host, size_t count) {
    return guard([&] {
        const Field& x = F(f);
        need(host, "host");
        copy_out(*x.ctx, x.buf, host, x.nx + 2, x.ny + 2, count);
    });
}
int ismg_field_fill(ismg_field* f, double value) {
    return guard([&] {
        Field& x = F(f);
        k_fill(*x.ctx, x.view(), value);
    });
}

int ismg_velocity_create(ismg_ctx* c, int nx, int ny, ismg_velocity** out) {
    return guard([&] {
        need(c, "ctx");
        need(out, "out");
        *out = new ismg_velocity(&c->impl, nx, ny);
    });
}
int ismg_velocity_destroy(ismg_velocity* v) {
    return guard([&] { delete v; });
}
int ismg_velocity_upload(ismg_velocity* v, const double* u_host, size_t uc, const double* v_host, size_t vc) {
    return guard([&] {
        need(v, "velocity");
        Velocity& V = v->impl;
        copy_in(*V.ctx, V.u, u_host, V.nx + 3, V.ny + 2, uc);
        copy_in(*V.ctx, V.v, v_host, V.nx + 2, V.ny + 3, vc);
    });
}
int ismg_velocity_download(const ismg_velocity* v, double* u_host, size_t uc, double* v_host, size_t vc) {
    return guard([&] {
        need(v, "velocity");
        const Velocity& V = v->impl;
        copy_out(*V.ctx, V.u, u_host, V.nx + 3, V.ny + 2, uc);
        copy_out(*V.ctx, V.v, v_host, V.nx + 2, V.ny + 3, vc);
    });
}

int ismg_solver_create(ismg_ctx* c, const ismg_grid_spec* g, const ismg_cycle_config* cf, ismg_solver** out) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        need(cf, "config");
        need(out, "out");
        *out = new ismg_solver(&c->impl, *g, *cf);
    });
}
int ismg_solver_destroy(ismg_solver* s) {
    return guard([&] { delete s; });
}
int ismg_solver_info(const ismg_solver* s, ismg_grid_spec* g_out, int32_t* ncx, int32_t* ncy, int32_t* singular) {
    return guard([&] {
        need(s, "solver");
        const Solver& v = s->impl;
        if (g_out) *g_out = v.g;
        if (ncx) *ncx = v.levels.empty() ? 0 : v.levels.front().h.ncx;
        if (ncy) *ncy = v.levels.empty() ? 0 : v.levels.front().h.ncy;
        if (singular) *singular = v.singular;
    });
}

int ismg_rbgs_sweep(ismg_solver* s, ismg_field* x, const ismg_field* b) {
    return guard([&] {
        Solver& v = S(s);
        fine_dims(v, F(x));
        fine_dims(v, F(b));
        v.rbgs_sweep(F(x), F(b));
    });
}
int ismg_fine_residual(ismg_solver* s, ismg_field* x, const ismg_field* b, ismg_field* out, double* rmax) {
    return guard([&] {
        Solver& v = S(s);
        fine_dims(v, F(x));
        fine_dims(v, F(b));
        if (out) fine_dims(v, F(out));
        double r = v.fine_residual(F(x), F(b), out ? &F(out) : nullptr, rmax != nullptr);
        if (rmax) *rmax = r;
    });
}
int ismg_anchor_mean(ismg_solver* s, ismg_field* x) {
    return guard([&] {
        Solver& v = S(s);
        fine_dims(v, F(x));
        v.anchor_mean(F(x));
    });
}
int ismg_zero_ghosts(ismg_solver* s, ismg_field* x) {
    return guard([&] {
        Solver& v = S(s);
        same_ctx(v, F(x));
        k_zero_ghosts(*v.ctx, F(x).view());
    });
}
int ismg_restrict_sum(ismg_solver* s, const ismg_field* fine, ismg_field* coarse) {
    return guard([&] {
        Solver& v = S(s);
        fine_dims(v, F(fine));
        const LevelDev& L = coarse_level(v, F(coarse));
        k_restrict_exact(*v.ctx, F(fine).view(), F(coarse).view(), L.h.ax.tile, L.h.ay.tile, L.h.ncx, L.h.ncy);
    });
}
int ismg_prolongate_bilinear(ismg_solver* s, const ismg_field* coarse, ismg_field* fine) {
    return guard([&] {
        Solver& v = S(s);
        fine_dims(v, F(fine));
        const LevelDev& L = coarse_level(v, F(coarse));
        k_prolong_bilinear(*v.ctx, F(coarse).view(), F(fine).view(), L.ax, L.ay);
    });
}
int ismg_coarse_residual(ismg_solver* s, const ismg_field* x, const ismg_field* b, ismg_field* out, double* rmax) {
    return guard([&] {
        Solver& v = S(s);
        const LevelDev& L = coarse_level(v, F(x));
        coarse_level(v, F(b));
        if (out) coarse_level(v, F(out));
        double r = v.coarse_residual(L, F(x), F(b), out ? &F(out) : nullptr, rmax != nullptr);
        if (rmax) *rmax = r;
    });
}
int ismg_gs_sweep_lex(ismg_solver* s, ismg_field* x, const ismg_field* b) {
    return guard([&] {
        Solver& v = S(s);
        const LevelDev& L = coarse_level(v, F(x));
        coarse_level(v, F(b));
        v.gs_sweep_lex(L, F(x), F(b));
    });
}
int ismg_coarse_anchor_mean(ismg_solver* s, ismg_field* x) {
    return guard([&] {
        Solver& v = S(s);
        const LevelDev& L = coarse_level(v, F(x));
        v.coarse_anchor(F(x), L.h.singular);
    });
}

int ismg_solve(ismg_solver* s, ismg_field* x, const ismg_field* b, ismg_report* rep, ismg_step_metrics* current,
               int64_t fine_cells) {
    return guard([&] {
        Solver& v = S(s);
        need(rep, "report");
        fine_dims(v, F(x));
        fine_dims(v, F(b));
        v.solve(F(x), F(b), *rep, current, fine_cells);
    });
}

int ismg_solve_host(ismg_solver* s, double* x_host, const double* b_host, size_t count, ismg_report* rep,
                    ismg_step_metrics* current, int64_t fine_cells) {
    return guard([&] {
        Solver& v = S(s);
        need(rep, "report");
        need(x_host, "x");
        need(b_host, "b");
        Field x(v.ctx, v.g.nx, v.g.ny), b(v.ctx, v.g.nx, v.g.ny);
        copy_in(*v.ctx, x.buf, x_host, v.g.nx + 2, v.g.ny + 2, count);
        copy_in(*v.ctx, b.buf, b_host, v.g.nx + 2, v.g.ny + 2, count);
        v.solve(x, b, *rep, current, fine_cells);
        copy_out(*v.ctx, x.buf, x_host, v.g.nx + 2, v.g.ny + 2, count);
    });
}

int ismg_solver_visit_log(const ismg_solver* s, int32_t* out, size_t cap, size_t* n) {
    return guard([&] {
        need(s, "solver");
        need(n, "n");
        const std::vector<int>& log = s->impl.visit_log;
        *n = log.size() / 2;
        if (out)
            for (size_t k = 0; k < std::min(cap, *n) * 2; ++k) out[k] = log[k];
    });
}

int ismg_bench_fine_pass(ismg_solver* s, ismg_field* x, const ismg_field* b, int iters, double* ms_per_pass) {
    return guard([&] {
        Solver& v = S(s);
        need(ms_per_pass, "ms_per_pass");
        fine_dims(v, F(x));
        fine_dims(v, F(b));
        if (!v.fused) fail(ISMG_ERR_INVALID_ARGUMENT, "bench_fine_pass: solver has no fused path");
        if (iters < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "bench_fine_pass: iters must be >= 1");
        ISMG_CUDA(cudaSetDevice(v.ctx->device));
        *ms_per_pass = fused_bench_fine_pass(v, F(x), F(b), iters);
    });
}

int ismg_bench_coarse_visit(ismg_solver* s, const ismg_field* cb, ismg_field* ce, int64_t budget, int first_group,
                            int64_t* sweeps, double* rc, double* ms) {
    return guard([&] {
        Solver& v = S(s);
        need(sweeps, "sweeps");
        need(rc, "rc");
        need(ms, "ms");
        if (!v.fused) fail(ISMG_ERR_INVALID_ARGUMENT, "bench_coarse_visit: solver has no fused path");
        ISMG_CUDA(cudaSetDevice(v.ctx->device));
        long long n = 0;
        *ms = fused_bench_coarse_visit(v, F(cb), F(ce), budget, first_group, &n, rc);
        *sweeps = n;
    });
}

int ismg_ctx_launch_count(const ismg_ctx* c, int64_t* out) {
    return guard([&] {
        need(c, "ctx");
        need(out, "out");
        *out = c->impl.launches;
    });
}

int ismg_solver_last_stats(const ismg_solver* s, ismg_solve_stats* out) {
    return guard([&] {
        need(s, "solver");
        need(out, "out");
        *out = s->impl.last;
    });
}

int ismg_apply_scalar_bc(ismg_ctx* c, const ismg_grid_spec* g, ismg_field* f) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        k_scalar_bc(c->impl, F(f).view(), pressure_bc(*g));
    });
}
int ismg_apply_velocity_bc(ismg_ctx* c, const ismg_grid_spec* g, ismg_velocity* vel) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        need(vel, "velocity");
        k_velocity_bc(c->impl, vel->impl, *g);
    });
}
int ismg_divergence(ismg_ctx* c, const ismg_grid_spec* g, const ismg_velocity* vel, ismg_field* out, double scale) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        need(vel, "velocity");
        k_divergence(c->impl, vel->impl, F(out).view(), 1.0 / g->h, scale, scale != 1.0);
    });
}
int ismg_correct(ismg_ctx* c, const ismg_grid_spec* g, ismg_velocity* vel, ismg_field* dp, double dt) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        need(vel, "velocity");
        k_scalar_bc(c->impl, F(dp).view(), pressure_bc(*g));
        k_correct(c->impl, vel->impl, F(dp).view(), dt / g->h);
    });
}
int ismg_predictor(ismg_ctx* c, const ismg_grid_spec* g, const ismg_velocity* vel, const ismg_field* p, double dt,
                   double nu, ismg_velocity* out) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        need(vel, "velocity");
        need(out, "out");
        const bool px = g->bc[ISMG_SIDE_WEST].kind == ISMG_BC_PERIODIC;
        const bool py = g->bc[ISMG_SIDE_SOUTH].kind == ISMG_BC_PERIODIC;
        k_predictor(c->impl, vel->impl, F(p).view(), dt, nu, 1.0 / g->h, 1.0 / (g->h * g->h), px, py, out->impl);
    });
}

int ismg_state_create(ismg_ctx* c, const ismg_grid_spec* g, ismg_state** out) {
    return guard([&] {
        need(c, "ctx");
        need(g, "grid");
        need(out, "out");
        *out = new ismg_state(&c->impl, *g);
    });
}
int ismg_state_destroy(ismg_state* st) {
    return guard([&] { delete st; });
}
int ismg_state_set_scalars(ismg_state* st, double t, double dt, double nu, int64_t step_count) {
    return guard([&] {
        need(st, "state");
        st->impl.t = t, st->impl.dt = dt, st->impl.nu = nu, st->impl.step_count = step_count;
    });
}
int ismg_state_get_scalars(const ismg_state* st, double* t, double* dt, double* nu, int64_t* step_count) {
    return guard([&] {
        need(st, "state");
        if (t) *t = st->impl.t;
        if (dt) *dt = st->impl.dt;
        if (nu) *nu = st->impl.nu;
        if (step_count) *step_count = st->impl.step_count;
    });
}
int ismg_state_upload(ismg_state* st, const double* u, size_t uc, const double* v, size_t vc, const double* p,
                      size_t pc) {
    return guard([&] {
        need(st, "state");
        State& S_ = st->impl;
        copy_in(*S_.ctx, S_.vel.u, u, S_.g.nx + 3, S_.g.ny + 2, uc);
        copy_in(*S_.ctx, S_.vel.v, v, S_.g.nx + 2, S_.g.ny + 3, vc);
        copy_in(*S_.ctx, S_.p.buf, p, S_.g.nx + 2, S_.g.ny + 2, pc);
    });
}
int ismg_state_download(const ismg_state* st, double* u, size_t uc, double* v, size_t vc, double* p, size_t pc) {
    return guard([&] {
        need(st, "state");
        const State& S_ = st->impl;
        if (u) copy_out(*S_.ctx, S_.vel.u, u, S_.g.nx + 3, S_.g.ny + 2, uc);
        if (v) copy_out(*S_.ctx, S_.vel.v, v, S_.g.nx + 2, S_.g.ny + 3, vc);
        if (p) copy_out(*S_.ctx, S_.p.buf, p, S_.g.nx + 2, S_.g.ny + 2, pc);
    });
}
int ismg_step(ismg_state* st, ismg_solver* s, ismg_report* rep, ismg_step_metrics* current, int64_t fine_cells) {
    return guard([&] {
        need(st, "state");
        need(rep, "report");
        Solver& v = S(s);
        if (st->impl.g.nx != v.g.nx || st->impl.g.ny != v.g.ny)
            fail(ISMG_ERR_INVALID_ARGUMENT, "state and solver grids differ");
        st->impl.step(v, *rep, current, fine_cells);
    });
}

int ismg_nccl_unique_id(void* out, size_t bytes) {
    return guard([&] {
        need(out, "out");
        if (bytes < 128) fail(ISMG_ERR_INVALID_ARGUMENT, "unique id buffer must hold 128 bytes");
        nccl_unique_id(out);
    });
}

int ismg_ctx_attach_comm(ismg_ctx* c, const void* id, int rank, int nranks) {
    return guard([&] {
        need(c, "ctx");
        need(id, "unique id");
        Ctx& x = c->impl;
        if (x.comm) fail(ISMG_ERR_INVALID_ARGUMENT, "context already has a communicator");
        x.comm = make_comm(x.device, id, rank, nranks);
    });
}

int ismg_strip_rows(int ny, int tile, int nranks, int rank, int32_t* r0, int32_t* r1) {
    return guard([&] {
        need(r0, "r0");
        need(r1, "r1");
        int a = 0, b = 0;
        strip_rows(ny, tile, nranks, rank, &a, &b);
        *r0 = a, *r1 = b;
    });
}

}  // extern "C"

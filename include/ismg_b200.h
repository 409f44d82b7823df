/*
 * ismg_b200.h — C-ABI of the B200-native ISM pressure solve.
 *
 * Drop-in boundary for the pressure path of the reference's header-only C++
 * library `ismg` (arXiv 1309.7128 reference, /root/reference/proj/include/ismg).
 * Every entry point below names the reference interface it replaces
 * (path:line relative to the reference root). Plain pointers and sizes only:
 * no CUDA, torch or C++ types cross this boundary.
 *
 * Conventions:
 *   - every function returns an int status (ISMG_OK = 0); the message of the
 *     last failure on the calling thread is returned by ismg_last_error();
 *   - status codes map to the reference's exception types:
 *       ISMG_ERR_INVALID_ARGUMENT -> std::invalid_argument
 *       ISMG_ERR_DOMAIN           -> std::domain_error
 *       ISMG_ERR_LOGIC            -> std::logic_error
 *     plus device-side failures (CUDA / NCCL / no device);
 *   - op-level calls are stream-ordered and asynchronous; calls returning a
 *     host scalar (residual max, reports) synchronise the context stream;
 *   - fields live on the device with the reference's logical layout (one
 *     ghost ring around an nx x ny interior); host arrays passed to
 *     upload/download use exactly the reference layout:
 *       scalar  (nx+2)*(ny+2), index (j+1)*(nx+2) + (i+1)     field.hpp:24-31
 *       u       (nx+3)*(ny+2), index (j+1)*(nx+3) + (i+1)     field.hpp:108-117
 *       v       (nx+2)*(ny+3), index (j+1)*(nx+2) + (i+1)     field.hpp:108-117
 *   - one context per host thread; there is no global mutable state apart
 *     from the thread-local error string.
 *
 * Arithmetic is fp64 (T = double in the reference templates).
 */
#ifndef ISMG_B200_H
#define ISMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define ISMG_B200_ABI_VERSION 2

/* ---- status codes -------------------------------------------------------- */
enum {
    ISMG_OK = 0,
    ISMG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    ISMG_ERR_DOMAIN = 2,           /* std::domain_error     */
    ISMG_ERR_LOGIC = 3,            /* std::logic_error      */
    ISMG_ERR_CUDA = 4,
    ISMG_ERR_NCCL = 5,
    ISMG_ERR_NO_DEVICE = 6,
    ISMG_ERR_INTERNAL = 7
};

/* ---- enums (grid.hpp:18-28, grid.hpp:119, coarsening.hpp:27) ------------- */
enum { ISMG_SIDE_WEST = 0, ISMG_SIDE_EAST = 1, ISMG_SIDE_SOUTH = 2, ISMG_SIDE_NORTH = 3 };
enum {
    ISMG_BC_DIRICHLET_VELOCITY = 0,
    ISMG_BC_SYMMETRY_FIXED_PRESSURE = 1,
    ISMG_BC_PERIODIC = 2,
    ISMG_BC_INLET = 3
};
enum { ISMG_PBC_NEUMANN = 0, ISMG_PBC_DIRICHLET_ZERO = 1, ISMG_PBC_PERIODIC = 2 };
enum {
    ISMG_SCHEME_PLAIN_GS = 0,
    ISMG_SCHEME_ISMG = 1,
    ISMG_SCHEME_GMG = 2,
    ISMG_SCHEME_ACM = 3
};

/* ---- value types --------------------------------------------------------- */
/* BoundaryCondition — grid.hpp:30-65 */
typedef struct ismg_bc {
    int32_t kind; /* ISMG_BC_* */
    int32_t inlet_start;
    int32_t inlet_width;
    int32_t reserved;
    double u_wall;
    double v_wall;
    double p_wall;
    double v_inflow;
} ismg_bc;

/* GridSpec — grid.hpp:67-97 (bc indexed by ISMG_SIDE_*) */
typedef struct ismg_grid_spec {
    int32_t nx;
    int32_t ny;
    double h;
    int32_t tile;
    int32_t reserved;
    ismg_bc bc[4];
} ismg_grid_spec;

/* CycleConfig — cycles.hpp:20-45 */
typedef struct ismg_cycle_config {
    int32_t scheme; /* ISMG_SCHEME_* */
    int32_t tile;
    int32_t depth;
    int32_t acm_pre_smooth;
    int32_t acm_post_smooth;
    int32_t reserved;
    double tol_fine;
    double tol_coarse;
    int64_t max_total_sweeps;
    double stall_factor;
} ismg_cycle_config;

/* ConvergenceReport — cycles.hpp:47-52 (+ a NaN side channel that never
 * alters control flow). */
typedef struct ismg_report {
    int32_t converged;
    int32_t nan_seen;
    int64_t fine_sweeps;
    int64_t coarse_sweeps;
    double residual;
} ismg_report;

/* StepMetrics — metrics.hpp:22-35 (the running `current` row). */
typedef struct ismg_step_metrics {
    int64_t step;
    int64_t fine_sweeps;   /* I_f   */
    int64_t coarse_sweeps; /* I_c   */
    int64_t sync_fine;     /* NCC_f */
    int64_t sync_coarse;   /* NCC_c */
    double lap_equiv;      /* N_Lap */
    int64_t restrictions;
    int64_t prolongations;
    double residual_final;
    int32_t converged;
    int32_t reserved;
} ismg_step_metrics;

/* Measured synchronisation events and device timing of the last solve
 * (extension: the model counts above are the reference's NCC; these are the
 * B200 implementation's real kernel boundaries / host round trips). */
typedef struct ismg_solve_stats {
    int64_t fine_passes;        /* fused fine-grid passes launched with work */
    int64_t prolong_passes;     /* prolongation + residual passes            */
    int64_t coarse_visits;      /* coarse-solve kernel launches with work    */
    int64_t kernel_launches;    /* all kernels launched by the solve          */
    int64_t host_syncs;         /* host <-> device round trips                */
    int64_t collectives;        /* NCCL calls (multi-GPU; not the per-pass exchange) */
    double fine_pass_ms;        /* summed CUDA-event time of fine passes      */
    double coarse_ms;           /* summed CUDA-event time of coarse visits    */
    double solve_ms;            /* CUDA-event time of the whole solve         */
    int64_t coarse_steps;       /* wavefront steps of the coarse visits       */
    int64_t coarse_engine;      /* coarse-visit kernel of the fused path: 0 global
                                   wavefront, 1 shared-memory iterate, 2 TMEM rhs,
                                   3 cluster bands, 4 register wavefront,
                                   5 sweep pipeline, 6 sweep pipeline with several
                                   blocks per warp; -1 op-level */
} ismg_solve_stats;

/* ---- opaque handles ------------------------------------------------------ */
typedef struct ismg_ctx ismg_ctx;
typedef struct ismg_field ismg_field;       /* ScalarField<double>  field.hpp:18-71   */
typedef struct ismg_velocity ismg_velocity; /* MacVelocity<double>  field.hpp:102-137 */
typedef struct ismg_solver ismg_solver;     /* PressureSolver<double> cycles.hpp:286-333 */
typedef struct ismg_state ismg_state;       /* FluidState<double>  projection.hpp:26-36 */

/* ---- library / context ---------------------------------------------------- */
const char* ismg_last_error(void);
int ismg_abi_version(void);
int ismg_device_count(int* out);
/* stream: a cudaStream_t (NULL = the context creates its own non-blocking stream) */
int ismg_ctx_create(int device, void* stream, ismg_ctx** out);
int ismg_ctx_destroy(ismg_ctx* ctx);
int ismg_ctx_synchronize(ismg_ctx* ctx);
/* multi-GPU (strip decomposition along y; no reference
 * counterpart — the reference is single-core). Rank 0 makes a 128-byte
 * ncclUniqueId, the caller shares it, every rank attaches it to its context
 * BEFORE creating solvers (collective: every rank creates the same solvers in
 * the same order). Fused solves on that context then own the rank's strip of
 * fine rows and exchange halo rows / scalars / coarse rhs inside the fine pass
 * through peer memory (CUDA IPC over NVLink; the ranks must be on one node with
 * peer access), and return the full solution on every rank (NCCL, once per
 * solve). At most 8 ranks. */
int ismg_nccl_unique_id(void* out, size_t bytes);
int ismg_ctx_attach_comm(ismg_ctx* ctx, const void* nccl_unique_id, int rank, int nranks);
/* rows [r0, r1) of a rank: whole coarse tiles, as even as possible (host only) */
int ismg_strip_rows(int ny, int tile, int nranks, int rank, int32_t* r0, int32_t* r1);

/* ---- host-side geometry (no device needed) -------------------------------- */
/* GridSpec::validate — grid.hpp:79-96 */
int ismg_grid_validate(const ismg_grid_spec* g);
/* CycleConfig::validate — cycles.hpp:31-44 */
int ismg_cycle_validate(const ismg_cycle_config* c);
/* pressure_bc + pressure_singular — grid.hpp:124-149 */
int ismg_pressure_bc(const ismg_grid_spec* g, int32_t out[4], int32_t* singular);
/* build_fine_stage diag — smoother.hpp:36-67; diag has the scalar layout */
int ismg_build_fine_diag(const ismg_grid_spec* g, double* diag_host, size_t count);
/* build_ismg_operator — coarsening.hpp:196-305. Call with w == NULL to query
 * (ncx, ncy); then w receives 9 planes of ncx*ncy coefficients in slot order
 * C,E,W,N,S,NE,NW,SE,SW (coarsening.hpp:121-125), plane-major. */
int ismg_build_ismg_operator(const ismg_grid_spec* g, int32_t* ncx, int32_t* ncy, double* w,
                             size_t count);
/* build_gmg_operator — coarsening.hpp:311-360 (same output convention) */
int ismg_build_gmg_operator(const ismg_grid_spec* g, int32_t* ncx, int32_t* ncy, double* w,
                            size_t count);

/* ---- device fields -------------------------------------------------------- */
int ismg_field_create(ismg_ctx* ctx, int nx, int ny, ismg_field** out); /* zero-filled */
int ismg_field_destroy(ismg_field* f);
int ismg_field_dims(const ismg_field* f, int32_t* nx, int32_t* ny);
int ismg_field_upload(ismg_field* f, const double* host, size_t count);
int ismg_field_download(const ismg_field* f, double* host, size_t count);
int ismg_field_fill(ismg_field* f, double value); /* ScalarField::fill field.hpp:184-186 */

int ismg_velocity_create(ismg_ctx* ctx, int nx, int ny, ismg_velocity** out);
int ismg_velocity_destroy(ismg_velocity* v);
int ismg_velocity_upload(ismg_velocity* v, const double* u_host, size_t u_count,
                         const double* v_host, size_t v_count);
int ismg_velocity_download(const ismg_velocity* v, double* u_host, size_t u_count,
                           double* v_host, size_t v_count);

/* ---- solver --------------------------------------------------------------- */
/* PressureSolver(grid, cfg) — cycles.hpp:289-308 */
int ismg_solver_create(ismg_ctx* ctx, const ismg_grid_spec* g, const ismg_cycle_config* c,
                       ismg_solver** out);
int ismg_solver_destroy(ismg_solver* s);
/* effective grid (tile adopted from the cycle config) and coarse dims */
int ismg_solver_info(const ismg_solver* s, ismg_grid_spec* g_out, int32_t* ncx, int32_t* ncy,
                     int32_t* singular);

/* op-level calls (stream-ordered). `x`/`b` are fine fields unless noted. */
/* rbgs_sweep — smoother.hpp:101-117 */
int ismg_rbgs_sweep(ismg_solver* s, ismg_field* x, const ismg_field* b);
/* fine_residual — smoother.hpp:121-141; out may be NULL; rmax may be NULL
 * (then the call does not synchronise). */
int ismg_fine_residual(ismg_solver* s, ismg_field* x, const ismg_field* b, ismg_field* out,
                       double* rmax);
/* anchor_mean (fine) — smoother.hpp:145-148 */
int ismg_anchor_mean(ismg_solver* s, ismg_field* x);
/* zero_ghosts — smoother.hpp:71-81 */
int ismg_zero_ghosts(ismg_solver* s, ismg_field* x);
/* restrict_sum — coarsening.hpp:471-480 (coarse is ncx x ncy) */
int ismg_restrict_sum(ismg_solver* s, const ismg_field* fine, ismg_field* coarse);
/* prolongate_bilinear — coarsening.hpp:485-503 (adds into fine) */
int ismg_prolongate_bilinear(ismg_solver* s, const ismg_field* coarse, ismg_field* fine);
/* coarse_residual — coarsening.hpp:531-549 (coarse fields) */
int ismg_coarse_residual(ismg_solver* s, const ismg_field* x, const ismg_field* b,
                         ismg_field* out, double* rmax);
/* gs_sweep_lex — coarsening.hpp:552-567 (coarse fields) */
int ismg_gs_sweep_lex(ismg_solver* s, ismg_field* x, const ismg_field* b);
/* anchor_mean (coarse) — coarsening.hpp:592-595 */
int ismg_coarse_anchor_mean(ismg_solver* s, ismg_field* x);

/* PressureSolver::solve — cycles.hpp:310-321 (solve_two_level :101-165 for
 * ISMG/GMG). `current` (may be NULL) accumulates the RunMetrics counters of
 * metrics.hpp:46-58 exactly as record_* would; fine_cells is RunMetrics::fine_cells. */
int ismg_solve(ismg_solver* s, ismg_field* x, const ismg_field* b, ismg_report* rep,
               ismg_step_metrics* current, int64_t fine_cells);
/* Same, on host arrays (scalar layout): one upload of x and b, one download of x. */
int ismg_solve_host(ismg_solver* s, double* x_host, const double* b_host, size_t count,
                    ismg_report* rep, ismg_step_metrics* current, int64_t fine_cells);
/* stats of the last solve on this solver */
int ismg_solver_last_stats(const ismg_solver* s, ismg_solve_stats* out);
/* Coarse-visit log of the last solve: per outer iteration (restriction) the
 * number of coarse sweeps and of fine sweeps that followed, interleaved
 * (c0, f0, c1, f1, ...). *n receives the number of visits; at most cap visits
 * are written (out may be NULL to query). */
int ismg_solver_visit_log(const ismg_solver* s, int32_t* out, size_t cap, size_t* n);
/* Measurement hook: run `iters` fused fine passes (red + black half-sweeps,
 * residual, tile-sum restriction, anchor sum; 24 algorithmic bytes per cell)
 * back to back on (x, b) with CUDA events around each on the context stream;
 * *ms_per_pass = mean event time. Requires the fused path (ISMG/GMG,
 * non-periodic, power-of-two tile <= 64). x is relaxed in place. */
int ismg_bench_fine_pass(ismg_solver* s, ismg_field* x, const ismg_field* b, int iters,
                         double* ms_per_pass);
/* Measurement / parity hook (no reference counterpart): ONE coarse visit
 * (cycles.hpp:120-137: gs_sweep_lex + coarse_residual until tol_coarse, then
 * the coarse anchor when singular) of the fused path's coarse-visit kernel on
 * rhs cb (coarse extent ncx x ncy), from ce = 0, with at most `budget` sweeps;
 * the first sweep group holds `first_group` sweeps (the visit-length
 * prediction). ce receives the iterate, *sweeps the sweeps run, *rc the final
 * coarse residual max, *ms the kernel's CUDA-event time. Requires the fused
 * path. */
int ismg_bench_coarse_visit(ismg_solver* s, const ismg_field* cb, ismg_field* ce, int64_t budget, int first_group,
                            int64_t* sweeps, double* rc, double* ms);
/* kernels launched through this context so far (stream order) */
int ismg_ctx_launch_count(const ismg_ctx* ctx, int64_t* out);

/* ---- projection step ------------------------------------------------------ */
/* apply_scalar_bc — field.hpp:77-96 */
int ismg_apply_scalar_bc(ismg_ctx* ctx, const ismg_grid_spec* g, ismg_field* f);
/* apply_velocity_bc — field.hpp:143-228 */
int ismg_apply_velocity_bc(ismg_ctx* ctx, const ismg_grid_spec* g, ismg_velocity* vel);
/* divergence — projection.hpp:38-46; if scale != 1 the result is multiplied
 * by `scale` as a separate rounding (projection.hpp:174-178). */
int ismg_divergence(ismg_ctx* ctx, const ismg_grid_spec* g, const ismg_velocity* vel,
                    ismg_field* out, double scale);
/* correct — projection.hpp:121-133 (refreshes dp's ghost ring) */
int ismg_correct(ismg_ctx* ctx, const ismg_grid_spec* g, ismg_velocity* vel, ismg_field* dp,
                 double dt);
/* predictor — projection.hpp:75-119 (writes the owned faces of out) */
int ismg_predictor(ismg_ctx* ctx, const ismg_grid_spec* g, const ismg_velocity* vel,
                   const ismg_field* p, double dt, double nu, ismg_velocity* out);

/* FluidState — projection.hpp:26-36 */
int ismg_state_create(ismg_ctx* ctx, const ismg_grid_spec* g, ismg_state** out);
int ismg_state_destroy(ismg_state* st);
int ismg_state_set_scalars(ismg_state* st, double t, double dt, double nu, int64_t step_count);
int ismg_state_get_scalars(const ismg_state* st, double* t, double* dt, double* nu,
                           int64_t* step_count);
int ismg_state_upload(ismg_state* st, const double* u, size_t u_count, const double* v,
                      size_t v_count, const double* p, size_t p_count);
int ismg_state_download(const ismg_state* st, double* u, size_t u_count, double* v,
                        size_t v_count, double* p, size_t p_count);
/* step — projection.hpp:139-190. `current` accumulates this step's counters;
 * closing the row (RunMetrics::close_timestep) is left to the caller, who
 * receives the step number through ismg_state_get_scalars. */
int ismg_step(ismg_state* st, ismg_solver* s, ismg_report* rep, ismg_step_metrics* current,
              int64_t fine_cells);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* ISMG_B200_H */

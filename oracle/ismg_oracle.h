/*
 * ismg_oracle.h — CPU oracle for the ISM pressure path (TEST INFRASTRUCTURE).
 *
 * A plain-C restatement of the reference's algorithm (arXiv 1309.7128
 * reference, /root/reference/proj/include/ismg). Only tests/, the smoke()
 * check of __graft_entry__.py and bench.py's cpu_baseline / reference legs may
 * load it, and only as the checker — never as the product path.
 *
 * Pinned against (a) the reference itself, compiled from its headers into
 * oracle/_ref (oracle/ref_shim.cpp), bit-for-bit on random cases, and
 * (b) the reference's own known-answer tests, restated in
 * tests/test_oracle_golden.py, plus committed golden vectors in tests/golden/.
 *
 * Value types are shared with the product C-ABI (include/ismg_b200.h) so the
 * same ctypes structs drive both. Fields use the reference's ghosted layout.
 */
#ifndef ISMG_ORACLE_H
#define ISMG_ORACLE_H

#include "../include/ismg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* geometry */
int orc_pressure_bc(const ismg_grid_spec* g, int32_t out[4], int32_t* singular);
int orc_build_fine_diag(const ismg_grid_spec* g, double* diag);

/* fine-level smoother (scalar layout (nx+2)*(ny+2)) */
void orc_zero_ghosts(int nx, int ny, double* x);
int orc_rbgs_sweep(const ismg_grid_spec* g, double* x, const double* b);
double orc_fine_residual(const ismg_grid_spec* g, double* x, const double* b, double* out);
void orc_anchor_mean(const ismg_grid_spec* g, double* x);
double orc_interior_sum(int nx, int ny, const double* x);

/* tile axis (coarsening.hpp:42-105): per-cell locate tables */
int orc_tile_axis(int n, int tile, int periodic, int32_t* nc, int32_t* start, int32_t* width,
                  double* center, int32_t* k0, int32_t* k1, double* t, double* dk);

/* coarse operators: 9 planes of ncx*ncy, slot order C,E,W,N,S,NE,NW,SE,SW */
int orc_ismg_dims(const ismg_grid_spec* g, int32_t* ncx, int32_t* ncy);
int orc_build_ismg_operator(const ismg_grid_spec* g, double* w);
int orc_build_gmg_operator(const ismg_grid_spec* g, double* w);

/* transfers; fine (nx,ny) <-> coarse (ncx,ncy) with the grid's tile/periodicity */
void orc_restrict_sum(const ismg_grid_spec* g, const double* fine, double* coarse);
void orc_prolongate_bilinear(const ismg_grid_spec* g, const double* coarse, double* fine);

/* coarse relaxation on a 9-plane operator (five_point != 0 -> 5 slots) */
double orc_coarse_residual(int ncx, int ncy, int px, int py, int five_point, const double* w,
                           const double* x, const double* b, double* out);
int orc_gs_sweep_lex(int ncx, int ncy, int px, int py, int five_point, const double* w,
                     double* x, const double* b);
void orc_coarse_anchor(int ncx, int ncy, int singular, double* x);

/* PressureSolver::solve (all four schemes); returns status */
int orc_solve(const ismg_grid_spec* g, const ismg_cycle_config* c, double* x, const double* b,
              ismg_report* rep, ismg_step_metrics* current, int64_t fine_cells);

/* projection */
void orc_apply_scalar_bc(const ismg_grid_spec* g, double* f);
void orc_apply_velocity_bc(const ismg_grid_spec* g, double* u, double* v);
void orc_divergence(const ismg_grid_spec* g, const double* u, const double* v, double* out);
void orc_correct(const ismg_grid_spec* g, double* u, double* v, double* dp, double dt);
void orc_predictor(const ismg_grid_spec* g, const double* u, const double* v, const double* p,
                   double dt, double nu, double* out_u, double* out_v);
/* step(): state arrays updated in place; scal = {t, dt, nu, step_count} */
int orc_step(const ismg_grid_spec* g, const ismg_cycle_config* c, double* u, double* v,
             double* p, double* scal, ismg_report* rep, ismg_step_metrics* current,
             int64_t fine_cells);
/* run N steps of a case (bench.hpp:127-158 with seed = 0, steady_tol = 0);
 * rows receives N closed step rows. */
int orc_run_steps(const ismg_grid_spec* g, const ismg_cycle_config* c, double* u, double* v,
                  double* p, double* scal, long nsteps, ismg_step_metrics* rows);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif

/*
 * ismg_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see ismg_oracle.h).
 *
 * Plain-C restatement of the reference ISM pressure path. Each function cites
 * the reference function it restates (paths relative to
 * /root/reference/proj/include/ismg). Arithmetic is written to follow the
 * reference's expression order exactly, so that with FMA contraction off
 * (-ffp-contract=off, no -march, as proj/CMakeLists.txt:14 builds it) the
 * results are bit-identical to the reference (checked against oracle/_ref).
 */
#include "ismg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

#define SAT(f, nx, i, j) (f)[(size_t)((j) + 1) * (size_t)((nx) + 2) + (size_t)((i) + 1)]
#define UAT(f, nx, i, j) (f)[(size_t)((j) + 1) * (size_t)((nx) + 3) + (size_t)((i) + 1)]
#define VAT(f, nx, i, j) (f)[(size_t)((j) + 1) * (size_t)((nx) + 2) + (size_t)((i) + 1)]

/* std::max(a, b) semantics: returns a unless a < b (NaN b is dropped). */
static inline double stdmax(double a, double b) { return (a < b) ? b : a; }

/* ------------------------------------------------------------------------ */
/* grid.hpp:79-96 GridSpec::validate                                          */
static int grid_validate(const ismg_grid_spec* g) {
    if (g->nx < 1 || g->ny < 1) return fail(ISMG_ERR_INVALID_ARGUMENT, "grid: nx, ny must be >= 1");
    if (g->h <= 0.0) return fail(ISMG_ERR_INVALID_ARGUMENT, "grid: h must be positive");
    if (g->tile < 2) return fail(ISMG_ERR_INVALID_ARGUMENT, "grid: tile must be >= 2");
    int pw = g->bc[0].kind == ISMG_BC_PERIODIC, pe = g->bc[1].kind == ISMG_BC_PERIODIC;
    int ps = g->bc[2].kind == ISMG_BC_PERIODIC, pn = g->bc[3].kind == ISMG_BC_PERIODIC;
    if (pw != pe) return fail(ISMG_ERR_INVALID_ARGUMENT, "grid: periodic west/east must pair");
    if (ps != pn) return fail(ISMG_ERR_INVALID_ARGUMENT, "grid: periodic south/north must pair");
    for (int s = 0; s < 4; ++s) {
        const ismg_bc* b = &g->bc[s];
        if (b->kind != ISMG_BC_INLET) continue;
        int extent = (s == ISMG_SIDE_SOUTH || s == ISMG_SIDE_NORTH) ? g->nx : g->ny;
        if (b->inlet_width < 1 || b->inlet_start < 0 || b->inlet_start + b->inlet_width > extent)
            return fail(ISMG_ERR_INVALID_ARGUMENT, "grid: inlet span out of range");
    }
    return ISMG_OK;
}

/* grid.hpp:124-149 pressure_bc / pressure_singular */
int orc_pressure_bc(const ismg_grid_spec* g, int32_t out[4], int32_t* singular) {
    int sing = 1;
    for (int s = 0; s < 4; ++s) {
        switch (g->bc[s].kind) {
            case ISMG_BC_DIRICHLET_VELOCITY:
            case ISMG_BC_INLET: out[s] = ISMG_PBC_NEUMANN; break;
            case ISMG_BC_SYMMETRY_FIXED_PRESSURE: out[s] = ISMG_PBC_DIRICHLET_ZERO; break;
            default: out[s] = ISMG_PBC_PERIODIC; break;
        }
        if (out[s] == ISMG_PBC_DIRICHLET_ZERO) sing = 0;
    }
    if (singular) *singular = sing;
    return ISMG_OK;
}

/* smoother.hpp:47-54 face_weight */
static double face_weight(int32_t pbc) {
    switch (pbc) {
        case ISMG_PBC_NEUMANN: return 0.0;
        case ISMG_PBC_DIRICHLET_ZERO: return 2.0;
        case ISMG_PBC_PERIODIC: return 1.0;
    }
    return 0.0;
}

/* smoother.hpp:55-61: d = open faces + 2 * fixed-pressure faces (+ wraps) */
static double fine_diag(const int32_t pbc[4], int nx, int ny, int i, int j) {
    double d = 0;
    d += (i > 0) ? 1.0 : face_weight(pbc[ISMG_SIDE_WEST]);
    d += (i < nx - 1) ? 1.0 : face_weight(pbc[ISMG_SIDE_EAST]);
    d += (j > 0) ? 1.0 : face_weight(pbc[ISMG_SIDE_SOUTH]);
    d += (j < ny - 1) ? 1.0 : face_weight(pbc[ISMG_SIDE_NORTH]);
    return d;
}

/* smoother.hpp:36-67 build_fine_stage (diag plane, scalar layout) */
int orc_build_fine_diag(const ismg_grid_spec* g, double* diag) {
    int32_t pbc[4];
    orc_pressure_bc(g, pbc, NULL);
    for (int j = 0; j < g->ny; ++j)
        for (int i = 0; i < g->nx; ++i) {
            double d = fine_diag(pbc, g->nx, g->ny, i, j);
            if (d <= 0.0) return fail(ISMG_ERR_DOMAIN, "smoother: fine row has empty stencil");
            if (diag) SAT(diag, g->nx, i, j) = d;
        }
    return ISMG_OK;
}

/* smoother.hpp:71-81 zero_ghosts */
void orc_zero_ghosts(int nx, int ny, double* x) {
    for (int j = -1; j <= ny; ++j) {
        SAT(x, nx, -1, j) = 0.0;
        SAT(x, nx, nx, j) = 0.0;
    }
    for (int i = -1; i <= nx; ++i) {
        SAT(x, nx, i, -1) = 0.0;
        SAT(x, nx, i, ny) = 0.0;
    }
}

/* smoother.hpp:83-96 refresh_periodic_ghosts */
static void refresh_periodic(int nx, int ny, double* x, int px, int py) {
    if (px)
        for (int j = 0; j < ny; ++j) {
            SAT(x, nx, -1, j) = SAT(x, nx, nx - 1, j);
            SAT(x, nx, nx, j) = SAT(x, nx, 0, j);
        }
    if (py)
        for (int i = 0; i < nx; ++i) {
            SAT(x, nx, i, -1) = SAT(x, nx, i, ny - 1);
            SAT(x, nx, i, ny) = SAT(x, nx, i, 0);
        }
}

/* smoother.hpp:101-117 rbgs_sweep: x = (((W + E) + S) + N - b) / d per colour */
int orc_rbgs_sweep(const ismg_grid_spec* g, double* x, const double* b) {
    int32_t pbc[4];
    orc_pressure_bc(g, pbc, NULL);
    const int nx = g->nx, ny = g->ny;
    const int px = pbc[ISMG_SIDE_WEST] == ISMG_PBC_PERIODIC;
    const int py = pbc[ISMG_SIDE_SOUTH] == ISMG_PBC_PERIODIC;
    for (int color = 0; color < 2; ++color) {
        refresh_periodic(nx, ny, x, px, py);
        for (int j = 0; j < ny; ++j)
            for (int i = (color + j) & 1; i < nx; i += 2) {
                double s = SAT(x, nx, i - 1, j) + SAT(x, nx, i + 1, j) + SAT(x, nx, i, j - 1) +
                           SAT(x, nx, i, j + 1);
                SAT(x, nx, i, j) = (s - SAT(b, nx, i, j)) / fine_diag(pbc, nx, ny, i, j);
            }
    }
    return ISMG_OK;
}

/* smoother.hpp:121-141 fine_residual: r = b - ((((W+E)+S)+N) - d*x) */
double orc_fine_residual(const ismg_grid_spec* g, double* x, const double* b, double* out) {
    int32_t pbc[4];
    orc_pressure_bc(g, pbc, NULL);
    const int nx = g->nx, ny = g->ny;
    refresh_periodic(nx, ny, x, pbc[0] == ISMG_PBC_PERIODIC, pbc[2] == ISMG_PBC_PERIODIC);
    double rmax = 0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            double ax = SAT(x, nx, i - 1, j) + SAT(x, nx, i + 1, j) + SAT(x, nx, i, j - 1) +
                        SAT(x, nx, i, j + 1) - fine_diag(pbc, nx, ny, i, j) * SAT(x, nx, i, j);
            double r = SAT(b, nx, i, j) - ax;
            if (out) SAT(out, nx, i, j) = r;
            rmax = stdmax(rmax, fabs(r));
        }
    return rmax;
}

/* field.hpp:41-48 interior_sum (serial, row-major) */
double orc_interior_sum(int nx, int ny, const double* x) {
    double s = 0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) s += SAT(x, nx, i, j);
    return s;
}

/* field.hpp:49 interior_mean + :53-59 shift_interior */
static void shift_by_mean(int nx, int ny, double* x) {
    double mean = orc_interior_sum(nx, ny, x) / (double)((size_t)nx * (size_t)ny);
    double c = -mean;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) SAT(x, nx, i, j) += c;
}

/* smoother.hpp:145-148 anchor_mean */
void orc_anchor_mean(const ismg_grid_spec* g, double* x) {
    int32_t pbc[4], sing;
    orc_pressure_bc(g, pbc, &sing);
    if (sing) shift_by_mean(g->nx, g->ny, x);
}

/* ------------------------------------------------------------------------ */
/* coarsening.hpp:42-105 TileAxis                                            */
typedef struct {
    int n, tile, periodic, nc;
    int *start, *width;
    double *center, *rect, rect_wrap;
    int *k0, *k1; /* cached locate(i + 0.5) */
    double *t, *dk;
} axis_t;

typedef struct {
    int k0, k1;
    double t, dk;
} locate_t;

/* coarsening.hpp:85-97 locate */
static locate_t axis_locate(const axis_t* a, double c) {
    locate_t L;
    if (a->nc == 1) {
        L.k0 = 0, L.k1 = 0, L.t = 0.0, L.dk = 1.0;
        return L;
    }
    if (a->periodic && (c < a->center[0] || c >= a->center[a->nc - 1])) {
        double t = c - a->center[a->nc - 1];
        if (t < 0) t += a->n;
        L.k0 = a->nc - 1, L.k1 = 0, L.t = t, L.dk = a->rect_wrap;
        return L;
    }
    if (c <= a->center[0]) {
        L.k0 = 0, L.k1 = 1, L.t = 0.0, L.dk = a->rect[0];
        return L;
    }
    if (c >= a->center[a->nc - 1]) {
        L.k0 = a->nc - 2, L.k1 = a->nc - 1, L.t = a->rect[a->nc - 2], L.dk = a->rect[a->nc - 2];
        return L;
    }
    int k = 0;
    while (a->center[k + 1] <= c) ++k;
    L.k0 = k, L.k1 = k + 1, L.t = c - a->center[k], L.dk = a->rect[k];
    return L;
}

static void axis_free(axis_t* a) {
    free(a->start), free(a->width), free(a->center), free(a->rect);
    free(a->k0), free(a->k1), free(a->t), free(a->dk);
    memset(a, 0, sizeof *a);
}

/* coarsening.hpp:60-76 constructor */
static int axis_init(axis_t* a, int n, int tile, int periodic) {
    memset(a, 0, sizeof *a);
    if (n < 1 || tile < 1) return fail(ISMG_ERR_INVALID_ARGUMENT, "tile axis: need n >= 1, tile >= 1");
    a->n = n, a->tile = tile, a->periodic = periodic;
    a->nc = (n + tile - 1) / tile;
    int nc = a->nc;
    a->start = malloc(sizeof(int) * nc);
    a->width = malloc(sizeof(int) * nc);
    a->center = malloc(sizeof(double) * nc);
    a->rect = malloc(sizeof(double) * (nc > 1 ? nc - 1 : 1));
    a->k0 = malloc(sizeof(int) * n);
    a->k1 = malloc(sizeof(int) * n);
    a->t = malloc(sizeof(double) * n);
    a->dk = malloc(sizeof(double) * n);
    for (int k = 0; k < nc; ++k) {
        a->start[k] = k * tile;
        a->width[k] = (k == nc - 1) ? n - (nc - 1) * tile : tile;
        a->center[k] = a->start[k] + a->width[k] / 2.0;
    }
    for (int k = 0; k + 1 < nc; ++k) a->rect[k] = a->center[k + 1] - a->center[k];
    if (periodic) a->rect_wrap = (a->width[nc - 1] + a->width[0]) / 2.0;
    for (int i = 0; i < n; ++i) {
        locate_t L = axis_locate(a, i + 0.5);
        a->k0[i] = L.k0, a->k1[i] = L.k1, a->t[i] = L.t, a->dk[i] = L.dk;
    }
    return ISMG_OK;
}

int orc_tile_axis(int n, int tile, int periodic, int32_t* nc, int32_t* start, int32_t* width,
                  double* center, int32_t* k0, int32_t* k1, double* t, double* dk) {
    axis_t a;
    int rc = axis_init(&a, n, tile, periodic);
    if (rc) return rc;
    if (nc) *nc = a.nc;
    for (int k = 0; k < a.nc; ++k) {
        if (start) start[k] = a.start[k];
        if (width) width[k] = a.width[k];
        if (center) center[k] = a.center[k];
    }
    for (int i = 0; i < n; ++i) {
        if (k0) k0[i] = a.k0[i];
        if (k1) k1[i] = a.k1[i];
        if (t) t[i] = a.t[i];
        if (dk) dk[i] = a.dk[i];
    }
    axis_free(&a);
    return ISMG_OK;
}

/* coarsening.hpp:110-119 wrap_delta */
static int wrap_delta(int k_to, int k_from, int nc, int periodic) {
    int d = k_to - k_from;
    if (periodic) {
        if (d > nc / 2) d -= nc;
        if (d < -nc / 2) d += nc;
        if (d == nc - 1) d = -1;
        if (d == -(nc - 1)) d = 1;
    }
    return d;
}

/* coarsening.hpp:122-132 slot tables: C,E,W,N,S,NE,NW,SE,SW */
static const int slot_di[9] = {0, 1, -1, 0, 0, 1, -1, 1, -1};
static const int slot_dj[9] = {0, 0, 0, 1, -1, 1, 1, -1, -1};
static int slot_index(int di, int dj) {
    static const int lut[9] = {8, 4, 7, 2, 0, 1, 6, 3, 5};
    if (di < -1 || di > 1 || dj < -1 || dj > 1) return -1;
    return lut[(dj + 1) * 3 + (di + 1)];
}

/* coarsening.hpp:137-159 CoarseOperator */
typedef struct {
    int ncx, ncy;
    axis_t ax, ay;
    int px, py, five_point, singular;
    double* w[9];
} cop_t;

static void cop_free(cop_t* op) {
    axis_free(&op->ax), axis_free(&op->ay);
    for (int s = 0; s < 9; ++s) free(op->w[s]);
    memset(op, 0, sizeof *op);
}

static void cop_init(cop_t* op) {
    op->ncx = op->ax.nc, op->ncy = op->ay.nc;
    op->px = op->ax.periodic, op->py = op->ay.periodic;
    for (int s = 0; s < 9; ++s) op->w[s] = calloc((size_t)op->ncx * op->ncy, sizeof(double));
}

typedef struct {
    cop_t* op;
    int err;
} adder_t;

/* coarsening.hpp:212-216 add() */
static void op_add(adder_t* A, int I, int J, int Ic, int Jc, double wgt) {
    cop_t* op = A->op;
    int di = wrap_delta(Ic, I, op->ncx, op->px);
    int dj = wrap_delta(Jc, J, op->ncy, op->py);
    int sl = slot_index(di, dj);
    if (sl < 0) {
        A->err = fail(ISMG_ERR_LOGIC, "coarsening: coupling beyond the 9-point neighborhood");
        return;
    }
    op->w[sl][(size_t)J * op->ncx + I] += wgt;
}

/* coarsening.hpp:221-237 vface */
static void vface(adder_t* A, int I, int Inb, int J) {
    cop_t* op = A->op;
    double dx = (Inb == I + 1) ? op->ax.rect[I] : op->ax.rect_wrap;
    int j0 = op->ay.start[J], hJ = op->ay.width[J];
    for (int j = j0; j < j0 + hJ; ++j) {
        double gw = 1.0 / (dx * op->ay.dk[j]);
        const double t = op->ay.t[j], dy = op->ay.dk[j];
        const double ws[4] = {-gw * (dy - t), gw * (dy - t), -gw * t, gw * t};
        const int ic[4] = {I, Inb, I, Inb};
        const int jc[4] = {op->ay.k0[j], op->ay.k0[j], op->ay.k1[j], op->ay.k1[j]};
        for (int q = 0; q < 4; ++q) {
            op_add(A, I, J, ic[q], jc[q], ws[q]);
            op_add(A, Inb, J, ic[q], jc[q], -ws[q]);
        }
    }
}

/* coarsening.hpp:239-254 hface */
static void hface(adder_t* A, int I, int J, int Jnb) {
    cop_t* op = A->op;
    double dy = (Jnb == J + 1) ? op->ay.rect[J] : op->ay.rect_wrap;
    int i0 = op->ax.start[I], wI = op->ax.width[I];
    for (int i = i0; i < i0 + wI; ++i) {
        double gw = 1.0 / (op->ax.dk[i] * dy);
        const double s = op->ax.t[i], dx = op->ax.dk[i];
        const double ws[4] = {-gw * (dx - s), -gw * s, gw * (dx - s), gw * s};
        const int ic[4] = {op->ax.k0[i], op->ax.k1[i], op->ax.k0[i], op->ax.k1[i]};
        const int jc[4] = {J, J, Jnb, Jnb};
        for (int q = 0; q < 4; ++q) {
            op_add(A, I, J, ic[q], jc[q], ws[q]);
            op_add(A, I, Jnb, ic[q], jc[q], -ws[q]);
        }
    }
}

/* coarsening.hpp:268-303 fixed-pressure closures (one fine boundary cell) */
static void dclose_cell(adder_t* A, int I, int J, int i, int j) {
    cop_t* op = A->op;
    double gw = 1.0 / (op->ax.dk[i] * op->ay.dk[j]);
    const double s = op->ax.t[i], dx = op->ax.dk[i], t = op->ay.t[j], dy = op->ay.dk[j];
    int kx0 = op->ax.k0[i], kx1 = op->ax.k1[i], ky0 = op->ay.k0[j], ky1 = op->ay.k1[j];
    op_add(A, I, J, kx0, ky0, -2.0 * gw * (dx - s) * (dy - t));
    op_add(A, I, J, kx1, ky0, -2.0 * gw * s * (dy - t));
    op_add(A, I, J, kx0, ky1, -2.0 * gw * (dx - s) * t);
    op_add(A, I, J, kx1, ky1, -2.0 * gw * s * t);
}

static int build_ismg(const ismg_grid_spec* g, cop_t* op) {
    memset(op, 0, sizeof *op);
    if (g->tile < 2) return fail(ISMG_ERR_INVALID_ARGUMENT, "ismg operator: tile must be >= 2");
    int32_t bc[4], sing;
    orc_pressure_bc(g, bc, &sing);
    int rc = axis_init(&op->ax, g->nx, g->tile, bc[ISMG_SIDE_WEST] == ISMG_PBC_PERIODIC);
    if (!rc) rc = axis_init(&op->ay, g->ny, g->tile, bc[ISMG_SIDE_SOUTH] == ISMG_PBC_PERIODIC);
    if (rc) {
        cop_free(op);
        return rc;
    }
    if (op->ax.nc < 2 || op->ay.nc < 2) {
        cop_free(op);
        return fail(ISMG_ERR_INVALID_ARGUMENT, "ismg operator: need at least 2 coarse cells per axis");
    }
    cop_init(op);
    op->five_point = 0;
    op->singular = sing;
    adder_t A = {op, 0};
    const int ncx = op->ncx, ncy = op->ncy;
    for (int J = 0; J < ncy; ++J) { /* coarsening.hpp:256-259 */
        for (int I = 0; I < ncx - 1; ++I) vface(&A, I, I + 1, J);
        if (op->px) vface(&A, ncx - 1, 0, J);
    }
    for (int I = 0; I < ncx; ++I) { /* :260-263 */
        for (int J = 0; J < ncy - 1; ++J) hface(&A, I, J, J + 1);
        if (op->py) hface(&A, I, ncy - 1, 0);
    }
    /* :300-303 closures in W, E, S, N order */
    for (int side = 0; side < 2; ++side) {
        if (bc[side] != ISMG_PBC_DIRICHLET_ZERO) continue;
        int I = side == ISMG_SIDE_WEST ? 0 : ncx - 1;
        int i = side == ISMG_SIDE_WEST ? 0 : g->nx - 1;
        for (int J = 0; J < ncy; ++J)
            for (int j = op->ay.start[J]; j < op->ay.start[J] + op->ay.width[J]; ++j)
                dclose_cell(&A, I, J, i, j);
    }
    for (int side = 2; side < 4; ++side) {
        if (bc[side] != ISMG_PBC_DIRICHLET_ZERO) continue;
        int J = side == ISMG_SIDE_SOUTH ? 0 : ncy - 1;
        int j = side == ISMG_SIDE_SOUTH ? 0 : g->ny - 1;
        for (int I = 0; I < ncx; ++I)
            for (int i = op->ax.start[I]; i < op->ax.start[I] + op->ax.width[I]; ++i)
                dclose_cell(&A, I, J, i, j);
    }
    if (A.err) {
        cop_free(op);
        return A.err;
    }
    return ISMG_OK;
}

/* coarsening.hpp:311-360 build_gmg_operator */
static int build_gmg(const ismg_grid_spec* g, cop_t* op) {
    memset(op, 0, sizeof *op);
    if (g->tile < 2) return fail(ISMG_ERR_INVALID_ARGUMENT, "gmg operator: tile must be >= 2");
    int32_t bc[4], sing;
    orc_pressure_bc(g, bc, &sing);
    int rc = axis_init(&op->ax, g->nx, g->tile, bc[ISMG_SIDE_WEST] == ISMG_PBC_PERIODIC);
    if (!rc) rc = axis_init(&op->ay, g->ny, g->tile, bc[ISMG_SIDE_SOUTH] == ISMG_PBC_PERIODIC);
    if (rc) {
        cop_free(op);
        return rc;
    }
    if (op->ax.nc < 2 || op->ay.nc < 2) {
        cop_free(op);
        return fail(ISMG_ERR_INVALID_ARGUMENT, "gmg operator: need at least 2 coarse cells per axis");
    }
    cop_init(op);
    op->five_point = 1;
    op->singular = sing;
    const axis_t *ax = &op->ax, *ay = &op->ay;
    for (int J = 0; J < op->ncy; ++J)
        for (int I = 0; I < op->ncx; ++I) {
            size_t k = (size_t)J * op->ncx + I;
            double face_x = ay->width[J], face_y = ax->width[I], diag = 0.0, c;
#define COUPLE(slot, face, dist) (c = (face) / (dist), op->w[slot][k] += c, diag += c)
#define CLOSE(side, face, half_w) \
    if (bc[side] == ISMG_PBC_DIRICHLET_ZERO) diag += (face) / (half_w)
            if (I < op->ncx - 1) COUPLE(1, face_x, ax->rect[I]);
            else if (ax->periodic) COUPLE(1, face_x, ax->rect_wrap);
            else { CLOSE(ISMG_SIDE_EAST, face_x, ax->width[I] / 2.0); }
            if (I > 0) COUPLE(2, face_x, ax->rect[I - 1]);
            else if (ax->periodic) COUPLE(2, face_x, ax->rect_wrap);
            else { CLOSE(ISMG_SIDE_WEST, face_x, ax->width[I] / 2.0); }
            if (J < op->ncy - 1) COUPLE(3, face_y, ay->rect[J]);
            else if (ay->periodic) COUPLE(3, face_y, ay->rect_wrap);
            else { CLOSE(ISMG_SIDE_NORTH, face_y, ay->width[J] / 2.0); }
            if (J > 0) COUPLE(4, face_y, ay->rect[J - 1]);
            else if (ay->periodic) COUPLE(4, face_y, ay->rect_wrap);
            else { CLOSE(ISMG_SIDE_SOUTH, face_y, ay->width[J] / 2.0); }
#undef COUPLE
#undef CLOSE
            op->w[0][k] = -diag;
        }
    return ISMG_OK;
}

/* coarsening.hpp:367-406 fine_as_operator */
static int fine_as_operator(const ismg_grid_spec* g, cop_t* op) {
    memset(op, 0, sizeof *op);
    int32_t bc[4], sing;
    orc_pressure_bc(g, bc, &sing);
    int rc = axis_init(&op->ax, g->nx, 1, bc[ISMG_SIDE_WEST] == ISMG_PBC_PERIODIC);
    if (!rc) rc = axis_init(&op->ay, g->ny, 1, bc[ISMG_SIDE_SOUTH] == ISMG_PBC_PERIODIC);
    if (rc) return rc;
    cop_init(op);
    op->five_point = 1;
    op->singular = sing;
    for (int j = 0; j < g->ny; ++j)
        for (int i = 0; i < g->nx; ++i) {
            size_t k = (size_t)j * op->ncx + i;
            double diag = 0.0;
            const int open[4] = {i < g->nx - 1, i > 0, j < g->ny - 1, j > 0};
            const int side[4] = {ISMG_SIDE_EAST, ISMG_SIDE_WEST, ISMG_SIDE_NORTH, ISMG_SIDE_SOUTH};
            for (int f = 0; f < 4; ++f) {
                if (open[f] || bc[side[f]] == ISMG_PBC_PERIODIC) {
                    op->w[1 + f][k] = 1.0;
                    diag += 1.0;
                } else {
                    diag += face_weight(bc[side[f]]);
                }
            }
            op->w[0][k] = -diag;
        }
    return ISMG_OK;
}

/* coarsening.hpp:411-441 agglomerate2 */
static int agglomerate2(const cop_t* f, cop_t* c) {
    memset(c, 0, sizeof *c);
    if (!f->five_point) return fail(ISMG_ERR_INVALID_ARGUMENT, "agglomerate2: expected a 5-point level");
    int rc = axis_init(&c->ax, f->ncx, 2, f->px);
    if (!rc) rc = axis_init(&c->ay, f->ncy, 2, f->py);
    if (rc) return rc;
    cop_init(c);
    c->five_point = 1;
    c->singular = f->singular;
    for (int j = 0; j < f->ncy; ++j) {
        int BJ = j / 2;
        for (int i = 0; i < f->ncx; ++i) {
            int BI = i / 2;
            size_t kf = (size_t)j * f->ncx + i, kc = (size_t)BJ * c->ncx + BI;
            for (int sl = 0; sl < 5; ++sl) {
                double wgt = f->w[sl][kf];
                if (wgt == 0.0) continue;
                int ii = i + slot_di[sl], jj = j + slot_dj[sl];
                if (f->px) ii = (ii + f->ncx) % f->ncx;
                if (f->py) jj = (jj + f->ncy) % f->ncy;
                if (ii < 0 || ii >= f->ncx || jj < 0 || jj >= f->ncy) continue;
                int di = wrap_delta(ii / 2, BI, c->ncx, c->px);
                int dj = wrap_delta(jj / 2, BJ, c->ncy, c->py);
                int s = slot_index(di, dj);
                if (s < 0) return fail(ISMG_ERR_LOGIC, "coarsening: coupling beyond the 9-point neighborhood");
                c->w[s][kc] += wgt;
            }
        }
    }
    return ISMG_OK;
}

int orc_ismg_dims(const ismg_grid_spec* g, int32_t* ncx, int32_t* ncy) {
    if (g->tile < 1) return fail(ISMG_ERR_INVALID_ARGUMENT, "tile must be >= 1");
    *ncx = (g->nx + g->tile - 1) / g->tile;
    *ncy = (g->ny + g->tile - 1) / g->tile;
    return ISMG_OK;
}

static void copy_planes(const cop_t* op, double* w) {
    size_t n = (size_t)op->ncx * op->ncy;
    for (int s = 0; s < 9; ++s) memcpy(w + s * n, op->w[s], n * sizeof(double));
}

int orc_build_ismg_operator(const ismg_grid_spec* g, double* w) {
    cop_t op;
    int rc = build_ismg(g, &op);
    if (rc) return rc;
    if (w) copy_planes(&op, w);
    cop_free(&op);
    return ISMG_OK;
}

int orc_build_gmg_operator(const ismg_grid_spec* g, double* w) {
    cop_t op;
    int rc = build_gmg(g, &op);
    if (rc) return rc;
    if (w) copy_planes(&op, w);
    cop_free(&op);
    return ISMG_OK;
}

/* ------------------------------------------------------------------------ */
/* coarsening.hpp:471-480 restrict_sum (serial row-major accumulation)        */
static void restrict_axes(const axis_t* ax, const axis_t* ay, const double* fine, double* coarse) {
    const int nx = ax->n, ncx = ax->nc;
    for (int J = 0; J < ay->nc; ++J)
        for (int I = 0; I < ncx; ++I) SAT(coarse, ncx, I, J) = 0.0;
    for (int j = 0; j < ay->n; ++j) {
        int J = j / ay->tile;
        for (int i = 0; i < nx; ++i) SAT(coarse, ncx, i / ax->tile, J) += SAT(fine, nx, i, j);
    }
}

/* coarsening.hpp:485-503 prolongate_bilinear (adds into fine) */
static void prolong_axes(const axis_t* ax, const axis_t* ay, const double* coarse, double* fine) {
    const int nx = ax->n, ncx = ax->nc;
    for (int j = 0; j < ay->n; ++j) {
        const double t = ay->t[j], dy = ay->dk[j];
        const int J0 = ay->k0[j], J1 = ay->k1[j];
        for (int i = 0; i < nx; ++i) {
            const double s = ax->t[i], dx = ax->dk[i];
            const int I0 = ax->k0[i], I1 = ax->k1[i];
            double val = ((dx - s) * ((dy - t) * SAT(coarse, ncx, I0, J0) + t * SAT(coarse, ncx, I0, J1)) +
                          s * ((dy - t) * SAT(coarse, ncx, I1, J0) + t * SAT(coarse, ncx, I1, J1))) /
                         (dx * dy);
            SAT(fine, nx, i, j) += val;
        }
    }
}

/* coarsening.hpp:506-514 prolongate_constant */
static void prolong_const_axes(const axis_t* ax, const axis_t* ay, const double* coarse, double* fine) {
    const int nx = ax->n, ncx = ax->nc;
    for (int j = 0; j < ay->n; ++j)
        for (int i = 0; i < nx; ++i)
            SAT(fine, nx, i, j) += SAT(coarse, ncx, i / ax->tile, j / ay->tile);
}

static int grid_axes(const ismg_grid_spec* g, axis_t* ax, axis_t* ay) {
    int32_t bc[4];
    orc_pressure_bc(g, bc, NULL);
    int rc = axis_init(ax, g->nx, g->tile, bc[0] == ISMG_PBC_PERIODIC);
    if (!rc) rc = axis_init(ay, g->ny, g->tile, bc[2] == ISMG_PBC_PERIODIC);
    return rc;
}

void orc_restrict_sum(const ismg_grid_spec* g, const double* fine, double* coarse) {
    axis_t ax, ay;
    if (grid_axes(g, &ax, &ay)) return;
    restrict_axes(&ax, &ay, fine, coarse);
    axis_free(&ax), axis_free(&ay);
}

void orc_prolongate_bilinear(const ismg_grid_spec* g, const double* coarse, double* fine) {
    axis_t ax, ay;
    if (grid_axes(g, &ax, &ay)) return;
    prolong_axes(&ax, &ay, coarse, fine);
    axis_free(&ax), axis_free(&ay);
}

/* ------------------------------------------------------------------------ */
/* coarsening.hpp:520-528 coarse_neighbor                                     */
static inline double coarse_nb(int ncx, int ncy, int px, int py, const double* x, int I, int J,
                               int sl) {
    int II = I + slot_di[sl], JJ = J + slot_dj[sl];
    if (px) II = (II + ncx) % ncx;
    if (py) JJ = (JJ + ncy) % ncy;
    if (II < 0 || II >= ncx || JJ < 0 || JJ >= ncy) return 0.0;
    return SAT(x, ncx, II, JJ);
}

/* coarsening.hpp:531-549 coarse_residual */
double orc_coarse_residual(int ncx, int ncy, int px, int py, int five_point, const double* w,
                           const double* x, const double* b, double* out) {
    const int ns = five_point ? 5 : 9;
    const size_t n = (size_t)ncx * ncy;
    double rmax = 0;
    for (int J = 0; J < ncy; ++J)
        for (int I = 0; I < ncx; ++I) {
            size_t k = (size_t)J * ncx + I;
            double ax = w[k] * SAT(x, ncx, I, J);
            for (int sl = 1; sl < ns; ++sl) {
                double wgt = w[sl * n + k];
                if (wgt != 0.0) ax += wgt * coarse_nb(ncx, ncy, px, py, x, I, J, sl);
            }
            double r = SAT(b, ncx, I, J) - ax;
            if (out) SAT(out, ncx, I, J) = r;
            rmax = stdmax(rmax, fabs(r));
        }
    return rmax;
}

/* coarsening.hpp:552-567 gs_sweep_lex */
int orc_gs_sweep_lex(int ncx, int ncy, int px, int py, int five_point, const double* w, double* x,
                     const double* b) {
    const int ns = five_point ? 5 : 9;
    const size_t n = (size_t)ncx * ncy;
    for (int J = 0; J < ncy; ++J)
        for (int I = 0; I < ncx; ++I) {
            size_t k = (size_t)J * ncx + I;
            double s = 0;
            for (int sl = 1; sl < ns; ++sl) {
                double wgt = w[sl * n + k];
                if (wgt != 0.0) s += wgt * coarse_nb(ncx, ncy, px, py, x, I, J, sl);
            }
            if (w[k] == 0.0) return fail(ISMG_ERR_DOMAIN, "coarsening: singular stencil row");
            SAT(x, ncx, I, J) = (SAT(b, ncx, I, J) - s) / w[k];
        }
    return ISMG_OK;
}

/* coarsening.hpp:571-588 rbgs_sweep on a stored 5-point level */
static int rbgs_op(const cop_t* op, double* x, const double* b) {
    if (!op->five_point)
        return fail(ISMG_ERR_INVALID_ARGUMENT, "rbgs_sweep: red-black relaxation expects a 5-point level");
    const int ncx = op->ncx, ncy = op->ncy;
    for (int color = 0; color < 2; ++color)
        for (int J = 0; J < ncy; ++J)
            for (int I = (color + J) & 1; I < ncx; I += 2) {
                size_t k = (size_t)J * ncx + I;
                double s = 0;
                for (int sl = 1; sl < 5; ++sl) {
                    double wgt = op->w[sl][k];
                    if (wgt != 0.0) s += wgt * coarse_nb(ncx, ncy, op->px, op->py, x, I, J, sl);
                }
                if (op->w[0][k] == 0.0) return fail(ISMG_ERR_DOMAIN, "coarsening: singular stencil row");
                SAT(x, ncx, I, J) = (SAT(b, ncx, I, J) - s) / op->w[0][k];
            }
    return ISMG_OK;
}

/* coarsening.hpp:592-595 anchor_mean(op) */
void orc_coarse_anchor(int ncx, int ncy, int singular, double* x) {
    if (singular) shift_by_mean(ncx, ncy, x);
}

/* planes of a cop_t as one contiguous buffer view */
static double* cop_flat(const cop_t* op) {
    size_t n = (size_t)op->ncx * op->ncy;
    double* w = malloc(9 * n * sizeof(double));
    copy_planes(op, w);
    return w;
}

static double cres(const cop_t* op, const double* wf, const double* x, const double* b, double* out) {
    return orc_coarse_residual(op->ncx, op->ncy, op->px, op->py, op->five_point, wf, x, b, out);
}

/* ------------------------------------------------------------------------ */
/* metrics.hpp:46-58 record_sweep / record_restriction / record_prolongation  */
static void record_sweep(ismg_step_metrics* m, int fine, int stencil, int64_t cells, int64_t fine_cells) {
    if (!m) return;
    if (fine) {
        m->fine_sweeps += 1;
        m->sync_fine += 2;
    } else {
        m->coarse_sweeps += 1;
        m->sync_coarse += 1;
    }
    m->lap_equiv += ((double)cells / (double)fine_cells) * ((double)stencil / 5.0);
}

/* cycles.hpp:31-44 CycleConfig::validate */
static int cycle_validate(const ismg_cycle_config* c) {
    if (!(c->tol_fine > 0) || !(c->tol_coarse > 0))
        return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: tolerances must be positive");
    if (c->tol_coarse < c->tol_fine)
        return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: tol_coarse must be >= tol_fine");
    if (c->max_total_sweeps < 1)
        return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: max_total_sweeps must be positive");
    if (!(c->stall_factor > 0.0 && c->stall_factor < 1.0))
        return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: stall_factor must lie in (0,1)");
    if (c->acm_pre_smooth < 0 || c->acm_post_smooth < 0)
        return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: smoothing counts must be non-negative");
    if (c->depth < 2) return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: depth must be >= 2");
    if (c->tile < 2) return fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: tile must be >= 2");
    return ISMG_OK;
}

/* cycles.hpp:71-94 solve_plain_gs */
static void solve_plain(const ismg_grid_spec* g, const ismg_cycle_config* c, double* x,
                        const double* b, ismg_report* rep, ismg_step_metrics* m, int64_t fc) {
    const int nx = g->nx, ny = g->ny;
    const int64_t cells = (int64_t)nx * ny;
    orc_zero_ghosts(nx, ny, x);
    double r = orc_fine_residual(g, x, b, NULL);
    orc_anchor_mean(g, x);
    long total = 0;
    while (r > c->tol_fine) {
        if (total >= c->max_total_sweeps) {
            rep->converged = 0;
            break;
        }
        orc_rbgs_sweep(g, x, b);
        record_sweep(m, 1, 5, cells, fc);
        ++rep->fine_sweeps;
        ++total;
        r = orc_fine_residual(g, x, b, NULL);
        orc_anchor_mean(g, x);
    }
    rep->residual = r;
}

/* cycles.hpp:101-165 solve_two_level */
static int solve_two_level(const ismg_grid_spec* g, const ismg_cycle_config* c, const cop_t* op,
                           double* x, const double* b, ismg_report* rep, ismg_step_metrics* m,
                           int64_t fc) {
    const int nx = g->nx, ny = g->ny, ncx = op->ncx, ncy = op->ncy;
    const int64_t cells = (int64_t)nx * ny, ccells = (int64_t)ncx * ncy;
    const int stencil = op->five_point ? 5 : 9;
    double* wf = cop_flat(op);
    orc_zero_ghosts(nx, ny, x);
    double* res = calloc((size_t)(nx + 2) * (ny + 2), sizeof(double));
    double* cb = calloc((size_t)(ncx + 2) * (ncy + 2), sizeof(double));
    double* ce = calloc((size_t)(ncx + 2) * (ncy + 2), sizeof(double));
    long total = 0;
    int rc = ISMG_OK;
    double r = orc_fine_residual(g, x, b, res);
    orc_anchor_mean(g, x);

    while (r > c->tol_fine) {
        if (total >= c->max_total_sweeps) {
            rep->converged = 0;
            break;
        }
        restrict_axes(&op->ax, &op->ay, res, cb);
        if (m) m->restrictions += 1;
        memset(ce, 0, (size_t)(ncx + 2) * (ncy + 2) * sizeof(double));
        double rc_ = cres(op, wf, ce, cb, NULL);
        long coarse_visit = 0;
        while (rc_ > c->tol_coarse && total < c->max_total_sweeps) {
            rc = orc_gs_sweep_lex(ncx, ncy, op->px, op->py, op->five_point, wf, ce, cb);
            if (rc) goto out;
            record_sweep(m, 0, stencil, ccells, fc);
            ++rep->coarse_sweeps;
            ++total;
            ++coarse_visit;
            rc_ = cres(op, wf, ce, cb, NULL);
            orc_coarse_anchor(ncx, ncy, op->singular, ce);
        }
        if (rc_ > c->tol_coarse) {
            rep->converged = 0;
            break;
        }
        if (coarse_visit > 0) {
            prolong_axes(&op->ax, &op->ay, ce, x);
            if (m) m->prolongations += 1;
            r = orc_fine_residual(g, x, b, res);
            orc_anchor_mean(g, x);
            if (r <= c->tol_fine) break;
        }
        double prev = r;
        while (total < c->max_total_sweeps) {
            orc_rbgs_sweep(g, x, b);
            record_sweep(m, 1, 5, cells, fc);
            ++rep->fine_sweeps;
            ++total;
            r = orc_fine_residual(g, x, b, res);
            orc_anchor_mean(g, x);
            if (r <= c->tol_fine) break;
            if (r > c->stall_factor * prev) break;
            prev = r;
        }
        if (r > c->tol_fine && total >= c->max_total_sweeps) {
            rep->converged = 0;
            break;
        }
    }
    rep->residual = r;
out:
    free(wf), free(res), free(cb), free(ce);
    return rc;
}

/* cycles.hpp:172-282 v_cycle_acm; levels[k] ties level k into level k+1 */
static int v_cycle_acm(const ismg_grid_spec* g, const ismg_cycle_config* c, cop_t* levels, int L,
                       double* x, const double* b, ismg_report* rep, ismg_step_metrics* m,
                       int64_t fc) {
    const int nx = g->nx, ny = g->ny;
    const int64_t cells = (int64_t)nx * ny;
    orc_zero_ghosts(nx, ny, x);
    double **xs = calloc(L, sizeof(double*)), **bs = calloc(L, sizeof(double*)),
           **rs = calloc(L, sizeof(double*)), **wf = calloc(L, sizeof(double*));
    for (int k = 0; k < L; ++k) {
        size_t sz = (size_t)(levels[k].ncx + 2) * (levels[k].ncy + 2);
        xs[k] = calloc(sz, sizeof(double));
        bs[k] = calloc(sz, sizeof(double));
        rs[k] = calloc(sz, sizeof(double));
        wf[k] = cop_flat(&levels[k]);
    }
    double* rs0 = calloc((size_t)(nx + 2) * (ny + 2), sizeof(double));
    int rc = ISMG_OK;
    long total = 0;
    double r = orc_fine_residual(g, x, b, rs0);
    orc_anchor_mean(g, x);

    while (r > c->tol_fine) {
        if (total >= c->max_total_sweeps) {
            rep->converged = 0;
            break;
        }
        int capped = 0;
        for (int k = 1; k <= L && !capped; ++k) { /* descend */
            cop_t* op = &levels[k - 1];
            const double* res_above = (k == 1) ? rs0 : rs[k - 2];
            restrict_axes(&op->ax, &op->ay, res_above, bs[k - 1]);
            if (m) m->restrictions += 1;
            memset(xs[k - 1], 0, (size_t)(op->ncx + 2) * (op->ncy + 2) * sizeof(double));
            if (k < L) {
                for (int s = 0; s < c->acm_pre_smooth; ++s) {
                    if (total >= c->max_total_sweeps) {
                        capped = 1;
                        break;
                    }
                    if ((rc = rbgs_op(op, xs[k - 1], bs[k - 1]))) goto out;
                    record_sweep(m, 1, 5, (int64_t)op->ncx * op->ncy, fc);
                    ++rep->fine_sweeps;
                    ++total;
                }
                cres(op, wf[k - 1], xs[k - 1], bs[k - 1], rs[k - 1]);
            } else {
                double rcv = cres(op, wf[k - 1], xs[k - 1], bs[k - 1], NULL);
                while (rcv > c->tol_coarse) {
                    if (total >= c->max_total_sweeps) {
                        capped = 1;
                        break;
                    }
                    if ((rc = orc_gs_sweep_lex(op->ncx, op->ncy, op->px, op->py, 1, wf[k - 1], xs[k - 1], bs[k - 1])))
                        goto out;
                    record_sweep(m, 0, 5, (int64_t)op->ncx * op->ncy, fc);
                    ++rep->coarse_sweeps;
                    ++total;
                    rcv = cres(op, wf[k - 1], xs[k - 1], bs[k - 1], NULL);
                    orc_coarse_anchor(op->ncx, op->ncy, op->singular, xs[k - 1]);
                }
            }
        }
        if (capped) {
            rep->converged = 0;
            break;
        }
        for (int k = L - 1; k >= 1 && !capped; --k) { /* ascend */
            const cop_t* below = &levels[k];
            prolong_const_axes(&below->ax, &below->ay, xs[k], xs[k - 1]);
            if (m) m->prolongations += 1;
            cop_t* op = &levels[k - 1];
            for (int s = 0; s < c->acm_post_smooth; ++s) {
                if (total >= c->max_total_sweeps) {
                    capped = 1;
                    break;
                }
                if ((rc = rbgs_op(op, xs[k - 1], bs[k - 1]))) goto out;
                record_sweep(m, 1, 5, (int64_t)op->ncx * op->ncy, fc);
                ++rep->fine_sweeps;
                ++total;
            }
        }
        if (!capped) {
            prolong_const_axes(&levels[0].ax, &levels[0].ay, xs[0], x);
            if (m) m->prolongations += 1;
            for (int s = 0; s < c->acm_post_smooth; ++s) {
                if (total >= c->max_total_sweeps) {
                    capped = 1;
                    break;
                }
                orc_rbgs_sweep(g, x, b);
                record_sweep(m, 1, 5, cells, fc);
                ++rep->fine_sweeps;
                ++total;
            }
        }
        r = orc_fine_residual(g, x, b, rs0);
        orc_anchor_mean(g, x);
        if (capped && r > c->tol_fine) {
            rep->converged = 0;
            break;
        }
    }
    rep->residual = r;
out:
    for (int k = 0; k < L; ++k) free(xs[k]), free(bs[k]), free(rs[k]), free(wf[k]);
    free(xs), free(bs), free(rs), free(wf), free(rs0);
    return rc;
}

/* cycles.hpp:289-321 PressureSolver construction + solve dispatch */
int orc_solve(const ismg_grid_spec* g0, const ismg_cycle_config* c, double* x, const double* b,
              ismg_report* rep, ismg_step_metrics* current, int64_t fine_cells) {
    int rc = cycle_validate(c);
    if (rc) return rc;
    ismg_grid_spec g = *g0;
    if (c->scheme == ISMG_SCHEME_ISMG || c->scheme == ISMG_SCHEME_GMG) g.tile = c->tile;
    if ((rc = grid_validate(&g))) return rc;
    if ((rc = orc_build_fine_diag(&g, NULL))) return rc;
    rep->converged = 1, rep->nan_seen = 0, rep->fine_sweeps = 0, rep->coarse_sweeps = 0;
    rep->residual = 0.0;
    if (c->scheme == ISMG_SCHEME_PLAIN_GS) {
        solve_plain(&g, c, x, b, rep, current, fine_cells);
        return ISMG_OK;
    }
    if (c->scheme == ISMG_SCHEME_ISMG || c->scheme == ISMG_SCHEME_GMG) {
        cop_t op;
        rc = c->scheme == ISMG_SCHEME_ISMG ? build_ismg(&g, &op) : build_gmg(&g, &op);
        if (rc) return rc;
        rc = solve_two_level(&g, c, &op, x, b, rep, current, fine_cells);
        cop_free(&op);
        return rc;
    }
    if (c->scheme == ISMG_SCHEME_ACM) { /* coarsening.hpp:452-465 build_acm_hierarchy */
        int L = c->depth - 1;
        cop_t* levels = calloc(L, sizeof(cop_t));
        cop_t cur;
        if ((rc = fine_as_operator(&g, &cur))) {
            free(levels);
            return rc;
        }
        int built = 0;
        for (int k = 1; k < c->depth; ++k) {
            const cop_t* prev = (k == 1) ? &cur : &levels[k - 2];
            if (prev->ncx < 2 || prev->ncy < 2) {
                rc = fail(ISMG_ERR_INVALID_ARGUMENT, "acm hierarchy: grid too small for depth");
                break;
            }
            if ((rc = agglomerate2(prev, &levels[k - 1]))) break;
            ++built;
        }
        cop_free(&cur);
        if (!rc) rc = v_cycle_acm(&g, c, levels, L, x, b, rep, current, fine_cells);
        for (int k = 0; k < built; ++k) cop_free(&levels[k]);
        free(levels);
        return rc;
    }
    return fail(ISMG_ERR_LOGIC, "pressure solver: unknown scheme");
}

/* ------------------------------------------------------------------------ */
/* field.hpp:77-96 apply_scalar_bc                                            */
static inline double ghost_val(int32_t k, double inner, double wrapped) {
    switch (k) {
        case ISMG_PBC_NEUMANN: return inner;
        case ISMG_PBC_DIRICHLET_ZERO: return -inner;
        default: return wrapped;
    }
}

void orc_apply_scalar_bc(const ismg_grid_spec* g, double* f) {
    int32_t bc[4];
    orc_pressure_bc(g, bc, NULL);
    const int nx = g->nx, ny = g->ny;
    for (int j = 0; j < ny; ++j) {
        SAT(f, nx, -1, j) = ghost_val(bc[0], SAT(f, nx, 0, j), SAT(f, nx, nx - 1, j));
        SAT(f, nx, nx, j) = ghost_val(bc[1], SAT(f, nx, nx - 1, j), SAT(f, nx, 0, j));
    }
    for (int i = -1; i <= nx; ++i) {
        SAT(f, nx, i, -1) = ghost_val(bc[2], SAT(f, nx, i, 0), SAT(f, nx, i, ny - 1));
        SAT(f, nx, i, ny) = ghost_val(bc[3], SAT(f, nx, i, ny - 1), SAT(f, nx, i, 0));
    }
}

/* field.hpp:302-311 normal_value */
static double normal_value(const ismg_bc* b, int x_side, int k) {
    switch (b->kind) {
        case ISMG_BC_DIRICHLET_VELOCITY: return x_side ? b->u_wall : b->v_wall;
        case ISMG_BC_INLET:
            return (k >= b->inlet_start && k < b->inlet_start + b->inlet_width) ? b->v_inflow : 0.0;
        default: return 0.0;
    }
}

/* field.hpp:334-341 tangential_ghost */
static double tangential_ghost(const ismg_bc* b, double wall_speed, double inner) {
    switch (b->kind) {
        case ISMG_BC_DIRICHLET_VELOCITY: return 2.0 * wall_speed - inner;
        case ISMG_BC_INLET: return -inner;
        default: return inner;
    }
}

/* field.hpp:143-228 apply_velocity_bc */
void orc_apply_velocity_bc(const ismg_grid_spec* g, double* u, double* v) {
    const int nx = g->nx, ny = g->ny;
    const ismg_bc *W = &g->bc[0], *E = &g->bc[1], *S = &g->bc[2], *N = &g->bc[3];
    const int per_x = W->kind == ISMG_BC_PERIODIC, per_y = S->kind == ISMG_BC_PERIODIC;
    if (!per_x)
        for (int j = 0; j < ny; ++j) {
            UAT(u, nx, 0, j) = W->kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? UAT(u, nx, 1, j) : normal_value(W, 1, j);
            UAT(u, nx, nx, j) = E->kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? UAT(u, nx, nx - 1, j) : normal_value(E, 1, j);
        }
    if (!per_y)
        for (int i = 0; i < nx; ++i) {
            VAT(v, nx, i, 0) = S->kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? VAT(v, nx, i, 1) : normal_value(S, 0, i);
            VAT(v, nx, i, ny) = N->kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? VAT(v, nx, i, ny - 1) : normal_value(N, 0, i);
        }
    if (!per_x)
        for (int j = 0; j <= ny; ++j) {
            VAT(v, nx, -1, j) = tangential_ghost(W, W->v_wall, VAT(v, nx, 0, j));
            VAT(v, nx, nx, j) = tangential_ghost(E, E->v_wall, VAT(v, nx, nx - 1, j));
        }
    if (!per_y)
        for (int i = 0; i <= nx; ++i) {
            UAT(u, nx, i, -1) = tangential_ghost(S, S->u_wall, UAT(u, nx, i, 0));
            UAT(u, nx, i, ny) = tangential_ghost(N, N->u_wall, UAT(u, nx, i, ny - 1));
        }
    if (per_y) {
        for (int i = 0; i <= nx; ++i) {
            UAT(u, nx, i, -1) = UAT(u, nx, i, ny - 1);
            UAT(u, nx, i, ny) = UAT(u, nx, i, 0);
        }
        for (int i = 0; i < nx; ++i) {
            VAT(v, nx, i, ny) = VAT(v, nx, i, 0);
            VAT(v, nx, i, -1) = VAT(v, nx, i, ny - 1);
            VAT(v, nx, i, ny + 1) = VAT(v, nx, i, 1);
        }
    }
    if (per_x) {
        for (int j = -1; j <= ny; ++j) {
            UAT(u, nx, nx, j) = UAT(u, nx, 0, j);
            UAT(u, nx, -1, j) = UAT(u, nx, nx - 1, j);
            UAT(u, nx, nx + 1, j) = UAT(u, nx, 1, j);
        }
        for (int j = -1; j <= ny + 1; ++j) {
            VAT(v, nx, -1, j) = VAT(v, nx, nx - 1, j);
            VAT(v, nx, nx, j) = VAT(v, nx, 0, j);
        }
    }
}

/* projection.hpp:38-46 divergence */
void orc_divergence(const ismg_grid_spec* g, const double* u, const double* v, double* out) {
    const int nx = g->nx, ny = g->ny;
    const double invh = 1.0 / g->h;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            SAT(out, nx, i, j) = (UAT(u, nx, i + 1, j) - UAT(u, nx, i, j) + VAT(v, nx, i, j + 1) -
                                  VAT(v, nx, i, j)) * invh;
}

/* projection.hpp:121-133 correct */
void orc_correct(const ismg_grid_spec* g, double* u, double* v, double* dp, double dt) {
    orc_apply_scalar_bc(g, dp);
    const int nx = g->nx, ny = g->ny;
    const double c = dt / g->h;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i <= nx; ++i) UAT(u, nx, i, j) -= c * (SAT(dp, nx, i, j) - SAT(dp, nx, i - 1, j));
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i < nx; ++i) VAT(v, nx, i, j) -= c * (SAT(dp, nx, i, j) - SAT(dp, nx, i, j - 1));
}

/* projection.hpp:75-119 predictor */
void orc_predictor(const ismg_grid_spec* g, const double* U, const double* V, const double* p,
                   double dt, double nu, double* ou, double* ov) {
    const int nx = g->nx, ny = g->ny;
    const int px = g->bc[0].kind == ISMG_BC_PERIODIC, py = g->bc[2].kind == ISMG_BC_PERIODIC;
    const double invh = 1.0 / g->h, invh2 = 1.0 / (g->h * g->h), half = 0.5;
#define Uc(i, j) UAT(U, nx, i, j)
#define Vc(i, j) VAT(V, nx, i, j)
    for (int j = 0; j < ny; ++j)
        for (int i = px ? 0 : 1; i < nx; ++i) {
            double uE = half * (Uc(i, j) + Uc(i + 1, j));
            double uW = half * (Uc(i - 1, j) + Uc(i, j));
            double uN = half * (Uc(i, j) + Uc(i, j + 1));
            double uS = half * (Uc(i, j - 1) + Uc(i, j));
            double vN = half * (Vc(i - 1, j + 1) + Vc(i, j + 1));
            double vS = half * (Vc(i - 1, j) + Vc(i, j));
            double adv = (uE * uE - uW * uW + uN * vN - uS * vS) * invh;
            double lap = (Uc(i + 1, j) + Uc(i - 1, j) + Uc(i, j + 1) + Uc(i, j - 1) - 4.0 * Uc(i, j)) * invh2;
            double gpx = (SAT(p, nx, i, j) - SAT(p, nx, i - 1, j)) * invh;
            UAT(ou, nx, i, j) = Uc(i, j) + dt * (-adv + nu * lap - gpx);
        }
    for (int j = py ? 0 : 1; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            double vN = half * (Vc(i, j) + Vc(i, j + 1));
            double vS = half * (Vc(i, j - 1) + Vc(i, j));
            double vE = half * (Vc(i, j) + Vc(i + 1, j));
            double vW = half * (Vc(i - 1, j) + Vc(i, j));
            double uE = half * (Uc(i + 1, j - 1) + Uc(i + 1, j));
            double uW = half * (Uc(i, j - 1) + Uc(i, j));
            double adv = (vN * vN - vS * vS + vE * uE - vW * uW) * invh;
            double lap = (Vc(i + 1, j) + Vc(i - 1, j) + Vc(i, j + 1) + Vc(i, j - 1) - 4.0 * Vc(i, j)) * invh2;
            double gpy = (SAT(p, nx, i, j) - SAT(p, nx, i, j - 1)) * invh;
            VAT(ov, nx, i, j) = Vc(i, j) + dt * (-adv + nu * lap - gpy);
        }
#undef Uc
#undef Vc
}

/* projection.hpp:139-190 step (CFL warnings are diagnostics only) */
int orc_step(const ismg_grid_spec* g, const ismg_cycle_config* c, double* u, double* v, double* p,
             double* scal, ismg_report* rep, ismg_step_metrics* current, int64_t fine_cells) {
    const int nx = g->nx, ny = g->ny;
    const size_t nu_ = (size_t)(nx + 3) * (ny + 2), nv_ = (size_t)(nx + 2) * (ny + 3),
                 ns = (size_t)(nx + 2) * (ny + 2);
    const double dt = scal[1], nu = scal[2];
    orc_apply_scalar_bc(g, p);
    orc_apply_velocity_bc(g, u, v);
    rep->converged = 1, rep->nan_seen = 0, rep->fine_sweeps = 0, rep->coarse_sweeps = 0;
    rep->residual = 0.0;
    if (dt == 0.0) {
        scal[3] += 1;
        return ISMG_OK;
    }
    double* us = malloc(nu_ * sizeof(double));
    double* vs = malloc(nv_ * sizeof(double));
    memcpy(us, u, nu_ * sizeof(double));
    memcpy(vs, v, nv_ * sizeof(double));
    orc_predictor(g, u, v, p, dt, nu, us, vs);
    orc_apply_velocity_bc(g, us, vs);
    double* rhs = calloc(ns, sizeof(double));
    orc_divergence(g, us, vs, rhs);
    const double scale = g->h * g->h / dt;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) SAT(rhs, nx, i, j) *= scale;
    double* dp = calloc(ns, sizeof(double));
    int rc = orc_solve(g, c, dp, rhs, rep, current, fine_cells);
    if (!rc) {
        orc_correct(g, us, vs, dp, dt);
        memcpy(u, us, nu_ * sizeof(double));
        memcpy(v, vs, nv_ * sizeof(double));
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) SAT(p, nx, i, j) += SAT(dp, nx, i, j);
        scal[0] += dt;
        scal[3] += 1;
    }
    free(us), free(vs), free(rhs), free(dp);
    return rc;
}

/* bench.hpp:127-158 run_case restricted to seed = 0, steady_tol = 0, t_max = 0;
 * metrics.hpp:61-67 close_timestep per row */
int orc_run_steps(const ismg_grid_spec* g, const ismg_cycle_config* c, double* u, double* v,
                  double* p, double* scal, long nsteps, ismg_step_metrics* rows) {
    const int64_t fc = (int64_t)g->nx * g->ny;
    for (long s = 0; s < nsteps; ++s) {
        ismg_step_metrics cur;
        memset(&cur, 0, sizeof cur);
        ismg_report rep;
        int rc = orc_step(g, c, u, v, p, scal, &rep, &cur, fc);
        if (rc) return rc;
        cur.step = (int64_t)scal[3];
        cur.residual_final = scal[1] == 0.0 ? 0.0 : rep.residual;
        cur.converged = rep.converged;
        if (rows) rows[s] = cur;
    }
    return ISMG_OK;
}

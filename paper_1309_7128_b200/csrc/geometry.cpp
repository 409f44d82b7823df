// geometry.cpp — host-side setup of the pressure path, run once per solver:
// validation, pressure closures, tile axes and the coarse operators.
//
// The coarse operator is assembled face segment by face segment in the same
// order as the reference (coarsening.hpp:196-305) so the nine coefficient
// planes are bit-identical to build_ismg_operator<double>; they are uploaded
// to HBM once and stay resident.
#include <cmath>

#include "common.h"

namespace ismgb {

void grid_validate(const ismg_grid_spec& g) {  // grid.hpp:79-96
    if (g.nx < 1 || g.ny < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "grid: nx, ny must be >= 1");
    if (g.h <= 0.0) fail(ISMG_ERR_INVALID_ARGUMENT, "grid: h must be positive");
    if (g.tile < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "grid: tile must be >= 2");
    auto per = [&](int s) { return g.bc[s].kind == ISMG_BC_PERIODIC; };
    if (per(ISMG_SIDE_WEST) != per(ISMG_SIDE_EAST))
        fail(ISMG_ERR_INVALID_ARGUMENT, "grid: periodic west/east must pair");
    if (per(ISMG_SIDE_SOUTH) != per(ISMG_SIDE_NORTH))
        fail(ISMG_ERR_INVALID_ARGUMENT, "grid: periodic south/north must pair");
    for (int s = 0; s < 4; ++s) {
        const ismg_bc& b = g.bc[s];
        if (b.kind != ISMG_BC_INLET) continue;
        int extent = (s == ISMG_SIDE_SOUTH || s == ISMG_SIDE_NORTH) ? g.nx : g.ny;
        if (b.inlet_width < 1 || b.inlet_start < 0 || b.inlet_start + b.inlet_width > extent)
            fail(ISMG_ERR_INVALID_ARGUMENT, "grid: inlet span out of range");
    }
}

void cycle_validate(const ismg_cycle_config& c) {  // cycles.hpp:31-44
    if (!(c.tol_fine > 0) || !(c.tol_coarse > 0))
        fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: tolerances must be positive");
    if (c.tol_coarse < c.tol_fine) fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: tol_coarse must be >= tol_fine");
    if (c.max_total_sweeps < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: max_total_sweeps must be positive");
    if (!(c.stall_factor > 0.0 && c.stall_factor < 1.0))
        fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: stall_factor must lie in (0,1)");
    if (c.acm_pre_smooth < 0 || c.acm_post_smooth < 0)
        fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: smoothing counts must be non-negative");
    if (c.depth < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: depth must be >= 2");
    if (c.tile < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "cycle: tile must be >= 2");
    if (c.scheme < ISMG_SCHEME_PLAIN_GS || c.scheme > ISMG_SCHEME_ACM)
        fail(ISMG_ERR_LOGIC, "pressure solver: unknown scheme");
}

PBC pressure_bc(const ismg_grid_spec& g, bool* singular) {  // grid.hpp:124-149
    PBC p;
    bool sing = true;
    for (int s = 0; s < 4; ++s) {
        switch (g.bc[s].kind) {
            case ISMG_BC_DIRICHLET_VELOCITY:
            case ISMG_BC_INLET: p.k[s] = ISMG_PBC_NEUMANN; break;
            case ISMG_BC_SYMMETRY_FIXED_PRESSURE: p.k[s] = ISMG_PBC_DIRICHLET_ZERO; break;
            default: p.k[s] = ISMG_PBC_PERIODIC; break;
        }
        if (p.k[s] == ISMG_PBC_DIRICHLET_ZERO) sing = false;
    }
    if (singular) *singular = sing;
    return p;
}

void check_fine_stage(const ismg_grid_spec& g) {  // smoother.hpp:55-65
    // d(i,j) = sum of four face weights; only a 1-cell extent can leave a row
    // without any open face, so checking the four corner cells suffices.
    PBC p = pressure_bc(g);
    auto w = [](int k) { return k == ISMG_PBC_NEUMANN ? 0.0 : k == ISMG_PBC_DIRICHLET_ZERO ? 2.0 : 1.0; };
    for (int j : {0, g.ny - 1})
        for (int i : {0, g.nx - 1}) {
            double d = 0;
            d += (i > 0) ? 1.0 : w(p.k[ISMG_SIDE_WEST]);
            d += (i < g.nx - 1) ? 1.0 : w(p.k[ISMG_SIDE_EAST]);
            d += (j > 0) ? 1.0 : w(p.k[ISMG_SIDE_SOUTH]);
            d += (j < g.ny - 1) ? 1.0 : w(p.k[ISMG_SIDE_NORTH]);
            if (d <= 0.0) fail(ISMG_ERR_DOMAIN, "smoother: fine row has empty stencil");
        }
}

// coarsening.hpp:60-97: tile starts/widths/centres and the per-cell bracketing
// rectangle of cell centre i + 0.5 (clamped at non-periodic ends, wrapped on
// periodic axes).
TileAxisH::TileAxisH(int n_, int tile_, bool periodic_) : n(n_), tile(tile_), periodic(periodic_) {
    if (n < 1 || tile < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "tile axis: need n >= 1, tile >= 1");
    nc = (n + tile - 1) / tile;
    start.resize(nc);
    width.resize(nc);
    center.resize(nc);
    for (int k = 0; k < nc; ++k) {
        start[k] = k * tile;
        width[k] = (k == nc - 1) ? n - (nc - 1) * tile : tile;
        center[k] = start[k] + width[k] / 2.0;
    }
    rect.assign(nc > 1 ? nc - 1 : 0, 0.0);
    for (int k = 0; k + 1 < nc; ++k) rect[k] = center[k + 1] - center[k];
    if (periodic) rect_wrap = (width[nc - 1] + width[0]) / 2.0;
    k0.resize(n);
    k1.resize(n);
    t.resize(n);
    dk.resize(n);
    int k = 0;  // centres are increasing: walk them once
    for (int i = 0; i < n; ++i) {
        const double c = i + 0.5;
        if (nc == 1) {
            k0[i] = 0, k1[i] = 0, t[i] = 0.0, dk[i] = 1.0;
        } else if (periodic && (c < center[0] || c >= center[nc - 1])) {
            double tt = c - center[nc - 1];
            if (tt < 0) tt += n;
            k0[i] = nc - 1, k1[i] = 0, t[i] = tt, dk[i] = rect_wrap;
        } else if (c <= center[0]) {
            k0[i] = 0, k1[i] = 1, t[i] = 0.0, dk[i] = rect[0];
        } else if (c >= center[nc - 1]) {
            k0[i] = nc - 2, k1[i] = nc - 1, t[i] = rect[nc - 2], dk[i] = rect[nc - 2];
        } else {
            while (center[k + 1] <= c) ++k;
            k0[i] = k, k1[i] = k + 1, t[i] = c - center[k], dk[i] = rect[k];
        }
    }
}

namespace {

// coarsening.hpp:110-119: coarse index delta folded onto {-1,0,1} on periodic axes.
int fold_delta(int to, int from, int nc, bool periodic) {
    int d = to - from;
    if (periodic) {
        if (d > nc / 2) d -= nc;
        if (d < -nc / 2) d += nc;
        if (d == nc - 1) d = -1;
        if (d == -(nc - 1)) d = 1;
    }
    return d;
}

// (di, dj) -> slot in C,E,W,N,S,NE,NW,SE,SW order (coarsening.hpp:121-132)
int slot_of(int di, int dj) {
    if (di < -1 || di > 1 || dj < -1 || dj > 1)
        fail(ISMG_ERR_LOGIC, "coarsening: coupling beyond the 9-point neighborhood");
    static const int lut[9] = {8, 4, 7, 2, 0, 1, 6, 3, 5};
    return lut[(dj + 1) * 3 + (di + 1)];
}

struct Assembler {
    CoarseOpH& op;
    // Row (I,J) gains `wgt` times the unknown of coarse cell (Ic,Jc).
    void couple(int I, int J, int Ic, int Jc, double wgt) {
        int s = slot_of(fold_delta(Ic, I, op.ncx, op.px), fold_delta(Jc, J, op.ncy, op.py));
        op.at(s, I, J) += wgt;
    }
    // One fine face segment: flux weights on the 4 rectangle corners leave
    // `from` and enter `to` with the opposite sign (coarsening.hpp:221-254).
    void segment(int from_I, int from_J, int to_I, int to_J, const double ws[4], const int ic[4],
                 const int jc[4]) {
        for (int q = 0; q < 4; ++q) {
            couple(from_I, from_J, ic[q], jc[q], ws[q]);
            couple(to_I, to_J, ic[q], jc[q], -ws[q]);
        }
    }
};

}  // namespace

// Interpolated 9-point operator = R A P (coarsening.hpp:196-305).
CoarseOpH build_ismg_operator(const ismg_grid_spec& g) {
    if (g.tile < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "ismg operator: tile must be >= 2");
    bool singular = false;
    PBC bc = pressure_bc(g, &singular);
    CoarseOpH op;
    op.ax = TileAxisH(g.nx, g.tile, bc.px());
    op.ay = TileAxisH(g.ny, g.tile, bc.py());
    if (op.ax.nc < 2 || op.ay.nc < 2)
        fail(ISMG_ERR_INVALID_ARGUMENT, "ismg operator: need at least 2 coarse cells per axis");
    op.ncx = op.ax.nc, op.ncy = op.ay.nc;
    op.px = bc.px(), op.py = bc.py();
    op.five_point = false;
    op.singular = singular;
    op.w.assign(size_t(9) * op.ncx * op.ncy, 0.0);
    Assembler A{op};
    const TileAxisH &ax = op.ax, &ay = op.ay;

    // x-flux through the vertical coarse face (I | Ie), row J: the
    // interpolant's x-rectangle spans the two centres, the y-rectangle
    // follows each fine segment.
    auto x_face = [&](int I, int Ie, int J) {
        const double dx = (Ie == I + 1) ? ax.rect[I] : ax.rect_wrap;
        for (int j = ay.start[J]; j < ay.start[J] + ay.width[J]; ++j) {
            const double gw = 1.0 / (dx * ay.dk[j]), t = ay.t[j], dy = ay.dk[j];
            const double ws[4] = {-gw * (dy - t), gw * (dy - t), -gw * t, gw * t};
            const int ic[4] = {I, Ie, I, Ie};
            const int jc[4] = {ay.k0[j], ay.k0[j], ay.k1[j], ay.k1[j]};
            A.segment(I, J, Ie, J, ws, ic, jc);
        }
    };
    // y-flux through the horizontal coarse face (J | Jn), column I.
    auto y_face = [&](int I, int J, int Jn) {
        const double dy = (Jn == J + 1) ? ay.rect[J] : ay.rect_wrap;
        for (int i = ax.start[I]; i < ax.start[I] + ax.width[I]; ++i) {
            const double gw = 1.0 / (ax.dk[i] * dy), s = ax.t[i], dx = ax.dk[i];
            const double ws[4] = {-gw * (dx - s), -gw * s, gw * (dx - s), gw * s};
            const int ic[4] = {ax.k0[i], ax.k1[i], ax.k0[i], ax.k1[i]};
            const int jc[4] = {J, J, Jn, Jn};
            A.segment(I, J, I, Jn, ws, ic, jc);
        }
    };
    for (int J = 0; J < op.ncy; ++J) {
        for (int I = 0; I + 1 < op.ncx; ++I) x_face(I, I + 1, J);
        if (op.px) x_face(op.ncx - 1, 0, J);
    }
    for (int I = 0; I < op.ncx; ++I) {
        for (int J = 0; J + 1 < op.ncy; ++J) y_face(I, J, J + 1);
        if (op.py) y_face(I, op.ncy - 1, 0);
    }
    // Fixed-pressure closures: the fine ghost (-inner) folds through P as
    // -2 x the interpolated value of the boundary cell (coarsening.hpp:268-303).
    auto close_cell = [&](int I, int J, int i, int j) {
        const double gw = 1.0 / (ax.dk[i] * ay.dk[j]);
        const double s = ax.t[i], dx = ax.dk[i], t = ay.t[j], dy = ay.dk[j];
        A.couple(I, J, ax.k0[i], ay.k0[j], -2.0 * gw * (dx - s) * (dy - t));
        A.couple(I, J, ax.k1[i], ay.k0[j], -2.0 * gw * s * (dy - t));
        A.couple(I, J, ax.k0[i], ay.k1[j], -2.0 * gw * (dx - s) * t);
        A.couple(I, J, ax.k1[i], ay.k1[j], -2.0 * gw * s * t);
    };
    for (int side : {ISMG_SIDE_WEST, ISMG_SIDE_EAST}) {
        if (bc.k[side] != ISMG_PBC_DIRICHLET_ZERO) continue;
        const int I = side == ISMG_SIDE_WEST ? 0 : op.ncx - 1, i = side == ISMG_SIDE_WEST ? 0 : g.nx - 1;
        for (int J = 0; J < op.ncy; ++J)
            for (int j = ay.start[J]; j < ay.start[J] + ay.width[J]; ++j) close_cell(I, J, i, j);
    }
    for (int side : {ISMG_SIDE_SOUTH, ISMG_SIDE_NORTH}) {
        if (bc.k[side] != ISMG_PBC_DIRICHLET_ZERO) continue;
        const int J = side == ISMG_SIDE_SOUTH ? 0 : op.ncy - 1, j = side == ISMG_SIDE_SOUTH ? 0 : g.ny - 1;
        for (int I = 0; I < op.ncx; ++I)
            for (int i = ax.start[I]; i < ax.start[I] + ax.width[I]; ++i) close_cell(I, J, i, j);
    }
    return op;
}

// Re-discretised 5-point operator (coarsening.hpp:311-360).
CoarseOpH build_gmg_operator(const ismg_grid_spec& g) {
    if (g.tile < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "gmg operator: tile must be >= 2");
    bool singular = false;
    PBC bc = pressure_bc(g, &singular);
    CoarseOpH op;
    op.ax = TileAxisH(g.nx, g.tile, bc.px());
    op.ay = TileAxisH(g.ny, g.tile, bc.py());
    if (op.ax.nc < 2 || op.ay.nc < 2)
        fail(ISMG_ERR_INVALID_ARGUMENT, "gmg operator: need at least 2 coarse cells per axis");
    op.ncx = op.ax.nc, op.ncy = op.ay.nc;
    op.px = bc.px(), op.py = bc.py();
    op.five_point = true;
    op.singular = singular;
    op.w.assign(size_t(9) * op.ncx * op.ncy, 0.0);
    const TileAxisH &ax = op.ax, &ay = op.ay;
    for (int J = 0; J < op.ncy; ++J)
        for (int I = 0; I < op.ncx; ++I) {
            const double face_x = ay.width[J], face_y = ax.width[I];
            double diag = 0.0;
            // one face: open neighbour (slot), periodic wrap, or a boundary closure
            auto face = [&](int slot, bool inner, double inner_dist, bool per, double wrap_dist, int side,
                            double face_len, double half_w) {
                if (inner || per) {
                    const double c = face_len / (inner ? inner_dist : wrap_dist);
                    op.at(slot, I, J) += c;
                    diag += c;
                } else if (bc.k[side] == ISMG_PBC_DIRICHLET_ZERO) {
                    diag += face_len / half_w;
                }
            };
            face(1, I < op.ncx - 1, I < op.ncx - 1 ? ax.rect[I] : 0.0, ax.periodic, ax.rect_wrap, ISMG_SIDE_EAST,
                 face_x, ax.width[I] / 2.0);
            face(2, I > 0, I > 0 ? ax.rect[I - 1] : 0.0, ax.periodic, ax.rect_wrap, ISMG_SIDE_WEST, face_x,
                 ax.width[I] / 2.0);
            face(3, J < op.ncy - 1, J < op.ncy - 1 ? ay.rect[J] : 0.0, ay.periodic, ay.rect_wrap, ISMG_SIDE_NORTH,
                 face_y, ay.width[J] / 2.0);
            face(4, J > 0, J > 0 ? ay.rect[J - 1] : 0.0, ay.periodic, ay.rect_wrap, ISMG_SIDE_SOUTH, face_y,
                 ay.width[J] / 2.0);
            op.at(0, I, J) = -diag;
        }
    return op;
}

// Summed (additive-correction) hierarchy: factor-2 agglomeration of the fine
// flux matrix (coarsening.hpp:367-465). Level k's axes tile level k-1.
std::vector<CoarseOpH> build_acm_hierarchy(const ismg_grid_spec& g, int depth) {
    if (depth < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "acm hierarchy: depth must be >= 2");
    bool singular = false;
    PBC bc = pressure_bc(g, &singular);
    // level 0: the fine matrix in stencil form (fine_as_operator)
    CoarseOpH cur;
    cur.ax = TileAxisH(g.nx, 1, bc.px());
    cur.ay = TileAxisH(g.ny, 1, bc.py());
    cur.ncx = g.nx, cur.ncy = g.ny;
    cur.px = bc.px(), cur.py = bc.py();
    cur.five_point = true;
    cur.singular = singular;
    cur.w.assign(size_t(9) * g.nx * g.ny, 0.0);
    auto closure = [](int k) { return k == ISMG_PBC_NEUMANN ? 0.0 : k == ISMG_PBC_DIRICHLET_ZERO ? 2.0 : 1.0; };
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i) {
            double diag = 0.0;
            const bool open[4] = {i < g.nx - 1, i > 0, j < g.ny - 1, j > 0};
            const int side[4] = {ISMG_SIDE_EAST, ISMG_SIDE_WEST, ISMG_SIDE_NORTH, ISMG_SIDE_SOUTH};
            for (int f = 0; f < 4; ++f) {
                if (open[f] || bc.k[side[f]] == ISMG_PBC_PERIODIC) {
                    cur.at(1 + f, i, j) = 1.0;
                    diag += 1.0;
                } else {
                    diag += closure(bc.k[side[f]]);
                }
            }
            cur.at(0, i, j) = -diag;
        }
    static const int sdi[5] = {0, 1, -1, 0, 0}, sdj[5] = {0, 0, 0, 1, -1};
    std::vector<CoarseOpH> levels;
    for (int k = 1; k < depth; ++k) {
        const CoarseOpH& f = levels.empty() ? cur : levels.back();
        if (f.ncx < 2 || f.ncy < 2) fail(ISMG_ERR_INVALID_ARGUMENT, "acm hierarchy: grid too small for depth");
        CoarseOpH c;
        c.ax = TileAxisH(f.ncx, 2, f.px);
        c.ay = TileAxisH(f.ncy, 2, f.py);
        c.ncx = c.ax.nc, c.ncy = c.ay.nc;
        c.px = f.px, c.py = f.py;
        c.five_point = true;
        c.singular = f.singular;
        c.w.assign(size_t(9) * c.ncx * c.ncy, 0.0);
        for (int j = 0; j < f.ncy; ++j)
            for (int i = 0; i < f.ncx; ++i)
                for (int sl = 0; sl < 5; ++sl) {
                    const double wgt = f.at(sl, i, j);
                    if (wgt == 0.0) continue;
                    int ii = i + sdi[sl], jj = j + sdj[sl];
                    if (f.px) ii = (ii + f.ncx) % f.ncx;
                    if (f.py) jj = (jj + f.ncy) % f.ncy;
                    if (ii < 0 || ii >= f.ncx || jj < 0 || jj >= f.ncy) continue;
                    const int s = slot_of(fold_delta(ii / 2, i / 2, c.ncx, c.px), fold_delta(jj / 2, j / 2, c.ncy, c.py));
                    c.at(s, i / 2, j / 2) += wgt;
                }
        levels.push_back(std::move(c));
    }
    return levels;
}

}  // namespace ismgb

// ops.cu — op-level sm_100a kernels behind the reference's operator API
// (smoother.hpp, coarsening.hpp, field.hpp, projection.hpp). Each kernel is
// bit-identical to the reference function it replaces (compiled -fmad=false,
// same association order); the interior-sum of anchor_mean is a fixed-order
// tree (deterministic, not serial-order).
#include <algorithm>

#include "engine.h"
#include "kernels.cuh"

namespace ismgb {

namespace {

inline int blocks_for(int64_t n, int threads, int cap) {
    int64_t b = (n + threads - 1) / threads;
    return int(std::max<int64_t>(1, std::min<int64_t>(b, cap)));
}

// ---- generic field kernels ----------------------------------------------
__global__ void fill_kernel(View f, int w, int h, double v) {  // logical [-1, w) x [-1, h)
    int i = blockIdx.x * blockDim.x + threadIdx.x - 1;
    int j = blockIdx.y - 1;
    if (i < w) f.at(i, j) = v;
}

__global__ void copy_kernel(View d, View s, int w, int h) {
    int i = blockIdx.x * blockDim.x + threadIdx.x - 1;
    int j = blockIdx.y - 1;
    if (i < w) d.at(i, j) = s.at(i, j);
}

__global__ void zero_ghosts_kernel(View f) {  // smoother.hpp:71-81
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k <= f.ny + 1) {
        f.at(-1, k - 1) = 0.0;
        f.at(f.nx, k - 1) = 0.0;
    }
    if (k <= f.nx + 1) {
        f.at(k - 1, -1) = 0.0;
        f.at(k - 1, f.ny) = 0.0;
    }
}

__global__ void refresh_periodic_kernel(View f, bool px, bool py) {  // smoother.hpp:83-96
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (px && k < f.ny) {
        f.at(-1, k) = f.at(f.nx - 1, k);
        f.at(f.nx, k) = f.at(0, k);
    }
    if (py && k < f.nx) {
        f.at(k, -1) = f.at(k, f.ny - 1);
        f.at(k, f.ny) = f.at(k, 0);
    }
}

// smoother.hpp:101-117, one colour: x = (((W + E) + S) + N - b) / d.
// Same-colour cells never read each other (periodic images come from the
// ghost ring refreshed before the half-sweep), so the parallel update is the
// serial one.
__global__ void rbgs_half_kernel(View x, View b, PBC bc, int color) {
    const int j = blockIdx.y;
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x) + ((color + j) & 1);
    if (i >= x.nx) return;
    const double s = x.at(i - 1, j) + x.at(i + 1, j) + x.at(i, j - 1) + x.at(i, j + 1);
    x.at(i, j) = div_by_diag(s - b.at(i, j), fine_diag(bc, x.nx, x.ny, i, j));
}

// atomic max on non-negative doubles through their ordered bit patterns
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

// smoother.hpp:121-141: r = b - ((((W + E) + S) + N) - d x).
__global__ void fine_residual_kernel(View x, View b, View out, PBC bc, double* rmax, double* nan_count) {
    __shared__ double red[32];
    const int64_t n = int64_t(x.nx) * x.ny;
    double m = 0.0, nans = 0.0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(k / x.nx), i = int(k - int64_t(j) * x.nx);
        const double ax = x.at(i - 1, j) + x.at(i + 1, j) + x.at(i, j - 1) + x.at(i, j + 1) -
                          fine_diag(bc, x.nx, x.ny, i, j) * x.at(i, j);
        const double r = b.at(i, j) - ax;
        if (out.p) out.at(i, j) = r;
        m = max_drop_nan(m, fabs(r));
        if (r != r) nans += 1.0;
    }
    m = block_max(m, red);
    if (threadIdx.x == 0) atomic_max_nonneg(rmax, m);
    if (nan_count) {
        nans = block_sum(nans, red);
        if (threadIdx.x == 0 && nans > 0) atomicAdd(nan_count, nans);
    }
}

__global__ void sum_partials_kernel(View x, double* part) {
    __shared__ double red[32];
    const int64_t n = int64_t(x.nx) * x.ny;
    double s = 0.0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(k / x.nx), i = int(k - int64_t(j) * x.nx);
        s += x.at(i, j);
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// field.hpp:49 + smoother.hpp:147: out[0] = sum, out[1] = -(sum / N)
__global__ void finish_mean_kernel(const double* part, int nparts, double ncells, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int k = threadIdx.x; k < nparts; k += blockDim.x) s += part[k];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
        out[0] = s;
        out[1] = -(s / ncells);
    }
}

__global__ void shift_kernel(View x, const double* c) {  // field.hpp:53-59
    const double v = *c;
    const int64_t n = int64_t(x.nx) * x.ny;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(k / x.nx), i = int(k - int64_t(j) * x.nx);
        x.at(i, j) += v;
    }
}

// coarsening.hpp:471-480 in the reference's own order: each coarse cell sums
// its tile row-major from 0 (bit-identical to the serial loop).
__global__ void restrict_exact_kernel(View fine, View coarse, int tx, int ty, int ncx, int ncy) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y;
    if (I >= ncx) return;
    const int i0 = I * tx, i1 = min(i0 + tx, fine.nx), j0 = J * ty, j1 = min(j0 + ty, fine.ny);
    double s = 0.0;
    for (int j = j0; j < j1; ++j)
        for (int i = i0; i < i1; ++i) s += fine.at(i, j);
    coarse.at(I, J) = s;
}

// coarsening.hpp:485-503
__global__ void prolong_bilinear_kernel(View coarse, View fine, AxisDev ax, AxisDev ay) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= fine.nx) return;
    const double t = ay.t[j], dy = ay.dk[j], s = ax.t[i], dx = ax.dk[i];
    const int J0 = ay.k0[j], J1 = ay.k1[j], I0 = ax.k0[i], I1 = ax.k1[i];
    const double val = ((dx - s) * ((dy - t) * coarse.at(I0, J0) + t * coarse.at(I0, J1)) +
                        s * ((dy - t) * coarse.at(I1, J0) + t * coarse.at(I1, J1))) /
                       (dx * dy);
    fine.at(i, j) += val;
}

// coarsening.hpp:506-514
__global__ void prolong_constant_kernel(View coarse, View fine, int tx, int ty) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= fine.nx) return;
    fine.at(i, j) += coarse.at(i / tx, j / ty);
}

// coarsening.hpp:531-549
__global__ void coarse_residual_kernel(View x, View b, View out, const double* __restrict__ w, int ncx, int ncy,
                                       bool px, bool py, int nslots, double* rmax) {
    __shared__ double red[32];
    const int64_t n = int64_t(ncx) * ncy;
    double m = 0.0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
        double ax = w[k] * x.at(I, J);
        for (int sl = 1; sl < nslots; ++sl) {
            const double wg = w[sl * n + k];
            if (wg != 0.0) ax += wg * coarse_neighbor(x, ncx, ncy, px, py, I, J, slot_di(sl), slot_dj(sl));
        }
        const double r = b.at(I, J) - ax;
        if (out.p) out.at(I, J) = r;
        m = max_drop_nan(m, fabs(r));
    }
    m = block_max(m, red);
    if (threadIdx.x == 0) atomic_max_nonneg(rmax, m);
}

__device__ __forceinline__ void gs_cell(View x, View b, const double* __restrict__ w, int ncx, int ncy, bool px,
                                        bool py, int nslots, int I, int J) {
    const int64_t n = int64_t(ncx) * ncy, k = int64_t(J) * ncx + I;
    double s = 0;
    for (int sl = 1; sl < nslots; ++sl) {
        const double wg = w[sl * n + k];
        if (wg != 0.0) s += wg * coarse_neighbor(x, ncx, ncy, px, py, I, J, slot_di(sl), slot_dj(sl));
    }
    x.at(I, J) = (b.at(I, J) - s) / w[k];
}

// coarsening.hpp:552-567 lexicographic GS. Without an x-wrap, cell (I,J)
// reads new values only from cells with smaller t = I + 2J and old values only
// from cells with larger t, so the anti-diagonal wavefront over t reproduces
// the serial order exactly. An x-wrap couples the end of row J-1 to the
// start of row J, making the order fully serial (one cell per step).
__global__ void gs_lex_kernel(View x, View b, const double* __restrict__ w, int ncx, int ncy, bool px, bool py,
                              int nslots) {
    if (px) {
        if (threadIdx.x == 0)
            for (int J = 0; J < ncy; ++J)
                for (int I = 0; I < ncx; ++I) gs_cell(x, b, w, ncx, ncy, px, py, nslots, I, J);
        return;
    }
    const int tmax = (ncx - 1) + 2 * (ncy - 1);
    for (int t = 0; t <= tmax; ++t) {
        const int jlo = max(0, (t - (ncx - 1) + 1) / 2), jhi = min(ncy - 1, t / 2);
        for (int J = jlo + int(threadIdx.x); J <= jhi; J += blockDim.x) gs_cell(x, b, w, ncx, ncy, px, py, nslots, t - 2 * J, J);
        __syncthreads();
    }
}

// coarsening.hpp:571-588 one colour of red-black on a stored 5-point level.
// With an odd periodic extent same-colour cells touch across the seam and the
// serial order matters; that (small) case runs in one thread.
__global__ void rbgs_op_kernel(View x, View b, const double* __restrict__ w, int ncx, int ncy, bool px, bool py,
                               int color, bool serial) {
    if (serial) {
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
            for (int J = 0; J < ncy; ++J)
                for (int I = (color + J) & 1; I < ncx; I += 2) gs_cell(x, b, w, ncx, ncy, px, py, 5, I, J);
        return;
    }
    const int J = blockIdx.y;
    const int I = 2 * (blockIdx.x * blockDim.x + threadIdx.x) + ((color + J) & 1);
    if (I < ncx) gs_cell(x, b, w, ncx, ncy, px, py, 5, I, J);
}

// ---- projection kernels (projection.hpp, field.hpp) -----------------------
__device__ __forceinline__ double ghost_of(int k, double inner, double wrapped) {
    return k == ISMG_PBC_NEUMANN ? inner : (k == ISMG_PBC_DIRICHLET_ZERO ? -inner : wrapped);
}

__global__ void scalar_bc_x_kernel(View f, PBC bc) {  // field.hpp:239-242
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= f.ny) return;
    const double a = f.at(0, j), z = f.at(f.nx - 1, j);
    f.at(-1, j) = ghost_of(bc.k[ISMG_SIDE_WEST], a, z);
    f.at(f.nx, j) = ghost_of(bc.k[ISMG_SIDE_EAST], z, a);
}

__global__ void scalar_bc_y_kernel(View f, PBC bc) {  // field.hpp:243-246
    const int i = blockIdx.x * blockDim.x + threadIdx.x - 1;
    if (i > f.nx) return;
    const double a = f.at(i, 0), z = f.at(i, f.ny - 1);
    f.at(i, -1) = ghost_of(bc.k[ISMG_SIDE_SOUTH], a, z);
    f.at(i, f.ny) = ghost_of(bc.k[ISMG_SIDE_NORTH], z, a);
}

struct BcDev {
    int kind;
    int start, width;
    double u_wall, v_wall;
    double v_inflow;
};

__device__ __forceinline__ double normal_value(const BcDev& b, bool x_side, int k) {  // field.hpp:302-311
    if (b.kind == ISMG_BC_DIRICHLET_VELOCITY) return x_side ? b.u_wall : b.v_wall;
    if (b.kind == ISMG_BC_INLET) return (k >= b.start && k < b.start + b.width) ? b.v_inflow : 0.0;
    return 0.0;
}

__device__ __forceinline__ double tangential_ghost(const BcDev& b, double wall, double inner) {  // :334-341
    if (b.kind == ISMG_BC_DIRICHLET_VELOCITY) return 2.0 * wall - inner;
    if (b.kind == ISMG_BC_INLET) return -inner;
    return inner;
}

struct VelBc {
    BcDev s[4];
};

// field.hpp:313-331 wall-normal faces
__global__ void vel_normal_kernel(View u, View v, VelBc bc, int nx, int ny, bool per_x, bool per_y) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const BcDev &W = bc.s[0], &E = bc.s[1], &S = bc.s[2], &N = bc.s[3];
    if (!per_x && k < ny) {
        u.at(0, k) = W.kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? u.at(1, k) : normal_value(W, true, k);
        u.at(nx, k) = E.kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? u.at(nx - 1, k) : normal_value(E, true, k);
    }
    if (!per_y && k < nx) {
        v.at(k, 0) = S.kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? v.at(k, 1) : normal_value(S, false, k);
        v.at(k, ny) = N.kind == ISMG_BC_SYMMETRY_FIXED_PRESSURE ? v.at(k, ny - 1) : normal_value(N, false, k);
    }
}

// field.hpp:342-353 tangential ghost layers
__global__ void vel_tangential_kernel(View u, View v, VelBc bc, int nx, int ny, bool per_x, bool per_y) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const BcDev &W = bc.s[0], &E = bc.s[1], &S = bc.s[2], &N = bc.s[3];
    if (!per_x && k <= ny) {
        v.at(-1, k) = tangential_ghost(W, W.v_wall, v.at(0, k));
        v.at(nx, k) = tangential_ghost(E, E.v_wall, v.at(nx - 1, k));
    }
    if (!per_y && k <= nx) {
        u.at(k, -1) = tangential_ghost(S, S.u_wall, u.at(k, 0));
        u.at(k, ny) = tangential_ghost(N, N.u_wall, u.at(k, ny - 1));
    }
}

// field.hpp:357-367 periodic images in y (core columns)
__global__ void vel_wrap_y_kernel(View u, View v, int nx, int ny) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k <= nx) {
        u.at(k, -1) = u.at(k, ny - 1);
        u.at(k, ny) = u.at(k, 0);
    }
    if (k < nx) {
        v.at(k, ny) = v.at(k, 0);
        v.at(k, -1) = v.at(k, ny - 1);
        v.at(k, ny + 1) = v.at(k, 1);
    }
}

// field.hpp:368-378 periodic images in x (full rows, after y)
__global__ void vel_wrap_x_kernel(View u, View v, int nx, int ny) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x - 1;
    if (k <= ny) {
        u.at(nx, k) = u.at(0, k);
        u.at(-1, k) = u.at(nx - 1, k);
        u.at(nx + 1, k) = u.at(1, k);
    }
    if (k <= ny + 1) {
        v.at(-1, k) = v.at(nx - 1, k);
        v.at(nx, k) = v.at(0, k);
    }
}

// projection.hpp:38-46 (+ the separate h^2/dt rounding of :174-178)
__global__ void divergence_kernel(View u, View v, View out, double invh, double scale, bool do_scale) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= out.nx) return;
    double d = (u.at(i + 1, j) - u.at(i, j) + v.at(i, j + 1) - v.at(i, j)) * invh;
    if (do_scale) d *= scale;
    out.at(i, j) = d;
}

// projection.hpp:128-132 (dp's ghost ring applied first)
__global__ void correct_kernel(View u, View v, View dp, double c, int nx, int ny) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (j < ny && i <= nx) u.at(i, j) -= c * (dp.at(i, j) - dp.at(i - 1, j));
    if (j <= ny && i < nx) v.at(i, j) -= c * (dp.at(i, j) - dp.at(i, j - 1));
}

// projection.hpp:86-118 predictor
__global__ void predictor_kernel(View U, View V, View p, View ou, View ov, double dt, double nu, double invh,
                                 double invh2, bool px, bool py, int nx, int ny) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    const double half = 0.5;
    if (j < ny && i < nx && i >= (px ? 0 : 1)) {
        const double uc = U.at(i, j);
        const double uE = half * (uc + U.at(i + 1, j));
        const double uW = half * (U.at(i - 1, j) + uc);
        const double uN = half * (uc + U.at(i, j + 1));
        const double uS = half * (U.at(i, j - 1) + uc);
        const double vN = half * (V.at(i - 1, j + 1) + V.at(i, j + 1));
        const double vS = half * (V.at(i - 1, j) + V.at(i, j));
        const double adv = (uE * uE - uW * uW + uN * vN - uS * vS) * invh;
        const double lap = (U.at(i + 1, j) + U.at(i - 1, j) + U.at(i, j + 1) + U.at(i, j - 1) - 4.0 * uc) * invh2;
        const double gpx = (p.at(i, j) - p.at(i - 1, j)) * invh;
        ou.at(i, j) = uc + dt * (-adv + nu * lap - gpx);
    }
    if (j < ny && j >= (py ? 0 : 1) && i < nx) {
        const double vc = V.at(i, j);
        const double vN = half * (vc + V.at(i, j + 1));
        const double vS = half * (V.at(i, j - 1) + vc);
        const double vE = half * (vc + V.at(i + 1, j));
        const double vW = half * (V.at(i - 1, j) + vc);
        const double uE = half * (U.at(i + 1, j - 1) + U.at(i + 1, j));
        const double uW = half * (U.at(i, j - 1) + U.at(i, j));
        const double adv = (vN * vN - vS * vS + vE * uE - vW * uW) * invh;
        const double lap = (V.at(i + 1, j) + V.at(i - 1, j) + V.at(i, j + 1) + V.at(i, j - 1) - 4.0 * vc) * invh2;
        const double gpy = (p.at(i, j) - p.at(i, j - 1)) * invh;
        ov.at(i, j) = vc + dt * (-adv + nu * lap - gpy);
    }
}

__global__ void add_interior_kernel(View d, View s) {  // field.hpp:60-66
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i < d.nx) d.at(i, j) += s.at(i, j);
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
#define LAUNCH_CHECK()                  \
    do {                                \
        ISMG_CUDA(cudaGetLastError());  \
        c.launches += 1;                \
    } while (0)

void k_fill(Ctx& c, View f, double v) {
    dim3 grid((f.nx + 2 + 255) / 256, f.ny + 2);
    fill_kernel<<<grid, 256, 0, c.stream>>>(f, f.nx + 1, f.ny + 1, v);
    LAUNCH_CHECK();
}

void k_copy_field(Ctx& c, View d, View s, int w, int h) {
    dim3 grid((w + 1 + 255) / 256, h + 1);
    copy_kernel<<<grid, 256, 0, c.stream>>>(d, s, w, h);
    LAUNCH_CHECK();
}

void k_zero_ghosts(Ctx& c, View f) {
    int n = std::max(f.nx, f.ny) + 2;
    zero_ghosts_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(f);
    LAUNCH_CHECK();
}

void k_refresh_periodic(Ctx& c, View f, bool px, bool py) {
    if (!px && !py) return;
    int n = std::max(f.nx, f.ny);
    refresh_periodic_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(f, px, py);
    LAUNCH_CHECK();
}

void k_rbgs_half(Ctx& c, View x, View b, PBC bc, int color) {
    dim3 grid(((x.nx + 1) / 2 + 127) / 128, x.ny);
    rbgs_half_kernel<<<grid, 128, 0, c.stream>>>(x, b, bc, color);
    LAUNCH_CHECK();
}

void k_fine_residual(Ctx& c, View x, View b, View out, PBC bc, double* d_rmax, double* d_nan) {
    ISMG_CUDA(cudaMemsetAsync(d_rmax, 0, sizeof(double), c.stream));
    if (d_nan) ISMG_CUDA(cudaMemsetAsync(d_nan, 0, sizeof(double), c.stream));
    int nb = blocks_for(int64_t(x.nx) * x.ny, 256, 8 * c.sms);
    fine_residual_kernel<<<nb, 256, 0, c.stream>>>(x, b, out, bc, d_rmax, d_nan);
    LAUNCH_CHECK();
}

void k_mean_shift(Ctx& c, View x, double* d_out) {
    int nb = blocks_for(int64_t(x.nx) * x.ny, 256, 4 * c.sms);
    sum_partials_kernel<<<nb, 256, 0, c.stream>>>(x, c.s.part);
    LAUNCH_CHECK();
    finish_mean_kernel<<<1, 1024, 0, c.stream>>>(c.s.part, nb, double(int64_t(x.nx) * x.ny), d_out);
    LAUNCH_CHECK();
}

void k_shift_interior(Ctx& c, View x, const double* d_shift) {
    int nb = blocks_for(int64_t(x.nx) * x.ny, 256, 8 * c.sms);
    shift_kernel<<<nb, 256, 0, c.stream>>>(x, d_shift);
    LAUNCH_CHECK();
}

void k_restrict_exact(Ctx& c, View fine, View coarse, int tx, int ty, int ncx, int ncy) {
    dim3 grid((ncx + 127) / 128, ncy);
    restrict_exact_kernel<<<grid, 128, 0, c.stream>>>(fine, coarse, tx, ty, ncx, ncy);
    LAUNCH_CHECK();
}

void k_prolong_bilinear(Ctx& c, View coarse, View fine, const AxisDev& ax, const AxisDev& ay) {
    dim3 grid((fine.nx + 255) / 256, fine.ny);
    prolong_bilinear_kernel<<<grid, 256, 0, c.stream>>>(coarse, fine, ax, ay);
    LAUNCH_CHECK();
}

void k_prolong_constant(Ctx& c, View coarse, View fine, int tx, int ty) {
    dim3 grid((fine.nx + 255) / 256, fine.ny);
    prolong_constant_kernel<<<grid, 256, 0, c.stream>>>(coarse, fine, tx, ty);
    LAUNCH_CHECK();
}

void k_coarse_residual(Ctx& c, View x, View b, View out, const double* w, int ncx, int ncy, bool px, bool py,
                       int nslots, double* d_rmax) {
    ISMG_CUDA(cudaMemsetAsync(d_rmax, 0, sizeof(double), c.stream));
    int nb = blocks_for(int64_t(ncx) * ncy, 256, 4 * c.sms);
    coarse_residual_kernel<<<nb, 256, 0, c.stream>>>(x, b, out, w, ncx, ncy, px, py, nslots, d_rmax);
    LAUNCH_CHECK();
}

void k_gs_lex(Ctx& c, View x, View b, const double* w, int ncx, int ncy, bool px, bool py, int nslots) {
    gs_lex_kernel<<<1, 1024, 0, c.stream>>>(x, b, w, ncx, ncy, px, py, nslots);
    LAUNCH_CHECK();
}

void k_rbgs_op(Ctx& c, View x, View b, const double* w, int ncx, int ncy, bool px, bool py, int color) {
    const bool serial = (px && (ncx & 1)) || (py && (ncy & 1));
    dim3 grid(((ncx + 1) / 2 + 127) / 128, ncy);
    rbgs_op_kernel<<<grid, 128, 0, c.stream>>>(x, b, w, ncx, ncy, px, py, color, serial);
    LAUNCH_CHECK();
}

void k_scalar_bc(Ctx& c, View f, PBC bc) {
    scalar_bc_x_kernel<<<(f.ny + 255) / 256, 256, 0, c.stream>>>(f, bc);
    LAUNCH_CHECK();
    scalar_bc_y_kernel<<<(f.nx + 2 + 255) / 256, 256, 0, c.stream>>>(f, bc);
    LAUNCH_CHECK();
}

void k_velocity_bc(Ctx& c, Velocity& vel, const ismg_grid_spec& g) {
    VelBc bc;
    for (int s = 0; s < 4; ++s) {
        const ismg_bc& b = g.bc[s];
        bc.s[s] = BcDev{b.kind, b.inlet_start, b.inlet_width, b.u_wall, b.v_wall, b.v_inflow};
    }
    const bool per_x = g.bc[ISMG_SIDE_WEST].kind == ISMG_BC_PERIODIC;
    const bool per_y = g.bc[ISMG_SIDE_SOUTH].kind == ISMG_BC_PERIODIC;
    const int nx = g.nx, ny = g.ny, n = std::max(nx, ny) + 3;
    View u = vel.uv(), v = vel.vv();
    vel_normal_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(u, v, bc, nx, ny, per_x, per_y);
    LAUNCH_CHECK();
    vel_tangential_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(u, v, bc, nx, ny, per_x, per_y);
    LAUNCH_CHECK();
    if (per_y) {
        vel_wrap_y_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(u, v, nx, ny);
        LAUNCH_CHECK();
    }
    if (per_x) {
        vel_wrap_x_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(u, v, nx, ny);
        LAUNCH_CHECK();
    }
}

void k_divergence(Ctx& c, const Velocity& vel, View out, double invh, double scale, bool do_scale) {
    dim3 grid((out.nx + 255) / 256, out.ny);
    divergence_kernel<<<grid, 256, 0, c.stream>>>(vel.uv(), vel.vv(), out, invh, scale, do_scale);
    LAUNCH_CHECK();
}

void k_correct(Ctx& c, Velocity& vel, View dp, double cdt) {
    dim3 grid((vel.nx + 1 + 255) / 256, vel.ny + 1);
    correct_kernel<<<grid, 256, 0, c.stream>>>(vel.uv(), vel.vv(), dp, cdt, vel.nx, vel.ny);
    LAUNCH_CHECK();
}

void k_predictor(Ctx& c, const Velocity& vel, View p, double dt, double nu, double invh, double invh2, bool px,
                 bool py, Velocity& out) {
    dim3 grid((vel.nx + 255) / 256, vel.ny);
    predictor_kernel<<<grid, 256, 0, c.stream>>>(vel.uv(), vel.vv(), p, out.uv(), out.vv(), dt, nu, invh, invh2, px,
                                                 py, vel.nx, vel.ny);
    LAUNCH_CHECK();
}

void k_add_interior(Ctx& c, View d, View s) {
    dim3 grid((d.nx + 255) / 256, d.ny);
    add_interior_kernel<<<grid, 256, 0, c.stream>>>(d, s);
    LAUNCH_CHECK();
}

}  // namespace ismgb

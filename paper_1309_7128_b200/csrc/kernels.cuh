// kernels.cuh — device helpers shared by the sm_100a kernels.
//
// Arithmetic discipline: the library is compiled with
// -fmad=false so no multiply-add is contracted; every expression below keeps
// the reference's association order so op-level results are bit-identical to
// the CPU reference.
#pragma once

#include <cuda_runtime.h>

#include "common.h"

namespace ismgb {

constexpr unsigned kFull = 0xffffffffu;

// smoother.hpp:47-54: face weight of a boundary face by pressure closure.
__host__ __device__ __forceinline__ double face_weight(int k) {
    return k == ISMG_PBC_NEUMANN ? 0.0 : (k == ISMG_PBC_DIRICHLET_ZERO ? 2.0 : 1.0);
}

// smoother.hpp:55-61: d(i,j) summed W, E, S, N from 0 (integer valued).
__host__ __device__ __forceinline__ double fine_diag(const PBC& bc, int nx, int ny, int i, int j) {
    double d = 0;
    d += (i > 0) ? 1.0 : face_weight(bc.k[ISMG_SIDE_WEST]);
    d += (i < nx - 1) ? 1.0 : face_weight(bc.k[ISMG_SIDE_EAST]);
    d += (j > 0) ? 1.0 : face_weight(bc.k[ISMG_SIDE_SOUTH]);
    d += (j < ny - 1) ? 1.0 : face_weight(bc.k[ISMG_SIDE_NORTH]);
    return d;
}

// num / d for integer-valued d in 1..8. Division by a power of two equals the
// exact scaling, so those cases use a multiply (bit-identical); the others
// keep the IEEE-rounded division.
__device__ __forceinline__ double div_by_diag(double num, double d) {
    if (d == 4.0) return num * 0.25;
    if (d == 2.0) return num * 0.5;
    if (d == 8.0) return num * 0.125;
    if (d == 1.0) return num;
    return __ddiv_rn(num, d);
}

// Correctly rounded num / w with y = RN(1 / w), no DDIV sequence. Two Markstein
// corrections: q0 = RN(num y) is within 1.5 ulp of num / w; q1 = RN(q0 + RN(num -
// w q0) y) is within one ulp (the residual's rounding error is 2^-53 relative);
// by Markstein's theorem (y within half an ulp of 1/w, q1 within one ulp of
// num/w, r1 = num - w q1 exact by FMA) q2 = RN(q1 + r1 y) = RN(num / w). The
// theorem needs the residuals clear of underflow / overflow: numerators outside
// [2^-900, 2^1000] (zero and subnormal-adjacent included) and non-finite ones
// take IEEE division on a warp-uniform branch. Used by every coarse engine.
static __device__ __noinline__ double div_ieee_lanes(double num, double w, double q, bool bad) {
    return bad ? __ddiv_rn(num, w) : q;
}
__device__ __forceinline__ double div_cr(double num, double w, double y) {
    const unsigned e = unsigned(__double2hiint(num)) & 0x7ff00000u;
    const bool bad = e - (123u << 20) > (1900u << 20);
    const double q0 = __dmul_rn(num, y);
    const double e0 = __fma_rn(-q0, w, num);
    const double q1 = __fma_rn(e0, y, q0);
    const double e1 = __fma_rn(-q1, w, num);
    double q = __fma_rn(e1, y, q1);
    if (__any_sync(__activemask(), bad)) q = div_ieee_lanes(num, w, q, bad);
    return q;
}

// std::max(m, v) with the reference's NaN behaviour: a NaN v is dropped.
__device__ __forceinline__ double max_drop_nan(double m, double v) { return (m < v) ? v : m; }

// Warp reductions folding into lane 0 in a fixed order (deterministic).
__device__ __forceinline__ double warp_sum_down(double v) {
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_down_sync(kFull, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// Block reductions (blockDim.x a multiple of 32, <= 1024). Result valid in
// thread 0. `scratch` holds >= 32 doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum_down(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? scratch[lane] : 0.0;
        v = warp_sum_down(v);
    }
    return v;
}
__device__ __forceinline__ double block_max(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? scratch[lane] : 0.0;
        v = warp_max(v);
    }
    return v;
}

// Slot offsets in C,E,W,N,S,NE,NW,SE,SW order (coarsening.hpp:121-123).
__host__ __device__ constexpr int slot_di(int s) {
    return (s == 1 || s == 5 || s == 7) ? 1 : ((s == 2 || s == 6 || s == 8) ? -1 : 0);
}
__host__ __device__ constexpr int slot_dj(int s) {
    return (s == 3 || s == 5 || s == 6) ? 1 : ((s == 4 || s == 7 || s == 8) ? -1 : 0);
}

// coarsening.hpp:520-528: stored-stencil neighbour with wrap; out of range -> 0.
__device__ __forceinline__ double coarse_neighbor(const View& x, int ncx, int ncy, bool px, bool py, int I,
                                                  int J, int di, int dj) {
    int II = I + di, JJ = J + dj;
    if (px) II = (II + ncx) % ncx;
    if (py) JJ = (JJ + ncy) % ncy;
    if (II < 0 || II >= ncx || JJ < 0 || JJ >= ncy) return 0.0;
    return x.at(II, JJ);
}

}  // namespace ismgb

// coarse.cu — coarse visits of the fused hot path: lexicographic Gauss-Seidel
// on the interpolated 9-point operator until tol_coarse (cycles.hpp:120-137,
// coarsening.hpp:531-567, 592-595).
#include <cmath>

#include "fused_impl.cuh"

namespace ismgb {
namespace fz {

// ---- coarse visit: lexicographic GS to tol_coarse (cycles.hpp:120-137) ------
// One CTA. Cell (I,J) of a sweep reads new values only from cells with a
// smaller t = I + 2J and old values from larger t, so the anti-diagonal
// wavefront reproduces gs_sweep_lex bit for bit. Residual and anchor follow
// every sweep exactly as the reference orders them.
__device__ __forceinline__ void coarse_cell(const Params& P, View x, int I, int J) {
    const int64_t n = int64_t(P.ncx) * P.ncy, k = int64_t(J) * P.ncx + I;
    double s = 0;
    for (int sl = 1; sl < P.nslots; ++sl) {
        const double wg = P.w[sl * n + k];
        if (wg != 0.0) s += wg * coarse_neighbor(x, P.ncx, P.ncy, false, false, I, J, slot_di(sl), slot_dj(sl));
    }
    x.at(I, J) = (P.cb.at(I, J) - s) / P.w[k];
}

__global__ void __launch_bounds__(kCoarseThreads) coarse_visit_kernel(Params P) {
    __shared__ double red[32];
    __shared__ double bc[2];
    Ctl* s = P.ctl;
    if (s->phase != kCoarse) return;
    const int ncx = P.ncx, ncy = P.ncy;
    const int64_t n = int64_t(ncx) * ncy;
    View x = P.ce;
    // ce = 0 (ghosts included); rc = coarse_residual(ce = 0) = max|cb|
    double m = 0.0;
    for (int64_t k = threadIdx.x; k < int64_t(ncx + 2) * (ncy + 2); k += blockDim.x) {
        const int J = int(k / (ncx + 2)) - 1, I = int(k % (ncx + 2)) - 1;
        x.at(I, J) = 0.0;
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
        double ax = P.w[k] * 0.0;
        for (int sl = 1; sl < P.nslots; ++sl) {
            const double wg = P.w[sl * n + k];
            if (wg != 0.0) ax += wg * 0.0;
        }
        m = max_drop_nan(m, fabs(P.cb.at(I, J) - ax));
    }
    double rc = block_max(m, red);
    if (threadIdx.x == 0) bc[0] = rc;
    __syncthreads();
    rc = bc[0];
    const long long budget = P.max_total - s->total;
    long long sweeps = 0;
    const int tmax = (ncx - 1) + 2 * (ncy - 1);
    while (rc > P.tol_coarse && sweeps < budget) {
        for (int t = 0; t <= tmax; ++t) {
            const int jlo = max(0, (t - (ncx - 1) + 1) / 2), jhi = min(ncy - 1, t / 2);
            for (int J = jlo + int(threadIdx.x); J <= jhi; J += blockDim.x) coarse_cell(P, x, t - 2 * J, J);
            __syncthreads();
        }
        ++sweeps;
        // coarse_residual (coarsening.hpp:531-549)
        m = 0.0;
        double sum = 0.0;
        for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
            const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
            double ax = P.w[k] * x.at(I, J);
            for (int sl = 1; sl < P.nslots; ++sl) {
                const double wg = P.w[sl * n + k];
                if (wg != 0.0) ax += wg * coarse_neighbor(x, ncx, ncy, false, false, I, J, slot_di(sl), slot_dj(sl));
            }
            m = max_drop_nan(m, fabs(P.cb.at(I, J) - ax));
            sum += x.at(I, J);
        }
        rc = block_max(m, red);
        if (threadIdx.x == 0) bc[0] = rc;
        __syncthreads();
        rc = bc[0];
        if (P.singular) {  // anchor_mean(op, ce) coarsening.hpp:592-595
            sum = block_sum(sum, red);
            if (threadIdx.x == 0) bc[1] = -(sum / double(n));
            __syncthreads();
            const double cs = bc[1];
            for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
                const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
                x.at(I, J) += cs;
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        s->coarse_launches += 1;
        s->total += sweeps;
        s->coarse += sweeps;
        s->rc = rc;
        if (s->nvisits > 0 && s->nvisits <= P.visit_cap) P.visit_log[2 * (s->nvisits - 1)] = int(sweeps);
        if (rc > P.tol_coarse) {  // cycles.hpp:134-137
            s->phase = kDone, s->converged = 0;
        } else if (sweeps > 0) {
            s->phase = kProlong;
        } else {
            s->prev = s->r;
            s->phase = kFine;
        }
    }
}

// ---- pipelined coarse visit: the coarse iterate lives in shared memory -------
// Sweep s of cell (I,J) runs at wavefront step tau = I + 2J + 8s. Within one
// sweep the order is the lexicographic one (see coarse_visit_kernel); across
// sweeps, sweep s+1 reads sweep-s values of (I+1,J), (I-1,J+1), (I,J+1),
// (I+1,J+1), all written at steps <= tau - 5, and none of them is overwritten
// by sweep s+2 before tau + 3. The residual of (I,J) after sweep s is formed at
// step tau + 4: every neighbour then holds its sweep-s value (the last, NE,
// written at tau + 3; sweep s+1 reaches the first neighbour, SW, at tau + 5),
// so update and residual share one barrier per step. Sweeps run in groups
// with a checkpoint; when a group overshoots the first sweep whose residual
// passes tol_coarse, the iterate is restored and replayed exactly that far.
// Singular operators anchor once at the end of the visit (the sweeps commute
// with a constant shift).
constexpr int kLag = 8;
constexpr int kMaxGroup = 128;

struct CoarseSmem {
    unsigned long long rmax[kMaxGroup];
    double red[32];
    double bcast[4];
    int ictl[4];
};

__device__ __forceinline__ double cx(const double* xs, int ld, int I, int J) { return xs[(J + 1) * ld + (I + 1)]; }

// one coarse cell update, reference order (coarsening.hpp:557-565)
__device__ __forceinline__ double coarse_update(const Params& P, const double* xs, int ld, int I, int J,
                                                double bIJ) {
    const int64_t n = int64_t(P.ncx) * P.ncy, k = int64_t(J) * P.ncx + I;
    double s = 0;
    for (int sl = 1; sl < P.nslots; ++sl) {
        const double wg = __ldg(&P.w[sl * n + k]);
        if (wg != 0.0) s += wg * cx(xs, ld, I + slot_di(sl), J + slot_dj(sl));
    }
    return (bIJ - s) / __ldg(&P.w[k]);
}

__device__ __forceinline__ double coarse_res(const Params& P, const double* xs, int ld, int I, int J, double bIJ) {
    const int64_t n = int64_t(P.ncx) * P.ncy, k = int64_t(J) * P.ncx + I;
    double ax = __ldg(&P.w[k]) * cx(xs, ld, I, J);
    for (int sl = 1; sl < P.nslots; ++sl) {
        const double wg = __ldg(&P.w[sl * n + k]);
        if (wg != 0.0) ax += wg * cx(xs, ld, I + slot_di(sl), J + slot_dj(sl));
    }
    return bIJ - ax;
}

// Run sweeps [0, G) of a group on the shared-memory iterate. With residuals,
// rmax[g] receives max|r| after sweep g (NaN dropped).
__device__ void coarse_group(const Params& P, double* xs, int ld, CoarseSmem& cs, int G, bool residuals) {
    const int ncx = P.ncx, ncy = P.ncy, dmax = (ncx - 1) + 2 * (ncy - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    if (residuals)
        for (int g = threadIdx.x; g < G; g += blockDim.x) cs.rmax[g] = 0ull;
    __syncthreads();
    const int tau_end = dmax + kLag * (G - 1) + (residuals ? 4 : 0);
    for (int tau = 0; tau <= tau_end; ++tau) {
        for (int phase = 0; phase < (residuals ? 2 : 1); ++phase) {
            const int base = phase == 0 ? tau : tau - 4;
            if (base < 0) continue;
            // sweeps with diagonal d = base - 8g in [0, dmax]
            const int g_lo = max(0, (base - dmax + kLag - 1) / kLag), g_hi = min(G - 1, base / kLag);
            for (int g = g_lo + warp; g <= g_hi; g += nwarps) {
                const int d = base - kLag * g;
                const int jlo = max(0, (d - (ncx - 1) + 1) / 2), jhi = min(ncy - 1, d / 2);
                double m = 0.0;
                for (int J = jlo + lane; J <= jhi; J += 32) {
                    {
                        const int I = d - 2 * J;
                        const double bIJ = P.cb.at(I, J);
                        if (phase == 0) {
                            xs[(J + 1) * ld + (I + 1)] = coarse_update(P, xs, ld, I, J, bIJ);
                        } else {
                            m = max_drop_nan(m, fabs(coarse_res(P, xs, ld, I, J, bIJ)));
                        }
                    }
                }
                if (phase == 1) {
                    m = warp_max(m);
                    if (lane == 0) atomicMax(&cs.rmax[g], (unsigned long long)__double_as_longlong(m));
                }
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kCoarseSmemThreads) coarse_visit_smem_kernel(Params P, double* backup) {
    extern __shared__ __align__(16) double xs[];
    __shared__ CoarseSmem cs;
    Ctl* s = P.ctl;
    if (s->phase != kCoarse) return;
    const int ncx = P.ncx, ncy = P.ncy, ld = ncx + 2;
    const int64_t n = int64_t(ncx) * ncy, ntot = int64_t(ld) * (ncy + 2);
    for (int64_t k = threadIdx.x; k < ntot; k += blockDim.x) xs[k] = 0.0;  // ce = 0, zero ghost ring
    // rc = coarse_residual(ce = 0) = max|cb| (exactly: b - (+-0) == b)
    double m = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
        m = max_drop_nan(m, fabs(P.cb.at(I, J)));
    }
    m = block_max(m, cs.red);
    if (threadIdx.x == 0) cs.bcast[0] = m;
    __syncthreads();
    double rc = cs.bcast[0];
    const long long budget = P.max_total - s->total;
    long long done = 0;
    int G = 1;
    while (rc > P.tol_coarse && done < budget) {
        if (budget - done < G) G = int(budget - done);
        for (int64_t k = threadIdx.x; k < ntot; k += blockDim.x) backup[k] = xs[k];  // checkpoint
        coarse_group(P, xs, ld, cs, G, true);
        if (threadIdx.x == 0) {
            int first = -1;
            for (int g = 0; g < G; ++g)
                if (!(__longlong_as_double((long long)cs.rmax[g]) > P.tol_coarse)) {
                    first = g;
                    break;
                }
            cs.ictl[0] = first;
            cs.bcast[1] = __longlong_as_double((long long)cs.rmax[first >= 0 ? first : G - 1]);
        }
        __syncthreads();
        const int first = cs.ictl[0];
        rc = cs.bcast[1];
        if (first >= 0 && first < G - 1) {  // overshoot: restore and replay first+1 sweeps
            for (int64_t k = threadIdx.x; k < ntot; k += blockDim.x) xs[k] = backup[k];
            __syncthreads();
            coarse_group(P, xs, ld, cs, first + 1, false);
            done += first + 1;
            break;
        }
        done += G;
        if (first >= 0) break;
        G = min(2 * G, kMaxGroup);
    }
    if (P.singular && done > 0) {  // anchor_mean(op, ce) of the visit's result
        double sum = 0.0;
        for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
            const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
            sum += xs[(J + 1) * ld + (I + 1)];
        }
        sum = block_sum(sum, cs.red);
        if (threadIdx.x == 0) cs.bcast[2] = -(sum / double(n));
        __syncthreads();
        const double c = cs.bcast[2];
        for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
            const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
            xs[(J + 1) * ld + (I + 1)] += c;
        }
        __syncthreads();
    }
    for (int64_t k = threadIdx.x; k < ntot; k += blockDim.x) {  // ce for the prolongation
        const int J = int(k / ld) - 1, I = int(k % ld) - 1;
        P.ce.at(I, J) = xs[k];
    }
    if (threadIdx.x == 0) {
        s->coarse_launches += 1;
        s->total += done;
        s->coarse += done;
        s->rc = rc;
        if (s->nvisits > 0 && s->nvisits <= P.visit_cap) P.visit_log[2 * (s->nvisits - 1)] = int(done);
        if (rc > P.tol_coarse) {  // cycles.hpp:134-137
            s->phase = kDone, s->converged = 0;
        } else if (done > 0) {
            s->phase = kProlong;
        } else {
            s->prev = s->r;
            s->phase = kFine;
        }
    }
}


// ---- TMEM-resident coarse visit (coarse grids up to 256 x 128) --------------
// Same pipelined schedule as coarse_visit_smem_kernel, laid out for the SM:
//  * lane l of warp w owns coarse row J = 32 (w % 4) + l; the kTmH warps that
//    share a row quadrant split the in-flight sweeps (g = h mod kTmH);
//  * the iterate sits in shared memory in diagonal coordinates,
//    xs[J][(I + 2J + 4) mod PP] with PP = 1 (mod 16): the cells a warp touches
//    at one wavefront step share the diagonal I + 2J, so the 32 lanes hit 32
//    distinct bank pairs, and the zero slots of each row are its ghost cells;
//  * the coarse rhs lives in Tensor Memory: TMEM lane J holds b(I, J) at
//    column pair 2 ((I + 2J) mod 256), so every tcgen05.ld of a wavefront step
//    reads one warp-uniform column;
//  * interior rows use the operator's interior stencil held in registers, the
//    boundary ring reads its nine coefficients from a shared-memory table.
constexpr int kTmH = 4;
constexpr int kTmThreads = 128 * kTmH;

struct TmSmem {
    unsigned long long rmax[kMaxGroup];
    double red[32];
    double bcast[4];
    int ictl[4];
    uint32_t tmem_base;
};

__device__ __forceinline__ void tm_ld2(uint32_t taddr, uint32_t& lo, uint32_t& hi) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(taddr));
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, uint32_t lo, uint32_t hi) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(lo), "r"(hi));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ int wrapP(int s, int PP) { return s >= PP ? s - PP : (s < 0 ? s + PP : s); }

// ring index of a boundary cell (rows 0 / ncy-1 first, then columns 0 / ncx-1)
__device__ __forceinline__ int ring_index(const TmGeom& T, int I, int J) {
    if (J == 0) return I;
    if (J == T.ncy - 1) return T.ncx + I;
    if (I == 0) return 2 * T.ncx + J;
    return 2 * T.ncx + T.ncy + J;
}

// Update (or residual) of cell (I, J) whose diagonal slot in row J is sc.
template <bool kResidual>
__device__ __forceinline__ double tm_cell(const TmGeom& T, const double* xs, const double* spec, int I, int J,
                                          int sc, double bIJ) {
    const double* rowC = xs + (J + 1) * T.PP;
    const double* rowN = rowC + T.PP;
    const double* rowS = rowC - T.PP;
    const bool special = (I == 0) | (I == T.ncx - 1) | (J == 0) | (J == T.ncy - 1);
    const int ri = special ? ring_index(T, I, J) : 0;
    auto W = [&](int sl) { return special ? spec[sl * T.ring + ri] : T.stdw[sl]; };
    // neighbour (I + di, J + dj) sits in row J + dj at slot sc + di + 2 dj
    double acc = kResidual ? W(0) * rowC[sc] : 0.0;
    double wg;
    wg = W(1);
    if (wg != 0.0) acc += wg * rowC[wrapP(sc + 1, T.PP)];  // E
    wg = W(2);
    if (wg != 0.0) acc += wg * rowC[wrapP(sc - 1, T.PP)];  // W
    wg = W(3);
    if (wg != 0.0) acc += wg * rowN[wrapP(sc + 2, T.PP)];  // N
    wg = W(4);
    if (wg != 0.0) acc += wg * rowS[wrapP(sc - 2, T.PP)];  // S
    if (!T.five) {
        wg = W(5);
        if (wg != 0.0) acc += wg * rowN[wrapP(sc + 3, T.PP)];  // NE
        wg = W(6);
        if (wg != 0.0) acc += wg * rowN[wrapP(sc + 1, T.PP)];  // NW
        wg = W(7);
        if (wg != 0.0) acc += wg * rowS[wrapP(sc - 1, T.PP)];  // SE
        wg = W(8);
        if (wg != 0.0) acc += wg * rowS[wrapP(sc - 3, T.PP)];  // SW
    }
    return kResidual ? bIJ - acc : (bIJ - acc) / W(0);
}

__device__ void tm_group(const Params& P, const TmGeom& T, double* xs, const double* spec, uint32_t tq,
                         TmSmem& cs, int G, bool residuals) {
    const int dmax = (T.ncx - 1) + 2 * (T.ncy - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, h = warp >> 2;
    const int J = 32 * q + lane;
    const bool rowok = J < T.ncy;
    if (residuals)
        for (int g = threadIdx.x; g < G; g += blockDim.x) cs.rmax[g] = 0ull;
    __syncthreads();
    const int tau_end = dmax + kLag * (G - 1) + (residuals ? 4 : 0);
    for (int tau = 0; tau <= tau_end; ++tau) {
        for (int phase = 0; phase < (residuals ? 2 : 1); ++phase) {
            const int base = phase == 0 ? tau : tau - 4;
            if (base < 0) continue;
            const int g_lo = max(0, (base - dmax + kLag - 1) / kLag), g_hi = min(G - 1, base / kLag);
            const int g0 = g_lo + (((h - g_lo) % kTmH) + kTmH) % kTmH;
            for (int g = g0; g <= g_hi; g += kTmH) {
                const int d = base - kLag * g;
                uint32_t lo, hi;
                tm_ld2(tq + 2u * uint32_t(d & 255), lo, hi);
                tm_wait_ld();
                const double bIJ = __hiloint2double(int(hi), int(lo));
                const int I = d - 2 * J;
                const bool ok = rowok && I >= 0 && I < T.ncx;
                const int sc = (d + 4) % T.PP;
                if (phase == 0) {
                    if (ok) xs[(J + 1) * T.PP + sc] = tm_cell<false>(T, xs, spec, I, J, sc, bIJ);
                } else {
                    double m = ok ? fabs(tm_cell<true>(T, xs, spec, I, J, sc, bIJ)) : 0.0;
                    if (m != m) m = 0.0;
                    m = warp_max(m);
                    if (lane == 0) atomicMax(&cs.rmax[g], (unsigned long long)__double_as_longlong(m));
                }
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kTmThreads) coarse_visit_tmem_kernel(Params P, TmGeom T, const double* spec_g,
                                                                        double* backup) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ TmSmem cs;
    Ctl* s = P.ctl;
    if (s->phase != kCoarse) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, h = warp >> 2;
    const int J = 32 * q + lane;
    const bool rowok = J < T.ncy;
    const int nxs = (T.ncy + 2) * T.PP;
    double* xs = dyn;
    double* spec = dyn + nxs;
    // TMEM: 512 columns = 256 fp64 diagonal slots per lane (row)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            uint32_t(__cvta_generic_to_shared(&cs.tmem_base))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int k = threadIdx.x; k < nxs; k += blockDim.x) xs[k] = 0.0;  // ce = 0 with zero ghost slots
    for (int k = threadIdx.x; k < 9 * T.ring; k += blockDim.x) spec[k] = spec_g[k];
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tq = cs.tmem_base + (uint32_t(32 * q) << 16);
    // b -> TMEM (warps of a quadrant split the 256 slots); rc = max|cb|
    double m = 0.0;
    for (int slot = h; slot < 256; slot += kTmH) {
        const int I = (slot - 2 * J) & 255;
        double v = 0.0;
        if (rowok && I < T.ncx) {
            v = P.cb.at(I, J);
            m = max_drop_nan(m, fabs(v));
        }
        tm_st2(tq + 2u * uint32_t(slot), uint32_t(__double2loint(v)), uint32_t(__double2hiint(v)));
    }
    tm_wait_st();
    tm_fence_before();
    m = block_max(m, cs.red);
    if (threadIdx.x == 0) cs.bcast[0] = m;
    __syncthreads();
    tm_fence_after();
    double rc = cs.bcast[0];
    const long long budget = P.max_total - s->total;
    long long done = 0;
    int G = 1;
    while (rc > P.tol_coarse && done < budget) {
        if (budget - done < G) G = int(budget - done);
        if (G > 1)
            for (int k = threadIdx.x; k < nxs; k += blockDim.x) backup[k] = xs[k];  // checkpoint
        tm_group(P, T, xs, spec, tq, cs, G, true);
        if (threadIdx.x == 0) {
            int first = -1;
            for (int g = 0; g < G; ++g)
                if (!(__longlong_as_double((long long)cs.rmax[g]) > P.tol_coarse)) {
                    first = g;
                    break;
                }
            cs.ictl[0] = first;
            cs.bcast[1] = __longlong_as_double((long long)cs.rmax[first >= 0 ? first : G - 1]);
        }
        __syncthreads();
        const int first = cs.ictl[0];
        rc = cs.bcast[1];
        if (first >= 0 && first < G - 1) {  // overshoot: restore and replay first+1 sweeps
            for (int k = threadIdx.x; k < nxs; k += blockDim.x) xs[k] = backup[k];
            __syncthreads();
            tm_group(P, T, xs, spec, tq, cs, first + 1, false);
            done += first + 1;
            break;
        }
        done += G;
        if (first >= 0) break;
        G = min(2 * G, kMaxGroup);
    }
    // anchor once (singular) and hand ce to the prolongation, row J by its owner
    if (P.singular && done > 0) {
        double sum = 0.0;
        if (rowok && h == 0)
            for (int I = 0; I < T.ncx; ++I) sum += xs[(J + 1) * T.PP + (I + 2 * J + 4) % T.PP];
        sum = block_sum(sum, cs.red);
        if (threadIdx.x == 0) cs.bcast[2] = -(sum / double(int64_t(T.ncx) * T.ncy));
        __syncthreads();
        const double c = cs.bcast[2];
        if (rowok && h == 0)
            for (int I = 0; I < T.ncx; ++I) xs[(J + 1) * T.PP + (I + 2 * J + 4) % T.PP] += c;
    }
    if (rowok && h == 0)
        for (int I = 0; I < T.ncx; ++I) P.ce.at(I, J) = xs[(J + 1) * T.PP + (I + 2 * J + 4) % T.PP];
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(cs.tmem_base));
    if (threadIdx.x == 0) {
        s->coarse_launches += 1;
        s->total += done;
        s->coarse += done;
        s->rc = rc;
        if (s->nvisits > 0 && s->nvisits <= P.visit_cap) P.visit_log[2 * (s->nvisits - 1)] = int(done);
        if (rc > P.tol_coarse) {
            s->phase = kDone, s->converged = 0;
        } else if (done > 0) {
            s->phase = kProlong;
        } else {
            s->prev = s->r;
            s->phase = kFine;
        }
    }
}

// Host: can the TMEM kernel run this operator? (interior rows all equal the
// interior stencil; only the boundary ring is special.) Fills geometry + table.
bool tmem_coarse_plan(const CoarseOpH& op, TmGeom& T, std::vector<double>& spec, size_t& smem) {
    if (op.px || op.py || op.ncx > 256 || op.ncy > 128 || op.ncx < 3 || op.ncy < 3) return false;
    T.ncx = op.ncx, T.ncy = op.ncy, T.five = op.five_point;
    T.PP = ((op.ncx + 2 + 14) / 16) * 16 + 1;
    T.ring = 2 * op.ncx + 2 * op.ncy;
    for (int sl = 0; sl < 9; ++sl) T.stdw[sl] = op.at(sl, 1, 1);
    for (int J = 1; J < op.ncy - 1; ++J)
        for (int I = 1; I < op.ncx - 1; ++I)
            for (int sl = 0; sl < 9; ++sl)
                if (!(op.at(sl, I, J) == T.stdw[sl]) || std::signbit(op.at(sl, I, J)) != std::signbit(T.stdw[sl]))
                    return false;
    if (T.stdw[0] == 0.0) return false;
    spec.assign(size_t(9) * T.ring, 0.0);
    auto put = [&](int r, int I, int J) {
        for (int sl = 0; sl < 9; ++sl) spec[size_t(sl) * T.ring + r] = op.at(sl, I, J);
    };
    for (int I = 0; I < op.ncx; ++I) put(I, I, 0), put(op.ncx + I, I, op.ncy - 1);
    for (int J = 0; J < op.ncy; ++J) put(2 * op.ncx + J, 0, J), put(2 * op.ncx + op.ncy + J, op.ncx - 1, J);
    for (size_t r = 0; r < size_t(T.ring); ++r)
        if (spec[r] == 0.0) return false;  // singular ring row: op-level path raises
    smem = (size_t(op.ncy + 2) * T.PP + size_t(9) * T.ring) * sizeof(double);
    return smem <= 200 * 1024;
}

void launch_coarse_tmem(const Params& P, const TmGeom& T, const double* spec, double* backup, size_t smem,
                        cudaStream_t st) {
    coarse_visit_tmem_kernel<<<1, kTmThreads, smem, st>>>(P, T, spec, backup);
}
void set_coarse_tmem_smem(size_t bytes) {
    ISMG_CUDA(cudaFuncSetAttribute(coarse_visit_tmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

void launch_coarse_global(const Params& P, cudaStream_t st) { coarse_visit_kernel<<<1, kCoarseThreads, 0, st>>>(P); }
void launch_coarse_smem(const Params& P, double* backup, size_t smem, cudaStream_t st) {
    coarse_visit_smem_kernel<<<1, kCoarseSmemThreads, smem, st>>>(P, backup);
}
void set_coarse_smem(size_t bytes) {
    ISMG_CUDA(cudaFuncSetAttribute(coarse_visit_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

}  // namespace fz
}  // namespace ismgb

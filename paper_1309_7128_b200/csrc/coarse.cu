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
        publish_phase(P, s->phase);
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
        publish_phase(P, s->phase);
    }
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

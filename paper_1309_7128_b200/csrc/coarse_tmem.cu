// coarse_tmem.cu — TMEM-resident coarse visit (coarse grids up to 256 x 128).
//
// Same pipelined schedule as coarse_visit_smem_kernel (coarse.cu: sweep s of
// cell (I,J) at wavefront step tau = I + 2J + 8s, residual of sweep s at tau+4,
// one CTA barrier per step, grouped sweeps with checkpoint/replay), laid out
// for one SM:
//  * lane l of warp w owns coarse row J = 32 (w % 4) + l (the TMEM lane
//    quadrant of the warp); the kTmH warps sharing a quadrant split the
//    in-flight sweeps g = h (mod kTmH);
//  * the iterate sits in shared memory in diagonal coordinates: cell (I,J) at
//    slot (I + 2J + 4) mod PP of row J. The cells a warp touches at one step
//    share the diagonal I + 2J, so with a row pitch = 1 (mod 16) doubles the 32
//    lanes hit 32 distinct bank pairs; the 3 slots at each end of a row are
//    mirrored so neighbour slots never wrap; unused slots are the zero ghosts;
//  * the coarse rhs lives in Tensor Memory: TMEM lane J holds b(I, J) at the
//    column pair of slot (I + 2J) mod 256, so every tcgen05.ld of a step reads
//    one warp-uniform column;
//  * the interior stencil is a compile-time constant when the operator's
//    interior rows are the ISMG (-3; 1/2; 1/4) or five-point (-4; 1) stencil bit
//    for bit; boundary-ring cells take a divergent path with their nine
//    coefficients from shared memory.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "fused_impl.cuh"

namespace ismgb {
namespace fz {

namespace {

constexpr int kLagT = 8;         // wavefront steps between consecutive sweeps
constexpr int kMaxGroupT = 512;  // sweeps per checkpointed group
constexpr int kTmH = 8;          // warps per TMEM lane quadrant
constexpr int kTmU = 2;          // cells per warp-iteration
constexpr int kPredCap = 32;     // cap of the predicted first group of a visit
constexpr int kTmThreads = 128 * kTmH;

struct TmSmem {
    double wmax[4][kMaxGroupT];  // residual max per (quadrant, sweep of the group)
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

__device__ __forceinline__ int ring_index(const TmGeom& T, int I, int J) {
    if (J == 0) return I;
    if (J == T.ncy - 1) return T.ncx + I;
    if (I == 0) return 2 * T.ncx + J;
    return 2 * T.ncx + T.ncy + J;
}

// slot 0 of coarse row J (J in [-1, ncy])
__device__ __forceinline__ double* row_ptr(double* xs, const TmGeom& T, int J) { return xs + (J + 1) * T.pitch + 3; }

// The neighbour values of the cell at slot s of row pointer rc.
struct Nbr {
    double c, e, w, n, s, ne, nw, se, sw;
};
__device__ __forceinline__ Nbr gather(const double* rc, int pitch, int s, bool with_c, bool five) {
    const double* rn = rc + pitch;
    const double* rs = rc - pitch;
    Nbr v;
    v.c = with_c ? rc[s] : 0.0;
    v.e = rc[s + 1];
    v.w = rc[s - 1];
    v.n = rn[s + 2];
    v.s = rs[s - 2];
    if (!five) {
        v.ne = rn[s + 3];
        v.nw = rn[s + 1];
        v.se = rs[s - 1];
        v.sw = rs[s - 3];
    } else {
        v.ne = v.nw = v.se = v.sw = 0.0;
    }
    return v;
}

// Reference order (coarsening.hpp:539-543 residual, :558-565 update): slots
// E, W, N, S, NE, NW, SE, SW, each skipped when its weight is zero.
template <bool kResidual>
__device__ __forceinline__ double apply_w(const double* w, const Nbr& v, double bIJ, bool five) {
    double acc = kResidual ? w[0] * v.c : 0.0;
    if (w[1] != 0.0) acc += w[1] * v.e;
    if (w[2] != 0.0) acc += w[2] * v.w;
    if (w[3] != 0.0) acc += w[3] * v.n;
    if (w[4] != 0.0) acc += w[4] * v.s;
    if (!five) {
        if (w[5] != 0.0) acc += w[5] * v.ne;
        if (w[6] != 0.0) acc += w[6] * v.nw;
        if (w[7] != 0.0) acc += w[7] * v.se;
        if (w[8] != 0.0) acc += w[8] * v.sw;
    }
    return kResidual ? bIJ - acc : (bIJ - acc) / w[0];
}

// a / -3 correctly rounded, without the DDIV sequence (~115-cycle latency):
// div_cr (kernels.cuh), two Markstein corrections with y = RN(-1/3).
__device__ __forceinline__ double div_m3(double a) {
    constexpr double y = -1.0 / 3.0;
    return div_cr(a, -3.0, y);
}

// Compile-time interior stencils (host-verified against the built operator).
template <bool kResidual, int Kind>
__device__ __forceinline__ double apply_std(const TmGeom& T, const Nbr& v, double bIJ) {
    if constexpr (Kind == 1) {  // ISMG interior row: C -3, E/W/N/S 1/2, corners 1/4
        double acc = kResidual ? -3.0 * v.c : 0.0;
        acc += 0.5 * v.e;
        acc += 0.5 * v.w;
        acc += 0.5 * v.n;
        acc += 0.5 * v.s;
        acc += 0.25 * v.ne;
        acc += 0.25 * v.nw;
        acc += 0.25 * v.se;
        acc += 0.25 * v.sw;
        return kResidual ? bIJ - acc : div_m3(bIJ - acc);
    } else if constexpr (Kind == 2) {  // five-point interior row: C -4, E/W/N/S 1
        double acc = kResidual ? -4.0 * v.c : 0.0;
        acc += 1.0 * v.e;
        acc += 1.0 * v.w;
        acc += 1.0 * v.n;
        acc += 1.0 * v.s;
        return kResidual ? bIJ - acc : (bIJ - acc) * -0.25;  // exact: power-of-two divisor
    } else {
        return apply_w<kResidual>(T.stdw, v, bIJ, T.five);
    }
}

template <bool kResidual, int Kind>
__device__ __forceinline__ double tm_cell(const TmGeom& T, const double* rc, const double* spec, int I, int J, int s,
                                          double bIJ) {
    const Nbr v = gather(rc, T.pitch, s, kResidual, T.five);
    const bool special = (I == 0) | (I == T.ncx - 1) | (J == 0) | (J == T.ncy - 1);
    if (!special) return apply_std<kResidual, Kind>(T, v, bIJ);
    // boundary ring: stencil class table, 9 weights + RN(1/w0) per class
    const int* ring_cls = reinterpret_cast<const int*>(spec + 10 * T.ncls);
    const double* wc = spec + 10 * ring_cls[ring_index(T, I, J)];
    double w[9];
#pragma unroll
    for (int sl = 0; sl < 9; ++sl) w[sl] = wc[sl];
    if (kResidual) return apply_w<true>(w, v, bIJ, T.five);
    double acc = 0.0;  // update: coarsening.hpp:558-565
    if (w[1] != 0.0) acc += w[1] * v.e;
    if (w[2] != 0.0) acc += w[2] * v.w;
    if (w[3] != 0.0) acc += w[3] * v.n;
    if (w[4] != 0.0) acc += w[4] * v.s;
    if (!T.five) {
        if (w[5] != 0.0) acc += w[5] * v.ne;
        if (w[6] != 0.0) acc += w[6] * v.nw;
        if (w[7] != 0.0) acc += w[7] * v.se;
        if (w[8] != 0.0) acc += w[8] * v.sw;
    }
    const double num = bIJ - acc;
    if (!T.fastdiv) return num / w[0];
    return div_cr(num, w[0], wc[9]);  // correctly rounded (kernels.cuh)
}

// max over the warp of non-negative doubles through two 32-bit REDUX steps
// (ordering of non-negative doubles = ordering of their (hi, lo) words)
__device__ __forceinline__ double warp_max_nonneg(double m) {
    const unsigned hi = unsigned(__double2hiint(m)), lo = unsigned(__double2loint(m));
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    return __hiloint2double(int(mh), int(ml));
}

// U independent cells per warp-iteration: the cells one warp handles at one
// step lie on diagonals 8 kTmH apart, so none reads another's slot; their
// TMEM loads, gathers, arithmetic and stores are issued as batches and the
// fp64 dependency chains overlap.
template <int Kind, int U>
__device__ void tm_group(const TmGeom& T, double* xs, const double* spec, uint32_t tq, TmSmem& cs, int G,
                         bool residuals) {
    const int dmax = (T.ncx - 1) + 2 * (T.ncy - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, h = warp >> 2;
    const int J = 32 * q + lane;
    const bool rowok = J < T.ncy;
    double* rc = row_ptr(xs, T, J);
    const int PP = T.PP;
    const int jmin = 32 * q, jmax = min(32 * q + 31, T.ncy - 1);
    const int dlo = 2 * jmin, dhi = min(dmax, 2 * jmax + T.ncx - 1);
    if (residuals)
        for (int k = threadIdx.x; k < 4 * kMaxGroupT; k += blockDim.x) (&cs.wmax[0][0])[k] = 0.0;
    __syncthreads();
    const int tau_end = dmax + kLagT * (G - 1) + (residuals ? 4 : 0);
    constexpr int kStride = kLagT * kTmH;  // diagonal distance of consecutive cells of one warp
    for (int tau = 0; tau <= tau_end; ++tau) {
        if (jmin < T.ncy) {
            for (int phase = 0; phase < (residuals ? 2 : 1); ++phase) {
                const int base = phase == 0 ? tau : tau - 4;
                if (base < dlo) continue;
                const int g_lo = max(0, (base - dhi + kLagT - 1) / kLagT), g_hi = min(G - 1, (base - dlo) / kLagT);
                const int g0 = g_lo + (((h - g_lo) % kTmH) + kTmH) % kTmH;
                if (g0 > g_hi) continue;
                const int d0 = base - kLagT * g0;
                int s0 = (d0 + 4) % PP;
                for (int gb = g0; gb <= g_hi; gb += U * kTmH) {
                    uint32_t lo[U], hi[U];
                    int I[U], s[U];
                    bool ok[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int g = gb + u * kTmH;
                        const int d = base - kLagT * g;
                        s[u] = s0;
                        s0 -= kStride;
                        s0 += s0 < 0 ? PP : 0;  // kStride < PP (plan)
                        I[u] = d - 2 * J;
                        ok[u] = (g <= g_hi) && rowok && I[u] >= 0 && I[u] < T.ncx;
                        if (g <= g_hi) tm_ld2(tq + 2u * uint32_t(d & 255), lo[u], hi[u]);  // warp-uniform
                    }
                    tm_wait_ld();
                    double out[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const double bIJ = __hiloint2double(int(hi[u]), int(lo[u]));
                        out[u] = 0.0;
                        if (ok[u]) {
                            out[u] = phase == 0 ? tm_cell<false, Kind>(T, rc, spec, I[u], J, s[u], bIJ)
                                                : tm_cell<true, Kind>(T, rc, spec, I[u], J, s[u], bIJ);
                        }
                    }
                    if (phase == 0) {
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (ok[u]) {
                                const int su = s[u];
                                rc[su] = out[u];
                                if (su < 3) rc[su + PP] = out[u];  // mirrored end slots
                                if (su >= PP - 3) rc[su - PP] = out[u];
                            }
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int g = gb + u * kTmH;
                            if (g > g_hi) break;
                            double m = fabs(out[u]);
                            m = (m != m) ? 0.0 : m;  // std::max drops NaN
                            m = warp_max_nonneg(m);
                            // (q, g) belongs to this warp alone: accumulate over steps
                            if (lane == 0) cs.wmax[q][g] = fmax(cs.wmax[q][g], m);
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
}

template <int Kind>
__device__ void tm_group_v1(const TmGeom& T, double* xs, const double* spec, uint32_t tq, TmSmem& cs, int G,
                            bool residuals) {
    const int dmax = (T.ncx - 1) + 2 * (T.ncy - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, h = warp >> 2;
    const int J = 32 * q + lane;
    const bool rowok = J < T.ncy;
    double* rc = row_ptr(xs, T, J);
    const int PP = T.PP;
    // diagonals that cross this quadrant's rows
    const int jmin = 32 * q, jmax = min(32 * q + 31, T.ncy - 1);
    const int dlo = 2 * jmin, dhi = min(dmax, 2 * jmax + T.ncx - 1);
    if (residuals)
        for (int k = threadIdx.x; k < 4 * kMaxGroupT; k += blockDim.x) (&cs.wmax[0][0])[k] = 0.0;
    __syncthreads();
    const int tau_end = dmax + kLagT * (G - 1) + (residuals ? 4 : 0);
    for (int tau = 0; tau <= tau_end; ++tau) {
        if (jmin < T.ncy) {
            for (int phase = 0; phase < (residuals ? 2 : 1); ++phase) {
                const int base = phase == 0 ? tau : tau - 4;
                if (base < dlo) continue;
                const int g_lo = max(0, (base - dhi + kLagT - 1) / kLagT), g_hi = min(G - 1, (base - dlo) / kLagT);
                const int g0 = g_lo + (((h - g_lo) % kTmH) + kTmH) % kTmH;
                if (g0 > g_hi) continue;
                int d = base - kLagT * g0;
                int s = (d + 4) % PP;  // warp-uniform slot of diagonal d
                for (int g = g0; g <= g_hi; g += kTmH) {
                    uint32_t lo, hi;
                    tm_ld2(tq + 2u * uint32_t(d & 255), lo, hi);
                    const int I = d - 2 * J;
                    const bool ok = rowok && I >= 0 && I < T.ncx;
                    tm_wait_ld();
                    const double bIJ = __hiloint2double(int(hi), int(lo));
                    if (phase == 0) {
                        if (ok) {
                            const double v = tm_cell<false, Kind>(T, rc, spec, I, J, s, bIJ);
                            rc[s] = v;
                            if (s < 3) rc[s + PP] = v;  // mirrored end slots
                            if (s >= PP - 3) rc[s - PP] = v;
                        }
                    } else {
                        double m = ok ? fabs(tm_cell<true, Kind>(T, rc, spec, I, J, s, bIJ)) : 0.0;
                        m = warp_max(m);  // fmax: NaN dropped as std::max does
                        // (q, g) belongs to this warp alone: accumulate over steps
                        if (lane == 0) cs.wmax[q][g] = fmax(cs.wmax[q][g], m);
                    }
                    d -= kLagT * kTmH;
                    s -= kLagT * kTmH;
                    while (s < 0) s += PP;
                }
            }
        }
        __syncthreads();
    }
}

template <int Kind>
__global__ void __launch_bounds__(kTmThreads) coarse_visit_tmem_kernel(Params P, TmGeom T, const double* spec_g,
                                                                        double* backup) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ TmSmem cs;
    Ctl* st = P.ctl;
    if (st->phase != kCoarse) return;
    const long long t_start = gtimer();
    long long steps = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, h = warp >> 2;
    const int J = 32 * q + lane;
    const bool rowok = J < T.ncy;
    const int ncx = T.ncx, ncy = T.ncy, PP = T.PP;
    const int dmax = (ncx - 1) + 2 * (ncy - 1);
    const int nxs = (ncy + 2) * T.pitch;
    double* xs = dyn;
    double* spec = dyn + max(nxs, ncx * ncy);
    if (warp == 0) {  // TMEM: 512 columns = 256 fp64 diagonal slots per lane (row)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            uint32_t(__cvta_generic_to_shared(&cs.tmem_base))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // stage cb through shared memory (coalesced), then into TMEM row by row
    for (int k = threadIdx.x; k < ncx * ncy; k += blockDim.x) {
        const int JJ = k / ncx, II = k - JJ * ncx;
        xs[k] = P.cb.at(II, JJ);
    }
    // class table (10 doubles per class) followed by the ring's class ids
    const int spec_words = 10 * T.ncls + (T.ring + 1) / 2;
    for (int k = threadIdx.x; k < spec_words; k += blockDim.x) spec[k] = spec_g[k];
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tq = cs.tmem_base + (uint32_t(32 * q) << 16);
    for (int slot = h; slot < 256; slot += kTmH) {
        const int I = (slot - 2 * J) & 255;
        const double v = (rowok && I < ncx) ? xs[J * ncx + I] : 0.0;
        tm_st2(tq + 2u * uint32_t(slot), uint32_t(__double2loint(v)), uint32_t(__double2hiint(v)));
    }
    tm_wait_st();
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    for (int k = threadIdx.x; k < nxs; k += blockDim.x) xs[k] = 0.0;  // ce = 0 with zero ghost slots
    __syncthreads();
    double rc = st->rc;  // max|cb|, formed by the fine pass that restricted
    const long long budget = P.max_total - st->total;
    long long done = 0;
    // first group = the previous visit's sweep count (visits of one solve
    // have similar lengths), then doubling
    int G = max(1, min(st->pred, kPredCap));
    while (rc > P.tol_coarse && done < budget) {
        if (budget - done < G) G = int(budget - done);
        if (G > 1)
            for (int k = threadIdx.x; k < nxs; k += blockDim.x) backup[k] = xs[k];  // checkpoint
        tm_group<Kind, kTmU>(T, xs, spec, tq, cs, G, true);
        steps += dmax + kLagT * (G - 1) + 5;
        if (threadIdx.x == 0) {
            int first = -1;
            double rg = 0.0;
            for (int g = 0; g < G; ++g) {
                rg = fmax(fmax(cs.wmax[0][g], cs.wmax[1][g]), fmax(cs.wmax[2][g], cs.wmax[3][g]));
                if (!(rg > P.tol_coarse)) {
                    first = g;
                    break;
                }
            }
            cs.ictl[0] = first;
            cs.bcast[1] = rg;
        }
        __syncthreads();
        const int first = cs.ictl[0];
        rc = cs.bcast[1];
        if (first >= 0 && first < G - 1) {  // overshoot: restore and replay first+1 sweeps
            for (int k = threadIdx.x; k < nxs; k += blockDim.x) xs[k] = backup[k];
            __syncthreads();
            tm_group<Kind, kTmU>(T, xs, spec, tq, cs, first + 1, false);
            steps += dmax + kLagT * first + 1;
            done += first + 1;
            break;
        }
        done += G;
        if (first >= 0) break;
        G = min(2 * G, kMaxGroupT);
    }
    // anchor once (singular) and hand ce to the prolongation
    if (P.singular && done > 0) {
        double sum = 0.0;
        double* r = row_ptr(xs, T, J);
        if (rowok && h == 0)
            for (int I = 0; I < ncx; ++I) sum += r[(I + 2 * J + 4) % PP];
        sum = block_sum(sum, cs.red);
        if (threadIdx.x == 0) cs.bcast[2] = -(sum / double(int64_t(ncx) * ncy));
        __syncthreads();
        const double c = cs.bcast[2];
        if (rowok && h == 0)
            for (int I = 0; I < ncx; ++I) r[(I + 2 * J + 4) % PP] += c;
        __syncthreads();
    }
    for (int k = threadIdx.x; k < ncx * ncy; k += blockDim.x) {  // coalesced write-out
        const int JJ = k / ncx, II = k - JJ * ncx;
        P.ce.at(II, JJ) = row_ptr(xs, T, JJ)[(II + 2 * JJ + 4) % PP];
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(cs.tmem_base));
    if (threadIdx.x == 0) {
        st->coarse_launches += 1;
        st->coarse_ns += gtimer() - t_start;
        st->coarse_steps += steps;
        if (done > 0) st->pred = int(done);
        st->total += done;
        st->coarse += done;
        st->rc = rc;
        if (st->nvisits > 0 && st->nvisits <= P.visit_cap) P.visit_log[2 * (st->nvisits - 1)] = int(done);
        if (rc > P.tol_coarse) {  // cycles.hpp:134-137
            st->phase = kDone, st->converged = 0;
        } else if (done > 0) {
            st->phase = kProlong;
        } else {
            st->prev = st->r;
            st->phase = kFine;
        }
        publish_phase(P, st->phase);
    }
}

bool same_bits(double a, double b) { return a == b && std::signbit(a) == std::signbit(b); }

}  // namespace

// Host: can the TMEM kernel run this operator? (every interior cell carries
// the interior stencil bit for bit; the boundary ring is tabulated.)
bool tmem_coarse_plan(const CoarseOpH& op, TmGeom& T, std::vector<double>& spec, size_t& smem) {
    if (op.px || op.py || op.ncx > 256 || op.ncy > 128 || op.ncx < 3 || op.ncy < 3) return false;
    T.ncx = op.ncx, T.ncy = op.ncy, T.five = op.five_point;
    // PP >= ncx + 2 (distinct ghost slots), > 8 kTmH (one fold per step), and
    // PP = 11 (mod 16) so the row pitch PP + 6 = 1 (mod 16) doubles
    const int pp_min = std::max(op.ncx + 2, kLagT * kTmH + 1);
    T.PP = pp_min + ((11 - pp_min % 16) + 16) % 16;
    T.pitch = T.PP + 6;
    T.ring = 2 * op.ncx + 2 * op.ncy;
    for (int sl = 0; sl < 9; ++sl) T.stdw[sl] = op.at(sl, 1, 1);
    for (int J = 1; J < op.ncy - 1; ++J)
        for (int I = 1; I < op.ncx - 1; ++I)
            for (int sl = 0; sl < 9; ++sl)
                if (!same_bits(op.at(sl, I, J), T.stdw[sl])) return false;
    if (T.stdw[0] == 0.0) return false;
    static const double ismg[9] = {-3.0, 0.5, 0.5, 0.5, 0.5, 0.25, 0.25, 0.25, 0.25};
    static const double five[9] = {-4.0, 1.0, 1.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0};
    T.kind = 0;
    bool is_ismg = !op.five_point, is_five = op.five_point;
    for (int sl = 0; sl < 9; ++sl) {
        is_ismg = is_ismg && same_bits(T.stdw[sl], ismg[sl]);
        is_five = is_five && (sl >= 5 || same_bits(T.stdw[sl], five[sl]));
    }
    if (is_ismg) T.kind = 1;
    if (is_five) T.kind = 2;
    // boundary ring -> classes of identical stencils (walls are translation invariant)
    std::vector<std::array<double, 9>> cls;
    std::vector<int> ring_cls(size_t(T.ring), 0);
    auto classify = [&](int r, int I, int J) {
        std::array<double, 9> w;
        for (int sl = 0; sl < 9; ++sl) w[sl] = op.at(sl, I, J);
        size_t c = 0;
        for (; c < cls.size(); ++c) {
            bool eq = true;
            for (int sl = 0; sl < 9 && eq; ++sl) eq = same_bits(cls[c][sl], w[sl]);
            if (eq) break;
        }
        if (c == cls.size()) cls.push_back(w);
        ring_cls[size_t(r)] = int(c);
    };
    for (int I = 0; I < op.ncx; ++I) classify(I, I, 0), classify(op.ncx + I, I, op.ncy - 1);
    for (int J = 0; J < op.ncy; ++J) classify(2 * op.ncx + J, 0, J), classify(2 * op.ncx + op.ncy + J, op.ncx - 1, J);
    T.ncls = int(cls.size());
    if (T.ncls > 1024) return false;
    // Markstein's correction RN(q + r y) == RN(a / w0) for y = RN(1/w0): spot-check
    // every class divisor on random operands before trusting it
    T.fastdiv = 1;
    uint64_t st = 0x9E3779B97F4A7C15ull;
    for (const auto& w : cls) {
        if (w[0] == 0.0) return false;  // singular ring row: the op-level path raises
        const double b = w[0], y = 1.0 / b;
        for (int k = 0; k < 20000 && T.fastdiv; ++k) {
            st ^= st << 13, st ^= st >> 7, st ^= st << 17;
            const double a = std::ldexp(double(st >> 11) * 0x1.0p-53 + 0.5, int((st >> 3) % 120) - 60) *
                             ((st & 1) ? -1.0 : 1.0);
            const double q = a * y, r = std::fma(-q, b, a), mk = std::fma(r, y, q);
            if (!same_bits(mk, a / b)) T.fastdiv = 0;
        }
    }
    spec.assign(size_t(10) * T.ncls + size_t(T.ring + 1) / 2, 0.0);
    for (int c = 0; c < T.ncls; ++c) {
        for (int sl = 0; sl < 9; ++sl) spec[size_t(10) * c + sl] = cls[size_t(c)][size_t(sl)];
        spec[size_t(10) * c + 9] = 1.0 / cls[size_t(c)][0];
    }
    std::memcpy(spec.data() + size_t(10) * T.ncls, ring_cls.data(), sizeof(int) * ring_cls.size());
    const size_t xs_doubles = std::max(size_t(op.ncy + 2) * T.pitch, size_t(op.ncx) * op.ncy);
    smem = (xs_doubles + spec.size()) * sizeof(double);
    return smem <= 200 * 1024;
}

void launch_coarse_tmem(const Params& P, const TmGeom& T, const double* spec, double* backup, size_t smem,
                        cudaStream_t st) {
    if (T.kind == 1)
        coarse_visit_tmem_kernel<1><<<1, kTmThreads, smem, st>>>(P, T, spec, backup);
    else if (T.kind == 2)
        coarse_visit_tmem_kernel<2><<<1, kTmThreads, smem, st>>>(P, T, spec, backup);
    else
        coarse_visit_tmem_kernel<0><<<1, kTmThreads, smem, st>>>(P, T, spec, backup);
}
void set_coarse_tmem_smem(size_t bytes) {
    ISMG_CUDA(cudaFuncSetAttribute(coarse_visit_tmem_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    ISMG_CUDA(cudaFuncSetAttribute(coarse_visit_tmem_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    ISMG_CUDA(cudaFuncSetAttribute(coarse_visit_tmem_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

}  // namespace fz
}  // namespace ismgb

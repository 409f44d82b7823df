// coarse_cl.cu — the coarse visit on a thread-block cluster (cycles.hpp:120-137,
// coarsening.hpp:531-567): lexicographic Gauss-Seidel sweeps on the 9-point
// interpolated operator until tol_coarse, bit for bit the reference's order.
//
// Schedule (as coarse_visit_smem_kernel, coarse.cu): sweep g of cell (I,J)
// runs at wavefront step tau = I + 2J + 8g and its residual at tau + 4, one
// barrier per step; sweeps run in checkpointed groups, a group that overshoots
// the first converged sweep is restored and replayed exactly that far.
//
// Layout, B200-first:
//  * the coarse rows are split into bands over the C CTAs of ONE cluster
//    (C = 1..16 SMs); a CTA keeps its band of the iterate, plus one mirrored
//    halo row on each side, in shared memory in natural row-major order; the
//    row pitch is 3 (mod 16) doubles, so the 32 lanes of a warp (32
//    consecutive rows, one cell each on a wavefront I = t - 2J) touch 32
//    distinct bank pairs;
//  * a band's first / last row is also stored into the neighbour CTA's halo
//    row through distributed shared memory, and every step ends with one
//    cluster barrier (release / acquire);
//  * the rhs sits in shared memory when the band fits, else it is read
//    through L1 (read-only path);
//  * warps of a 32-row block split the sweeps in flight (g = h mod kH); the
//    per-cell index work is one subtract, one compare and one add;
//  * the interior stencil is a compile-time constant when the operator's
//    interior rows are the ISMG or five-point stencil bit for bit; the
//    boundary ring takes a divergent path through a class table.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "fused_impl.cuh"

namespace cg = cooperative_groups;
#ifndef ISMG_CL_TRACE_WARPS
#define ISMG_CL_TRACE_WARPS 1
#endif

namespace ismgb {
namespace fz {

namespace {

constexpr int kLag = 8;            // wavefront steps between consecutive sweeps
constexpr int kMaxGroup = 512;     // sweeps per checkpointed group
constexpr int kPredCap = 32;       // cap of the predicted first group of a visit
constexpr int kHandG = 4;          // role 1: largest group run on one SM
#ifndef ISMG_CL_S4
#define ISMG_CL_S4 3  // barrier interval on a 4-SM cluster (tuning hook)
#endif
#ifndef ISMG_CL_S8
// ... on 8 or more SMs. Same-box A/B at 16384^2 (coarse 512^2, 16 SMs; tools/
// visit_hist.py, coarse ms of steps 1-3): S = 8 1702 / 663 / 785 against 1790 /
// 701 / 829 at S = 4, 1862 / 693 / 817 at 6, 1794 / 678 / 800 at 12.
#define ISMG_CL_S8 8
#endif
#ifndef ISMG_CLX_WARPS
#define ISMG_CLX_WARPS 16
#endif
constexpr int kIntWarps = ISMG_CLX_WARPS;  // warps: 4 row blocks x 4 sweeps in flight
constexpr int kClThreads = 32 * kIntWarps;

constexpr int kMaxRowBlocks = 4;  // 32-row blocks per CTA band

// The CTA's dynamic shared memory, addressed by offsets (doubles) so every
// access compiles to a 32-bit LDS/STS: [iterate band | rhs band | class table].
extern __shared__ __align__(16) double cl_dyn[];

struct ClShared {
    double cmax[kMaxRowBlocks][kMaxGroup];  // residual max per (row block, sweep of the group)
    double gmax[kMaxGroup];                 // ... all reduced over the CTA
    double red[32];
    double bcast[4];
    int ictl[4];
    int first;
};

struct Nbr {
    double c, e, w, n, s, ne, nw, se, sw;
};
// neighbours of the cell at shared offset o (row pitch `pitch`; N = row J+1)
__device__ __forceinline__ Nbr gather(int o, int pitch, bool with_c, bool five) {
    const double* p = cl_dyn + o;
    Nbr v;
    v.c = with_c ? p[0] : 0.0;
    v.e = p[1];
    v.w = p[-1];
    v.n = p[pitch];
    v.s = p[-pitch];
    if (!five) {
        v.ne = p[pitch + 1];
        v.nw = p[pitch - 1];
        v.se = p[1 - pitch];
        v.sw = p[-1 - pitch];
    } else {
        v.ne = v.nw = v.se = v.sw = 0.0;
    }
    return v;
}

// max over the warp of non-negative doubles (their order = the order of the
// (hi, lo) words): two 32-bit REDUX steps
__device__ __forceinline__ double warp_max_nonneg(double m) {
    const unsigned hi = unsigned(__double2hiint(m)), lo = unsigned(__double2loint(m));
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    return __hiloint2double(int(mh), int(ml));
}

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

struct Band {
    int c, C;       // cluster rank, cluster size
    int J0, J1;     // rows [J0, J1) of this CTA
    double* xs;     // iterate: row J at xs + (J - J0 + 1) * pitch + 1 (halo rows J0-1, J1); xs = cl_dyn
    int bo;         // rhs band (BM == 1): row J at cl_dyn[bo + (J - J0) * bpitch]
    int bpitch;
    int so;         // class table offset in cl_dyn
    double* south;  // neighbour CTA's halo row that mirrors row J0 (nullptr at the bottom)
    double* north;  // neighbour CTA's halo row that mirrors row J1 - 1
    uint32_t tmem;  // TMEM base (BM == 2): lane J - J0, column pair (I + 2J) mod 256 holds b(I, J)
};

__device__ __forceinline__ void step_sync(const Band& B) {
    if (B.C > 1) cg::this_cluster().sync();
    else __syncthreads();
}

// Weights of one cell in slot order C, E, W, N, S, NE, NW, SE, SW; y = RN(1 / w[0]).
struct Wts {
    double w[9], y;
};
__device__ __forceinline__ void load_wts(int off, Wts& W) {  // off even: 16-byte loads
    const double2* p = reinterpret_cast<const double2*>(cl_dyn + off);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const double2 v = p[k];
        if (2 * k < 9) W.w[2 * k] = v.x;
        if (2 * k + 1 < 9) W.w[2 * k + 1] = v.y;
        else W.y = v.y;
    }
}

// Term of one slot. The reference skips a zero weight's slot (coarsening.hpp:
// 539-543 residual, :558-565 update). When every zero weight faces a ghost
// (value +0.0), w * v is a signed zero, an exact identity of the update's sum
// (it starts at +0.0, so it is never -0.0) and at most flips the sign of a
// zero residual, whose |r| is all that is used: kSel = false multiplies
// straight through. Otherwise (kSel) the slot's term is -0.0, the identity of +.
template <bool kSel>
__device__ __forceinline__ double term(double w, double v) {
    if constexpr (kSel) return w != 0.0 ? w * v : -0.0;
    return w * v;
}

// Update (num / w0) or residual (b - A x) of one cell with per-lane weights.
template <bool kResidual, bool kFive, bool kSel>
__device__ __forceinline__ double apply_lane(const Wts& W, const Nbr& v, double bIJ, bool fastdiv) {
    double acc = kResidual ? W.w[0] * v.c : 0.0;
    acc += term<kSel>(W.w[1], v.e);
    acc += term<kSel>(W.w[2], v.w);
    acc += term<kSel>(W.w[3], v.n);
    acc += term<kSel>(W.w[4], v.s);
    if (!kFive) {
        acc += term<kSel>(W.w[5], v.ne);
        acc += term<kSel>(W.w[6], v.nw);
        acc += term<kSel>(W.w[7], v.se);
        acc += term<kSel>(W.w[8], v.sw);
    }
    const double num = bIJ - acc;
    if (kResidual) return num;
    if (!fastdiv) return num / W.w[0];
#ifdef ISMG_CLX_NODIV
    return num * W.y;
#endif
    return div_cr(num, W.w[0], W.y);  // correctly rounded (kernels.cuh)
}

// One group of G sweeps (residuals: also form the residual max of every sweep).
// Lane = row J of a 32-row block; the warps of a row block split the sweeps in
// flight (g = h mod kH). Sweep g updates diagonal I + 2J = tau - 8g at step tau
// and forms its residual on tau - 4 - 8g; one loop iteration carries one of
// each, so their independent fp64 chains overlap. Every lane keeps the weights
// of its current update and residual cells in registers and reloads them from
// the class table only when the cell's class changes (ring cells: first / last
// row and column; the interior is class ncls), so ring cells cost no extra pass.
template <int Kind, int BM, int S>
__device__ int cl_group(const ClGeom& T, const Band& B, const View& cbg, ClShared& cs, int G, bool residuals) {
    constexpr bool kFive = (Kind & 1) != 0, kSel = (Kind & 2) != 0;
    const int dmax = (T.ncx - 1) + 2 * (T.ncy - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nrb = (B.J1 - B.J0 + 31) >> 5;  // 32-row blocks of the band (1, 2 or 4)
    // TMEM rhs: a warp may only read its own lane quadrant, so row block = warp mod 4
    const int nq = BM == 2 ? 4 : nrb;
    // warps per row block (power of two; nrb = 3 idles some). One cell-pair
    // iteration is a long dependent chain, so the sweeps in flight are spread
    // over all warps even when few are in flight.
    const int kH = 1 << (31 - __clz(kIntWarps / nq));
    const int rb = warp % nq, h = warp / nq;
    const int Jw = B.J0 + 32 * rb;  // first row of the warp
    const int J = Jw + lane;
    const int jlast = min(Jw + 31, B.J1 - 1);
    const bool w_on = rb < nrb && h < kH;
    const bool rowin = w_on && J <= jlast;  // this lane's row lies in the band
    const bool ringrow = J == 0 || J == T.ncy - 1;
    const int pitch = T.pitch;
    // offsets of cell (0, J) of this lane's row (rows outside the band read row J0)
    const int Jc = rowin ? J : B.J0;
    const int rowo = (Jc - B.J0 + 1) * pitch + 1;
    const int browo = B.bo + (Jc - B.J0) * B.bpitch;
    const double* brow = cbg.p + int64_t(Jc) * cbg.pitch;
    const uint32_t tq = B.tmem + (uint32_t(32 * rb) << 16);  // TMEM lane quadrant of this warp (BM == 2)
    const bool mirror_s = rowin && J == B.J0 && B.south != nullptr;
    const bool mirror_n = rowin && J == B.J1 - 1 && B.north != nullptr;
    const unsigned ncx = unsigned(T.ncx);
    const bool fastdiv = T.fastdiv != 0;
    // class table: 10 doubles per class (interior = class ncls), then the ring's class ids
    const int icls = T.ncls;
    const int* ring_cls = reinterpret_cast<const int*>(cl_dyn + B.so + 10 * (T.ncls + 1));
    // table offsets of this lane's classes: interior, first / last column of its
    // row; a first / last row's cells look theirs up by column (ring order:
    // row 0 by I, row ncy-1 by ncx + I, column 0 by 2 ncx + J, column ncx-1 by
    // 2 ncx + ncy + J)
    const int rbase = J == 0 ? 0 : T.ncx;
    const int off_i = B.so + 10 * icls;
    const int off_w = rowin && !ringrow ? B.so + 10 * ring_cls[2 * T.ncx + J] : off_i;
    const int off_e = rowin && !ringrow ? B.so + 10 * ring_cls[2 * T.ncx + T.ncy + J] : off_i;
    if (residuals) {
        for (int k = threadIdx.x; k < nrb * kMaxGroup; k += blockDim.x) (&cs.cmax[0][0])[k] = 0.0;
    }
    __syncthreads();
    // Schedule: sweep g updates cell (I, J) of band c at step I + 2J + L g + D c and
    // forms its residual R steps later. One SM, or bands of several row blocks: a
    // barrier every step, L = 8, R = 4, D = 0. A cluster of 32-row bands keeps every
    // sweep of a band in one warp, so only other sweeps and the band edges need the
    // cluster. Skewing the bands by D steps and stretching R and L puts every such
    // dependency (RAW and WAR, the mirrored halo rows included) >= S steps apart,
    // so a cluster barrier every S steps suffices, with a warp barrier in between.
    // (S = 2: D = 1, R = 6, L = 12; the binding constraints are the last row's
    // residual reading the next band's NE, R >= 3 + D + S, and the next sweep
    // overwriting the previous band's SW after the residual read it,
    // L >= R + D + S + 3.)
    // A barrier every S steps (S > 1: clusters of 32-row bands only):
    // D = S - 1, R = 3 + D + S, L = R + D + S + 3; compile-time, so the sweep-range
    // divisions by L and the step test are shifts and masks where they can be.
    constexpr int D = S - 1, R = S > 1 ? 3 + D + S : 4, L = S > 1 ? R + D + S + 3 : kLag;
    const int toff = D * B.c;
    const int tau_end = dmax + D * (B.C - 1) + L * (G - 1) + (residuals ? R : 0);
    const int dlo = 2 * Jw, dhi = 2 * jlast + T.ncx - 1;
    // G <= kH: every warp of a row block owns at most one sweep (g = h) for the
    // whole group, so its residual max stays in a register until the group ends
    const bool one_g = G <= kH;
#ifndef ISMG_CL_SPLIT
#define ISMG_CL_SPLIT 1
#endif
    const bool split = ISMG_CL_SPLIT && residuals && 2 * G <= kH;
    const int sg = h & (kH / 2 - 1);
    double lmax = 0.0;
#ifdef ISMG_CL_TRACE
    long long tr_int = 0, tr_bar = 0;
    const long long tr_l0 = clock64();
#endif
    for (int tau = 0; tau <= tau_end; ++tau) {
#ifdef ISMG_CL_TRACE
        const long long c0 = clock64();
#endif
        // one update (diagonal dU) and one residual (diagonal dR, sweep gr) per lane
        auto pair = [&](bool du, bool dres, int dU, int dR, int gr) {
            const int Iu = dU - 2 * J, Ir = dR - 2 * J;
            const bool oku = du && rowin && unsigned(Iu) < ncx;
            const bool okr = dres && rowin && unsigned(Ir) < ncx;
            const int Iuc = oku ? Iu : 0, Irc = okr ? Ir : 0;  // clamped: every lane reads a valid cell
            // weights of the two cells: interior, first / last column, or (first /
            // last row) by column from the ring's class ids
            const int offu = ringrow ? B.so + 10 * ring_cls[rbase + Iuc]
                                     : (Iu == 0 ? off_w : Iu == T.ncx - 1 ? off_e : off_i);
            const int offr = ringrow ? B.so + 10 * ring_cls[rbase + Irc]
                                     : (Ir == 0 ? off_w : Ir == T.ncx - 1 ? off_e : off_i);
            Wts Wu, Wr;
            load_wts(offu, Wu);
            load_wts(offr, Wr);
            double bu, br_;
            if constexpr (BM == 2) {  // rhs of the cells on diagonals d: TMEM column (d mod 256), warp-uniform
                uint32_t lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
                if (du) tm_ld2(tq + 2u * uint32_t(dU & 255), lo0, hi0);
                if (dres) tm_ld2(tq + 2u * uint32_t(dR & 255), lo1, hi1);
                tm_wait_ld();
                bu = __hiloint2double(int(hi0), int(lo0));
                br_ = __hiloint2double(int(hi1), int(lo1));
            } else if constexpr (BM == 1) {
                bu = cl_dyn[browo + Iuc];
                br_ = cl_dyn[browo + Irc];
            } else {
#ifdef ISMG_CLX_NOB
                bu = 0.5, br_ = 0.25;
#else
                bu = __ldg(brow + Iuc);
                br_ = __ldg(brow + Irc);
#endif
            }
            // both cells, branch-free, so their independent fp64 chains interleave
            const Nbr vr = gather(rowo + Irc, pitch, true, kFive);
            const Nbr vu = gather(rowo + Iuc, pitch, false, kFive);
            const double rres = apply_lane<true, kFive, kSel>(Wr, vr, br_, fastdiv);
            const double out = apply_lane<false, kFive, kSel>(Wu, vu, bu, fastdiv);
            if (oku) {  // update of sweep gu
                cl_dyn[rowo + Iu] = out;
                if (mirror_s) B.south[Iu] = out;
                if (mirror_n) B.north[Iu] = out;
            }
            if (dres) {  // residual of sweep gr (inputs final since step tau - 1)
                double m = okr ? fabs(rres) : 0.0;
                m = (m != m) ? 0.0 : m;  // std::max drops NaN
                if (one_g) {  // the warp's only sweep: keep a per-lane max, fold once per group
                    lmax = fmax(lmax, m);
                } else {
                    m = warp_max_nonneg(m);
                    if (lane == 0) cs.cmax[rb][gr] = fmax(cs.cmax[rb][gr], m);  // (rb, gr): this warp alone
                }
            }
        };
        // split (G <= kH / 2): warp h < kH / 2 updates sweep h, warp h + kH / 2 forms
        // its residuals, so the two fp64 chains run on separate warps
        auto upd_only = [&](int dU) {
            const int Iu = dU - 2 * J;
            const bool oku = rowin && unsigned(Iu) < ncx;
            const int Iuc = oku ? Iu : 0;
            const int offu = ringrow ? B.so + 10 * ring_cls[rbase + Iuc]
                                     : (Iu == 0 ? off_w : Iu == T.ncx - 1 ? off_e : off_i);
            Wts Wu;
            load_wts(offu, Wu);
            double bu;
            if constexpr (BM == 2) {
                uint32_t lo0 = 0, hi0 = 0;
                tm_ld2(tq + 2u * uint32_t(dU & 255), lo0, hi0);
                tm_wait_ld();
                bu = __hiloint2double(int(hi0), int(lo0));
            } else if constexpr (BM == 1) {
                bu = cl_dyn[browo + Iuc];
            } else {
#ifdef ISMG_CLX_NOB
                bu = 0.5;
#else
                bu = __ldg(brow + Iuc);
#endif
            }
            const Nbr vu = gather(rowo + Iuc, pitch, false, kFive);
            const double out = apply_lane<false, kFive, kSel>(Wu, vu, bu, fastdiv);
            if (oku) {
                cl_dyn[rowo + Iu] = out;
                if (mirror_s) B.south[Iu] = out;
                if (mirror_n) B.north[Iu] = out;
            }
        };
        auto res_only = [&](int dR) {
            const int Ir = dR - 2 * J;
            const bool okr = rowin && unsigned(Ir) < ncx;
            const int Irc = okr ? Ir : 0;
            const int offr = ringrow ? B.so + 10 * ring_cls[rbase + Irc]
                                     : (Ir == 0 ? off_w : Ir == T.ncx - 1 ? off_e : off_i);
            Wts Wr;
            load_wts(offr, Wr);
            double br_;
            if constexpr (BM == 2) {
                uint32_t lo1 = 0, hi1 = 0;
                tm_ld2(tq + 2u * uint32_t(dR & 255), lo1, hi1);
                tm_wait_ld();
                br_ = __hiloint2double(int(hi1), int(lo1));
            } else if constexpr (BM == 1) {
                br_ = cl_dyn[browo + Irc];
            } else {
#ifdef ISMG_CLX_NOB
                br_ = 0.25;
#else
                br_ = __ldg(brow + Irc);
#endif
            }
            const Nbr vr = gather(rowo + Irc, pitch, true, kFive);
            const double rres = apply_lane<true, kFive, kSel>(Wr, vr, br_, fastdiv);
            double m = okr ? fabs(rres) : 0.0;
            m = (m != m) ? 0.0 : m;  // std::max drops NaN
            lmax = fmax(lmax, m);
        };
        if (w_on) {
            if (split) {
                const int dU = tau - toff - L * sg, dR = dU - R;
                if (h < kH / 2) {
                    if (sg < G && dU >= dlo && dU <= dhi) upd_only(dU);
                } else if (sg < G && dR >= dlo && dR <= dhi) {
                    res_only(dR);
                }
            } else if (one_g) {  // this warp's only sweep is g = h
                const int dU = tau - toff - L * h, dR = dU - R;
                const bool du = h < G && dU >= dlo && dU <= dhi;
                const bool dres = residuals && h < G && dR >= dlo && dR <= dhi;
                if (du || dres) pair(du, dres, dU, dR, h);
            } else {
                const int bu0 = tau - toff, br0 = residuals ? tau - toff - R : -1;
                int gu = 0, guh = -1, gr = 0, grh = -1;
                if (bu0 >= dlo) {
                    const int g_lo = max(0, (bu0 - dhi + L - 1) / L);
                    guh = min(G - 1, (bu0 - dlo) / L);
                    gu = g_lo + ((h - g_lo) & (kH - 1));
                }
                if (br0 >= dlo) {
                    const int g_lo = max(0, (br0 - dhi + L - 1) / L);
                    grh = min(G - 1, (br0 - dlo) / L);
                    gr = g_lo + ((h - g_lo) & (kH - 1));
                }
#pragma unroll 1
                while (gu <= guh || gr <= grh) {
                    pair(gu <= guh, gr <= grh, bu0 - L * gu, br0 - L * gr, gr);
                    gu += kH, gr += kH;
                }
            }
        }
#ifdef ISMG_CL_TRACE
        const long long c1 = clock64();
        tr_int += c1 - c0;
#endif
#ifdef ISMG_CLX_NOSYNC
        if (tau == tau_end) step_sync(B);
#else
        if (S == 1 || tau % S == S - 1 || tau == tau_end) step_sync(B);  // S: template constant
#endif
        else __syncwarp();
#ifdef ISMG_CL_TRACE
        tr_bar += clock64() - c1;
#endif
    }
    const int fold_g = split ? (h >= kH / 2 ? sg : -1) : h;  // the sweep whose residuals this warp formed
    if (one_g && residuals && w_on && fold_g >= 0 && fold_g < G) {  // fold the per-lane maxima
        const double m = warp_max_nonneg(lmax);
        if (lane == 0) cs.cmax[rb][fold_g] = fmax(cs.cmax[rb][fold_g], m);
    }
    __syncthreads();
#ifdef ISMG_CL_TRACE
    const long long tr_loop = clock64() - tr_l0;
    if (lane == 0 && (G == 1 || (G >= 4 && G <= 8)) && residuals && ISMG_CL_TRACE_WARPS)
        printf("TRACE G=%d steps=%d warp=%2d loop=%lld int=%lld bar=%lld\n", G, tau_end + 1, warp, tr_loop, tr_int,
               tr_bar);
#endif
    return tau_end + 1;
}

// The barrier interval of a group: 1 on one SM or with multi-block bands; on a
// cluster of 32-row bands 2 on 2 SMs, 3 on 4, 4 from 8. Measured (same box, A/B):
// 4096^2 (4 SMs) coarse per step 1 / 2: 214 / 85 ms at S = 3, 219 / 89 at S = 2,
// 213 / 84 at S = 4; 16384^2 (16 SMs) per 200-sweep visit: 22.1 ms at S = 4,
// 21.4 at S = 5, 32.9 at S = 1.
template <int Kind, int BM>
__device__ __forceinline__ int cl_group_s(const ClGeom& T, const Band& B, const View& cbg, ClShared& cs, int G,
                                          bool residuals) {
    const bool bands = B.C > 1 && B.J1 - B.J0 <= 32;
    if (!bands) return cl_group<Kind, BM, 1>(T, B, cbg, cs, G, residuals);
    if (B.C >= 8) return cl_group<Kind, BM, ISMG_CL_S8>(T, B, cbg, cs, G, residuals);
    if (B.C >= 4) return cl_group<Kind, BM, ISMG_CL_S4>(T, B, cbg, cs, G, residuals);
    return cl_group<Kind, BM, 2>(T, B, cbg, cs, G, residuals);
}

template <int Kind, int BM>
__global__ void __launch_bounds__(kClThreads, 1) coarse_cl_kernel(Params P, ClGeom T, const double* spec_g,
                                                               double* backup) {
    __shared__ ClShared cs;
    Ctl* st = P.ctl;
    if (st->phase != kCoarse) return;
    if (T.role == 2 && st->cl_hand == 0) return;  // the one-SM kernel finished this visit
    if (T.role == 1 && max(1, min(st->pred, kPredCap)) > kHandG) {  // a long visit: all of it on the cluster
        __syncthreads();
        if (threadIdx.x == 0) {
            st->cl_hand_G = max(1, min(st->pred, kPredCap)), st->cl_hand_done = 0, st->cl_hand_rc = st->rc;
            st->cl_hand = 1;
        }
        return;
    }
    const long long t_start = gtimer();
    cg::cluster_group cluster = cg::this_cluster();
    double* dyn = cl_dyn;
    Band B;
    B.C = int(cluster.num_blocks());
    B.c = int(cluster.block_rank());
    const int R = T.band;
    B.J0 = B.c * R, B.J1 = min(T.ncy, B.J0 + R);
    const int pitch = T.pitch;
    const int rows = R + 2;
    B.xs = dyn;
    B.bo = rows * pitch;
    double* bsm = dyn + B.bo;
    B.bpitch = T.bpitch;
    B.so = B.bo + (BM == 1 ? R * T.bpitch : 0);
    double* spec = dyn + B.so;
    // mirrors: my row J0 is row (R + 1) of the CTA below's buffer; my row J1-1 is row 0 of the CTA above
    B.south = (B.c > 0) ? cluster.map_shared_rank(B.xs, B.c - 1) + size_t(R + 1) * pitch + 1 : nullptr;
    B.north = (B.c + 1 < B.C && B.J1 < T.ncy) ? cluster.map_shared_rank(B.xs, B.c + 1) + 1 : nullptr;
    const int nxs = rows * pitch;
    if (BM != 2)  // (BM == 2: zeroed after the rhs staging that borrows the area)
        for (int k = threadIdx.x; k < nxs; k += blockDim.x) B.xs[k] = 0.0;  // ce = 0, zero ghosts and halos
    B.tmem = 0;
    if constexpr (BM == 2) {  // rhs into Tensor Memory: 512 columns = 256 fp64 diagonal slots per row
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                uint32_t(__cvta_generic_to_shared(&cs.ictl[3]))));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
        B.tmem = uint32_t(cs.ictl[3]);
        // the band's rhs rows through the (not yet zeroed) iterate area with
        // coalesced loads, then from shared memory along the diagonal slots
        double* tmp = B.xs;  // row jj at tmp + jj * T.bpitch
        for (int k = threadIdx.x; k < (B.J1 - B.J0) * T.ncx; k += blockDim.x) {
            const int jj = k / T.ncx, I = k - jj * T.ncx;
            tmp[jj * T.bpitch + I] = P.cb.at(I, B.J0 + jj);
        }
        __syncthreads();
        const int q = warp & 3, nh = int(blockDim.x >> 7);
        const int J = B.J0 + 32 * q + lane;
        const uint32_t tq = B.tmem + (uint32_t(32 * q) << 16);
        for (int slot = warp >> 2; slot < 256; slot += nh) {
            const int I = (slot - 2 * J) & 255;
            const double v = (J < B.J1 && I < T.ncx) ? tmp[(J - B.J0) * T.bpitch + I] : 0.0;
            tm_st2(tq + 2u * uint32_t(slot), uint32_t(__double2loint(v)), uint32_t(__double2hiint(v)));
        }
        tm_wait_st();
        __syncthreads();
        for (int k = threadIdx.x; k < nxs; k += blockDim.x) B.xs[k] = 0.0;
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
    }
    if (BM == 1)
        for (int k = threadIdx.x; k < (B.J1 - B.J0) * T.ncx; k += blockDim.x) {
            const int jj = k / T.ncx, I = k - jj * T.ncx;
            bsm[jj * T.bpitch + I] = P.cb.at(I, B.J0 + jj);
        }
    const int spec_words = 10 * (T.ncls + 1) + (T.ring + 1) / 2;
    for (int k = threadIdx.x; k < spec_words; k += blockDim.x) spec[k] = spec_g[k];
    const bool resume = T.role == 2;
    if (resume && st->cl_hand_done > 0)  // the handed-over iterate, band and halo rows
        for (int k = threadIdx.x; k < rows * T.ncx; k += blockDim.x) {
            const int jj = k / T.ncx, I = k - jj * T.ncx, J = B.J0 - 1 + jj;
            if (J >= 0 && J < T.ncy && J <= B.J1) B.xs[jj * pitch + 1 + I] = P.ce.at(I, J);
        }
    cluster.sync();
    double* my_backup = backup + size_t(B.c) * nxs;
    double rc = resume ? st->cl_hand_rc : st->rc;  // max|cb|, formed by the fine pass that restricted
    const long long budget = P.max_total - st->total;
    long long done = resume ? st->cl_hand_done : 0, steps = 0, gns = 0;
    int G = resume ? st->cl_hand_G : max(1, min(st->pred, kPredCap));
    if (resume) {
        cluster.sync();  // every CTA has read the hand-over before it is cleared
        if (B.c == 0 && threadIdx.x == 0) st->cl_hand = 0;
    }
    bool handoff = false;
    while (rc > P.tol_coarse && done < budget) {
        if (budget - done < G) G = int(budget - done);
        // one SM is faster while every warp owns one sweep (G <= 4 at 128 rows); larger
        // groups go to the cluster kernel that follows in the same graph slot
        if (T.role == 1 && G > kHandG) {
            handoff = true;
            break;
        }
        if (G > 1)
            for (int k = threadIdx.x; k < nxs; k += blockDim.x) my_backup[k] = B.xs[k];  // checkpoint
        const long long tg0 = gtimer();
#ifdef ISMG_CL_TRACE
        const long long ck0 = clock64();
#endif
        const int gsteps = cl_group_s<Kind, BM>(T, B, P.cb, cs, G, true);
        gns += gtimer() - tg0;
#ifdef ISMG_CL_TRACE
        if (threadIdx.x == 0 && B.c == 0) printf("GROUP G=%d ns=%lld cycles=%lld\n", G, gtimer() - tg0, clock64() - ck0);
#endif
        steps += gsteps;
        // cluster-wide first sweep whose residual passes tol_coarse
        {
            const int nrb = (B.J1 - B.J0 + 31) >> 5;
            for (int g = threadIdx.x; g < G; g += blockDim.x) {
                double m = cs.cmax[0][g];
                for (int r = 1; r < nrb; ++r) m = fmax(m, cs.cmax[r][g]);
                cs.gmax[g] = m;
            }
            if (threadIdx.x == 0) cs.first = G;
            cluster.sync();
            if (B.c == 0) {
                for (int g = threadIdx.x; g < G; g += blockDim.x) {
                    double rg = 0.0;
                    for (int r = 0; r < B.C; ++r) rg = fmax(rg, cluster.map_shared_rank(&cs.gmax[0], r)[g]);
                    cs.cmax[0][g] = rg;
                    if (!(rg > P.tol_coarse)) atomicMin(&cs.first, g);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    const int first = cs.first < G ? cs.first : -1;
                    cs.ictl[0] = first;
                    cs.bcast[1] = cs.cmax[0][first >= 0 ? first : G - 1];
                }
            }
        }
        cluster.sync();
        const int first = *cluster.map_shared_rank(&cs.ictl[0], 0);
        rc = *cluster.map_shared_rank(&cs.bcast[1], 0);
        cluster.sync();  // everyone has read CTA 0's decision before it can change
        if (first >= 0 && first < G - 1) {  // overshoot: restore and replay first+1 sweeps
            for (int k = threadIdx.x; k < nxs; k += blockDim.x) B.xs[k] = my_backup[k];
            cluster.sync();
            const long long tg0 = gtimer();
            steps += cl_group_s<Kind, BM>(T, B, P.cb, cs, first + 1, false);
            gns += gtimer() - tg0;
#ifdef ISMG_CL_TRACE
            if (threadIdx.x == 0 && B.c == 0) printf("REPLAY G=%d ns=%lld\n", first + 1, gtimer() - tg0);
#endif
            done += first + 1;
            break;
        }
        done += G;
        if (first >= 0) break;
        G = min(2 * G, kMaxGroup);
    }
    // anchor once (singular) and hand ce to the prolongation
    if (P.singular && done > 0 && !handoff) {
        double sum = 0.0;
        for (int J = B.J0 + int(threadIdx.x >> 5); J < B.J1; J += int(blockDim.x >> 5)) {
            const double* r = B.xs + (J - B.J0 + 1) * pitch + 1;
            double s = 0.0;
            for (int I = int(threadIdx.x & 31); I < T.ncx; I += 32) s += r[I];
            sum += warp_sum_down(s);
        }
        sum = block_sum((threadIdx.x & 31) == 0 ? sum : 0.0, cs.red);
        if (threadIdx.x == 0) cs.bcast[2] = sum;
        cluster.sync();
        double tot = 0.0;
        for (int r = 0; r < B.C; ++r) tot += *cluster.map_shared_rank(&cs.bcast[2], r);
        const double c = -(tot / double(int64_t(T.ncx) * T.ncy));
        for (int k = threadIdx.x; k < (B.J1 - B.J0) * T.ncx; k += blockDim.x) {
            const int jj = k / T.ncx, I = k - jj * T.ncx;
            B.xs[(jj + 1) * pitch + 1 + I] += c;
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < (B.J1 - B.J0) * T.ncx; k += blockDim.x) {  // coalesced write-out
        const int jj = k / T.ncx, I = k - jj * T.ncx;
        P.ce.at(I, B.J0 + jj) = B.xs[(jj + 1) * pitch + 1 + I];
    }
    if constexpr (BM == 2) {
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
        if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(B.tmem));
    }
    cluster.sync();  // no CTA exits while another may still read its shared memory
    if (handoff) {
        if (B.c == 0 && threadIdx.x == 0) {
            st->coarse_ns += gtimer() - t_start;
            st->coarse_steps += steps;
            st->coarse_group_ns += gns;
            st->cl_hand_G = G, st->cl_hand_done = done, st->cl_hand_rc = rc;
            st->cl_hand = 1;
        }
        return;
    }
    if (B.c == 0 && threadIdx.x == 0) {
        st->coarse_launches += 1;
        st->coarse_ns += gtimer() - t_start;
        st->coarse_steps += steps;
        st->coarse_group_ns += gns;
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

template <int Kind, int BM>
void launch_one(const Params& P, const ClGeom& T, const double* spec, double* backup, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(T.csize);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(T.csize);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ISMG_CUDA(cudaLaunchKernelEx(&cfg, coarse_cl_kernel<Kind, BM>, P, T, spec, backup));
}

template <int Kind, int BM>
void set_attrs(size_t smem) {
    ISMG_CUDA(cudaFuncSetAttribute(coarse_cl_kernel<Kind, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
    ISMG_CUDA(cudaFuncSetAttribute(coarse_cl_kernel<Kind, BM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

}  // namespace

// Stencil classes of a non-periodic coarse operator: the interior rows' stencil
// (bit for bit one class), the boundary ring tabulated by class. Table layout
// (spec): classes 0..ncls-1 (ring), class ncls (interior), 10 doubles each (w0..w8,
// RN(1 / w0)), then the ring's class ids as ints (row 0 by I, row ncy-1 by ncx + I,
// column 0 by 2 ncx + J, column ncx-1 by 2 ncx + ncy + J). kind bit 0: five-point;
// bit 1: some zero weight faces a cell inside the grid (the engines then skip it).
bool stencil_classes(const CoarseOpH& op, StencilClasses& S) {
    if (op.px || op.py || op.ncx < 3 || op.ncy < 3) return false;
    S.five = op.five_point;
    S.ring = 2 * op.ncx + 2 * op.ncy;
    for (int sl = 0; sl < 9; ++sl) S.stdw[sl] = op.at(sl, 1, 1);
    for (int J = 1; J < op.ncy - 1; ++J)
        for (int I = 1; I < op.ncx - 1; ++I)
            for (int sl = 0; sl < 9; ++sl)
                if (!same_bits(op.at(sl, I, J), S.stdw[sl])) return false;
    if (S.stdw[0] == 0.0) return false;
    std::vector<std::array<double, 9>> cls;
    std::vector<int> ring_cls(size_t(S.ring), 0);
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
    S.ncls = int(cls.size());
    if (S.ncls > 1024) return false;
    S.fastdiv = 1;  // div_cr (kernels.cuh): correctly rounded for every divisor; the sample below is a sanity check
    uint64_t st = 0x9E3779B97F4A7C15ull;
    for (size_t c = 0; c <= cls.size(); ++c) {
        const double b = c < cls.size() ? cls[c][0] : S.stdw[0];
        if (b == 0.0) return false;  // singular ring row: the op-level path raises
        const double y = 1.0 / b;
        for (int k = 0; k < 20000 && S.fastdiv; ++k) {
            st ^= st << 13, st ^= st >> 7, st ^= st << 17;
            const double a = std::ldexp(double(st >> 11) * 0x1.0p-53 + 0.5, int((st >> 3) % 120) - 60) *
                             ((st & 1) ? -1.0 : 1.0);
            const double q = a * y, r = std::fma(-q, b, a), mk = std::fma(r, y, q);
            if (!same_bits(mk, a / b)) S.fastdiv = 0;
        }
    }
    // zero weights facing only ghosts (+0.0) need no skip (see term()); corners
    // of a five-point operator are never read
    static const int dx[9] = {0, 1, -1, 0, 0, 1, -1, 1, -1}, dy[9] = {0, 0, 0, 1, -1, 1, 1, -1, -1};
    const int nsl = S.five ? 5 : 9;
    bool zghost = true;
    for (int sl = 1; sl < nsl; ++sl) zghost = zghost && S.stdw[sl] != 0.0;
    for (int r = 0; r < S.ring && zghost; ++r) {
        int I, J;
        if (r < op.ncx) I = r, J = 0;
        else if (r < 2 * op.ncx) I = r - op.ncx, J = op.ncy - 1;
        else if (r < 2 * op.ncx + op.ncy) I = 0, J = r - 2 * op.ncx;
        else I = op.ncx - 1, J = r - 2 * op.ncx - op.ncy;
        for (int sl = 1; sl < nsl; ++sl) {
            const int In = I + dx[sl], Jn = J + dy[sl];
            const bool ghost = In < 0 || In >= op.ncx || Jn < 0 || Jn >= op.ncy;
            if (cls[size_t(ring_cls[size_t(r)])][size_t(sl)] == 0.0 && !ghost) zghost = false;
        }
    }
    S.kind = (S.five ? 1 : 0) | (zghost ? 0 : 2);
    S.spec.assign(size_t(10) * (S.ncls + 1) + size_t(S.ring + 1) / 2, 0.0);
    for (int c = 0; c <= S.ncls; ++c) {
        const double* w = c < S.ncls ? cls[size_t(c)].data() : S.stdw;
        for (int sl = 0; sl < 9; ++sl) S.spec[size_t(10) * c + sl] = w[sl];
        S.spec[size_t(10) * c + 9] = 1.0 / w[0];
    }
    std::memcpy(S.spec.data() + size_t(10) * (S.ncls + 1), ring_cls.data(), sizeof(int) * ring_cls.size());
    return true;
}

// Host plan: stencil classes (interior constant + tabulated boundary ring),
// cluster size and band height so the band fits shared memory.
bool cl_coarse_plan(const CoarseOpH& op, ClGeom& T, std::vector<double>& spec, size_t& smem, int band_min) {
    StencilClasses S;
    if (!stencil_classes(op, S)) return false;
    T.ncx = op.ncx, T.ncy = op.ncy, T.five = S.five;
    T.ring = S.ring, T.ncls = S.ncls, T.fastdiv = S.fastdiv, T.kind = S.kind;
    for (int sl = 0; sl < 9; ++sl) T.stdw[sl] = S.stdw[sl];
    T.stdy = 1.0 / T.stdw[0];
    T.role = 0;
    spec = S.spec;
    // pitches = 3 (mod 16) doubles (conflict-free wavefront lanes), >= ncx + 2
    T.pitch = (op.ncx + 2) + ((3 - (op.ncx + 2) % 16) + 16) % 16;
    T.bpitch = op.ncx + ((3 - op.ncx % 16) + 16) % 16;
    const size_t cap = 200 * 1024;
    const size_t spec_bytes = spec.size() * sizeof(double);
    // Band height: 32 rows per CTA when the cluster allows it. One 32-row band per
    // SM spreads a step's cells over C SMs; the cluster barrier per step (~600
    // cycles against ~50 for a CTA barrier) is repaid from about 5 sweeps in
    // flight up (measured at 128^2: 252 ms of coarse groups at C = 4 against 346 at
    // C = 1 over a 4096^2 step). rhs in shared memory if it fits, else in Tensor
    // Memory (bands <= 128 rows, ncx <= 256), else read through L1.
    int rmin = std::max(32, band_min / 32 * 32);  // tuning hook: ISMG_CL_BAND = smallest band height tried
    if (const char* e = getenv("ISMG_CL_BAND")) rmin = std::max(32, atoi(e) / 32 * 32);
    for (int R = rmin; R <= 32 * kMaxRowBlocks; R *= 2) {
        const int C = (op.ncy + R - 1) / R;
        if (C > 16) continue;
        for (int bm : {1, 2, 0}) {
            if (bm == 2 && (R > 128 || op.ncx > 256)) continue;
            const size_t bytes = (size_t(R + 2) * T.pitch + (bm == 1 ? size_t(R) * T.bpitch : 0)) * sizeof(double) +
                                 spec_bytes;
            if (bytes <= cap) {
                T.csize = C;
                T.band = R;
                T.bsmem = bm;
                smem = bytes;
                return true;
            }
        }
    }
    return false;
}

size_t cl_backup_doubles(const ClGeom& T) { return size_t(T.csize) * size_t(T.band + 2) * T.pitch; }

template <int Kind>
void launch_kind(const Params& P, const ClGeom& T, const double* spec, double* backup, size_t smem, cudaStream_t st) {
    if (T.bsmem == 2) launch_one<Kind, 2>(P, T, spec, backup, smem, st);
    else if (T.bsmem == 1) launch_one<Kind, 1>(P, T, spec, backup, smem, st);
    else launch_one<Kind, 0>(P, T, spec, backup, smem, st);
}
void launch_coarse_cl(const Params& P, const ClGeom& T, const double* spec, double* backup, size_t smem,
                      cudaStream_t st) {
    switch (T.kind) {
        case 0: launch_kind<0>(P, T, spec, backup, smem, st); break;
        case 1: launch_kind<1>(P, T, spec, backup, smem, st); break;
        case 2: launch_kind<2>(P, T, spec, backup, smem, st); break;
        default: launch_kind<3>(P, T, spec, backup, smem, st); break;
    }
}
template <int Kind>
void set_attrs_kind(size_t bytes) {
    set_attrs<Kind, 0>(bytes), set_attrs<Kind, 1>(bytes), set_attrs<Kind, 2>(bytes);
}
void set_coarse_cl_smem(size_t bytes) {
    set_attrs_kind<0>(bytes), set_attrs_kind<1>(bytes), set_attrs_kind<2>(bytes), set_attrs_kind<3>(bytes);
}

}  // namespace fz
}  // namespace ismgb

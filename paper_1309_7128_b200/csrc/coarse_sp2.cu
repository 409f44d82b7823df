// coarse_sp2.cu — the sweep pipeline of coarse_sp.cu for coarse grids of more
// than 16 blocks of 32 rows (config 4's 512 x 1024 level): the same schedule,
// rings and cross-CTA hand-off, but each compute warp takes several blocks in
// turn (warp w: blocks w, w + nw, ...; the plan makes the diagonal windows of a
// warp's blocks disjoint, ring reuse included), so <= 11 compute warps cover
// up to 32 blocks and a lane keeps its row's body weights in registers (168).
// At 512^2 the one-block-per-warp kernel is faster (0.80 against 1.11 ms per
// one-sweep visit), so this kernel only takes the grids that one cannot.
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include <type_traits>

#include "fused_impl.cuh"

namespace ismgb {
namespace fz {

namespace {

constexpr int kS = 4;                  // steps between named barriers of the compute warps
constexpr int kD = kS - 1;             // skew between consecutive 32-row blocks (steps)
constexpr int kR = 3 + kD + kS;        // residual lag (steps): row 32's mirror value is >= kS steps old
constexpr int kK = 7;                  // cp.async prefetch distance (steps)
constexpr int kQ = 24;                 // new-value ring slots (6 segments of 4)
constexpr int kQE = 8, kQB = 8;        // prefetch ring slots (old values; update / residual rhs)
constexpr int kRows = 34;              // ring rows: block rows -1 .. 32
constexpr int kMaxW = 16;              // compute warps
constexpr int kMaxB = 32;              // 32-row blocks (coarse rows <= 1024)
constexpr int kStride = 64 + kD;       // CTA steps between consecutive blocks
constexpr int kDLo = -4;               // first diagonal of a block's loop (ghost columns written as 0)
constexpr int kDHiPad = 63;            // last update diagonal: ncx + kDHiPad
constexpr int kDOff = 96;              // layouts: diagonal d of block b at [b][d + kDOff][lane]
constexpr int kDSpanPad = 192;         // diagonals per block: ncx + kDSpanPad
constexpr int kSpThreads = 32 * (kMaxW / 4 * 3);  // <= 12 warps: 168 registers
constexpr int kInf = INT_MAX;

// With a barrier every kS steps, block b+1 kD = kS-1 steps behind block b and
// the residual kR = 3 + kD + kS steps behind the update, every cross-block
// dependency (row -1 / row 32 mirrors, RAW and WAR) is >= kS steps apart.
// Live ring span: mirror writes kD ahead, residual reads kR + 1 behind, kS - 1
// of drift inside a barrier interval either way.
static_assert(kD + kR + 2 * kS <= kQ, "new-value ring: live span");
static_assert(kQ == 24 && kQE == 8 && kQB == 8, "ring segments: 6 / 2 of 4 slots");
static_assert(kR + 1 <= 16 && kD + 3 <= 7, "new-value ring offsets in segments -4 .. 1");
static_assert(kK + 1 <= kQE && kK + 1 <= kQB, "prefetch rings");
static_assert(kK - 2 >= 1, "prefetch must run ahead of the NE read (t + 2)");
static_assert(kDOff + kDLo - 2 * kR - 64 >= 0, "layout margin below the lowest prefetched diagonal");
static_assert(kDSpanPad - kDOff >= kDHiPad + kR + kK + 2, "layout margin above the highest prefetched diagonal");

__device__ unsigned g_sp2_stuck = 0u;  // watchdog: a wait ran past 2 s

}  // namespace

struct Sp2K {
    int ncx, ncy, nb;        // coarse grid, 32-row blocks
    int nw;                  // compute warps: warp w takes blocks w, w + nw, ... (disjoint diagonal windows)
    int P, B;                // CTAs (sweeps in flight), buffers
    int dspan;               // diagonals per block in the layouts
    int64_t bstride, bufsz;  // doubles per block / per buffer
    int ncls, ring, spec_words;
    int singular;
    int tend;                // last CTA step of a sweep
};

struct Sp2D {
    double* bufs;                // [B][nb][dspan][32] sweep outputs (diagonal layout)
    double* zero;                // one all-zero buffer: sweep -1 (ce = 0) and missing blocks
    double* bd;                  // rhs, diagonal layout
    const double* spec;          // class table (stencil_classes)
    unsigned long long* prog;    // [P] progress: (sweep << 32) | steps done (0xffffffff: sweep finished)
    unsigned* finw;              // [B] sweep g done: finw[g % B] = g + 1
    double* resw;                // [B] residual max of sweep g
    double* sumw;                // [B] Σ x of sweep g (anchor)
    int* st;                     // [0] first converged sweep (INT_MAX none), [1] sweeps finished
    unsigned* bar;               // grid barrier: [0] arrivals, [1] generation
};

namespace {

extern __shared__ __align__(16) double sp2_dyn[];

// ISMG_SP_CHECK builds: bounds of every ring slot and layout diagonal, trapping
// on the first violation (compute-sanitizer is not available on this pool).
#ifdef ISMG_SP_CHECK
#define SP_ASSERT(c, what)                                                                      \
    do {                                                                                        \
        if (!(c)) {                                                                             \
            printf("coarse_sp2 bounds: %s (block %d thread %d)\n", what, blockIdx.x, threadIdx.x); \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define SP_ASSERT(c, what) (void)0
#endif

__device__ __forceinline__ void cp8(uint32_t dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// shared-memory loads / stores by 32-bit address
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bar_compute(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }
__device__ __forceinline__ int ld_acq_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(su32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(su32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_vol_s(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ unsigned long long ld_acq_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acq_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_rlx_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rel_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool timed_out(long long t0) {
    if (gtimer() - t0 > 2000000000ll) {
        atomicExch(&g_sp2_stuck, 1u);
        return true;
    }
    return false;
}

__device__ void sp_grid_sync(unsigned* bar, unsigned n) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vb = bar;
        const unsigned gen = vb[1];
        __threadfence();
        if (atomicAdd(bar, 1u) == n - 1) {
            vb[0] = 0u;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            const long long t0 = gtimer();
            while (vb[1] == gen) {
                __nanosleep(32);
                if (timed_out(t0)) break;
            }
        }
        __threadfence();
    }
    __syncthreads();
}

struct Sp2Shared {
    int avail;      // steps of sweep g-1 available (from the comm warp)
    int abort_;     // sweep g > first converged sweep: stop
    int done_t;     // steps of this sweep done (for the comm warp to publish)
    int end;        // compute warps finished the sweep
    int aborted;
    int go;
    int dec[2];     // abort decision per barrier parity
    double wmax[kMaxW], wsum[kMaxB];
};

// Weights of one cell (slot order C, E, W, N, S, NE, NW, SE, SW) + RN(1 / w0).
struct Wt {
    double w[9], y;
};
__device__ __forceinline__ void load_wt(const double* tbl, int cls, Wt& W) {
    const double2* p = reinterpret_cast<const double2*>(tbl + 10 * cls);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const double2 v = p[k];
        W.w[2 * k] = v.x;
        if (2 * k + 1 < 9) W.w[2 * k + 1] = v.y;
        else W.y = v.y;
    }
}

// correctly rounded num / w with y = RN(1 / w) (kernels.cuh div_cr), every lane active
__device__ __forceinline__ double div_full(double num, double w, double y) {
#ifdef ISMG_SPX_NODIV
    return num * y;
#endif
    const unsigned e = unsigned(__double2hiint(num)) & 0x7ff00000u;
    const bool bad = e - (123u << 20) > (1900u << 20);
    const double q0 = __dmul_rn(num, y);
    const double e0 = __fma_rn(-q0, w, num);
    const double q1 = __fma_rn(e0, y, q0);
    const double e1 = __fma_rn(-q1, w, num);
    double q = __fma_rn(e1, y, q1);
    if (__any_sync(kFull, bad)) q = div_ieee_lanes(num, w, q, bad);
    return q;
}

// Shared-memory layout (offsets in doubles from sp2_dyn), per compute warp:
// new-value rings [nw][kQ][kRows] | old-value rings [nw][kQE][32] | rhs rings
// [nw][2][kQB][32] (update, residual) | X rings [nw][kQE] (lane 31's NE) | class table.
struct SmemMap {
    int e, bu, x, tbl;
};

// The lane state of block b (lane l owns row J = 32 b + l).
struct Blk {
    Wt W;                                           // the row's body class (column 1 .. ncx-2)
    double outP, seP, seP2, neP, neP2;              // update: W, S / SW (previous SE), N / NW (previous NE)
    double qSW, qS, qSE, qW, qC, qE, qNW, qN, qNE;  // residual window: rows r-1, r, r+1
    double lmax, rsum;
    int cls;   // classes of the row's column 0 | body | column ncx-1 (10 bits each)
};

// One step of block b at diagonal d (CTA step 4m + j): the update of column
// I = d - 2 l and the residual of column I - kR (sweep-g values on all nine
// points), two independent fp64 chains; nslot(q) / eslot(q) = ring offset / slot
// of step 4m + q in the new-value / prefetch rings. The row's body weights stay in registers; in the windows where some lane is
// at column 0 / ncx-1 those lanes load their class and restore the body after.
template <class Slot, class ESlot>
__device__ __forceinline__ void blk_step(Blk& B, int w, int b, bool rowok, int j, int d, const Sp2K& T, const SmemMap& M,
                                         int dn, int dp, double* xn_row, const Slot& nslot, const ESlot& eslot) {
    const int lane = threadIdx.x & 31;
    const int ncx = T.ncx;
    const int dhi = ncx + kDHiPad;
    const int I = d - 2 * lane, Ir = I - kR;
    const bool act_u = rowok && unsigned(I) < unsigned(ncx) && d <= dhi;
    const bool act_r = rowok && unsigned(Ir) < unsigned(ncx);
    const double* tbl = sp2_dyn + M.tbl;
    const uint32_t s0 = su32(sp2_dyn);
    const uint32_t sN = s0 + 8u * uint32_t(w * (kQ * kRows) + lane);  // this lane's column of the warp's ring
    const uint32_t sE = s0 + 8u * uint32_t(M.e + w * (kQE * 32) + lane);
    const uint32_t sB = s0 + 8u * uint32_t(M.bu + w * (2 * kQB * 32) + lane);
    SP_ASSERT(nslot(j - kR - 1) >= 0 && nslot(j + kD) + kRows <= kQ * kRows, "new-value ring slot");
    SP_ASSERT(d + kDOff >= 0 && d + kDOff < T.dspan, "output diagonal");
    // inputs of both cells (none is written by this step)
    const double E = lds64(sE + 8u * uint32_t(eslot(j) * 32));
    const double NE = lds64(lane < 31 ? sE + 8u * uint32_t(eslot(j + 2) * 32 + 1)
                                      : s0 + 8u * uint32_t(M.x + w * kQE + eslot(j)));
    const double SE = lds64(sN + 8u * uint32_t(nslot(j - 1)));
    const double bu = lds64(sB + 8u * uint32_t(eslot(j) * 32));
    const double rm1 = lds64(sN + 8u * uint32_t(nslot(j - kR - 1)));
    const double r0 = lds64(sN + 8u * uint32_t(nslot(j - kR + 1) + 1));
    const double rp1 = lds64(sN + 8u * uint32_t(nslot(j - kR + 3) + 2));
    const double br = lds64(sB + 8u * uint32_t(kQB * 32 + eslot(j) * 32));
    B.qSW = B.qS, B.qS = B.qSE, B.qSE = rm1;
    B.qW = B.qC, B.qC = B.qE, B.qE = r0;
    B.qNW = B.qN, B.qN = B.qNE, B.qNE = rp1;
    const int wcls = B.cls & 1023, bcls = (B.cls >> 10) & 1023, ecls = B.cls >> 20;
    // ---- update ----
    const bool endu = d <= 62 || (d >= ncx - 1 && d <= ncx + 61);  // warp-uniform: some lane may be at a row end
    const bool spu = endu && rowok && (I == 0 || I == ncx - 1);
    if (endu && spu) load_wt(tbl, I == 0 ? wcls : ecls, B.W);
    double acc = 0.0;
    acc += B.W.w[1] * E;
    acc += B.W.w[2] * B.outP;
    acc += B.W.w[3] * B.neP;
    acc += B.W.w[4] * B.seP;
    acc += B.W.w[5] * NE;
    acc += B.W.w[6] * B.neP2;
    acc += B.W.w[7] * SE;
    acc += B.W.w[8] * B.seP2;
    const double num = act_u ? bu - acc : 1.0;
    const double q = div_full(num, B.W.w[0], B.W.y);
    const double out = act_u ? q : 0.0;
    // ---- residual ----
    const bool endr = d - kR <= 62 || (d - kR >= ncx - 1 && d - kR <= ncx + 61);
    const bool spr = endr && rowok && (Ir == 0 || Ir == ncx - 1);
    if (endu || endr) {
        if (spr) load_wt(tbl, Ir == 0 ? wcls : ecls, B.W);
        else if (spu) load_wt(tbl, bcls, B.W);
    }
    double a = B.W.w[0] * B.qC;
    a += B.W.w[1] * B.qE;
    a += B.W.w[2] * B.qW;
    a += B.W.w[3] * B.qN;
    a += B.W.w[4] * B.qS;
    a += B.W.w[5] * B.qNE;
    a += B.W.w[6] * B.qNW;
    a += B.W.w[7] * B.qSE;
    a += B.W.w[8] * B.qSW;
    if (endr && spr) load_wt(tbl, bcls, B.W);
    double mm = act_r ? fabs(br - a) : 0.0;
    mm = (mm != mm) ? 0.0 : mm;  // std::max drops NaN
    B.lmax = fmax(B.lmax, mm);
    // ---- stores: own row, the neighbour blocks' mirror rows, the sweep's output ----
    sts64(sN + 8u * uint32_t(nslot(j) + 1), out);
    if (lane == 31 && b + 1 < T.nb) sts64(sN + 8u * uint32_t(dn + nslot(j + kD) - 31), out);  // row -1 of block b+1 (next warp's ring)
    if (lane == 0 && b > 0) sts64(sN + 8u * uint32_t(dp + nslot(j - kD) + 33), out);          // row 32 of block b-1 (previous warp's ring)
#ifndef ISMG_SPX_NOSTG
    if (d <= dhi) xn_row[(d + kDOff) * 32] = out;
#endif
    if (act_u) B.rsum += out;
    B.seP2 = B.seP, B.seP = SE, B.neP2 = B.neP, B.neP = NE, B.outP = out;
}

// prefetch (cp.async) of block b for the step kK ahead (diagonal dp = d + kK)
__device__ __forceinline__ void blk_prefetch(int w, int slot, int dp, const SmemMap& M, const double* xo_row,
                                             const double* xo_next, const double* bd_row) {
#ifndef ISMG_SPX_NOCP
    const int lane = threadIdx.x & 31;
    const uint32_t so = uint32_t(slot) * 256u;
    SP_ASSERT(slot >= 0 && slot < kQE, "prefetch ring slot");
    SP_ASSERT(dp - 61 + kDOff >= 0 && dp - kR + kDOff >= 0, "prefetch diagonal");
    cp8(su32(sp2_dyn + M.e + w * (kQE * 32) + lane) + so, xo_row + (dp + 1 + kDOff) * 32);
    cp8(su32(sp2_dyn + M.bu + w * (2 * kQB * 32) + lane) + so, bd_row + (dp + kDOff) * 32);
    cp8(su32(sp2_dyn + M.bu + w * (2 * kQB * 32) + kQB * 32 + lane) + so, bd_row + (dp - kR + kDOff) * 32);
    if (lane == 31)  // row 32 = block b+1's lane 0, column I + 1 (diagonal dp - 61 there)
        cp8(su32(sp2_dyn + M.x + w * kQE) + 8u * uint32_t(slot), xo_next + (dp - 61 + kDOff) * 32);
#endif
}

// The row state of lane l for block b (row J = 32 b + l): body weights, classes, zeroed windows.
__device__ __forceinline__ bool blk_begin(Blk& B, int b, const Sp2K& T, const SmemMap& M, const int* ring_cls) {
    const int lane = threadIdx.x & 31, ncx = T.ncx, ncy = T.ncy;
    const int J = 32 * b + lane;
    const bool rowok = b < T.nb && J < ncy;
    int wcls = T.ncls, bcls = T.ncls, ecls = T.ncls;  // column 0, columns 1 .. ncx-2 (one class, plan), column ncx-1
    if (rowok) {
        if (J == 0 || J == ncy - 1) {
            const int rb = J == 0 ? 0 : ncx;
            wcls = ring_cls[rb], bcls = ring_cls[rb + 1], ecls = ring_cls[rb + ncx - 1];
        } else {
            wcls = ring_cls[2 * ncx + J], ecls = ring_cls[2 * ncx + ncy + J];
        }
    }
    B.cls = wcls | (bcls << 10) | (ecls << 20);
    load_wt(sp2_dyn + M.tbl, bcls, B.W);
    B.outP = B.seP = B.seP2 = B.neP = B.neP2 = 0.0;
    B.qSW = B.qS = B.qSE = B.qW = B.qC = B.qE = B.qNW = B.qN = B.qNE = 0.0;
    B.rsum = 0.0;
    return rowok;
}

// One sweep of compute warp w over CTA steps -8 .. tend: blocks w, w + nw, ...
// in turn (block b works on diagonal d = t + kDLo - kStride b at step t; the
// plan makes the windows of a warp's blocks disjoint, ring reuse included),
// a named barrier of the compute warps every kS steps.
__device__ __forceinline__ void sp_sweep(const Sp2K& T, const Sp2D& D, Sp2Shared& sh, const SmemMap& M,
                                         const int* ring_cls, const double* __restrict__ xo,
                                         double* __restrict__ xn, int g) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NW = T.nw, nthr = 32 * NW;
    const int ncx = T.ncx;
    const int dhi = ncx + kDHiPad;
    // the rings of the warps holding blocks b+1 / b-1 (relative offsets in doubles)
    const int dn = ((w + 1 == NW) ? -w : 1) * (kQ * kRows);
    const int dp = ((w == 0) ? NW - 1 : -1) * (kQ * kRows);
    Blk B;
    B.lmax = 0.0;
    int b = w;
    bool rowok = blk_begin(B, b, T, M, ring_cls);
    const double* xo_row = xo + b * T.bstride + lane;
    const double* xo_next = b + 1 < T.nb ? xo + (b + 1) * T.bstride : D.zero;  // row 32 = block b+1's lane 0
    const double* bd_row = D.bd + b * T.bstride + lane;
    double* xn_row = xn + b * T.bstride + lane;
    int avail = g == 0 ? kInf : 0;
    int h = 0;
    bool aborted = false;
    const int mend = T.tend >> 2;
    int m6 = 4;  // m mod 6 (m = -2 at the start)
    for (int m = -2; m <= mend && !aborted; ++m, m6 = (m6 == 5 ? 0 : m6 + 1)) {
        // new-value ring: 6 segments of 4 slots; step 4m + q lives in segment (m + (q >> 2)) mod 6
        int segb[6];  // segb[k]: segment of q >> 2 == k - 4
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            int x = m6 + k + 2;
            x -= x >= 6 ? 6 : 0;
            x -= x >= 6 ? 6 : 0;
            segb[k] = x * 4 * kRows;
        }
        auto nslot = [&](int q) { return segb[(q >> 2) + 4] + (q & 3) * kRows; };  // q in [-16, 7]
        const int e0 = (m & 1) * 4, e1 = ((m + 1) & 1) * 4;  // prefetch rings: 2 segments of 4 slots
        auto eslot = [&](int q) { return (((q >> 2) & 1) ? e1 : e0) + (q & 3); };
        int d0 = 4 * m + kDLo - kStride * b;  // diagonal of step j = 0
        if (d0 > dhi + kR && b < T.nb) {     // block b done: fold its sum, take block b + nw
            const double s = warp_sum_down(B.rsum);
            if (lane == 0) sh.wsum[b] = s;
            b += NW;
            rowok = blk_begin(B, b, T, M, ring_cls);
            xo_row += NW * T.bstride, bd_row += NW * T.bstride, xn_row += NW * T.bstride;
            xo_next = b + 1 < T.nb ? xo + (b + 1) * T.bstride : D.zero;
            d0 = 4 * m + kDLo - kStride * b;
        }
        const bool live = b < T.nb;
        const bool pf_any = live && d0 + 3 + kK >= kDLo - kR && d0 + kK <= dhi + kR;
#ifndef ISMG_SP_NOIDLE
        if (!pf_any && !(live && d0 + 3 >= kDLo && d0 <= dhi + kR)) {  // an idle group: the barrier only
            if (w == 0 && lane == 0) sh.dec[h & 1] = ld_vol_s(&sh.abort_);
            bar_compute(nthr);
            if (w == 0 && lane == 0) st_rel_cta(&sh.done_t, max(0, 4 * m + 4));
            aborted = ld_vol_s(&sh.dec[h & 1]) != 0;
            ++h;
            continue;
        }
#endif
        // a group whose 4 steps all prefetch and update runs without the per-step window tests
        auto group = [&](auto fullc) {
            constexpr bool FULL = decltype(fullc)::value;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int t = 4 * m + j;
            const int d = d0 + j;
            if (j == 0 && pf_any && avail < t + 3 + kK + kD + 4) {  // sweep g-1 far enough for the next 4 steps
                const int need = t + 3 + kK + kD + 4;
                if (lane == 0) {
                    const long long tw = gtimer();
                    int a;
                    while ((a = ld_acq_cta(&sh.avail)) < need) {
                        if (ld_vol_s(&sh.abort_) || timed_out(tw)) break;
                    }
                    avail = a;
                }
                avail = __shfl_sync(kFull, avail, 0);
                __syncwarp();
            }
            if (FULL || (live && d + kK >= kDLo - kR && d + kK <= dhi + kR))
                blk_prefetch(w, eslot(j + kK), d + kK, M, xo_row, xo_next, bd_row);
            cp_commit();
            cp_wait<kK - 2>();
            __syncwarp();
            if (FULL || (live && d >= kDLo && d <= dhi + kR))
                blk_step(B, w, b, rowok, j, d, T, M, dn, dp, xn_row, nslot, eslot);
            if (j == 3) {  // named barrier of the compute warps every kS = 4 steps
                if (w == 0 && lane == 0) sh.dec[h & 1] = ld_vol_s(&sh.abort_);
                bar_compute(nthr);
                if (w == 0 && lane == 0) st_rel_cta(&sh.done_t, max(0, t + 1));
                aborted = ld_vol_s(&sh.dec[h & 1]) != 0;
                ++h;
            }
        }
        };
#ifndef ISMG_SP2_NOFULL
        if (live && d0 >= kDLo && d0 + 3 + kK <= dhi + kR) group(std::true_type{});
        else
#endif
            group(std::false_type{});
    }
    cp_wait<0>();
    if (b < T.nb) {  // the last block's sum
        const double s = warp_sum_down(B.rsum);
        if (lane == 0) sh.wsum[b] = s;
    }
    for (int o = 16; o > 0; o >>= 1) B.lmax = fmax(B.lmax, __shfl_xor_sync(kFull, B.lmax, o));
    if (lane == 0) sh.wmax[w] = B.lmax;
    bar_compute(nthr);
    if (w == 0 && lane == 0) {
        sh.aborted = aborted ? 1 : 0;
        *reinterpret_cast<volatile int*>(&sh.end) = 1;
    }
}

// The comm warp of a sweep: predecessor's progress in, this CTA's out, stop flag.
__device__ __forceinline__ void sp_comm(const Sp2D& D, Sp2Shared& sh, int g, int P) {
    if ((threadIdx.x & 31) == 0) {
        const unsigned long long prev_hi = (unsigned long long)(unsigned(g - 1)) << 32;
        const unsigned long long* pp = D.prog + (g > 0 ? (g - 1) % P : 0);
        unsigned long long* me = D.prog + blockIdx.x;
        int avail = g == 0 ? kInf : 0, last = -1;
        const long long t0 = gtimer();
        while (!ld_vol_s(&sh.end)) {
            if (avail < kInf) {
                const unsigned long long v = ld_acq_gpu(pp);
                if (v >= prev_hi) {
                    const unsigned lo = unsigned(v & 0xffffffffull);
                    const int a = ((v >> 32) > (unsigned long long)(g - 1) || lo == 0xffffffffu) ? kInf : int(lo);
                    if (a > avail) avail = a, st_rel_cta(&sh.avail, a);
                }
            }
            const int dt = ld_acq_cta(&sh.done_t);
            if (dt != last) {
                last = dt;
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(me),
                             "l"(((unsigned long long)(unsigned)g << 32) | unsigned(dt))
                             : "memory");
            }
            if (ld_rlx_gpu(D.st) < g) *reinterpret_cast<volatile int*>(&sh.abort_) = 1;
            if (timed_out(t0)) *reinterpret_cast<volatile int*>(&sh.abort_) = 1;
        }
    }
    __syncwarp();
}

// thread 0: may sweep g start? 1 go, 0 stop (past the first converged sweep or the budget)
__device__ int sp_start(const Sp2K& T, const Sp2D& D, int g, long long budget, int a0) {
    const long long t0 = gtimer();
    for (;;) {
        if (g >= budget || g > ld_rlx_gpu(D.st)) return 0;
        bool ok = g < a0 + 2 * ld_rlx_gpu(D.st + 1);  // at most a0 + 2 x (sweeps finished) in flight
        if (ok && g >= T.B)  // buffer g % B: sweep g-B decided, sweep g-B+1 done reading it
            ok = ld_acq_gpu(D.finw + g % T.B) == unsigned(g - T.B + 1) &&
                 ld_acq_gpu(D.finw + (g + 1) % T.B) == unsigned(g - T.B + 2);
        if (ok) return g > ld_rlx_gpu(D.st) ? 0 : 1;
        __nanosleep(64);
        if (timed_out(t0)) return 0;
    }
}

__global__ void __launch_bounds__(kSpThreads, 1) coarse_sp2_kernel(Params P, Sp2K T, Sp2D D) {
    Ctl* st = P.ctl;
    if (st->phase != kCoarse) return;
    const long long t_start = gtimer();
    __shared__ Sp2Shared sh;
    const int NW = T.nb;
    const int warp = threadIdx.x >> 5;
    const int NWc = T.nw;  // compute warps
    double* ringN = sp2_dyn;
    double* ringE = ringN + size_t(NWc) * kQ * kRows;
    double* ringB = ringE + size_t(NWc) * kQE * 32;
    double* ringX = ringB + size_t(NWc) * 2 * kQB * 32;
    double* tbl = ringX + size_t(NWc) * kQE;
    const int* ring_cls = reinterpret_cast<const int*>(tbl + 10 * (T.ncls + 1));
    SmemMap M;
    M.e = int(ringE - sp2_dyn), M.bu = int(ringB - sp2_dyn), M.x = int(ringX - sp2_dyn), M.tbl = int(tbl - sp2_dyn);
    const double rc0 = st->rc;  // max|cb|, formed by the fine pass that restricted
    const long long budget = P.max_total - st->total;
    const int pred = st->pred;
    const bool run = rc0 > P.tol_coarse && budget > 0;
    const unsigned nthreads = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x == 0) {  // per-visit state (nobody else touches it before the barrier)
        for (int k = threadIdx.x; k < T.P; k += blockDim.x) D.prog[k] = 0ull;
        for (int k = threadIdx.x; k < T.B; k += blockDim.x) D.finw[k] = 0u;
        if (threadIdx.x == 0) D.st[0] = kInf, D.st[1] = 0;
    }
    for (int k = threadIdx.x; k < T.spec_words; k += blockDim.x) tbl[k] = D.spec[k];
    for (int k = threadIdx.x; k < NWc * kQ * kRows; k += blockDim.x) ringN[k] = 0.0;  // rows -1 / 32 at the grid edge stay 0
    if (run) {  // the rhs into the diagonal layout: bd[b][d][l] = cb(d - 2 l, 32 b + l), 0 off the grid
        const int64_t n = int64_t(T.nb) * T.bstride;
        for (int64_t k = gtid; k < n; k += nthreads) {
            const int b = int(k / T.bstride);
            const int rem = int(k - int64_t(b) * T.bstride);
            const int l = rem & 31, d = (rem >> 5) - kDOff;
            const int I = d - 2 * l, J = 32 * b + l;
            D.bd[k] = (J < T.ncy && unsigned(I) < unsigned(T.ncx)) ? P.cb.at(I, J) : 0.0;
        }
    }
    sp_grid_sync(D.bar, gridDim.x);  // everyone has read Ctl; rhs and state ready
    const int a0 = 2 * max(1, pred) + 2;
    long long steps = 0;
    if (run) {
        for (int g = blockIdx.x;; g += gridDim.x) {
            if (threadIdx.x == 0) {
                sh.go = sp_start(T, D, g, budget, a0);
                sh.avail = g == 0 ? kInf : 0, sh.abort_ = 0, sh.done_t = 0, sh.end = 0, sh.aborted = 0;
                sh.dec[0] = sh.dec[1] = 0;
            }
            __syncthreads();
            if (!sh.go) break;
            const double* xo = g == 0 ? D.zero : D.bufs + size_t((g - 1) % T.B) * T.bufsz;
            double* xn = D.bufs + size_t(g % T.B) * T.bufsz;
            if (warp == NWc) sp_comm(D, sh, g, T.P);
            else sp_sweep(T, D, sh, M, ring_cls, xo, xn, g);
            __syncthreads();
            if (threadIdx.x == 0 && !sh.aborted) {
                double res = 0.0, sum = 0.0;
                for (int w = 0; w < NWc; ++w) res = fmax(res, sh.wmax[w]);
                for (int b = 0; b < NW; ++b) sum += sh.wsum[b];  // blocks in order
                D.resw[g % T.B] = res, D.sumw[g % T.B] = sum;
                if (!(res > P.tol_coarse)) atomicMin(D.st, g);
                __threadfence();
                st_rel_gpu(D.finw + g % T.B, unsigned(g + 1));
                atomicAdd(D.st + 1, 1);
                st_rel_gpu(D.prog + blockIdx.x, ((unsigned long long)(unsigned)g << 32) | 0xffffffffull);
            }
            __syncthreads();
        }
    }
    sp_grid_sync(D.bar, gridDim.x);
    int done = 0;
    double rc = rc0, sum = 0.0;
    const double* xk = nullptr;
    if (run) {
        const int first = *reinterpret_cast<volatile int*>(D.st);
        const int k = first < budget ? first : int(budget - 1);
        done = k + 1;
        rc = *reinterpret_cast<volatile double*>(D.resw + k % T.B);
        sum = *reinterpret_cast<volatile double*>(D.sumw + k % T.B);
        xk = D.bufs + size_t(k % T.B) * T.bufsz;
        steps = T.tend + 1;
    }
    // ce = the answer (anchored once when singular), natural layout
    const bool anchor = P.singular && done > 0;
    const double c = anchor ? -(sum / double(int64_t(T.ncx) * T.ncy)) : 0.0;
    const int64_t ncell = int64_t(T.ncx) * T.ncy;
    for (int64_t k = gtid; k < ncell; k += nthreads) {
        const int J = int(k / T.ncx), I = int(k - int64_t(J) * T.ncx);
        double v = 0.0;
        if (xk) {
            const int l = J & 31, b = J >> 5;
            v = xk[size_t(b) * T.bstride + size_t(I + 2 * l + kDOff) * 32 + l];
            if (anchor) v += c;
        }
        P.ce.at(I, J) = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->coarse_launches += 1;
        st->coarse_ns += gtimer() - t_start;
        st->coarse_steps += steps;
        st->coarse_group_ns += gtimer() - t_start;
        if (done > 0) st->pred = done;
        st->total += done;
        st->coarse += done;
        st->rc = rc;
        if (st->nvisits > 0 && st->nvisits <= P.visit_cap) P.visit_log[2 * (st->nvisits - 1)] = done;
        if (*(volatile unsigned*)&g_sp2_stuck) st->mp_error = 2;
        if (rc > P.tol_coarse || st->mp_error) {  // cycles.hpp:134-137
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

}  // namespace

struct Sp2Engine {
    Sp2K T{};
    Sp2D D{};
    void* mem = nullptr;
    size_t smem = 0;
};

// Host plan: a non-periodic 9-point operator whose zero weights face only ghosts
// (StencilClasses kind 0), at most 16 blocks of 32 rows, every CTA resident.
Sp2Engine* sp2_try_create(const CoarseOpH& op, int device) {
    if (const char* e = getenv("ISMG_COARSE_SP2"))
        if (e[0] == '0') return nullptr;
    StencilClasses S;
    if (!stencil_classes(op, S) || S.kind != 0 || !S.fastdiv) return nullptr;
    const int nb = (op.ncy + 31) / 32;
    if (nb > kMaxB) return nullptr;
    // compute warps: a warp's next block (b + nw) may start only after block b's
    // last ring access, nw - 1 block strides later
    const int nw = std::min(nb, 2 + (op.ncx + kDHiPad + kR - kDLo + kQ) / kStride);
    if (nw + 1 > kSpThreads / 32) return nullptr;
    {  // the first / last row: one class on columns 1 .. ncx-2 (the kernel's row body)
        const int* rc = reinterpret_cast<const int*>(S.spec.data() + size_t(10) * (S.ncls + 1));
        for (int I = 2; I < op.ncx - 1; ++I)
            if (rc[I] != rc[1] || rc[op.ncx + I] != rc[op.ncx + 1]) return nullptr;
    }
    Sp2K T{};
    T.ncx = op.ncx, T.ncy = op.ncy, T.nb = nb, T.nw = nw;
    T.dspan = op.ncx + kDSpanPad;
    T.bstride = int64_t(T.dspan) * 32;
    T.bufsz = T.bstride * nb;
    T.ncls = S.ncls, T.ring = S.ring;
    T.spec_words = int(S.spec.size());
    T.singular = op.singular ? 1 : 0;
    T.tend = (op.ncx + kDHiPad + kR - kDLo) + kStride * (nb - 1);
    const size_t smem = sizeof(double) * (size_t(nw) * (kQ * kRows + kQE * 32 + 2 * kQB * 32 + kQE) + S.spec.size());
    ISMG_CUDA(cudaFuncSetAttribute(coarse_sp2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0, sms = 0;
    ISMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_sp2_kernel, 32 * (nw + 1), smem));
    ISMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (per_sm < 1) return nullptr;
    int P = sms;
    if (const char* e = getenv("ISMG_SP_CTAS")) P = std::max(1, std::min(sms, atoi(e)));  // tuning hook
    T.P = P, T.B = P + 2;
    auto* e = new Sp2Engine();
    e->T = T;
    e->smem = smem;
    const size_t bufb = sizeof(double) * size_t(T.bufsz);
    const size_t bytes = bufb * size_t(T.B + 2) + sizeof(double) * S.spec.size() + sizeof(unsigned long long) * P +
                         sizeof(unsigned) * T.B + 2 * sizeof(double) * T.B + 64 + 1024;
    ISMG_CUDA(cudaMalloc(&e->mem, bytes));
    ISMG_ZERO(e->mem, bytes);
    char* p = static_cast<char*>(e->mem);
    e->D.bufs = reinterpret_cast<double*>(p), p += bufb * T.B;
    e->D.zero = reinterpret_cast<double*>(p), p += bufb;
    e->D.bd = reinterpret_cast<double*>(p), p += bufb;
    double* spec = reinterpret_cast<double*>(p);
    ISMG_H2D(spec, S.spec.data(), sizeof(double) * S.spec.size());
    e->D.spec = spec, p += sizeof(double) * S.spec.size();
    e->D.resw = reinterpret_cast<double*>(p), p += sizeof(double) * T.B;
    e->D.sumw = reinterpret_cast<double*>(p), p += sizeof(double) * T.B;
    e->D.prog = reinterpret_cast<unsigned long long*>(p), p += sizeof(unsigned long long) * P;
    e->D.finw = reinterpret_cast<unsigned*>(p), p += sizeof(unsigned) * T.B;
    p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 63) & ~uintptr_t(63));
    e->D.st = reinterpret_cast<int*>(p), p += 64;
    e->D.bar = reinterpret_cast<unsigned*>(p);
    return e;
}

void sp2_destroy(Sp2Engine* e) {
    if (!e) return;
    cudaFree(e->mem);
    delete e;
}

void launch_coarse_sp2(const Params& P, const Sp2Engine& e, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(e.T.P));
    cfg.blockDim = dim3(unsigned(32 * (e.T.nw + 1)));
    cfg.dynamicSmemBytes = e.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ISMG_CUDA(cudaLaunchKernelEx(&cfg, coarse_sp2_kernel, P, e.T, e.D));
}

}  // namespace fz
}  // namespace ismgb

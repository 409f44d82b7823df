// coarse_sp.cu — the coarse visit (cycles.hpp:120-137; coarsening.hpp:531-567)
// as a pipeline of whole sweeps over the SMs.
//
// gs_sweep_lex is lexicographic Gauss-Seidel: cell (I,J) of sweep g needs the
// sweep-g values of W, SW, S, SE and the sweep-(g-1) values of E, NW, N, NE.
// Within one sweep the cells on a diagonal I + 2J are independent, so a sweep
// is a wavefront of ncx + 2 ncy steps; between sweeps the only dependency is
// "sweep g reads what sweep g-1 wrote, a few columns ahead". This engine gives
// every sweep its own CTA (one per SM, cooperative launch):
//
//  * inside the CTA, lane l of compute warp b owns row J = 32 b + l; block b
//    runs kStride = 64 + kD steps behind block b-1 (the skew kD lets the warps
//    meet at a named barrier only every kS steps). The wavefront's critical
//    path never leaves the SM: in-warp neighbours through a shared-memory ring
//    of the sweep's new values, block edges mirrored into the neighbour warp's
//    ring;
//  * the sweep-(g-1) values and the rhs arrive by cp.async, kK steps ahead,
//    from L2 buffers in a diagonal layout (a warp's 32 lanes read 256
//    contiguous bytes per step); the sweep's own values go out the same way;
//  * CTA g runs ~30 steps behind CTA g-1: a comm warp per CTA publishes the
//    CTA's progress (release, gpu scope) and polls its predecessor's, so the
//    SM-to-SM latency (~1 us) sits in that lag, not in the wavefront;
//  * the residual of sweep g (coarse_residual, for the stop test after every
//    sweep) is formed kR steps behind the update from the same ring; the CTA
//    folds the sweep's max|r| and Σx (anchor) when the sweep ends.
//
// Sweeps are taken in order by the CTAs (CTA c: sweeps c, c + P, ...), each
// writing its own buffer (ring of B = P + 2), so no checkpoint and no replay:
// the first sweep whose residual passes tol_coarse is the answer; later sweeps
// in flight abort. A visit of G sweeps costs one wavefront plus G-1 lags; a
// long visit runs P sweeps at once. Results are the reference's bit for bit
// (same per-cell operation order; division correctly rounded, kernels.cuh).
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

#ifndef ISMG_SP_S
#define ISMG_SP_S 4
#endif
constexpr int kS = ISMG_SP_S;          // steps between named barriers of the compute warps (4 or 8)
constexpr int kD = kS - 1;             // skew between consecutive 32-row blocks (steps)
#ifdef ISMG_SP_INLINE_RES
constexpr int kR = 3 + kD + kS;        // residual lag (steps): row 32's mirror value is >= kS steps old
#else
constexpr int kR = 0;                  // the residual is a pass over the sweep's output (no lag)
#endif
#ifndef ISMG_SP_K
#define ISMG_SP_K 5
#endif
constexpr int kK = ISMG_SP_K;          // cp.async prefetch distance (steps)
constexpr int kQ = 24;                 // new-value ring slots (3 segments of 8)
constexpr int kQE = 8, kQB = 16;       // old-value / rhs ring slots
constexpr int kEW = 33;                // old-value ring row: lanes 0..31 + row 32 (the next block's row 0, lane 31's NE)
constexpr int kRows = 34;              // ring rows: block rows -1 .. 32
constexpr int kMaxW = 16;              // compute warps (32-row blocks)
constexpr int kStride = 64 + kD;       // CTA steps between consecutive blocks
constexpr int kDLo = -4;               // first diagonal of a block's loop (ghost columns written as 0)
constexpr int kDHiPad = 63;            // last update diagonal: ncx + kDHiPad
constexpr int kDOff = 72;              // layouts: diagonal d of block b at [b][d + kDOff][lane]
constexpr int kDSpanPad = 168;         // diagonals per block: ncx + kDSpanPad
constexpr int kSpThreads = 32 * (kMaxW + 1);
constexpr int kInf = INT_MAX;

static_assert(kS == 4 || kS == 8, "barrier interval divides the 8-step iteration");
static_assert(kK + kR + 1 <= kQB, "rhs ring: slots of the residual's rhs live until the update overwrites them");
static_assert(kK + 1 <= kQE, "old-value ring");
#ifdef ISMG_SP_INLINE_RES
static_assert(kD + kR + 2 * kS <= kQ, "new-value ring: live span (mirror writes ahead, residual reads behind)");
#else
static_assert(kD + kS < kQ, "new-value ring: a row -1 mirror slot is read before block b-1 rewrites it");
#endif
static_assert(kK - 2 >= 1, "prefetch must run ahead of the NE read (t + 2)");

__device__ unsigned g_sp_stuck = 0u;
#ifdef ISMG_SP_TRACE  // phase clock of CTA 0 (ns, accumulated): setup, sweep 0, loop rest, grid sync, write-out, visits
__device__ unsigned long long g_sp_trace[6];
#define SP_TRACE(i, t) (g_sp_trace[i] += (unsigned long long)(t))
#endif  // watchdog: a wait ran past 2 s

}  // namespace

struct SpK {
    int ncx, ncy, nb;        // coarse grid, 32-row blocks (= compute warps)
    int P, B;                // CTAs (sweeps in flight), buffers
    int dspan;               // diagonals per block in the layouts
    int64_t bstride, bufsz;  // doubles per block / per buffer
    int ncls, ring, spec_words;
    int singular;
    int tend;                // last CTA step of a sweep
    int nseg, seglen;        // residual chunks: nb blocks x nseg diagonal segments of seglen
};

struct SpD {
    double* bufs;                // [B][nb][dspan][32] sweep outputs (diagonal layout)
    double* zero;                // one all-zero buffer: sweep -1 (ce = 0) and missing blocks
    double* bd;                  // rhs, diagonal layout
    const double* spec;          // class table (stencil_classes)
    unsigned long long* prog;    // [P] progress: (sweep << 32) | steps done (0xffffffff: sweep finished)
    unsigned* finw;              // [B] sweep g done: finw[g % B] = g + 1
    double* resw;                // [B] residual max of sweep g
    double* sumw;                // [B] Σ x of sweep g (anchor)
    int* st;                     // [0] first converged sweep (INT_MAX none), [1] sweeps finished, [2] oldest
                                 // sweep whose residual chunks may be unclaimed
    unsigned* bar;               // grid barrier: [0] arrivals, [1] generation
    unsigned* rready;            // [B] sweep g's output complete, its residual chunks claimable: g + 1
    unsigned* rclaim;            // [B] residual chunks claimed
    unsigned* rdone;             // [B] residual chunks done
    unsigned long long* rbits;   // [B] residual max so far (bits of a non-negative double: ordered as integers)
};

namespace {

extern __shared__ __align__(16) double sp_dyn[];

// ISMG_SP_CHECK builds (tools/build_variant.sh): bounds of every ring slot and
// layout diagonal, trapping on the first violation (compute-sanitizer is not
// available on this pool).
#ifdef ISMG_SP_CHECK
#define SP_ASSERT(c, what)                                                                     \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("coarse_sp bounds: %s (block %d thread %d)\n", what, blockIdx.x, threadIdx.x); \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define SP_ASSERT(c, what) (void)0
#endif

__device__ __forceinline__ void cp8(uint32_t dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// shared-memory loads / stores by 32-bit address (the rings: no generic-to-shared
// conversion and no 64-bit address arithmetic per step)
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double2 lds128(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
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
        atomicExch(&g_sp_stuck, 1u);
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

struct SpShared {
    int avail;      // steps of sweep g-1 available (from the comm warp)
    int abort_;     // sweep g > first converged sweep: stop
    int done_t;     // steps of this sweep done (for the comm warp to publish)
    int end;        // compute warps finished the sweep
    int aborted;
    int go;
    int dec[2];     // abort decision per barrier parity
    int rs, rbase;  // residual chunks claimed: sweep, first chunk
    double wmax[kMaxW], wsum[kMaxW];
};

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

// One sweep of one compute warp (32-row block b) over CTA steps -8 .. tend.
// Lane l: row J = 32 b + l, update column I = d - 2 l, residual column I - kR,
// d = t + kDLo - kStride b. Per step: prefetch (cp.async) for step t + kK, the
// update (weights of the cell's class from the table: west column, row body,
// east column), the residual kR columns behind, a named barrier every kS steps.
__device__ __forceinline__ void sp_sweep(const SpK& T, const SpD& D, SpShared& sh, double* ringN, double* ringE,
                                         double* ringB, const double* tbl, const int* ring_cls,
                                         const double* __restrict__ xo, double* __restrict__ xn, int g) {
    const int b = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nthr = 32 * T.nb;
    const int ncx = T.ncx, ncy = T.ncy;
    const int J = 32 * b + lane;
    const bool rowok = J < ncy;
    const int dhi = ncx + kDHiPad;
    // classes of this lane's row: column 0, columns 1 .. ncx-2 (one class, checked by the plan), column ncx-1
    int wcls = T.ncls, bcls = T.ncls, ecls = T.ncls;
    if (rowok) {
        if (J == 0 || J == ncy - 1) {
            const int rb = J == 0 ? 0 : ncx;
            wcls = ring_cls[rb], bcls = ring_cls[rb + 1], ecls = ring_cls[rb + ncx - 1];
        } else {
            wcls = ring_cls[2 * ncx + J], ecls = ring_cls[2 * ncx + ncy + J];
        }
    }
    // rings of this warp (new values: [kQ][kRows]; the neighbour blocks' rings sit kQ kRows doubles away)
    double* rN = ringN + size_t(b) * kQ * kRows;
    double* rE = ringE + size_t(b) * kQE * kEW + lane;
    double* rB = ringB + size_t(b) * kQB * 32 + lane;
    const uint32_t sE = su32(rE), sB = su32(rB);
    const uint32_t sN = su32(rN) + 8u * uint32_t(lane), sT = su32(tbl);  // this lane's ring column, class table
    const bool has_n = b + 1 < T.nb;
#ifdef ISMG_SP_INLINE_RES
    const bool has_p = b > 0;
#endif
    const double* xo_b = xo + size_t(b) * T.bstride + lane;
    const double* xo_n = (has_n ? xo + size_t(b + 1) * T.bstride : D.zero);  // row 32 (b+1) = next block's lane 0
    const double* bd_b = D.bd + size_t(b) * T.bstride + lane;
    double* xn_b = xn + size_t(b) * T.bstride + lane;
    // update: W (own previous output), S / SW (previous SE), N / NW (previous NE)
    double outP = 0.0, seP = 0.0, seP2 = 0.0, neP = 0.0, neP2 = 0.0;
    // residual window: rows r-1 (S*), r (W C E), r+1 (N*)
#ifdef ISMG_SP_INLINE_RES
    double qSW = 0.0, qS = 0.0, qSE = 0.0, qW = 0.0, qC = 0.0, qE = 0.0, qNW = 0.0, qN = 0.0, qNE = 0.0;
#endif
    double lmax = 0.0, rsum = 0.0;
    int avail = g == 0 ? kInf : 0;
    int h = 0;
    bool aborted = false;
    const int mend = T.tend >> 3;
    for (int m = -1; m <= mend && !aborted; ++m) {
#ifndef ISMG_SP_NOIDLE
        // a group of 8 steps with neither a prefetch nor an update for this block (before or
        // after its diagonal window): only the barriers. Idle warps otherwise issue ~30
        // instructions per step, taking issue slots from the active warps on their SMSP.
        if (8 * m + kDLo - kStride * b + 7 + kK < kDLo || 8 * m + kDLo - kStride * b > dhi + kR) {
#pragma unroll
            for (int j = kS - 1; j < 8; j += kS) {
                if (b == 0 && lane == 0) sh.dec[h & 1] = ld_vol_s(&sh.abort_);
                bar_compute(nthr);
                if (b == 0 && lane == 0) st_rel_cta(&sh.done_t, max(0, 8 * m + j + 1));
                aborted = ld_vol_s(&sh.dec[h & 1]) != 0;
                ++h;
                if (aborted) break;
            }
            continue;
        }
#endif
        // new-value ring segments (8 slots each) of steps 8(m-1).., 8m.., 8(m+1).. (= 8(m-2)..)
        const int m3 = (m + 3) % 3;
        const int sA = ((m3 + 2) % 3) * 8 * kRows, sBn = m3 * 8 * kRows, sC = ((m3 + 1) % 3) * 8 * kRows;
        const int b0 = (m & 1) * 8 * 32, b1 = ((m + 1) & 1) * 8 * 32;  // rhs ring segments by parity
        const int d0 = 8 * m + kDLo - kStride * b;                       // diagonal of step j = 0
        const size_t o0 = size_t(d0 + kDOff) * 32;                        // layout offset of d0 (d0 + kDOff >= 0)
        const double* pE = xo_b + o0 + size_t(kK + 1) * 32;              // E of step j + kK: diagonal d + kK + 1
        const double* pB = bd_b + o0 + size_t(kK) * 32;
        const double* pX = xo_n + o0 + size_t(kK) * 32 - 61 * 32;        // lane 31: row 32, column I + 1
        double* pO = xn_b + o0;
        // a group whose 8 steps all prefetch and update (the common case) runs without the
        // per-step window tests, so the history registers rotate without copies
        auto group = [&](auto fullc) {
            constexpr bool FULL = decltype(fullc)::value;
    #pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int t = 8 * m + j;
                auto nslot = [&](int q) {  // ring offset of CTA step 8m + q (q folds to a constant)
                    const int seg = q >> 3;
                    return (seg == 0 ? sBn : (seg == -1 ? sA : sC)) + (q & 7) * kRows;
                };
                auto bslot = [&](int q) { return (((q >> 3) & 1) ? b1 : b0) + (q & 7) * 32; };
                if ((j & 3) == 0 && avail < min(t + 3 + kK + kD + 4, T.tend + 1)) {  // sweep g-1 far enough
                    const int need = min(t + 3 + kK + kD + 4, T.tend + 1);  // (its last step: no wait for its fold)
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
                const int d = d0 + j;
    #ifndef ISMG_SPX_NOCP
                if (FULL || (d + kK >= kDLo && d + kK <= dhi + kR)) {  // prefetch for step t + kK
                    SP_ASSERT(d + kK - 61 + kDOff >= 0 && d + kK + 1 + kDOff < T.dspan, "prefetch diagonal");
                    SP_ASSERT(bslot(j + kK) >= 0 && bslot(j + kK) < kQB * 32, "rhs ring slot");
                    cp8(sE + 8u * uint32_t(((j + kK) & 7) * kEW), pE + 32 * j);
                    cp8(sB + 8u * uint32_t(bslot(j + kK)), pB + 32 * j);
                    // lane 31: row 32 into position 32 of the slot its NE read of step t + kK uses
                    if (lane == 31) cp8(sE + 8u * uint32_t(((j + kK + 2) & 7) * kEW + 1), pX + 32 * j);
                }
    #endif
                cp_commit();
                cp_wait<kK - 2>();
                __syncwarp();
                if (FULL || (d >= kDLo && d <= dhi + kR)) {
                    // ---- update of column I (sweep g) ----
                    const int I = d - 2 * lane;
                    const bool act_u = rowok && unsigned(I) < unsigned(ncx) && d <= dhi;
                    SP_ASSERT(nslot(j - kR - 1) >= 0 && nslot(j + kD) + kRows <= kQ * kRows, "new-value ring slot");
                    SP_ASSERT(bslot(j - kR) >= 0 && bslot(j) < kQB * 32, "rhs ring slot");
                    SP_ASSERT(d + kDOff >= 0 && d + kDOff < T.dspan, "output diagonal");
                    SP_ASSERT(!has_n || b + 1 < T.nb, "mirror target");
                    const double E = lds64(sE + 8u * uint32_t((j & 7) * kEW));
                    const double NE = lds64(sE + 8u * uint32_t(((j + 2) & 7) * kEW + 1));  // lane 31: position 32
                    const double SE = lds64(sN + 8u * uint32_t(nslot(j - 1)));
                    const double bu = lds64(sB + 8u * uint32_t(bslot(j)));
                    const uint32_t wu = sT + 80u * uint32_t(I == 0 ? wcls : (I == ncx - 1 ? ecls : bcls));
                    const double2 u01 = lds128(wu), u23 = lds128(wu + 16), u45 = lds128(wu + 32), u67 = lds128(wu + 48),
                                  u89 = lds128(wu + 64);
                    double acc = 0.0;
                    acc += u01.y * E;
                    acc += u23.x * outP;
                    acc += u23.y * neP;
                    acc += u45.x * seP;
                    acc += u45.y * NE;
                    acc += u67.x * neP2;
                    acc += u67.y * SE;
                    acc += u89.x * seP2;
                    const double num = act_u ? bu - acc : 1.0;
                    const double q = div_full(num, u01.x, u89.y);
                    const double out = act_u ? q : 0.0;
                    sts64(sN + 8u * uint32_t(nslot(j) + 1), out);
                    if (lane == 31 && has_n) sts64(sN + 8u * uint32_t(kQ * kRows + nslot(j + kD) - 31), out);  // row -1 of the next block
    #ifdef ISMG_SP_INLINE_RES
                    if (lane == 0 && has_p) rN[nslot(j - kD) + 33 - kQ * kRows] = out;  // row 32 of the previous block
    #endif
    #ifndef ISMG_SPX_NOSTG
                    if (d <= dhi) pO[32 * j] = out;
    #endif
                    if (act_u) rsum += out;
                    seP2 = seP, seP = SE, neP2 = neP, neP = NE, outP = out;
    #ifdef ISMG_SP_INLINE_RES
                    // ---- residual of column I - kR (sweep g values on all nine points) ----
                    const int Ir = I - kR;
                    const bool act_r = rowok && unsigned(Ir) < unsigned(ncx);
                    qSW = qS, qS = qSE, qSE = rN[nslot(j - kR - 1) + lane];
                    qW = qC, qC = qE, qE = rN[nslot(j - kR + 1) + lane + 1];
                    qNW = qN, qN = qNE, qNE = rN[nslot(j - kR + 3) + lane + 2];
                    const double br = rB[bslot(j - kR)];
                    const double2* wr = reinterpret_cast<const double2*>(
                        tbl + 10 * (Ir == 0 ? wcls : (Ir == ncx - 1 ? ecls : bcls)));
                    const double2 r01 = wr[0], r23 = wr[1], r45 = wr[2], r67 = wr[3], r89 = wr[4];
                    double a = r01.x * qC;
                    a += r01.y * qE;
                    a += r23.x * qW;
                    a += r23.y * qN;
                    a += r45.x * qS;
                    a += r45.y * qNE;
                    a += r67.x * qNW;
                    a += r67.y * qSE;
                    a += r89.x * qSW;
                    double mm = act_r ? fabs(br - a) : 0.0;
                    mm = (mm != mm) ? 0.0 : mm;  // std::max drops NaN
                    lmax = fmax(lmax, mm);
    #endif
                }
    #ifdef ISMG_SPX_NOBAR
                if (false) {
    #else
                if ((j % kS) == kS - 1) {
    #endif  // named barrier of the compute warps every kS steps
                    if (b == 0 && lane == 0) sh.dec[h & 1] = ld_vol_s(&sh.abort_);
                    bar_compute(nthr);
                    if (b == 0 && lane == 0) st_rel_cta(&sh.done_t, max(0, t + 1));
                    aborted = ld_vol_s(&sh.dec[h & 1]) != 0;
                    ++h;
                    if (aborted) break;
                }
            }
        };
        if (d0 >= kDLo && d0 + 7 + kK <= dhi + kR) group(std::true_type{});
        else group(std::false_type{});
    }
    cp_wait<0>();
#ifndef ISMG_SP_INLINE_RES
    // (the sweep's residual: chunks over the SMs after the wavefront, sp_res_chunk)
#endif
    // fold: max|r| (order-free), Σx in a fixed order (lanes by tree, blocks in order)
    for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(kFull, lmax, o));
    rsum = warp_sum_down(rsum);
    if (lane == 0) sh.wmax[b] = lmax, sh.wsum[b] = rsum;
    bar_compute(nthr);
    if (b == 0 && lane == 0) {
        sh.aborted = aborted ? 1 : 0;
        *reinterpret_cast<volatile int*>(&sh.end) = 1;
    }
}

// The comm warp of a sweep: predecessor's progress in, this CTA's out, stop flag.
__device__ __forceinline__ void sp_comm(const SpD& D, SpShared& sh, int g, int P) {
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

// One residual chunk of sweep g (coarse_residual, the stop test after every sweep),
// by one warp: block bb's diagonals [d0, d1) of the sweep's output buffer. Lane l
// keeps x(d-3 .. d+3) of its row (J = 32 bb + l) in registers, one coalesced load
// per diagonal; rows J +- 1 come from lanes l +- 1 by shuffle and across the block
// edges from the neighbour blocks' lane 0 / 31 (zero buffer past the grid). Class
// weights and operation order are the update's. Returns the lanes' max |r|.
__device__ double sp_res_chunk(const SpK& T, const SpD& D, const double* tbl, const int* ring_cls, int g, int chunk) {
    const int lane = threadIdx.x & 31, ncx = T.ncx, ncy = T.ncy;
    const int bb = chunk / T.nseg, sg = chunk - bb * T.nseg;
    const int span = ncx + 62;
    const int d0 = sg * T.seglen, d1 = min(span, d0 + T.seglen);
    const double* xn = D.bufs + size_t(g % T.B) * T.bufsz;
    const int J = 32 * bb + lane;
    const bool rowok = J < ncy;
    int wcls = T.ncls, bcls = T.ncls, ecls = T.ncls;
    if (rowok && J != 0 && J != ncy - 1) wcls = ring_cls[2 * ncx + J], ecls = ring_cls[2 * ncx + ncy + J];
    const double* Xb = xn + int64_t(bb) * T.bstride + kDOff * 32 + lane;
    const double* Bb = D.bd + int64_t(bb) * T.bstride + kDOff * 32 + lane;
    const double* Xn = (bb + 1 < T.nb ? xn + int64_t(bb + 1) * T.bstride : D.zero) + kDOff * 32;      // lane 0
    const double* Xp = (bb > 0 ? xn + int64_t(bb - 1) * T.bstride : D.zero) + kDOff * 32 + 31;        // lane 31
    double lmax = 0.0;
    if (d0 >= d1) return lmax;
    double w0 = Xb[(d0 - 3) * 32], w1 = Xb[(d0 - 2) * 32], w2 = Xb[(d0 - 1) * 32], w3 = Xb[d0 * 32],
           w4 = Xb[(d0 + 1) * 32], w5 = Xb[(d0 + 2) * 32];
#pragma unroll 4
    for (int dd = d0; dd < d1; ++dd) {
        const double w6 = Xb[(dd + 3) * 32];  // x(d+3)
        const double bv = Bb[dd * 32];
        double N = __shfl_down_sync(kFull, w5, 1), NE = __shfl_down_sync(kFull, w6, 1),
               NW = __shfl_down_sync(kFull, w4, 1);
        double S = __shfl_up_sync(kFull, w1, 1), SE = __shfl_up_sync(kFull, w2, 1),
               SW = __shfl_up_sync(kFull, w0, 1);
        if (lane == 31 && dd >= 62) N = Xn[(dd - 62) * 32], NE = Xn[(dd - 61) * 32], NW = Xn[(dd - 63) * 32];
        if (lane == 0 && dd < ncx) S = Xp[(dd + 62) * 32], SE = Xp[(dd + 63) * 32], SW = Xp[(dd + 61) * 32];
        const int I = dd - 2 * lane;
        if (rowok && unsigned(I) < unsigned(ncx)) {
            const int cls = (J == 0 || J == ncy - 1) ? ring_cls[(J == 0 ? 0 : ncx) + I]
                                                      : (I == 0 ? wcls : (I == ncx - 1 ? ecls : bcls));
            const double2* w = reinterpret_cast<const double2*>(tbl + 10 * cls);
            const double2 r01 = w[0], r23 = w[1], r45 = w[2], r67 = w[3], r89 = w[4];
            double a = r01.x * w3;
            a += r01.y * w4;
            a += r23.x * w2;
            a += r23.y * N;
            a += r45.x * S;
            a += r45.y * NE;
            a += r67.x * NW;
            a += r67.y * SE;
            a += r89.x * SW;
            double mm = fabs(bv - a);
            mm = (mm != mm) ? 0.0 : mm;  // std::max drops NaN
            lmax = fmax(lmax, mm);
        }
        w0 = w1, w1 = w2, w2 = w3, w3 = w4, w4 = w5, w5 = w6;
    }
    return lmax;
}

// thread 0: claim up to `want` residual chunks of the oldest sweep that has some
// unclaimed (sweeps publish rready in order). Returns the sweep (or -1), *base the
// first chunk claimed.
__device__ int sp_claim(const SpK& T, const SpD& D, int want, int* base) {
    const int nchunk = T.nb * T.nseg;
    for (int tries = 0; tries < 4; ++tries) {
        const int s = ld_rlx_gpu(D.st + 2);
        if (ld_acq_gpu(D.rready + s % T.B) != unsigned(s + 1)) return -1;  // not published (yet)
        const unsigned c = atomicAdd(D.rclaim + s % T.B, unsigned(want));
        if (c < unsigned(nchunk)) {
            *base = int(c);
            return s;
        }
        atomicCAS(D.st + 2, s, s + 1);  // every chunk of s claimed: move on
    }
    return -1;
}

// every compute warp takes one chunk of sweep s (chunks base .. base + nw - 1); the
// warp that completes the sweep's last chunk decides it: residual, stop, done.
__device__ void sp_res_work(const SpK& T, const SpD& D, const Params& P, const double* tbl, const int* ring_cls,
                            int s, int base) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunk = T.nb * T.nseg;
    const int chunk = base + w;
    if (s < 0 || w >= T.nb || chunk >= nchunk) return;
    double m = sp_res_chunk(T, D, tbl, ring_cls, s, chunk);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) {
        atomicMax(D.rbits + s % T.B, (unsigned long long)__double_as_longlong(m));
        __threadfence();
        if (atomicAdd(D.rdone + s % T.B, 1u) == unsigned(nchunk - 1)) {  // the sweep's last chunk
            __threadfence();
            const double res = __longlong_as_double((long long)ld_acq_gpu(D.rbits + s % T.B));
            D.resw[s % T.B] = res;
            if (!(res > P.tol_coarse)) atomicMin(D.st, s);
            __threadfence();
            st_rel_gpu(D.finw + s % T.B, unsigned(s + 1));
            atomicAdd(D.st + 1, 1);
        }
    }
}

// thread 0: may sweep g start? 1 go, 0 stop (past the first converged sweep or the budget)
__device__ int sp_start(const SpK& T, const SpD& D, int g, long long budget, int a0) {
    if (g > ld_rlx_gpu(D.st)) return 0;
    if (g >= budget)  // no sweep to run: help until the sweeps below the budget have every chunk claimed
        return ld_rlx_gpu(D.st + 2) >= budget ? 0 : 2;
    bool ok = g < a0 + 2 * ld_rlx_gpu(D.st + 1);  // at most a0 + 2 x (sweeps finished) in flight
    if (ok && g >= T.B)  // buffer g % B: sweep g-B decided, sweep g-B+1 done reading it
        ok = ld_acq_gpu(D.finw + g % T.B) == unsigned(g - T.B + 1) &&
             ld_acq_gpu(D.finw + (g + 1) % T.B) == unsigned(g - T.B + 2);
    if (ok) return g > ld_rlx_gpu(D.st) ? 0 : 1;
    return 2;  // wait (and help with residual chunks)
}

__global__ void __launch_bounds__(kSpThreads, 1) coarse_sp_kernel(Params P, SpK T, SpD D) {
    Ctl* st = P.ctl;
    if (st->phase != kCoarse) return;
    const long long t_start = gtimer();
    __shared__ SpShared sh;
    const int NW = T.nb;
    const int warp = threadIdx.x >> 5;
    // shared memory: new-value rings [NW][kQ][kRows] | old [NW][kQE][kEW] | rhs [NW][kQB][32] | table
    double* ringN = sp_dyn;
    double* ringE = ringN + size_t(NW) * kQ * kRows;
    double* ringB = ringE + size_t(NW) * kQE * kEW;
    double* tbl = ringB + size_t(NW) * kQB * 32;
    const int* ring_cls = reinterpret_cast<const int*>(tbl + 10 * (T.ncls + 1));
    const double rc0 = st->rc;  // max|cb|, formed by the fine pass that restricted
    const long long budget = P.max_total - st->total;
    const int pred = st->pred;
    const bool run = rc0 > P.tol_coarse && budget > 0;
    const unsigned nthreads = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x == 0) {  // per-visit state (nobody else touches it before the barrier)
        for (int k = threadIdx.x; k < T.P; k += blockDim.x) D.prog[k] = 0ull;
        for (int k = threadIdx.x; k < T.B; k += blockDim.x) D.finw[k] = 0u, D.rready[k] = 0u;
        if (threadIdx.x == 0) D.st[0] = kInf, D.st[1] = 0, D.st[2] = 0;
    }
    for (int k = threadIdx.x; k < T.spec_words; k += blockDim.x) tbl[k] = D.spec[k];
    for (int k = threadIdx.x; k < NW * kQ * kRows; k += blockDim.x) ringN[k] = 0.0;  // rows -1 / 32 at the grid edge stay 0
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
#ifdef ISMG_SP_TRACE
    long long tr1 = gtimer(), tr2 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) SP_TRACE(0, tr1 - t_start), SP_TRACE(5, 1);
#endif
    const int a0 = 2 * max(1, pred) + 2;
    long long steps = 0;
    if (run) {
        for (int g = blockIdx.x;; g += gridDim.x) {
            // until sweep g may start: help with residual chunks of finished sweeps
            const long long tw = gtimer();
            for (;;) {
                if (threadIdx.x == 0) {
                    sh.go = sp_start(T, D, g, budget, a0);
                    sh.rs = -1;
                    if (sh.go == 2) {
                        int base = 0;
                        sh.rs = sp_claim(T, D, NW, &base);
                        sh.rbase = base;
                        if (sh.rs >= 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // also drops stale L1 lines
                        else if (timed_out(tw)) sh.go = 0;
                    }
                }
                __syncthreads();
                if (sh.go != 2) break;
                if (sh.rs >= 0) sp_res_work(T, D, P, tbl, ring_cls, sh.rs, sh.rbase);
                else if (threadIdx.x == 0) __nanosleep(64);
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                sh.avail = g == 0 ? kInf : 0, sh.abort_ = 0, sh.done_t = 0, sh.end = 0, sh.aborted = 0;
                sh.dec[0] = sh.dec[1] = 0;
            }
            __syncthreads();
            if (!sh.go) break;
            const double* xo = g == 0 ? D.zero : D.bufs + size_t((g - 1) % T.B) * T.bufsz;
            double* xn = D.bufs + size_t(g % T.B) * T.bufsz;
            if (warp == NW) sp_comm(D, sh, g, T.P);
            else sp_sweep(T, D, sh, ringN, ringE, ringB, tbl, ring_cls, xo, xn, g);
            __syncthreads();
#ifdef ISMG_SP_TRACE
            if (g == 0 && threadIdx.x == 0) tr2 = gtimer(), SP_TRACE(1, tr2 - tr1);
#endif
            if (threadIdx.x == 0 && !sh.aborted) {  // publish the sweep's residual chunks
                double sum = 0.0;
                for (int w = 0; w < NW; ++w) sum += sh.wsum[w];  // blocks in order
                D.sumw[g % T.B] = sum;
                D.rbits[g % T.B] = 0ull, D.rclaim[g % T.B] = 0u, D.rdone[g % T.B] = 0u;
                __threadfence();  // the sweep's output (every warp's stores: the CTA barrier above) first
                st_rel_gpu(D.rready + g % T.B, unsigned(g + 1));
                // the whole sweep to its consumer (the comm warp may have left before the last step's count)
                st_rel_gpu(D.prog + blockIdx.x, ((unsigned long long)(unsigned)g << 32) | 0xffffffffull);
            }
            __syncthreads();
            // work on this sweep's residual until every chunk is claimed (helpers take the rest)
            if (!sh.aborted) {
                for (;;) {
                    if (threadIdx.x == 0) {
                        int base = 0;
                        const int s2 = sp_claim(T, D, NW, &base);
                        sh.rs = s2, sh.rbase = base;
                        if (s2 >= 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        // done when this sweep's chunks are all claimed
                        sh.go = (s2 < 0 || s2 > g) ? 0 : 1;
                    }
                    __syncthreads();
                    if (sh.rs >= 0) sp_res_work(T, D, P, tbl, ring_cls, sh.rs, sh.rbase);  // whatever was claimed
                    const bool more = sh.go;
                    __syncthreads();
                    if (!more) break;
                }
            }
        }
    }
#ifdef ISMG_SP_TRACE
    const long long tr3 = gtimer();
    if (blockIdx.x == 0 && threadIdx.x == 0 && tr2) SP_TRACE(2, tr3 - tr2);
#endif
    sp_grid_sync(D.bar, gridDim.x);
#ifdef ISMG_SP_TRACE
    const long long tr4 = gtimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) SP_TRACE(3, tr4 - tr3);
#endif
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
#ifdef ISMG_SP_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) SP_TRACE(4, gtimer() - tr4);
#endif
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
        if (*(volatile unsigned*)&g_sp_stuck) st->mp_error = 2;
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

#ifdef ISMG_SP_TRACE
}  // namespace fz
}  // namespace ismgb
extern "C" __attribute__((visibility("default"))) void ismg_debug_sp_trace(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, ismgb::fz::g_sp_trace, sizeof(unsigned long long) * 6);
    const unsigned long long z[6] = {0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(ismgb::fz::g_sp_trace, z, sizeof(z));
}
namespace ismgb {
namespace fz {
#endif
struct SpEngine {
    SpK T{};
    SpD D{};
    void* mem = nullptr;
    size_t smem = 0;
};

// Host plan: a non-periodic 9-point operator whose zero weights face only ghosts
// (StencilClasses kind 0), at most 16 blocks of 32 rows, every CTA resident.
SpEngine* sp_try_create(const CoarseOpH& op, int device) {
    if (const char* e = getenv("ISMG_COARSE_SP"))
        if (e[0] == '0') return nullptr;
    StencilClasses S;
    if (!stencil_classes(op, S) || S.kind != 0 || !S.fastdiv) return nullptr;
    const int nb = (op.ncy + 31) / 32;
    if (nb > kMaxW) return nullptr;
    {  // the first / last row: one class on columns 1 .. ncx-2 (the kernel's row body)
        const int* rc = reinterpret_cast<const int*>(S.spec.data() + size_t(10) * (S.ncls + 1));
        for (int I = 2; I < op.ncx - 1; ++I)
            if (rc[I] != rc[1] || rc[op.ncx + I] != rc[op.ncx + 1]) return nullptr;
    }
    SpK T{};
    T.ncx = op.ncx, T.ncy = op.ncy, T.nb = nb;
    T.dspan = op.ncx + kDSpanPad;
    T.bstride = int64_t(T.dspan) * 32;
    T.bufsz = T.bstride * nb;
    T.ncls = S.ncls, T.ring = S.ring;
    T.spec_words = int(S.spec.size());
    T.singular = op.singular ? 1 : 0;
    T.tend = (op.ncx + kDHiPad + kR - kDLo) + kStride * (nb - 1);
    // residual chunks per block: 16 segments of the block's ncx + 62 diagonals. Same-box A/B
    // (tools/visit_hist.py 16384 32 3, coarse ms of steps 1-3): 16 -> 387 / 211 / 247,
    // 8 -> 406 / 236 / 285, 32 -> 430 / 241 / 286 (profiles/r02_ab_sp_nseg.txt)
    T.nseg = 16;
    if (const char* e = getenv("ISMG_SP_NSEG")) T.nseg = std::max(1, std::min(64, atoi(e)));  // tuning hook
    T.seglen = (op.ncx + 62 + T.nseg - 1) / T.nseg;
    const size_t smem = sizeof(double) * (size_t(nb) * (kQ * kRows + kQE * kEW + kQB * 32) + S.spec.size());
    ISMG_CUDA(cudaFuncSetAttribute(coarse_sp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0, sms = 0;
    ISMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_sp_kernel, 32 * (nb + 1), smem));
    ISMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (per_sm < 1) return nullptr;
    int P = sms;
    if (const char* e = getenv("ISMG_SP_CTAS")) P = std::max(1, std::min(sms, atoi(e)));  // tuning hook
    T.P = P, T.B = P + 2;
    auto* e = new SpEngine();
    e->T = T;
    e->smem = smem;
    const size_t bufb = sizeof(double) * size_t(T.bufsz);
    const size_t bytes = bufb * size_t(T.B + 2) + sizeof(double) * S.spec.size() + sizeof(unsigned long long) * P +
                         sizeof(unsigned) * T.B + 2 * sizeof(double) * T.B + 64 + 1024 +
                         3 * sizeof(unsigned) * T.B + sizeof(unsigned long long) * T.B + 64;
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
    e->D.rready = reinterpret_cast<unsigned*>(p), p += sizeof(unsigned) * T.B;
    e->D.rclaim = reinterpret_cast<unsigned*>(p), p += sizeof(unsigned) * T.B;
    e->D.rdone = reinterpret_cast<unsigned*>(p), p += sizeof(unsigned) * T.B;
    p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    e->D.rbits = reinterpret_cast<unsigned long long*>(p), p += sizeof(unsigned long long) * T.B;
    e->D.bar = reinterpret_cast<unsigned*>(p);
    return e;
}

void sp_destroy(SpEngine* e) {
    if (!e) return;
    cudaFree(e->mem);
    delete e;
}

void launch_coarse_sp(const Params& P, const SpEngine& e, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(e.T.P));
    cfg.blockDim = dim3(unsigned(32 * (e.T.nb + 1)));
    cfg.dynamicSmemBytes = e.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ISMG_CUDA(cudaLaunchKernelEx(&cfg, coarse_sp_kernel, P, e.T, e.D));
}

}  // namespace fz
}  // namespace ismgb

// coarse_rw.cu — the coarse visit (cycles.hpp:120-137; coarsening.hpp:531-567)
// as a register-resident wavefront spread over many SMs.
//
// gs_sweep_lex is a chain: cell (I,J) of sweep g needs the new values of W,
// SW, S, SE and the old ones of E, NW, N, NE. The linear schedule
//     tau(I, J, g) = I + 2J + L g
// respects every one of those dependencies, so all cells with equal tau can be
// relaxed at once and the result is the reference's lexicographic order bit
// for bit. The cost of a visit is its wavefront length, ncx + 2 ncy + L (G-1)
// steps for G sweeps, times the latency of one step. This engine makes a step
// as short as the fp64 dependency chain of one cell (~14 dependent DADD / DMUL
// / DFMA) by keeping the iterate in registers and never synchronising a whole
// block, cluster or grid inside a group of sweeps:
//
//  * lane s of a warp owns columns [32 s, 32 s + 32) of R = 2 coarse rows;
//    the warp holds the 2 x 32 values in registers. Every lane of a warp sits
//    at the same column offset c = tau - 2J (mod 32) of its segment, so the
//    register index is a compile-time constant of a 32-step unrolled loop;
//    lane s runs one sweep behind lane s-1 (L = 32 = the segment length), so
//    the value crossing a segment edge is one warp shuffle;
//  * the warps of the grid form a chain along J. Row 0 of a warp reads the new
//    values of the row below from a mailbox written by the warp below; its last
//    row reads the old values of the row above from the warp above. Mailboxes
//    live in L2 in NCCL's LL format (4-byte data + 4-byte tag per 8-byte word,
//    single-copy atomic), double-buffered by sweep parity, so a reader validates
//    every value by its tag: no fences, no flags, no barriers. Reads are
//    prefetched kA steps ahead with cp.async into shared memory;
//  * the residual of cell (I,J) after sweep g (coarse_residual, for the stop
//    test after every sweep) is formed in place kRl steps after its update,
//    when all nine neighbours hold their sweep-g values; each lane folds the
//    per-sweep maxima of its segment into a global atomicMax;
//  * warps drift into a skew that hides the mailbox latency: the dependencies
//    give a warp ~8 steps of slack against the warp below and ~15 against the
//    warp above. The chain cannot deadlock: the schedule tau + 6 w is valid
//    for every dependency, so the earliest unfinished step can always run.
//
// Sweeps run in groups (as coarse_cl.cu): a group of G sweeps records every
// sweep's residual max; a grid barrier ends it; a group that overshoots the
// first converged sweep is reloaded from its checkpoint (the coarse field) and
// replayed exactly that far, so the sweep count equals the reference's.
//
// Division x = num / w0 is correctly rounded: two Markstein corrections with
// y = RN(1/w0). q1 = RN(q0 + RN(num - w0 q0) y) is within one ulp of num/w0,
// and by Markstein's theorem (y within half an ulp of 1/w0, q1 within one ulp
// of num/w0, residual exact by FMA) q2 = RN(q1 + (num - w0 q1) y) = RN(num/w0).
// Numerators outside [2^-900, 2^1000] (zero, subnormal-adjacent, huge,
// non-finite), where the residual could underflow or overflow, take IEEE
// division.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "fused_impl.cuh"

namespace ismgb {
namespace fz {

namespace {

constexpr int kLS = 32;    // columns per lane segment = sweep lag
constexpr int kR = 2;      // rows per warp
constexpr int kRl = 28;    // residual lag (steps): the largest the in-warp overwrite allows (kLS - 4)
constexpr int kA = 4;      // mailbox prefetch distance (steps)
constexpr int kM = 1;      // (unused: wait-ahead after a stall, replaced by kTrail pacing)
constexpr int kTrail = 11; // steps the warp below leads by at a period's start (3 dependency + 2 L2 + 4 prefetch + 2)
constexpr int kNS = 8;     // prefetch slots per stream (power of two, > kA)
constexpr int kNStr = 4;   // mailbox streams: update-south, residual-south, update-north, residual-north
constexpr int kMaxG = 4096;
constexpr int kPredCap = 32;
constexpr int kRwWarps = 4;  // warps per CTA
constexpr int kRwThreads = 32 * kRwWarps;

static_assert(kRl >= 4 && kRl <= kLS - 4, "residual lag: all nine neighbours at sweep g, none at g+1");

}  // namespace

struct RwK {
    int ncx, ncy, K, nw, nctas;
    int bpitch;          // shared-memory rhs row pitch (doubles): K * (kLS + 1)
    int singular;
    int trace;           // ISMG_RW_TRACE: record every group's per-sweep residual maxima (debug)
    double w[9], y;      // interior stencil (slot order C, E, W, N, S, NE, NW, SE, SW), RN(1 / w0)
    double wa[9], ya;    // row 0 body (columns 1 .. ncx-2)
    double wb[9], yb;    // row ncy-1 body
};

struct RwD {
    const double* endw;          // [ncy][2][10]: classes of (0, J) and (ncx-1, J): w0..w8, RN(1 / w0)
    uint4* ms;                   // [nw][2][ncx] south mailboxes (written by the warp below)
    uint4* mn;                   // [nw][2][ncx] north mailboxes (written by the warp above)
    unsigned long long* cmax;    // [kMaxG] per-sweep residual max (bits of a non-negative double)
    unsigned* bar;               // grid barrier: [0] arrivals, [1] generation; [2] tag base
    double* part;                // [nw] anchor partial sums
    double* dec;                 // group decision: [0] first converged sweep, [1] residual
    unsigned long long* prog;    // [nw] progress per warp ((tag base << 32) | steps done)
};

namespace {

extern __shared__ __align__(16) double rw_dyn[];

__device__ __forceinline__ constexpr int cmod(int v) { return ((v % kLS) + kLS) % kLS; }
__device__ __forceinline__ constexpr int cdiv(int v) { return v >= 0 ? v / kLS : -((-v + kLS - 1) / kLS); }

__device__ __forceinline__ void ll_store(uint4* p, double v, unsigned tag) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(unsigned(__double2loint(v))),
                 "r"(tag), "r"(unsigned(__double2hiint(v))), "r"(tag)
                 : "memory");
}
__device__ __forceinline__ uint4 ll_load(const uint4* p) {
    uint4 u;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                 : "l"(p)
                 : "memory");
    return u;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// A slot's term. Interior weights are non-zero and face in-grid cells: the
// product as is. Ring / end weights may be zero (the reference then skips the
// slot, coarsening.hpp:539-543, :558-565): -0.0 is the exact identity of the
// accumulation in that case.
template <bool kSkip>
__device__ __forceinline__ double term(double w, double v) {
    if constexpr (kSkip) return w != 0.0 ? __dmul_rn(w, v) : -0.0;
    return __dmul_rn(w, v);
}

struct Nb {
    double c, e, w, n, s, ne, nw, se, sw;
};

// num = b - sum (update, acc from +0.0) or r = b - (w0 c + sum) (residual),
// slot order E, W, N, S, NE, NW, SE, SW.
template <bool kResid, bool kSkip, class Wt>
__device__ __forceinline__ double stencil(const Wt& w, const Nb& v, double b) {
    double acc = kResid ? __dmul_rn(w[0], v.c) : 0.0;
    acc = __dadd_rn(acc, term<kSkip>(w[1], v.e));
    acc = __dadd_rn(acc, term<kSkip>(w[2], v.w));
    acc = __dadd_rn(acc, term<kSkip>(w[3], v.n));
    acc = __dadd_rn(acc, term<kSkip>(w[4], v.s));
    acc = __dadd_rn(acc, term<kSkip>(w[5], v.ne));
    acc = __dadd_rn(acc, term<kSkip>(w[6], v.nw));
    acc = __dadd_rn(acc, term<kSkip>(w[7], v.se));
    acc = __dadd_rn(acc, term<kSkip>(w[8], v.sw));
    return __dsub_rn(b, acc);
}

// Per-warp state of a group (registers). Mailbox layout [warp][column][parity]
// (32 B per column): `par` is the parity of sweep g0 = q - lane this period,
// so a stream's word is base + 32 column + 16 (par ^ static parity).
struct Lane {
    int lane, K, G;
    unsigned base;          // tag of sweep 0
    bool live, has_l, has_r;
    const char* ms;         // south mailbox of this warp, column I0 (bytes)
    const char* mn;         // north mailbox of this warp, column I0
    char* pn;               // row 0 -> north mailbox of the warp below, column I0
    char* ps;               // row R-1 -> south mailbox of the warp above, column I0
    uint32_t slots;         // shared: this lane's prefetch slots ([kNStr][kNS][33] x 16 B, lane-offset)
    uint32_t b0, b1;        // shared: this lane's rhs segment of rows 0 / 1
    uint32_t ew;            // shared: end weights of this warp's rows [kR][2][10]
    unsigned long long* prog_me;           // this warp's published progress ((base << 32) | steps done)
    const unsigned long long* prog_south;  // ... of the warp below
};

// per-period values
struct Per {
    int q;          // period index (steps q * kLS ..)
    int g0;         // sweep of the lane's segment at offset 0 this period: q - lane
    unsigned tq;    // its tag
    int par;        // its parity
};

__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
    uint4 u;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(a) : "memory");
    return u;
}
__device__ __forceinline__ void sts_u4(uint32_t a, uint4 u) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w) : "memory");
}
__device__ __forceinline__ void cp_async16_s(uint32_t smem, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g) : "memory");
}

// stream s: row, lag, tag offset of the sweep read (update-north reads sweep g-1)
__device__ __forceinline__ constexpr int s_row(int s) { return s < 2 ? 0 : kR - 1; }
__device__ __forceinline__ constexpr int s_lag(int s) { return (s & 1) ? kRl : 0; }
__device__ __forceinline__ constexpr int s_toff(int s) { return s == 2 ? -1 : 0; }
// stream s exists in this warp variant (first warp: no row below; last: none above)
template <int S, bool kFirst, bool kLast>
__device__ __forceinline__ constexpr bool s_exists() { return S < 2 ? !kFirst : !kLast; }

__device__ __forceinline__ bool in_group(const Lane& L, int g) { return L.live && unsigned(g) < unsigned(L.G); }

template <int S>
__device__ __forceinline__ const char* mb_word(const Lane& L, const Per& p, int col, int d) {
    const char* m = S < 2 ? L.ms : L.mn;
    return m + 32 * col + 16 * ((p.par + d) & 1);
}
// shared slot of stream S for (static) step KS: own lane; +16 * 32 - 16 * lane: the extra slot (lane 0)
template <int S, int KS>
__device__ __forceinline__ constexpr uint32_t slot_off() {
    return 16u * uint32_t((S * kNS + (KS & (kNS - 1))) * 33);
}

// issue the prefetch of stream S for (static) step KS of the period
template <int S, int KS, bool kFirst, bool kLast>
__device__ __forceinline__ void pf_issue(const Lane& L, const Per& p, bool residuals) {
    if constexpr (s_exists<S, kFirst, kLast>()) {
        constexpr int kk = KS - 2 * s_row(S) - s_lag(S);
        constexpr int c = cmod(kk), d = cdiv(kk) + s_toff(S);
        if ((s_lag(S) != 0 && !residuals) || !in_group(L, p.g0 + cdiv(kk))) return;
        const uint32_t sl = L.slots + slot_off<S, KS>();
        if (c + 1 < kLS || L.has_r) cp_async16_s(sl, mb_word<S>(L, p, c + 1, d));
        if (c == 0 && L.lane == 0) cp_async16_s(sl + 16u * 32u, mb_word<S>(L, p, 0, d));
    }
}

// slow path: re-read stale mailbox words until the writer's tags show, and put
// the valid words back into the slots (read again by later steps / the next lane)
__device__ unsigned g_rw_stuck;  // a mailbox word or barrier never arrived (watchdog, ~2 s)

__device__ __forceinline__ bool ll_wait(const char* word, unsigned tag, long long t0) {
    for (;;) {
        const uint4 u = ll_load(reinterpret_cast<const uint4*>(word));
        if (((u.y ^ tag) | (u.w ^ tag)) == 0u) return true;
        if (gtimer() - t0 > 2000000000ll) {
            atomicExch(&g_rw_stuck, 1u);
            return false;
        }
    }
}

__device__ double g_rw_trace[8192];
__device__ unsigned g_rw_trace_n;
__device__ unsigned long long g_rw_slow[6];
// debug (ISMG_RW_TRACE): per warp [group cycles, slow-path cycles, pacing-spin cycles] of the last group
__device__ unsigned long long g_rw_cyc[3 * 1024];  // debug counters: slow-path entries by stream [0..3], own-column words [4], waits ahead [5]

// Slow path (warp-uniform): re-read a stale mailbox word until the writer's tag
// shows and put it back into its slot (read again by later steps / the lane
// beside). A stall on the row below (`ahead` set) means this warp caught up
// with the warp below, so the prefetches now in flight were issued too early:
// wait until the word kA + kM steps ahead has arrived, which restores kM steps
// of slack for the copies issued from here on.
__device__ __noinline__ void ll_settle(uint32_t slot, const char* word, unsigned tag, bool bad, const char* ahead,
                                       unsigned tag_ahead, bool wait_ahead, int stream) {
    const long long t0 = gtimer();
#ifdef ISMG_RW_COUNTERS
    const long long c0 = clock64();
    const bool any_wa = __any_sync(kFull, wait_ahead);
    if (threadIdx.x % 32 == 0) {
        atomicAdd(&g_rw_slow[stream], 1ull);
        if (any_wa) atomicAdd(&g_rw_slow[5], 1ull);
    }
#else
    (void)stream;
#endif
    if (bad) {
        uint4 u;
        for (;;) {
            u = ll_load(reinterpret_cast<const uint4*>(word));
            if (((u.y ^ tag) | (u.w ^ tag)) == 0u) break;
            if (gtimer() - t0 > 2000000000ll) {
                atomicExch(&g_rw_stuck, 1u);
                break;
            }
        }
        sts_u4(slot, u);
    }
    if (wait_ahead) ll_wait(ahead, tag_ahead, t0);
    __syncwarp();
#ifdef ISMG_RW_COUNTERS
    const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0 && wg < 1024) atomicAdd(&g_rw_cyc[3 * wg + 1], (unsigned long long)(clock64() - c0));
#endif
}

// validate the words delivered to stream S's slots at (static) step k
template <int S, int k, bool kFirst, bool kLast>
__device__ __forceinline__ void pf_check(const Lane& L, const Per& p, bool residuals) {
    if constexpr (s_exists<S, kFirst, kLast>()) {
        constexpr int kk = k - 2 * s_row(S) - s_lag(S);
        constexpr int c = cmod(kk), d = cdiv(kk) + s_toff(S);
        const bool act = (s_lag(S) == 0 || residuals) && in_group(L, p.g0 + cdiv(kk));
        const unsigned tag = p.tq + unsigned(d);
        const uint32_t sl = L.slots + slot_off<S, k>();
        const bool want = act && (c + 1 < kLS || L.has_r);
        // the word kA + kM steps ahead (update-south only: the row below leads)
        constexpr int ka = kk + kA + kM, ca = cmod(ka), da = cdiv(ka) + s_toff(S);
        const bool wa = false;  // (kept off: the period pacing in rw_group holds the lead instead)
        const char* ahead = mb_word<S>(L, p, ca + 1, da);
        const uint4 u = lds_u4(sl);
        const bool bad = want && ((u.y ^ tag) | (u.w ^ tag)) != 0u;
        if (__any_sync(kFull, bad)) ll_settle(sl, mb_word<S>(L, p, c + 1, d), tag, bad, ahead, p.tq + unsigned(da), wa, S);
        if constexpr (c == 0) {
            const bool own = act && L.lane == 0;
            const uint4 v = lds_u4(sl + 16u * 32u);
            const bool bad0 = own && ((v.y ^ tag) | (v.w ^ tag)) != 0u;
            if (__any_sync(kFull, bad0))
                ll_settle(sl + 16u * 32u, mb_word<S>(L, p, 0, d), tag, bad0, ahead, p.tq + unsigned(da), wa, 4);
        }
    }
}

// value of stream S's row at column I + j (j = -1, 0, 1; I = I0 + c) at (static)
// step k: delivered as the "column + 1" word of step k + j - 1, by this lane or
// (left of the segment) by the lane to the left; lane 0's column 0 in the extra slot
template <int S, int k, int j, bool kFirst, bool kLast>
__device__ __forceinline__ double wval(const Lane& L) {
    if constexpr (!s_exists<S, kFirst, kLast>()) {
        return 0.0;
    } else {
        constexpr int kk = k - 2 * s_row(S) - s_lag(S);
        constexpr int c = cmod(kk);
        constexpr int kd = k + j - 1;  // delivery step (may be in the previous period)
        constexpr uint32_t off = slot_off<S, (kd + kLS) % kLS>();
        if constexpr (c + j - 1 >= 0) {
            const uint4 u = lds_u4(L.slots + off);
            const double v = __hiloint2double(int(u.z), int(u.x));
            if constexpr (c + j >= kLS) return L.has_r ? v : 0.0;  // column ncx: ghost
            return v;
        } else {
            // column I0 + c + j <= I0: the left lane's delivery, or lane 0's column 0
            // (its extra slot, delivered at the step with offset 0) / ghost -1
            constexpr uint32_t off0 = slot_off<S, (k - c + kLS) % kLS>();
            const uint32_t a = L.lane == 0 ? L.slots + off0 + 16u * 32u : L.slots + off - 16u;
            const uint4 u = lds_u4(a);
            const double v = __hiloint2double(int(u.z), int(u.x));
            if constexpr (c + j < 0) return L.lane == 0 ? 0.0 : v;
            return v;
        }
    }
}

// Interior weights (slot order C, E, W, N, S, NE, NW, SE, SW): the ISMG
// interior row is tile-independent (coarsening.hpp:196-305;
// test_coarsening.cpp:136-149), so the plan requires it bit for bit and the
// kernel multiplies by immediates. kY = RN(1 / -3).
struct IsmgW {
    __device__ __forceinline__ double operator[](int k) const {
        return k == 0 ? -3.0 : (k < 5 ? 0.5 : 0.25);
    }
};
constexpr double kIsmgY = -0x1.5555555555555p-2;

// weights of row r's body cells: interior, or the first / last row's class
template <int r, bool kFirst, bool kLast>
__device__ __forceinline__ constexpr bool ring_row() {
    return (kFirst && r == 0) || (kLast && r == kR - 1);
}

// neighbours of the cell at column offset c (static) of row r: registers x,
// the lanes beside, and (first / last row of the warp) the mailbox streams
template <int r, int k, int c, int SS, int SN, bool kFirst, bool kLast>
__device__ __forceinline__ Nb gather(const Lane& L, const double (&x)[kR][kLS], bool with_c) {
    Nb v;
    v.c = with_c ? x[r][c] : 0.0;
    if constexpr (c + 1 < kLS) {
        v.e = x[r][c + 1];
    } else {
        const double t = __shfl_down_sync(kFull, x[r][0], 1);
        v.e = L.has_r ? t : 0.0;
    }
    if constexpr (c > 0) {
        v.w = x[r][c - 1];
    } else {
        const double t = __shfl_up_sync(kFull, x[r][kLS - 1], 1);
        v.w = L.has_l ? t : 0.0;
    }
    if constexpr (r + 1 < kR) {
        v.n = x[r + 1][c];
        if constexpr (c + 1 < kLS) {
            v.ne = x[r + 1][c + 1];
        } else {
            const double t = __shfl_down_sync(kFull, x[r + 1][0], 1);
            v.ne = L.has_r ? t : 0.0;
        }
        if constexpr (c > 0) {
            v.nw = x[r + 1][c - 1];
        } else {
            const double t = __shfl_up_sync(kFull, x[r + 1][kLS - 1], 1);
            v.nw = L.has_l ? t : 0.0;
        }
    } else {
        v.nw = wval<SN, k, -1, kFirst, kLast>(L);
        v.n = wval<SN, k, 0, kFirst, kLast>(L);
        v.ne = wval<SN, k, 1, kFirst, kLast>(L);
    }
    if constexpr (r > 0) {
        v.s = x[r - 1][c];
        if constexpr (c + 1 < kLS) {
            v.se = x[r - 1][c + 1];
        } else {
            const double t = __shfl_down_sync(kFull, x[r - 1][0], 1);
            v.se = L.has_r ? t : 0.0;
        }
        if constexpr (c > 0) {
            v.sw = x[r - 1][c - 1];
        } else {
            const double t = __shfl_up_sync(kFull, x[r - 1][kLS - 1], 1);
            v.sw = L.has_l ? t : 0.0;
        }
    } else {
        v.sw = wval<SS, k, -1, kFirst, kLast>(L);
        v.s = wval<SS, k, 0, kFirst, kLast>(L);
        v.se = wval<SS, k, 1, kFirst, kLast>(L);
    }
    return v;
}

// update (kResid = false) or residual (true) of row r at the cell with column
// offset c (static); the grid's first / last column takes its class weights,
// the first / last row its body class
template <bool kResid, int r, int c, bool kFirst, bool kLast>
__device__ __forceinline__ double cell(const RwK& T, const Lane& L, const Nb& v, double b) {
    if constexpr (c == 0 || c == kLS - 1) {
        const bool end = c == 0 ? L.lane == 0 : L.lane == L.K - 1;
        const uint32_t e = L.ew + 8u * uint32_t((r * 2 + (c == 0 ? 0 : 1)) * 10);
        double w[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            double bw;
            if constexpr (ring_row<r, kFirst, kLast>()) bw = (kFirst && r == 0) ? T.wa[k] : T.wb[k];
            else bw = IsmgW()[k];
            w[k] = end ? lds_f64(e + 8u * k) : bw;
        }
        const double num = stencil<kResid, true>(w, v, b);
        if constexpr (kResid) return num;
        double yb;
        if constexpr (ring_row<r, kFirst, kLast>()) yb = (kFirst && r == 0) ? T.ya : T.yb;
        else yb = kIsmgY;
        return div_cr(num, w[0], end ? lds_f64(e + 72u) : yb);
    } else if constexpr (ring_row<r, kFirst, kLast>()) {
        const double* bw = (kFirst && r == 0) ? T.wa : T.wb;
        const double num = stencil<kResid, true>(bw, v, b);
        if constexpr (kResid) return num;
        return div_cr(num, bw[0], (kFirst && r == 0) ? T.ya : T.yb);
    } else {
        const double num = stencil<kResid, false>(IsmgW(), v, b);
        if constexpr (kResid) return num;
        return div_cr(num, -3.0, kIsmgY);
    }
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double m) {
    atomicMax(p, (unsigned long long)__double_as_longlong(m));
}

template <int S, int KS, bool kFirst, bool kLast>
__device__ __forceinline__ void pf_issue_step(const Lane& L, const Per& p, const Per& pn, bool residuals) {
    if constexpr (KS < kLS) pf_issue<S, KS, kFirst, kLast>(L, p, residuals);
    else pf_issue<S, KS - kLS, kFirst, kLast>(L, pn, residuals);
}

// One step (static k of the period): prefetch, validate, residuals, updates.
template <int k, bool kFirst, bool kLast>
__device__ __forceinline__ void rw_step(const RwK& T, const Lane& L, const Per& p, const Per& pn, bool residuals,
                                        double (&x)[kR][kLS], double (&rmax)[kR], unsigned long long* cmax) {
    pf_issue_step<0, k + kA, kFirst, kLast>(L, p, pn, residuals);
    pf_issue_step<1, k + kA, kFirst, kLast>(L, p, pn, residuals);
    pf_issue_step<2, k + kA, kFirst, kLast>(L, p, pn, residuals);
    pf_issue_step<3, k + kA, kFirst, kLast>(L, p, pn, residuals);
    cp_commit();
    cp_wait<kA>();
    __syncwarp();  // every lane's delivered slots visible to the lane beside
    pf_check<0, k, kFirst, kLast>(L, p, residuals);
    pf_check<1, k, kFirst, kLast>(L, p, residuals);
    pf_check<2, k, kFirst, kLast>(L, p, residuals);
    pf_check<3, k, kFirst, kLast>(L, p, residuals);
    // residuals of the cells updated kRl steps ago (read before this step's updates)
    if (residuals) {
        auto res_row = [&](auto rc) {
            constexpr int r = decltype(rc)::value;
            constexpr int kk = k - 2 * r - kRl;
            constexpr int c = cmod(kk);
            const int g = p.g0 + cdiv(kk);
            const bool act = in_group(L, g);
            const Nb v = gather<r, k, c, 1, 3, kFirst, kLast>(L, x, true);
            const double b = lds_f64((r == 0 ? L.b0 : L.b1) + 8u * c);
            const double m = fabs(cell<true, r, c, kFirst, kLast>(T, L, v, b));
            if (act && m > rmax[r]) rmax[r] = m;  // std::max drops NaN (coarsening.hpp:545)
            if constexpr (c == kLS - 1) {
                if (act) atomic_max_nonneg(cmax + g, rmax[r]);
                rmax[r] = 0.0;
            }
        };
        res_row(std::integral_constant<int, 0>{});
        res_row(std::integral_constant<int, 1>{});
    }
    // updates: new values of both rows first (they read only older values), then store
    double nv[kR];
    bool act[kR];
    auto upd_row = [&](auto rc) {
        constexpr int r = decltype(rc)::value;
        constexpr int kk = k - 2 * r;
        constexpr int c = cmod(kk), d = cdiv(kk);
        act[r] = in_group(L, p.g0 + d);
        const Nb v = gather<r, k, c, 0, 2, kFirst, kLast>(L, x, false);
        const double b = lds_f64((r == 0 ? L.b0 : L.b1) + 8u * c);
        nv[r] = cell<false, r, c, kFirst, kLast>(T, L, v, b);
        if (act[r]) {
            const unsigned tag = p.tq + unsigned(d);
            const int po = 16 * ((p.par + d) & 1);
            if constexpr (r == 0 && !kFirst) ll_store(reinterpret_cast<uint4*>(L.pn + 32 * c + po), nv[r], tag);
            if constexpr (r == kR - 1 && !kLast) ll_store(reinterpret_cast<uint4*>(L.ps + 32 * c + po), nv[r], tag);
        }
    };
    upd_row(std::integral_constant<int, 0>{});
    upd_row(std::integral_constant<int, 1>{});
    {
        constexpr int c0 = cmod(k), c1 = cmod(k - 2);
        if (act[0]) x[0][c0] = nv[0];
        if (act[1]) x[1][c1] = nv[1];
    }
    if constexpr ((k & 3) == 3) {  // progress for the warp above's pacing: steps 0 .. q kLS + k done
        if (L.lane == 0) {
            const unsigned long long v = (static_cast<unsigned long long>(L.base) << 32) | unsigned(p.q * kLS + k + 1);
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(L.prog_me), "l"(v) : "memory");
        }
    }
}

template <int k, bool kFirst, bool kLast>
__device__ __forceinline__ void rw_period(const RwK& T, const Lane& L, const Per& p, const Per& pn, bool residuals,
                                          double (&x)[kR][kLS], double (&rmax)[kR], unsigned long long* cmax) {
    if constexpr (k < kLS) {
        rw_step<k, kFirst, kLast>(T, L, p, pn, residuals, x, rmax, cmax);
        rw_period<k + 1, kFirst, kLast>(T, L, p, pn, residuals, x, rmax, cmax);
    }
}

template <int k, bool kFirst, bool kLast>
__device__ __forceinline__ void rw_prologue(const Lane& L, const Per& p, bool residuals) {
    if constexpr (k < kA) {
        pf_issue<0, k, kFirst, kLast>(L, p, residuals);
        pf_issue<1, k, kFirst, kLast>(L, p, residuals);
        pf_issue<2, k, kFirst, kLast>(L, p, residuals);
        pf_issue<3, k, kFirst, kLast>(L, p, residuals);
        cp_commit();
        rw_prologue<k + 1, kFirst, kLast>(L, p, residuals);
    }
}

__device__ __forceinline__ Per period(const Lane& L, int q) {
    Per p;
    p.q = q;
    p.g0 = q - L.lane;
    p.tq = L.base + unsigned(p.g0);
    p.par = int(p.tq & 1u);
    return p;
}

// One group of G sweeps of this warp's rows (x in registers on entry and exit).
template <bool kFirst, bool kLast>
__device__ __forceinline__ void rw_group(const RwK& T, const Lane& L, double (&x)[kR][kLS], bool residuals,
                                         unsigned long long* cmax) {
    // the values of row 0 before sweep 0: read by the warp below (its north, sweep g - 1 = -1)
    if (!kFirst && L.live) {
        const unsigned tag = L.base - 1u;
#pragma unroll
        for (int c = 0; c < kLS; ++c) ll_store(reinterpret_cast<uint4*>(L.pn + 32 * c + 16 * (tag & 1u)), x[0][c], tag);
    }
    double rmax[kR] = {0.0, 0.0};
    // last step: the residual of lane K-1's last cell of sweep G-1 in row R-1
    const int tau_end = kLS * (L.K + L.G - 1) + 2 * kR - 3 + (residuals ? kRl : 0);
    const int qn = tau_end / kLS + 1;
    rw_prologue<0, kFirst, kLast>(L, period(L, 0), residuals);
    const unsigned long long gb = static_cast<unsigned long long>(L.base) << 32;
    const long long cg0 = clock64();
    if (L.lane == 0) {
        const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        if (wg < 1024) g_rw_cyc[3 * wg + 1] = 0, g_rw_cyc[3 * wg + 2] = 0;
    }
    __syncwarp();
#pragma unroll 1
    for (int q = 0; q < qn; ++q) {
        // pacing: start the period only once the warp below has done kTrail more
        // steps (its words this period's prefetches read are then in L2); the
        // lead stays in [kTrail, kTrail + 4 + jitter], inside the window the warp
        // above allows (its north words, kLS - 4 - kA - latency steps of slack)
        if (!kFirst) {
            const unsigned long long want = gb | unsigned(min(q * kLS + kTrail, tau_end + 1));
            if (L.lane == 0) {
                unsigned long long v;
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(L.prog_south) : "memory");
                if (v < want) {
                    const long long t0 = gtimer();
                    const long long c0 = clock64();
                    do {
                        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(L.prog_south) : "memory");
                        if (gtimer() - t0 > 2000000000ll) {
                            atomicExch(&g_rw_stuck, 1u);
                            break;
                        }
                    } while (v < want);
                    const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
                    if (wg < 1024) g_rw_cyc[3 * wg + 2] += (unsigned long long)(clock64() - c0);
                }
            }
            __syncwarp();
        }
        const Per p = period(L, q), pn = period(L, q + 1);
        rw_period<0, kFirst, kLast>(T, L, p, pn, residuals, x, rmax, cmax);
    }
    if (L.lane == 0) {  // the group's last step done (the pacing target of the warp above caps here)
        const unsigned long long v = gb | unsigned(tau_end + 1);
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(L.prog_me), "l"(v) : "memory");
        const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        if (wg < 1024) g_rw_cyc[3 * wg] = (unsigned long long)(clock64() - cg0);
    }
    cp_wait<0>();
    __threadfence();  // this thread's residual atomics performed before the group's grid barrier
}

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned n) {
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
                __nanosleep(20);
                if (gtimer() - t0 > 2000000000ll) {
                    atomicExch(&g_rw_stuck, 1u);
                    break;
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kRwThreads, 1) coarse_rw_kernel(Params P, RwK T, RwD D) {
    Ctl* st = P.ctl;
    if (st->phase != kCoarse) return;
    const long long t_start = gtimer();
    const int wic = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w = blockIdx.x * kRwWarps + wic;
    const bool wok = w < T.nw;
    const unsigned nct = gridDim.x;
    // shared memory: rhs rows [kRwWarps][kR][bpitch] | end weights [kRwWarps][kR][2][10] | slots
    double* bsm = rw_dyn;
    double* ewm = bsm + size_t(kRwWarps) * kR * T.bpitch;
    uint4* slots = reinterpret_cast<uint4*>(ewm + kRwWarps * kR * 20);
    Lane L;
    L.lane = lane, L.K = T.K, L.G = 0, L.base = 0;
    L.live = wok && lane < T.K;
    L.has_l = lane > 0;
    L.has_r = lane + 1 < T.K;
    const bool south = wok && w > 0, north = wok && w + 1 < T.nw;
    const size_t mrow = size_t(2) * T.ncx;  // uint4 words per mailbox ([ncx][2])
    const int I0 = lane * kLS;
    const int wq = wok ? w : 0;
    L.ms = reinterpret_cast<const char*>(D.ms + size_t(wq) * mrow + 2 * I0);
    L.mn = reinterpret_cast<const char*>(D.mn + size_t(wq) * mrow + 2 * I0);
    L.pn = south ? reinterpret_cast<char*>(D.mn + size_t(w - 1) * mrow + 2 * I0) : nullptr;
    L.ps = north ? reinterpret_cast<char*>(D.ms + size_t(w + 1) * mrow + 2 * I0) : nullptr;
    L.slots = su32(slots + size_t(wic) * kNStr * kNS * 33 + lane);
    L.b0 = su32(bsm + size_t(wic) * kR * T.bpitch + lane * (kLS + 1));
    L.b1 = L.b0 + 8u * uint32_t(T.bpitch);
    L.ew = su32(ewm + wic * kR * 20);
    L.prog_me = D.prog + (wok ? w : 0);
    L.prog_south = D.prog + (south ? w - 1 : 0);
    const int J0 = w * kR;
    // rhs and end classes of this warp's rows into shared memory (lane segments padded by one)
    if (wok) {
        for (int r = 0; r < kR; ++r) {
            for (int I = lane; I < T.ncx; I += 32)
                bsm[(wic * kR + r) * T.bpitch + (I / kLS) * (kLS + 1) + (I % kLS)] = P.cb.at(I, J0 + r);
            if (lane < 20) ewm[(wic * kR + r) * 20 + lane] = D.endw[size_t(J0 + r) * 20 + lane];
        }
    }
    // iterate: ce = 0 at the visit's start (cycles.hpp:122)
    double x[kR][kLS];
#pragma unroll
    for (int r = 0; r < kR; ++r)
#pragma unroll
        for (int c = 0; c < kLS; ++c) x[r][c] = 0.0;
    const double rc0 = st->rc;  // max|cb|, formed by the fine pass that restricted
    const long long budget = P.max_total - st->total;
    int G = max(1, min(st->pred, kPredCap));
    unsigned base = D.bar[2];
    grid_sync(D.bar, nct);  // everyone has read Ctl before block 0 may change it
    // ce = 0 is the checkpoint of the visit's first group (cycles.hpp:122)
    if (wok && lane < T.K)
#pragma unroll
        for (int r = 0; r < kR; ++r)
#pragma unroll
            for (int c = 0; c < kLS; ++c) P.ce.at(I0 + c, J0 + r) = 0.0;
    double rc = rc0;
    long long done = 0, steps = 0;
    bool replay = false;
    __shared__ double sdec[2];
    __shared__ int sfirst;
    while (replay || (rc > P.tol_coarse && done < budget)) {  // a replay runs whatever rc says
        if (budget - done < G) G = int(budget - done);
        L.G = G;
        L.base = base;
        if (wok) {
            if (w == 0) rw_group<true, false>(T, L, x, !replay, D.cmax);
            else if (w == T.nw - 1) rw_group<false, true>(T, L, x, !replay, D.cmax);
            else rw_group<false, false>(T, L, x, !replay, D.cmax);
        }
        base += unsigned(G) + 2u;
        steps += T.ncx + 2 * T.ncy + kLS * (G - 1) + (replay ? 0 : kRl);
        grid_sync(D.bar, nct);
        if (replay) {
            done += G;
            break;
        }
        if (blockIdx.x == 0) {  // first sweep whose residual passes tol_coarse, then clear the maxima
            if (threadIdx.x == 0) sfirst = G;
            __syncthreads();
            for (int g = threadIdx.x; g < G; g += blockDim.x)
                if (!(__longlong_as_double((long long)__ldcg(D.cmax + g)) > P.tol_coarse)) atomicMin(&sfirst, g);
            __syncthreads();
            if (threadIdx.x == 0) {
                const int first = sfirst < G ? sfirst : -1;
                D.dec[0] = double(first);
                D.dec[1] = __longlong_as_double((long long)__ldcg(D.cmax + (first >= 0 ? first : G - 1)));
            }
            __syncthreads();
            if (T.trace && threadIdx.x == 0) {
                unsigned n0 = g_rw_trace_n;
                if (n0 + 2 + G < 8192) {
                    g_rw_trace[n0] = -1.0, g_rw_trace[n0 + 1] = double(G);
                    for (int g = 0; g < G; ++g) g_rw_trace[n0 + 2 + g] = __longlong_as_double((long long)__ldcg(D.cmax + g));
                    g_rw_trace_n = n0 + 2 + G;
                }
            }
            __syncthreads();
            for (int g = threadIdx.x; g < G; g += blockDim.x) D.cmax[g] = 0ull;
            __threadfence();
        }
        grid_sync(D.bar, nct);
        if (threadIdx.x == 0) sdec[0] = __ldcg(D.dec), sdec[1] = __ldcg(D.dec + 1);
        __syncthreads();
        const int first = int(sdec[0]);
        rc = sdec[1];
        if (first >= 0 && first < G - 1) {  // overshoot: reload the checkpoint, replay first + 1 sweeps
            if (wok && lane < T.K)
#pragma unroll
                for (int r = 0; r < kR; ++r)
#pragma unroll
                    for (int c = 0; c < kLS; ++c) x[r][c] = P.ce.at(I0 + c, J0 + r);
            replay = true;
            G = first + 1;
            continue;
        }
        done += G;
        if (first >= 0) break;
        // accepted and not converged: checkpoint for the next group
        if (wok && lane < T.K)
#pragma unroll
            for (int r = 0; r < kR; ++r)
#pragma unroll
                for (int c = 0; c < kLS; ++c) P.ce.at(I0 + c, J0 + r) = x[r][c];
        G = min(2 * G, kMaxG);
    }
    // anchor once (singular), in a fixed order: lanes, then warps by index
    if (T.singular && done > 0) {
        double s = 0.0;
        if (wok && lane < T.K)
#pragma unroll
            for (int r = 0; r < kR; ++r)
#pragma unroll
                for (int c = 0; c < kLS; ++c) s += x[r][c];
        s = warp_sum_down(s);
        if (wok && lane == 0) D.part[w] = s;
        grid_sync(D.bar, nct);
        double tot = 0.0;
        for (int k = lane; k < T.nw; k += 32) tot += __ldcg(D.part + k);
        tot = __shfl_sync(kFull, warp_sum_down(tot), 0);
        const double c = -(tot / double(int64_t(T.ncx) * T.ncy));
#pragma unroll
        for (int r = 0; r < kR; ++r)
#pragma unroll
            for (int cc = 0; cc < kLS; ++cc) x[r][cc] += c;
    }
    if (wok && lane < T.K)
#pragma unroll
        for (int r = 0; r < kR; ++r)
#pragma unroll
            for (int c = 0; c < kLS; ++c) P.ce.at(I0 + c, J0 + r) = x[r][c];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        D.bar[2] = base;
        st->coarse_launches += 1;
        st->coarse_ns += gtimer() - t_start;
        st->coarse_steps += steps;
        if (done > 0) st->pred = int(done);
        st->total += done;
        st->coarse += done;
        st->rc = rc;
        if (st->nvisits > 0 && st->nvisits <= P.visit_cap) P.visit_log[2 * (st->nvisits - 1)] = int(done);
        if (*(volatile unsigned*)&g_rw_stuck) st->mp_error = 2;
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

bool same_bits(double a, double b) { return a == b && std::signbit(a) == std::signbit(b); }

}  // namespace

struct RwPlan {
    RwK T;
    std::vector<double> endw;
    size_t smem = 0;
};

// Host plan: the operator must be the ISMG 9-point stencil in the interior
// (every weight non-zero), each boundary row a single class on columns
// 1..ncx-2, non-periodic, ncx a multiple of 32 up to 1024, ncy even.
bool rw_coarse_plan(const CoarseOpH& op, RwPlan& p, int device) {
    if (const char* e = getenv("ISMG_COARSE_RW"))
        if (e[0] == '0') return false;
    if (op.px || op.py || op.five_point) return false;
    const int ncx = op.ncx, ncy = op.ncy;
    if (ncx % kLS != 0 || ncx / kLS > 32 || ncx < 2 * kLS || ncy % kR != 0 || ncy / kR < 2) return false;
    RwK& T = p.T;
    std::memset(&T, 0, sizeof(T));
    T.ncx = ncx, T.ncy = ncy, T.K = ncx / kLS, T.nw = ncy / kR;
    T.nctas = (T.nw + kRwWarps - 1) / kRwWarps;
    T.bpitch = T.K * (kLS + 1);
    T.singular = op.singular ? 1 : 0;
    T.trace = getenv("ISMG_RW_TRACE") ? 1 : 0;
    auto row_body = [&](int J, double* w) {
        for (int sl = 0; sl < 9; ++sl) w[sl] = op.at(sl, 1, J);
        for (int I = 2; I < ncx - 1; ++I)
            for (int sl = 0; sl < 9; ++sl)
                if (!same_bits(op.at(sl, I, J), w[sl])) return false;
        return w[0] != 0.0;
    };
    if (!row_body(1, T.w)) return false;
    static const double ismg[9] = {-3.0, 0.5, 0.5, 0.5, 0.5, 0.25, 0.25, 0.25, 0.25};
    for (int sl = 0; sl < 9; ++sl)
        if (!same_bits(T.w[sl], ismg[sl])) return false;  // the kernel's immediates
    for (int J = 2; J < ncy - 1; ++J) {
        double w[9];
        if (!row_body(J, w)) return false;
        for (int sl = 0; sl < 9; ++sl)
            if (!same_bits(w[sl], T.w[sl])) return false;
    }
    if (!row_body(0, T.wa) || !row_body(ncy - 1, T.wb)) return false;
    T.y = 1.0 / T.w[0], T.ya = 1.0 / T.wa[0], T.yb = 1.0 / T.wb[0];
    p.endw.assign(size_t(ncy) * 20, 0.0);
    for (int J = 0; J < ncy; ++J)
        for (int e = 0; e < 2; ++e) {
            const int I = e == 0 ? 0 : ncx - 1;
            double* d = p.endw.data() + size_t(J) * 20 + e * 10;
            for (int sl = 0; sl < 9; ++sl) d[sl] = op.at(sl, I, J);
            if (d[0] == 0.0) return false;
            d[9] = 1.0 / d[0];
        }
    p.smem = sizeof(double) * (size_t(kRwWarps) * kR * T.bpitch + size_t(kRwWarps) * kR * 20) +
             sizeof(uint4) * size_t(kRwWarps) * kNStr * kNS * 33;
    // every CTA must be resident at once (the mailboxes and grid barriers spin)
    ISMG_CUDA(cudaFuncSetAttribute(coarse_rw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem)));
    int per_sm = 0, sms = 0;
    ISMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_rw_kernel, kRwThreads, p.smem));
    ISMG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (long(per_sm) * sms < T.nctas) return false;
    return true;
}

struct RwEngine {
    RwPlan plan;
    RwD D{};
    void* mem = nullptr;
};

RwEngine* rw_create(const RwPlan& plan) {
    auto* e = new RwEngine();
    e->plan = plan;
    const RwK& T = plan.T;
    const size_t mail = sizeof(uint4) * size_t(T.nw) * 2 * T.ncx;
    const size_t bytes = 2 * mail + sizeof(unsigned long long) * kMaxG + 64 + sizeof(double) * (T.nw + 2) +
                         sizeof(double) * plan.endw.size() + sizeof(unsigned long long) * T.nw + 256;
    ISMG_CUDA(cudaMalloc(&e->mem, bytes));
    ISMG_ZERO(e->mem, bytes);
    char* p = static_cast<char*>(e->mem);
    e->D.ms = reinterpret_cast<uint4*>(p);
    p += mail;
    e->D.mn = reinterpret_cast<uint4*>(p);
    p += mail;
    e->D.cmax = reinterpret_cast<unsigned long long*>(p);
    p += sizeof(unsigned long long) * kMaxG;
    e->D.bar = reinterpret_cast<unsigned*>(p);
    p += 64;
    e->D.part = reinterpret_cast<double*>(p);
    p += sizeof(double) * T.nw;
    e->D.dec = reinterpret_cast<double*>(p);
    p += sizeof(double) * 2;
    double* endw = reinterpret_cast<double*>(p);
    ISMG_H2D(endw, plan.endw.data(), sizeof(double) * plan.endw.size());
    p += sizeof(double) * plan.endw.size();
    e->D.prog = reinterpret_cast<unsigned long long*>(p);
    e->D.endw = endw;
    const unsigned base0 = 16u;  // tags start above the zeroed mailboxes' 0
    ISMG_H2D(e->D.bar + 2, &base0, sizeof(unsigned));
    return e;
}

// debug: the recorded per-group residual maxima ([-1, G, cmax[0..G)]...), then reset
std::vector<double> rw_trace_take() {
    unsigned n = 0;
    ISMG_CUDA(cudaMemcpyFromSymbol(&n, g_rw_trace_n, sizeof(unsigned)));
    std::vector<double> v(n);
    if (n) ISMG_CUDA(cudaMemcpyFromSymbol(v.data(), g_rw_trace, sizeof(double) * n));
    const unsigned z = 0;
    ISMG_CUDA(cudaMemcpyToSymbol(g_rw_trace_n, &z, sizeof(unsigned)));
    unsigned long long slow[6] = {0, 0, 0, 0, 0, 0};
    ISMG_CUDA(cudaMemcpyFromSymbol(slow, g_rw_slow, sizeof(slow)));
    v.push_back(-2.0);
    for (unsigned long long c : slow) v.push_back(double(c));
    std::vector<unsigned long long> cyc(3 * 1024);
    ISMG_CUDA(cudaMemcpyFromSymbol(cyc.data(), g_rw_cyc, sizeof(unsigned long long) * cyc.size()));
    for (int w : {0, 1, 2, 3, 4, 5, 64, 127, 128, 200, 255}) {
        v.push_back(-3.0), v.push_back(double(w));
        for (int k = 0; k < 3; ++k) v.push_back(double(cyc[3 * w + k]));
    }
    const unsigned long long z2[6] = {0, 0, 0, 0, 0, 0};
    ISMG_CUDA(cudaMemcpyToSymbol(g_rw_slow, z2, sizeof(z2)));
    return v;
}

RwEngine* rw_try_create(const CoarseOpH& op, int device) {
    RwPlan p;
    if (!rw_coarse_plan(op, p, device)) return nullptr;
    return rw_create(p);
}

void rw_destroy(RwEngine* e) {
    if (!e) return;
    cudaFree(e->mem);
    delete e;
}

void launch_coarse_rw(const Params& P, const RwEngine& e, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(e.plan.T.nctas));
    cfg.blockDim = dim3(kRwThreads);
    cfg.dynamicSmemBytes = e.plan.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ISMG_CUDA(cudaLaunchKernelEx(&cfg, coarse_rw_kernel, P, e.plan.T, e.D));
}

}  // namespace fz
}  // namespace ismgb

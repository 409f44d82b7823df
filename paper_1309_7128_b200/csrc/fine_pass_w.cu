// fine_pass_w.cu — the fused fine pass on independent one-warp strips (tiles >= 4).
//
// Same pass as fine_pass.cu (anchor shift, red and black half-sweeps,
// residual, tile-sum restriction, anchor sum and max|r| in ONE HBM pass of
// 24 B/cell). Measured on B200, the pass is bound by the latency of each
// warp's in-order dependent instruction stream and by its slowest warps, so:
//   * a CTA is ONE warp owning a strip of nq column quads (lanes 1..nq;
//     4*nq a multiple of the tile, <= 120 columns); lanes 0 and nq+1 hold the
//     halo quads (a-4..a-1, a+4nq..a+4nq+3) and recompute the 2/1-cell
//     red / black halo; a finished strip frees its SM slot at once;
//   * the warp streams rows through its own shared-memory ring filled by TMA
//     bulk copies (issued from converged code by an elected lane) and
//     exchanges horizontal neighbours with shuffles; there is no CTA barrier;
//   * iteration k loads row k, relaxes the red cells of row k-1, the black
//     cells of row k-2 and forms the residual of row k-3 (vertical
//     neighbours in registers, slots compile-time in a 4-row unroll);
//   * every warp runs the SAME arithmetic: cells are relaxed with d = 4, and
//     boundary cases are fix-ups behind branches taken only where they apply:
//     lanes holding a boundary or out-of-domain column (lane-divergent, rare)
//     and boundary rows (warp-uniform). Out-of-domain lanes stay frozen at 0,
//     which is exactly the missing neighbour of the reference's stencil, so
//     boundary strips cost what interior strips cost.
#include <type_traits>

#include "fused_impl.cuh"

namespace ismgb {
namespace fz {

namespace {

// Minimum resident CTAs (= warps) per SM requested from ptxas, i.e. its register
// cap. 14 caps the single-GPU kernel at 128 registers without spills and runs
// 14 warps per SM instead of 12: 133 against 152 us per 4096^2 pass
// (tools/probe_fine.py; 12: 152, 13: 148, 15: 133, 16: 137, 20: 196 with spills).
#ifndef ISMG_FINE_MINB
#define ISMG_FINE_MINB 14
#endif
#ifndef ISMG_MP_FENCE_SC
#define ISMG_MP_FENCE_SC 0
#endif
#ifndef ISMG_FINE_MINB_PR
// the prolongation / residual kernel: 12 resident warps (168 registers, no spill,
// y-axis tables staged in shared memory). Same-box A/B (tools/visit_hist.py,
// solve ms): 16384^2 step 1 3127 at 12 against 3351 at 16 and 3461 at 14 with the
// staged tables; 4096^2 steps 1-3 437 / 232 / 245 against 458 / 245 / 257 at 14.
#define ISMG_FINE_MINB_PR 12
#endif
#ifndef ISMG_FINE_MINB_MP
#define ISMG_FINE_MINB_MP 1  // the multi-GPU all-phases variant spills at 14
#endif
#ifndef ISMG_FINE_MINB_MP_SW
#define ISMG_FINE_MINB_MP_SW 14  // multi-GPU sweep-only kernel (PH 1): 20 B of spills; 2 GPUs at 16384^2 127.3 G against 117.1 G at 12 (all-phases kernel 111.4 G)
#endif

constexpr int kRowW = 128;  // ring row: columns [a-4, a+124)
#ifndef ISMG_FINE_RING
#define ISMG_FINE_RING 6
#endif
constexpr int kRingW = ISMG_FINE_RING;  // rows in flight

struct SmemW {
    double x[kRingW][kRowW];
    double b[kRingW][kRowW];
    uint64_t bar[kRingW];
};

// TMA bulk copies of one row (x and b) into ring slot `slot`: called by the
// whole converged warp; one elected lane issues.
__device__ __forceinline__ void issue_row_w(SmemW& sm, const double* xrow, const double* brow, int slot,
                                            uint32_t bytes) {
    const uint32_t bar = su32(&sm.bar[slot]);
    const uint32_t dx = su32(&sm.x[slot][0]), db = su32(&sm.b[slot][0]);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %4, [%0];\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%5], [%6], %4, [%0];\n\t"
        "}" ::"r"(bar),
        "r"(2u * bytes), "r"(dx), "l"(xrow), "r"(bytes), "r"(db), "l"(brow)
        : "memory");
}

// Per-lane column geometry.
struct Lane {
    int l, c0;
    bool owned;   // lanes 1..nq: residual, store, tile sums
    bool frozen;  // no column of the lane in the domain (idle lanes, outside halos): values stay 0
    bool spec;    // a boundary column or a partly outside quad: exact per-cell fix-up
    bool dom[4], red[4], blk[4];
    double dc[4];  // column part of the diagonal (W + E faces)
    __device__ __forceinline__ Lane(const Params& P, int a, int nq) {
        l = threadIdx.x & 31;
        owned = l >= 1 && l <= nq;
        const bool active = l <= nq + 1;
        c0 = a - 4 + 4 * l;
        const int W = 4 * nq;
        bool any = false, all = true, interior = true;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = c0 + q;
            dom[q] = active && col >= 0 && col < P.nx;
            any = any || dom[q];
            all = all && dom[q];
            interior = interior && col >= 1 && col <= P.nx - 2;
            red[q] = dom[q] && col >= a - 2 && col < a + W + 2;
            blk[q] = dom[q] && col >= a - 1 && col < a + W + 1;
            dc[q] = col_diag(P, col);
        }
        frozen = !any;
        owned = owned && any;  // a quad entirely past the last column stores and sums nothing
        spec = any && !(all && interior);
    }
};

struct Acc {
    double mx = 0.0, sx = 0.0, tacc = 0.0, cm = 0.0;
    int nan = 0;
};

// Register window: at the top of iteration k (U = its index in a 4-row
// block) rows k-1, k-2, k-3, k-4 live in slots (U+3)&3, (U+2)&3, (U+1)&3, U.
struct Win {
    double x[4][4];
    double b[4][4];
};

struct Geo {
    int r0, r1, ny;
    double c, fwS, fwN;
    double* outp;
    int64_t pitch;
};

// release fence at system scope: orders this thread's peer stores before its
// later ticket / flag writes (no sequential-consistency fence needed)
__device__ __forceinline__ void fence_release_sys() {
#if ISMG_MP_FENCE_SC
    __threadfence_system();
#else
    asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
}

// a positive power of two (zero significand bits): its reciprocal is exact
__device__ __forceinline__ bool is_pow2(double d) {
    return d > 0.0 && (__double_as_longlong(d) & 0x000FFFFFFFFFFFFFll) == 0;
}
// 1 / d for a (normal) power of two d, exactly, from the exponent: no MUFU / DDIV
__device__ __forceinline__ double pow2_recip(double d) {
    return __hiloint2double((2046 << 20) - (__double2hiint(d) & 0x7ff00000), 0);
}
// IEEE num / den out of line: a branch the compiler cannot if-convert into
// computing the DDIV sequence for every cell (it did: MUFU.RCP64H was the
// prolongation pass's top stall at 16384^2, profiles/r02_fine_pass_w_ph2_16384_ncu_full.txt)
__device__ __noinline__ double div_slow(double num, double den) { return __ddiv_rn(num, den); }

// this rank's own pack slot of pass parity p in its exchange buffer
__device__ __forceinline__ double* my_pack(const Params& P, int p) {
    return P.xch[P.rank] + (int64_t(p) * P.nranks + P.rank) * P.pack_len;
}


// Multi-GPU, end of a CTA's pass: the boundary rows it relaxed (read back from
// x: the output of a sweep / prolongation, the unchanged input of a residual
// pass) go into this rank's pack slot of parity p on every rank, over NVLink for
// the peers, followed by a system-scope release fence. Only the CTAs holding
// the strip's first / last 3 rows push; tile sums and partials stay in the
// local slot, where mp_unpack_kernel on every rank pulls them from.
__device__ __forceinline__ void mp_push(const Params& P, const Lane& L, const Geo& G, int p, const double* xrows,
                                        int hb = 0) {
    const int64_t o0 = (int64_t(p) * P.nranks + P.rank) * P.pack_len;
    bool pushed = false;
    for (int h = 0; h < 2; ++h) {
        if (h == 0 ? P.row0 == 0 : P.row1 == P.ny) continue;
        const int hj = h == 0 ? P.row0 : P.row1 - 3;
        for (int j = max(hj, G.r0); j < min(hj + 3, G.r1); ++j) {
            pushed = true;
            if (!L.owned) continue;
            const double* src = xrows + int64_t(j) * P.pitch;
            const double2 v01 = *reinterpret_cast<const double2*>(src);
            const double2 v23 = *reinterpret_cast<const double2*>(src + 2);
            const int64_t off = o0 + P.h_off[hb + h] + int64_t(j - hj) * P.pitch + kXOff + L.c0;
            for (int q = 0; q < P.nranks; ++q) {
                reinterpret_cast<double2*>(P.xch[q] + off)[0] = v01;
                reinterpret_cast<double2*>(P.xch[q] + off)[1] = v23;
            }
        }
    }
    if (pushed) fence_release_sys();
}

// store a finished quad row j
__device__ __forceinline__ void put_row(const Geo& G, const Lane& L, int j, const double* v) {
    double* dst = G.outp + int64_t(j) * G.pitch;
    if (!L.spec) {
        reinterpret_cast<double2*>(dst)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(dst)[1] = make_double2(v[2], v[3]);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (L.dom[q]) dst[q] = v[q];
    }
}

__device__ __forceinline__ double row_part(const Geo& G, int j) {
    return ((j > 0) ? 1.0 : G.fwS) + ((j < G.ny - 1) ? 1.0 : G.fwN);  // smoother.hpp:60-61
}

__device__ __forceinline__ double sh_up(double v) { return __shfl_up_sync(kFull, v, 1); }
__device__ __forceinline__ double sh_dn(double v) { return __shfl_down_sync(kFull, v, 1); }

// Exact update of one cell (smoother.hpp:112-113) for the fix-up paths.
__device__ __forceinline__ double gs_exact(double W, double E, double S, double N, double b, double d) {
    return div_by_diag(((((W + E) + S) + N) - b), d);
}

// Iteration k; row k-1 has parity P1.
template <int U, int P1, bool MP>
__device__ __forceinline__ void step_w(const SmemW& sm, int slot, const Lane& L, const Geo& G, Win& w, Acc& A, int k) {
    constexpr int s0 = U, s1 = (U + 3) & 3, s2 = (U + 2) & 3, s3 = (U + 1) & 3;
    const int si = 4 * L.l;
    double t[4];
    {
        const double2 v01 = *reinterpret_cast<const double2*>(&sm.x[slot][si]);
        const double2 v23 = *reinterpret_cast<const double2*>(&sm.x[slot][si + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&sm.b[slot][si]);
        const double2 b23 = *reinterpret_cast<const double2*>(&sm.b[slot][si + 2]);
        t[0] = v01.x + G.c, t[1] = v01.y + G.c, t[2] = v23.x + G.c, t[3] = v23.y + G.c;
        if (k < 0 || k >= G.ny || L.frozen) {  // rows outside the domain / frozen lanes hold 0
#pragma unroll
            for (int q = 0; q < 4; ++q) t[q] = 0.0;
        } else if (L.spec) {  // columns outside the domain hold 0
#pragma unroll
            for (int q = 0; q < 4; ++q) t[q] = L.dom[q] ? t[q] : 0.0;
        }
        w.b[s0][0] = b01.x, w.b[s0][1] = b01.y, w.b[s0][2] = b23.x, w.b[s0][3] = b23.y;
    }
    double* x1 = w.x[s1];
    double* x2 = w.x[s2];
    double* x3 = w.x[s3];
    const double* x4 = w.x[s0];  // row k-4
    // neighbour exchanges (inputs final before this iteration)
    const double redW = sh_up(x1[3]), redE = sh_dn(x1[0]);  // raw black edges of row k-1
    const double blkW = sh_up(x2[3]), blkE = sh_dn(x2[0]);  // red edges of row k-2
    const double resW = sh_up(x3[3]), resE = sh_dn(x3[0]);  // final edges of row k-3
    // ---- red half-sweep of row j = k-1 (red cells: col + j even; S = row k-2, N = row k)
    {
        const int j = k - 1;
        if (j >= G.r0 - 2 && j >= 0 && j < G.ny) {
            const double* b = w.b[s1];
            constexpr int qa = P1, qb = qa + 2;
            const double Wa = qa == 0 ? redW : x1[0], Ea = x1[qa + 1];
            const double Wb = x1[qb - 1], Eb = qb == 3 ? redE : x1[3];
            double va = ((((Wa + Ea) + x2[qa]) + t[qa]) - b[qa]) * 0.25;
            double vb = ((((Wb + Eb) + x2[qb]) + t[qb]) - b[qb]) * 0.25;
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                va = L.red[qa] ? gs_exact(Wa, Ea, x2[qa], t[qa], b[qa], L.dc[qa] + dr) : x1[qa];
                vb = L.red[qb] ? gs_exact(Wb, Eb, x2[qb], t[qb], b[qb], L.dc[qb] + dr) : x1[qb];
            }
            if (!L.frozen) x1[qa] = va, x1[qb] = vb;
        }
    }
    // ---- black half-sweep of row j = k-2 (parity 1 - P1; S = row k-3, N = row k-1 relaxed)
    {
        const int j = k - 2;
        if (j >= G.r0 - 1 && j >= 0 && j < G.ny) {
            const double* b = w.b[s2];
            // black cells of row k-2 ((col + j) odd) sit in the columns of row k-1's red cells
            constexpr int qa = P1, qb = qa + 2;
            const double Wa = qa == 0 ? blkW : x2[0], Ea = x2[qa + 1];
            const double Wb = x2[qb - 1], Eb = qb == 3 ? blkE : x2[3];
            double va = ((((Wa + Ea) + x3[qa]) + x1[qa]) - b[qa]) * 0.25;
            double vb = ((((Wb + Eb) + x3[qb]) + x1[qb]) - b[qb]) * 0.25;
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                va = L.blk[qa] ? gs_exact(Wa, Ea, x3[qa], x1[qa], b[qa], L.dc[qa] + dr) : x2[qa];
                vb = L.blk[qb] ? gs_exact(Wb, Eb, x3[qb], x1[qb], b[qb], L.dc[qb] + dr) : x2[qb];
            }
            if (!L.frozen) x2[qa] = va, x2[qb] = vb;
        }
    }
    // ---- residual of row j = k-3 (smoother.hpp:121-141) and store
    {
        const int j = k - 3;
        if (j >= G.r0 && j < G.r1 && L.owned) {
            const double* b = w.b[s3];
            double r[4];
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                r[0] = b[0] - ((((resW + x3[1]) + x4[0]) + x2[0]) - (L.dc[0] + dr) * x3[0]);
                r[1] = b[1] - ((((x3[0] + x3[2]) + x4[1]) + x2[1]) - (L.dc[1] + dr) * x3[1]);
                r[2] = b[2] - ((((x3[1] + x3[3]) + x4[2]) + x2[2]) - (L.dc[2] + dr) * x3[2]);
                r[3] = b[3] - ((((x3[2] + resE) + x4[3]) + x2[3]) - (L.dc[3] + dr) * x3[3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) r[q] = L.dom[q] ? r[q] : 0.0;
            } else {
                r[0] = b[0] - ((((resW + x3[1]) + x4[0]) + x2[0]) - 4.0 * x3[0]);
                r[1] = b[1] - ((((x3[0] + x3[2]) + x4[1]) + x2[1]) - 4.0 * x3[1]);
                r[2] = b[2] - ((((x3[1] + x3[3]) + x4[2]) + x2[2]) - 4.0 * x3[2]);
                r[3] = b[3] - ((((x3[2] + resE) + x4[3]) + x2[3]) - 4.0 * x3[3]);
            }
            const double m01 = max_drop_nan(fabs(r[0]), fabs(r[1])), m23 = max_drop_nan(fabs(r[2]), fabs(r[3]));
            A.mx = max_drop_nan(A.mx, max_drop_nan(m01, m23));  // std::max(rmax, |r|): NaN dropped
            A.sx = A.sx + ((x3[0] + x3[1]) + (x3[2] + x3[3]));   // out-of-domain cells hold 0
            A.tacc = A.tacc + ((r[0] + r[1]) + (r[2] + r[3]));
            put_row(G, L, j, x3);
        }
    }
    // row k takes the slot of row k-4
#pragma unroll
    for (int q = 0; q < 4; ++q) w.x[s0][q] = t[q];
}

// tile row-block complete: fold the g = tile/4 lanes of every coarse cell
// (groups start at lane 1; the tile is a power of two)
template <bool MP>
__device__ __forceinline__ void tile_flush_w(const Params& P, const Lane& L, int j, int lg, Acc& A, double* mpk) {
    const int g = P.tile >> 2;
    double v = A.tacc;
    for (int o = g >> 1; o > 0; o >>= 1) v = v + __shfl_down_sync(kFull, v, o);
    if (L.owned && ((L.l - 1) & (g - 1)) == 0 && L.dom[0]) {
        if (MP) mpk[P.cb_off + int64_t(j >> lg) * P.cb_pitch + (L.c0 >> lg)] = v;  // multi-GPU: own pack slot
        else P.cbw.at(L.c0 >> lg, j >> lg) = v;
        A.cm = max_drop_nan(A.cm, fabs(v));
        A.nan |= (v != v);  // a NaN residual poisons its tile sum
    }
    A.tacc = 0.0;
}

__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Warp-level epilogue, a fixed two-level tree (deterministic sums): every warp
// (= CTA) stores its partial triple; the last warp of each group of 32 CTAs
// folds the group (one partial per lane); the last group folds the group
// partials and applies the reference's branch logic. (A single final warp
// folding all ~5500 partials serially added a multi-microsecond tail to every
// pass.) Scratch: part = [3 per CTA | 3 per group], ticket = [all | per group].
template <bool MP>
__device__ __forceinline__ void warp_epilogue(const Params& P, int mode, double mx, double sx, double cm, int nan,
                                              const Ctl& st) {
    const int nb = gridDim.x * gridDim.y;
    const int bid = blockIdx.y * gridDim.x + blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int ng = (nb + 31) >> 5, grp = bid >> 5;
    double* gpart = P.part + 3 * nb;
    mx = warp_max(mx);
    sx = warp_sum_down(sx);
    cm = warp_max(cm);
    const int anynan = __any_sync(kFull, nan);
    unsigned last = 0;
    if (lane == 0) {
        P.part[3 * bid] = mx;
        P.part[3 * bid + 1] = sx;
        P.part[3 * bid + 2] = cm;
        if (anynan) P.ctl->nan_seen = 1;
        // release: the partials before the ticket, without the full fence's L1
        // invalidation (CCTL.IVALL was the sweep pass's top stall line at 16384^2);
        // the group's last warp acquires with the fence below
        const unsigned gsize = unsigned(min(32, nb - 32 * grp));
        last = atom_add_release(&P.ticket[1 + grp], 1u) == gsize - 1;
    }
    if (!__shfl_sync(kFull, last, 0)) return;
    __threadfence();
    {  // fold the group: member 32 grp + lane
        const int k = 32 * grp + lane;
        double m = 0.0, s = 0.0, c = 0.0;
        if (k < nb) m = __ldcg(&P.part[3 * k]), s = __ldcg(&P.part[3 * k + 1]), c = __ldcg(&P.part[3 * k + 2]);
        m = warp_max(m);
        s = warp_sum_down(s);
        c = warp_max(c);
        last = 0;
        if (lane == 0) {
            gpart[3 * grp] = m, gpart[3 * grp + 1] = s, gpart[3 * grp + 2] = c;
            P.ticket[1 + grp] = 0u;
            __threadfence();
            last = atomicAdd(P.ticket, 1u) == unsigned(ng - 1);
        }
    }
    if (!__shfl_sync(kFull, last, 0)) return;
    __threadfence();
    double m = 0.0, s = 0.0, c = 0.0;
    for (int k = lane; k < ng; k += 32) {
        m = fmax(m, __ldcg(&gpart[3 * k]));
        s += __ldcg(&gpart[3 * k + 1]);
        c = fmax(c, __ldcg(&gpart[3 * k + 2]));
    }
    m = warp_max(m);
    s = warp_sum_down(s);
    c = warp_max(c);
    if (lane == 0) {
        if constexpr (MP) {  // to every rank's pack slot, then raise this rank's flag on every rank
            const int p = int(st.mp_seq & 1ull);
            double* mine = P.xch[P.rank] + (int64_t(p) * P.nranks + P.rank) * P.pack_len;
            mine[0] = m, mine[1] = c, mine[2] = 1.0, mine[3] = double(mode), mine[4] = s;
            fence_release_sys();  // with the tickets' chain: this pass's whole slot before the flags
#ifdef ISMG_MP_TRACE
            P.ctl->mp_t1 = (unsigned long long)gtimer();
#endif
            for (int q = 0; q < P.nranks; ++q)
                atomicExch(P.xflag[q] + P.rank, st.mp_seq + 1ull);  // mp_unpack_kernel waits for these
        } else {
            fine_decide(P, mode, m, s, c);
        }
        *P.ticket = 0u;
        __threadfence();
    }
}

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

template <bool MP>
__device__ __forceinline__ void sweep_w(SmemW& sm, const Params& P, const Ctl& st, int nq) {
    const int W = 4 * nq;
    const int a = blockIdx.x * W;
    const Lane L(P, a, nq);
    Geo G;
    G.r0 = P.row0 + blockIdx.y * P.H, G.r1 = min(G.r0 + P.H, P.row1), G.ny = P.ny;
    G.c = st.has_shift ? st.shift : -0.0;  // x + (-0.0) == x for every x
    G.fwS = face_weight(P.bc.k[ISMG_SIDE_SOUTH]), G.fwN = face_weight(P.bc.k[ISMG_SIDE_NORTH]);
    G.outp = st.buf[st.cur ^ 1] + L.c0;
    G.pitch = P.pitch;
    const int mpp = int(st.mp_seq & 1ull);  // multi-GPU: this pass's pack parity
    double* mpk = MP ? my_pack(P, mpp) : nullptr;
    const int tmask = P.tile - 1, lg = ilog2(P.tile);
    const uint32_t bytes = uint32_t(((min(a + W + 4, P.nx + 5) - (a - 4)) + 1) & ~1) * 8u;
    const double* xin = st.buf[st.cur];
    const double* brow0 = st.b + (a - 4);
    auto xsrc = [&](int k) {  // x row k (multi-GPU: the neighbours' rows from the gathered packs)
        return MP ? row_src(P, xin, k, a - 4, mpp ^ 1) : xin + int64_t(k) * G.pitch + (a - 4);
    };
    const int kfirst = G.r0 - 3, klast = G.r1 + 2;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < kRingW; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    for (int s = 0; s < kRingW && kfirst + s <= klast; ++s)
        issue_row_w(sm, xsrc(kfirst + s), brow0 + int64_t(kfirst + s) * G.pitch, s, bytes);
    Win w;
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) w.x[s][q] = w.b[s][q] = 0.0;
    Acc A;
    const uint32_t bar0 = su32(&sm.bar[0]);
    int slot = 0;
    uint32_t phase = 0;
    auto row = [&](auto u, int k) {
        constexpr int U = decltype(u)::value;
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), phase);
        step_w<U, (U & 1), MP>(sm, slot, L, G, w, A, k);
        const int j = k - 3;  // tile row-block of row k-3 complete
        if (j >= G.r0 && j < G.r1 && ((j & tmask) == tmask || j == P.ny - 1)) tile_flush_w<MP>(P, L, j, lg, A, mpk);
        __syncwarp();  // every lane has read the slot of row k
        if (k + kRingW <= klast)
            issue_row_w(sm, xsrc(k + kRingW), brow0 + int64_t(k + kRingW) * G.pitch, slot, bytes);
        if (++slot == kRingW) slot = 0, phase ^= 1u;
    };
    // kfirst = r0 - 3 = 1 (mod 4) (P.H is a multiple of 4), so in the block
    // starting at kb the row k-1 = kb - 1 + U has the parity of U
    for (int kb = kfirst; kb <= klast; kb += 4) {
        row(std::integral_constant<int, 0>{}, kb);
        if (kb + 1 <= klast) row(std::integral_constant<int, 1>{}, kb + 1);
        if (kb + 2 <= klast) row(std::integral_constant<int, 2>{}, kb + 2);
        if (kb + 3 <= klast) row(std::integral_constant<int, 3>{}, kb + 3);
    }
    if (MP) mp_push(P, L, G, mpp, G.outp);
    warp_epilogue<MP>(P, kFine, A.mx, A.sx, A.cm, A.nan, st);
}

// ---- PROLONG / RESID: x' = x + c + P ce (coarsening.hpp:495-500), residual and
// restriction of x'. Iteration k loads (and prolongs) row k and forms the
// residual of row k-1 with rows k-2, k-1 in registers.
template <bool MP>
__device__ __forceinline__ void prolong_w(SmemW& sm, const Params& P, const Ctl& st, int nq, bool prolong) {
    const int W = 4 * nq;
    const int a = blockIdx.x * W;
    const Lane L(P, a, nq);
    Geo G;
    G.r0 = P.row0 + blockIdx.y * P.H, G.r1 = min(G.r0 + P.H, P.row1), G.ny = P.ny;
    G.c = st.has_shift ? st.shift : -0.0;
    G.fwS = face_weight(P.bc.k[ISMG_SIDE_SOUTH]), G.fwN = face_weight(P.bc.k[ISMG_SIDE_NORTH]);
    G.outp = st.buf[st.cur ^ 1] + L.c0;
    G.pitch = P.pitch;
    const int mpp = int(st.mp_seq & 1ull);  // multi-GPU: this pass's pack parity
    double* mpk = MP ? my_pack(P, mpp) : nullptr;
    const int tmask = P.tile - 1, lg = ilog2(P.tile);
    const uint32_t bytes = uint32_t(((min(a + W + 4, P.nx + 5) - (a - 4)) + 1) & ~1) * 8u;
    const double* xin = st.buf[st.cur];
    const double* brow0 = st.b + (a - 4);
    auto xsrc = [&](int k) {  // x row k (multi-GPU: the neighbours' rows from the gathered packs)
        return MP ? row_src(P, xin, k, a - 4, mpp ^ 1) : xin + int64_t(k) * G.pitch + (a - 4);
    };
    Acc A;
    // TileAxis::locate_cell of the lane's columns
    int I0[4], I1[4];
    double sq[4], dxq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        I0[q] = I1[q] = 0, sq[q] = 0.0, dxq[q] = 1.0;
        if (prolong && L.dom[q]) {
            const int col = L.c0 + q;
            I0[q] = P.ax.k0[col], I1[q] = P.ax.k1[col], sq[q] = P.ax.t[col], dxq[q] = P.ax.dk[col];
        }
    }
    const int kfirst = G.r0 - 1, klast = G.r1;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < kRingW; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    for (int s = 0; s < kRingW && kfirst + s <= klast; ++s)
        issue_row_w(sm, xsrc(kfirst + s), brow0 + int64_t(kfirst + s) * G.pitch, s, bytes);
    const uint32_t bar0 = su32(&sm.bar[0]);
    double x1[4] = {0, 0, 0, 0}, x2[4] = {0, 0, 0, 0}, b1[4] = {0, 0, 0, 0};
    int slot = 0;
    uint32_t phase = 0;
    const int si = 4 * L.l;
    for (int k = kfirst; k <= klast; ++k) {
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), phase);
        double x0[4], b0[4];
        {
            const double2 v01 = *reinterpret_cast<const double2*>(&sm.x[slot][si]);
            const double2 v23 = *reinterpret_cast<const double2*>(&sm.x[slot][si + 2]);
            const double2 c01 = *reinterpret_cast<const double2*>(&sm.b[slot][si]);
            const double2 c23 = *reinterpret_cast<const double2*>(&sm.b[slot][si + 2]);
            const double raw[4] = {v01.x, v01.y, v23.x, v23.y};
            b0[0] = c01.x, b0[1] = c01.y, b0[2] = c23.x, b0[3] = c23.y;
            const bool rin = k >= 0 && k < G.ny;
            double tt = 0.0, dy = 1.0;
            int J0 = 0, J1 = 0;
            if (prolong && rin) tt = P.ay.t[k], dy = P.ay.dk[k], J0 = P.ay.k0[k], J1 = P.ay.k1[k];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double v = (rin && L.dom[q]) ? raw[q] + G.c : 0.0;
                if (prolong && rin && L.dom[q]) {
                    const double num =
                        (dxq[q] - sq[q]) * ((dy - tt) * P.ce.at(I0[q], J0) + tt * P.ce.at(I0[q], J1)) +
                        sq[q] * ((dy - tt) * P.ce.at(I1[q], J0) + tt * P.ce.at(I1[q], J1));
                    const double den = dxq[q] * dy;
                    // a power-of-two den (uniform tiles): the reciprocal product is the exact quotient
                    if ((__double_as_longlong(den) & 0x000FFFFFFFFFFFFFll) == 0) v += num * pow2_recip(den);
                    else v += div_slow(num, den);
                }
                x0[q] = v;
            }
        }
        const double W1 = sh_up(x1[3]), E1 = sh_dn(x1[0]);
        const int j = k - 1;
        if (L.owned && j >= G.r0 && j < G.r1) {
            const double dr = row_part(G, j);
            double r[4];
            r[0] = b1[0] - ((((W1 + x1[1]) + x2[0]) + x0[0]) - (L.dc[0] + dr) * x1[0]);
            r[1] = b1[1] - ((((x1[0] + x1[2]) + x2[1]) + x0[1]) - (L.dc[1] + dr) * x1[1]);
            r[2] = b1[2] - ((((x1[1] + x1[3]) + x2[2]) + x0[2]) - (L.dc[2] + dr) * x1[2]);
            r[3] = b1[3] - ((((x1[2] + E1) + x2[3]) + x0[3]) - (L.dc[3] + dr) * x1[3]);
#pragma unroll
            for (int q = 0; q < 4; ++q) r[q] = L.dom[q] ? r[q] : 0.0;
            const double m01 = max_drop_nan(fabs(r[0]), fabs(r[1])), m23 = max_drop_nan(fabs(r[2]), fabs(r[3]));
            A.mx = max_drop_nan(A.mx, max_drop_nan(m01, m23));
            A.sx = A.sx + ((x1[0] + x1[1]) + (x1[2] + x1[3]));
            A.tacc = A.tacc + ((r[0] + r[1]) + (r[2] + r[3]));
            if (prolong) put_row(G, L, j, x1);
        }
        if (j >= G.r0 && j < G.r1 && ((j & tmask) == tmask || j == P.ny - 1)) tile_flush_w<MP>(P, L, j, lg, A, mpk);
#pragma unroll
        for (int q = 0; q < 4; ++q) x2[q] = x1[q], x1[q] = x0[q], b1[q] = b0[q];
        __syncwarp();
        if (k + kRingW <= klast)
            issue_row_w(sm, xsrc(k + kRingW), brow0 + int64_t(k + kRingW) * G.pitch, slot, bytes);
        if (++slot == kRingW) slot = 0, phase ^= 1u;
    }
    if (MP) mp_push(P, L, G, mpp, prolong ? G.outp : xin + L.c0);
    warp_epilogue<MP>(P, prolong ? kProlong : kResid, A.mx, A.sx, A.cm, A.nan, st);
}

// ---- PROLONG / RESID, the split single-GPU kernel's version: the columns of a quad that
// share a coarse pair share its row terms (same values, bit for bit). x' = x + c + P ce
// (coarsening.hpp:495-500), residual and
// restriction of x'. Iteration k loads (and prolongs) row k and forms the
// residual of row k-1 with rows k-2, k-1 in registers.
template <bool MP>
__device__ __forceinline__ void prolong_w2(SmemW& sm, const Params& P, const Ctl& st, int nq, bool prolong) {
    const int W = 4 * nq;
    const int a = blockIdx.x * W;
    const Lane L(P, a, nq);
    Geo G;
    G.r0 = P.row0 + blockIdx.y * P.H, G.r1 = min(G.r0 + P.H, P.row1), G.ny = P.ny;
    G.c = st.has_shift ? st.shift : -0.0;
    G.fwS = face_weight(P.bc.k[ISMG_SIDE_SOUTH]), G.fwN = face_weight(P.bc.k[ISMG_SIDE_NORTH]);
    G.outp = st.buf[st.cur ^ 1] + L.c0;
    G.pitch = P.pitch;
    const int mpp = int(st.mp_seq & 1ull);  // multi-GPU: this pass's pack parity
    double* mpk = MP ? my_pack(P, mpp) : nullptr;
    const int tmask = P.tile - 1, lg = ilog2(P.tile);
    const uint32_t bytes = uint32_t(((min(a + W + 4, P.nx + 5) - (a - 4)) + 1) & ~1) * 8u;
    const double* xin = st.buf[st.cur];
    const double* brow0 = st.b + (a - 4);
    const bool alt = MP && st.no_fuse;  // redoing a fused pass's prolongation: the rows it read
    auto xsrc = [&](int k) {  // x row k (multi-GPU: the neighbours' rows from the gathered packs)
        return MP ? row_src(P, xin, k, a - 4, mpp ^ 1, alt) : xin + int64_t(k) * G.pitch + (a - 4);
    };
    Acc A;
    // TileAxis::locate_cell of the lane's columns
    int I0[4], I1[4];
    double sq[4], dxq[4], idx[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        I0[q] = I1[q] = 0, sq[q] = 0.0, dxq[q] = 1.0;
        if (prolong && L.dom[q]) {
            const int col = L.c0 + q;
            I0[q] = P.ax.k0[col], I1[q] = P.ax.k1[col], sq[q] = P.ax.t[col], dxq[q] = P.ax.dk[col];
        }
        idx[q] = is_pow2(dxq[q]) ? pow2_recip(dxq[q]) : 0.0;  // exact reciprocal, or 0: divide
    }
    // columns of a quad that share the previous column's coarse pair reuse its row terms
    // (a quad inside one half tile: one pair, 4 coarse loads per row instead of 16)
    bool same[4];
    same[0] = false;
#pragma unroll
    for (int q = 1; q < 4; ++q) same[q] = I0[q] == I0[q - 1] && I1[q] == I1[q - 1];
#ifndef ISMG_PH2_NOFAST
    // The fast row body (uniform power-of-two tiles, the whole interior of a
    // config-3 grid): every in-domain column of the lane has a power-of-two extent
    // and the quad's coarse pair, so the column weights can carry 1/dx and the
    // row weights 1/dy. Scaling by a power of two is exact, so
    //   ((dx-s)/dx) ((dy-t)/dy c00 + t/dy c01) + ...   ==   (...) / (dx dy)
    // bit for bit (as long as no product is subnormal), with 5 instead of 10
    // fp64 operations per cell and no per-cell reciprocal product.
    bool lok = true;
    double ar[4], sr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        ar[q] = (dxq[q] - sq[q]) * idx[q], sr[q] = sq[q] * idx[q];
        if (prolong && L.dom[q]) lok = lok && idx[q] != 0.0 && (q == 0 || same[q]);
    }
    bool fast = __all_sync(kFull, lok);
#else
    bool fast = false;
    double ar[4] = {0, 0, 0, 0}, sr[4] = {0, 0, 0, 0};
#endif
    const int kfirst = G.r0 - 1, klast = G.r1;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < kRingW; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    for (int s = 0; s < kRingW && kfirst + s <= klast; ++s)
        issue_row_w(sm, xsrc(kfirst + s), brow0 + int64_t(kfirst + s) * G.pitch, s, bytes);
    const uint32_t bar0 = su32(&sm.bar[0]);
#ifdef ISMG_PH2_ROLLED
    double x1[4] = {0, 0, 0, 0}, x2[4] = {0, 0, 0, 0}, b1[4] = {0, 0, 0, 0};
#endif
    int slot = 0;
    uint32_t phase = 0;
    const int si = 4 * L.l;
    // TileAxis::locate_cell of the rows, one row ahead (the loads leave the row's
    // critical path), and the lane's coarse values c(I0/I1, J0/J1) of the first
    // column pair, reloaded only when the row's coarse pair (J0, J1) changes (every
    // half tile) instead of four dependent L2 loads per row
    // the chunk's rows of the y-axis tables, staged once into shared memory with
    // coalesced loads (four dependent L2 loads per row were the pass's top stall)
    constexpr int kAxRows = 100;
    __shared__ double s_at[kAxRows], s_adk[kAxRows];
    __shared__ int s_ak0[kAxRows], s_ak1[kAxRows];
    const bool tab = prolong && klast - kfirst + 2 <= kAxRows;
    if (tab) {
        bool rok = true;  // every row of the chunk has a power-of-two extent
        for (int i = int(threadIdx.x & 31); i < klast - kfirst + 2; i += 32) {
            const int k = kfirst + i;
            if (k >= 0 && k < G.ny) rok = rok && is_pow2(P.ay.dk[k]);
        }
        fast = __all_sync(kFull, rok) && fast;
        for (int i = int(threadIdx.x & 31); i < klast - kfirst + 2; i += 32) {
            const int k = kfirst + i;
            const bool in = k >= 0 && k < G.ny;
            const double t = in ? P.ay.t[k] : 0.0, dk = in ? P.ay.dk[k] : 1.0;
            if (fast) {  // the row weights (dy - t) / dy and t / dy, exact
                const double idk = pow2_recip(dk);
                s_at[i] = (dk - t) * idk, s_adk[i] = t * idk;
            } else {
                s_at[i] = t, s_adk[i] = dk;
            }
            s_ak0[i] = in ? P.ay.k0[k] : 0, s_ak1[i] = in ? P.ay.k1[k] : 0;
        }
        __syncwarp();
    } else {
        fast = false;
    }
    auto row_axis = [&](int k, double& t_, double& d_, int& j0_, int& j1_) {
        t_ = 0.0, d_ = 1.0, j0_ = 0, j1_ = 0;
        if (tab) {
            const int i = k - kfirst;
            t_ = s_at[i], d_ = s_adk[i], j0_ = s_ak0[i], j1_ = s_ak1[i];
        } else if (prolong && k >= 0 && k < G.ny) {
            t_ = P.ay.t[k], d_ = P.ay.dk[k], j0_ = P.ay.k0[k], j1_ = P.ay.k1[k];
        }
    };
    double tt_n, dy_n;
    int J0_n, J1_n;
    row_axis(kfirst, tt_n, dy_n, J0_n, J1_n);
    int cJ0 = -1, cJ1 = -1;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#ifdef ISMG_PH2_ROLLED  // A/B hook: the row loop with register shifts (round-2 first version)
    for (int k = kfirst; k <= klast; ++k) {
        const double tt = tt_n, dy = dy_n;
        const int J0 = J0_n, J1 = J1_n;
        row_axis(k + 1, tt_n, dy_n, J0_n, J1_n);
        if (prolong && L.dom[0] && (J0 != cJ0 || J1 != cJ1)) {
            c00 = P.ce.at(I0[0], J0), c01 = P.ce.at(I0[0], J1), c10 = P.ce.at(I1[0], J0), c11 = P.ce.at(I1[0], J1);
            cJ0 = J0, cJ1 = J1;
        }
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), phase);
        double x0[4], b0[4];
        {
            const double2 v01 = *reinterpret_cast<const double2*>(&sm.x[slot][si]);
            const double2 v23 = *reinterpret_cast<const double2*>(&sm.x[slot][si + 2]);
            const double2 c01v = *reinterpret_cast<const double2*>(&sm.b[slot][si]);
            const double2 c23v = *reinterpret_cast<const double2*>(&sm.b[slot][si + 2]);
            const double raw[4] = {v01.x, v01.y, v23.x, v23.y};
            b0[0] = c01v.x, b0[1] = c01v.y, b0[2] = c23v.x, b0[3] = c23v.y;
            const bool rin = k >= 0 && k < G.ny;
            const double wy0 = dy - tt;
            // power-of-two extents (uniform tiles): num / (dx dy) is exactly num ((1/dx) (1/dy))
            const double idy = is_pow2(dy) ? pow2_recip(dy) : 0.0;
            double ca = 0.0, cb = 0.0;  // the column pair's row terms (dy-t) c(I,J0) + t c(I,J1)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double v = (rin && L.dom[q]) ? raw[q] + G.c : 0.0;
                if (prolong && rin && L.dom[q]) {
                    if (q == 0) {
                        ca = wy0 * c00 + tt * c01;
                        cb = wy0 * c10 + tt * c11;
                    } else if (!same[q]) {
                        ca = wy0 * P.ce.at(I0[q], J0) + tt * P.ce.at(I0[q], J1);
                        cb = wy0 * P.ce.at(I1[q], J0) + tt * P.ce.at(I1[q], J1);
                    }
                    const double num = (dxq[q] - sq[q]) * ca + sq[q] * cb;
                    const double r = idx[q] * idy;
                    if (r != 0.0) v += num * r;
                    else v += div_slow(num, dxq[q] * dy);
                }
                x0[q] = v;
            }
        }
        const double W1 = sh_up(x1[3]), E1 = sh_dn(x1[0]);
        const int j = k - 1;
        if (L.owned && j >= G.r0 && j < G.r1) {
            const double dr = row_part(G, j);
            double r[4];
            r[0] = b1[0] - ((((W1 + x1[1]) + x2[0]) + x0[0]) - (L.dc[0] + dr) * x1[0]);
            r[1] = b1[1] - ((((x1[0] + x1[2]) + x2[1]) + x0[1]) - (L.dc[1] + dr) * x1[1]);
            r[2] = b1[2] - ((((x1[1] + x1[3]) + x2[2]) + x0[2]) - (L.dc[2] + dr) * x1[2]);
            r[3] = b1[3] - ((((x1[2] + E1) + x2[3]) + x0[3]) - (L.dc[3] + dr) * x1[3]);
#pragma unroll
            for (int q = 0; q < 4; ++q) r[q] = L.dom[q] ? r[q] : 0.0;
            const double m01 = max_drop_nan(fabs(r[0]), fabs(r[1])), m23 = max_drop_nan(fabs(r[2]), fabs(r[3]));
            A.mx = max_drop_nan(A.mx, max_drop_nan(m01, m23));
            A.sx = A.sx + ((x1[0] + x1[1]) + (x1[2] + x1[3]));
            A.tacc = A.tacc + ((r[0] + r[1]) + (r[2] + r[3]));
            if (prolong) put_row(G, L, j, x1);
        }
        if (j >= G.r0 && j < G.r1 && ((j & tmask) == tmask || j == P.ny - 1)) tile_flush_w<MP>(P, L, j, lg, A, mpk);
#pragma unroll
        for (int q = 0; q < 4; ++q) x2[q] = x1[q], x1[q] = x0[q], b1[q] = b0[q];
        __syncwarp();
        if (k + kRingW <= klast)
            issue_row_w(sm, xsrc(k + kRingW), brow0 + int64_t(k + kRingW) * G.pitch, slot, bytes);
        if (++slot == kRingW) slot = 0, phase ^= 1u;
    }
#else
    // Rows in 4-row blocks with a compile-time register window (as the sweep pass):
    // same-box A/B (tools/visit_hist.py) 16384^2 steps 1-2 1811 / 1880 ms against
    // 1850 / 1920 with the shifting loop.
    // at row k (U = its index in the block) rows k, k-1, k-2 live in slots U,
    // (U+3)&3, (U+2)&3, so no row shifts through registers.
    double xw[4][4], bw[4][4];
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2)
#pragma unroll
        for (int q = 0; q < 4; ++q) xw[s2][q] = bw[s2][q] = 0.0;
    auto row = [&](auto u, auto fastc, int k) {
        constexpr int U = decltype(u)::value, U1 = (U + 3) & 3, U2 = (U + 2) & 3;
        constexpr bool FAST = decltype(fastc)::value;
        const double tt = tt_n, dy = dy_n;
        const int J0 = J0_n, J1 = J1_n;
        row_axis(k + 1, tt_n, dy_n, J0_n, J1_n);
        if (prolong && L.dom[0] && (J0 != cJ0 || J1 != cJ1)) {
            c00 = P.ce.at(I0[0], J0), c01 = P.ce.at(I0[0], J1), c10 = P.ce.at(I1[0], J0), c11 = P.ce.at(I1[0], J1);
            cJ0 = J0, cJ1 = J1;
        }
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), phase);
        if constexpr (FAST) {  // tt, dy hold the scaled row weights t / dy, (dy - t) / dy
            const double2 v01 = *reinterpret_cast<const double2*>(&sm.x[slot][si]);
            const double2 v23 = *reinterpret_cast<const double2*>(&sm.x[slot][si + 2]);
            const double2 c01v = *reinterpret_cast<const double2*>(&sm.b[slot][si]);
            const double2 c23v = *reinterpret_cast<const double2*>(&sm.b[slot][si + 2]);
            const double raw[4] = {v01.x, v01.y, v23.x, v23.y};
            bw[U][0] = c01v.x, bw[U][1] = c01v.y, bw[U][2] = c23v.x, bw[U][3] = c23v.y;
            const double ca = tt * c00 + dy * c01, cb = tt * c10 + dy * c11;
#pragma unroll
            for (int q = 0; q < 4; ++q) xw[U][q] = (raw[q] + G.c) + (ar[q] * ca + sr[q] * cb);
            if (k < 0 || k >= G.ny || L.frozen) {
#pragma unroll
                for (int q = 0; q < 4; ++q) xw[U][q] = 0.0;
            } else if (L.spec) {
#pragma unroll
                for (int q = 0; q < 4; ++q) xw[U][q] = L.dom[q] ? xw[U][q] : 0.0;
            }
        } else {
            const double2 v01 = *reinterpret_cast<const double2*>(&sm.x[slot][si]);
            const double2 v23 = *reinterpret_cast<const double2*>(&sm.x[slot][si + 2]);
            const double2 c01v = *reinterpret_cast<const double2*>(&sm.b[slot][si]);
            const double2 c23v = *reinterpret_cast<const double2*>(&sm.b[slot][si + 2]);
            const double raw[4] = {v01.x, v01.y, v23.x, v23.y};
            bw[U][0] = c01v.x, bw[U][1] = c01v.y, bw[U][2] = c23v.x, bw[U][3] = c23v.y;
            const bool rin = k >= 0 && k < G.ny;
            const double wy0 = dy - tt;
            const double idy = is_pow2(dy) ? pow2_recip(dy) : 0.0;
            double ca = 0.0, cb = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double v = (rin && L.dom[q]) ? raw[q] + G.c : 0.0;
                if (prolong && rin && L.dom[q]) {
                    if (q == 0) {
                        ca = wy0 * c00 + tt * c01;
                        cb = wy0 * c10 + tt * c11;
                    } else if (!same[q]) {
                        ca = wy0 * P.ce.at(I0[q], J0) + tt * P.ce.at(I0[q], J1);
                        cb = wy0 * P.ce.at(I1[q], J0) + tt * P.ce.at(I1[q], J1);
                    }
                    const double num = (dxq[q] - sq[q]) * ca + sq[q] * cb;
                    const double r = idx[q] * idy;
                    if (r != 0.0) v += num * r;
                    else v += div_slow(num, dxq[q] * dy);
                }
                xw[U][q] = v;
            }
        }
        const double W1 = sh_up(xw[U1][3]), E1 = sh_dn(xw[U1][0]);
        const int j = k - 1;
        if (L.owned && j >= G.r0 && j < G.r1) {
            double r[4];
            if (!FAST || (j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                r[0] = bw[U1][0] - ((((W1 + xw[U1][1]) + xw[U2][0]) + xw[U][0]) - (L.dc[0] + dr) * xw[U1][0]);
                r[1] = bw[U1][1] - ((((xw[U1][0] + xw[U1][2]) + xw[U2][1]) + xw[U][1]) - (L.dc[1] + dr) * xw[U1][1]);
                r[2] = bw[U1][2] - ((((xw[U1][1] + xw[U1][3]) + xw[U2][2]) + xw[U][2]) - (L.dc[2] + dr) * xw[U1][2]);
                r[3] = bw[U1][3] - ((((xw[U1][2] + E1) + xw[U2][3]) + xw[U][3]) - (L.dc[3] + dr) * xw[U1][3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) r[q] = L.dom[q] ? r[q] : 0.0;
            } else {  // interior cells of an interior row: d = 4 (col_diag + row_part, exact)
                r[0] = bw[U1][0] - ((((W1 + xw[U1][1]) + xw[U2][0]) + xw[U][0]) - 4.0 * xw[U1][0]);
                r[1] = bw[U1][1] - ((((xw[U1][0] + xw[U1][2]) + xw[U2][1]) + xw[U][1]) - 4.0 * xw[U1][1]);
                r[2] = bw[U1][2] - ((((xw[U1][1] + xw[U1][3]) + xw[U2][2]) + xw[U][2]) - 4.0 * xw[U1][2]);
                r[3] = bw[U1][3] - ((((xw[U1][2] + E1) + xw[U2][3]) + xw[U][3]) - 4.0 * xw[U1][3]);
            }
            const double m01 = max_drop_nan(fabs(r[0]), fabs(r[1])), m23 = max_drop_nan(fabs(r[2]), fabs(r[3]));
            A.mx = max_drop_nan(A.mx, max_drop_nan(m01, m23));
            A.sx = A.sx + ((xw[U1][0] + xw[U1][1]) + (xw[U1][2] + xw[U1][3]));
            A.tacc = A.tacc + ((r[0] + r[1]) + (r[2] + r[3]));
            if (prolong) put_row(G, L, j, xw[U1]);
        }
        if (j >= G.r0 && j < G.r1 && ((j & tmask) == tmask || j == P.ny - 1)) tile_flush_w<MP>(P, L, j, lg, A, mpk);
        __syncwarp();
        if (k + kRingW <= klast)
            issue_row_w(sm, xsrc(k + kRingW), brow0 + int64_t(k + kRingW) * G.pitch, slot, bytes);
        if (++slot == kRingW) slot = 0, phase ^= 1u;
    };
    auto rows = [&](auto fastc) {
        for (int kb = kfirst; kb <= klast; kb += 4) {
            row(std::integral_constant<int, 0>{}, fastc, kb);
            if (kb + 1 <= klast) row(std::integral_constant<int, 1>{}, fastc, kb + 1);
            if (kb + 2 <= klast) row(std::integral_constant<int, 2>{}, fastc, kb + 2);
            if (kb + 3 <= klast) row(std::integral_constant<int, 3>{}, fastc, kb + 3);
        }
    };
    if (fast) rows(std::true_type{});
    else rows(std::false_type{});
#endif
    if (MP) mp_push(P, L, G, mpp, prolong ? G.outp : xin + L.c0);
    warp_epilogue<MP>(P, prolong ? kProlong : kResid, A.mx, A.sx, A.cm, A.nan, st);
}

// ---- FUSED (kFused; single GPU, uniform power-of-two tiles): the prolongation pass
// and the first sweep after it in ONE HBM pass. Row k is loaded and prolonged,
// x' = (x + c) + P ce (coarsening.hpp:495-500; the fast rows of prolong_w2), then
// shifted by the prolonged field's anchor, x'' = x' + c' (cycles.hpp:142; c' from
// prolong_sum_kernel as -(sum of P ce) / cells, the field being anchored before).
// The prolongation's residual rp (cycles.hpp:141) is formed on the unrelaxed rows
// k-2 (a pristine copy), k-1, k; then the red / black sweep, its residual and tile
// sums run exactly as in sweep_w (cycles.hpp:148-152). The pass reads x, b and
// writes x once: the two passes it replaces moved 48 B per cell, it moves 24.
#ifndef ISMG_FINE_MINB_FU
// 11 resident warps (168 registers, no rematerialisation of the lane constants). Same-box
// A/B (tools/visit_hist.py 16384 32 3, solve ms of steps 1-3): 11 -> 1239 / 1385 / 1880,
// 12 (166 registers) -> 1308 / 1441 / 1943, 10 -> 1372 / 1495 / 2008 (profiles/r02_ab_fused_minb.txt)
#define ISMG_FINE_MINB_FU 11
#endif
constexpr int kFuRows = 104;  // staged y-axis rows: chunk + 3 + 3 halo + 1

struct ProW {
    double ar[4], sr[4];  // column weights (dx - s) / dx, s / dx (exact: dx is a power of two)
    int i0, i1;           // the quad's coarse pair (one per quad on uniform tiles)
};

template <int U, int P1>
__device__ __forceinline__ void step_f(const SmemW& sm, int slot, const Lane& L, const Geo& G, Win& w, Acc& A, int k,
                                       const ProW& pw, double cN, double ca, double cb, double* px, double& mxp) {
    constexpr int s0 = U, s1 = (U + 3) & 3, s2 = (U + 2) & 3, s3 = (U + 1) & 3;
    const int si = 4 * L.l;
    double t[4];
    {
        const double2 v01 = *reinterpret_cast<const double2*>(&sm.x[slot][si]);
        const double2 v23 = *reinterpret_cast<const double2*>(&sm.x[slot][si + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&sm.b[slot][si]);
        const double2 b23 = *reinterpret_cast<const double2*>(&sm.b[slot][si + 2]);
        const double raw[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = ((raw[q] + G.c) + (pw.ar[q] * ca + pw.sr[q] * cb)) + cN;
        if (k < 0 || k >= G.ny || L.frozen) {
#pragma unroll
            for (int q = 0; q < 4; ++q) t[q] = 0.0;
        } else if (L.spec) {
#pragma unroll
            for (int q = 0; q < 4; ++q) t[q] = L.dom[q] ? t[q] : 0.0;
        }
        w.b[s0][0] = b01.x, w.b[s0][1] = b01.y, w.b[s0][2] = b23.x, w.b[s0][3] = b23.y;
    }
    double* x1 = w.x[s1];
    double* x2 = w.x[s2];
    double* x3 = w.x[s3];
    const double* x4 = w.x[s0];  // row k-4
    const double redW = sh_up(x1[3]), redE = sh_dn(x1[0]);  // row k-1, unrelaxed
    const double blkW = sh_up(x2[3]), blkE = sh_dn(x2[0]);
    const double resW = sh_up(x3[3]), resE = sh_dn(x3[0]);
    // ---- rp: residual of the prolonged row j = k-1 (S = row k-2 before its red cells moved)
    {
        const int j = k - 1;
        if (j >= G.r0 && j < G.r1 && L.owned) {
            const double* b = w.b[s1];
            double r[4];
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                r[0] = b[0] - ((((redW + x1[1]) + px[0]) + t[0]) - (L.dc[0] + dr) * x1[0]);
                r[1] = b[1] - ((((x1[0] + x1[2]) + px[1]) + t[1]) - (L.dc[1] + dr) * x1[1]);
                r[2] = b[2] - ((((x1[1] + x1[3]) + px[2]) + t[2]) - (L.dc[2] + dr) * x1[2]);
                r[3] = b[3] - ((((x1[2] + redE) + px[3]) + t[3]) - (L.dc[3] + dr) * x1[3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) r[q] = L.dom[q] ? r[q] : 0.0;
            } else {
                r[0] = b[0] - ((((redW + x1[1]) + px[0]) + t[0]) - 4.0 * x1[0]);
                r[1] = b[1] - ((((x1[0] + x1[2]) + px[1]) + t[1]) - 4.0 * x1[1]);
                r[2] = b[2] - ((((x1[1] + x1[3]) + px[2]) + t[2]) - 4.0 * x1[2]);
                r[3] = b[3] - ((((x1[2] + redE) + px[3]) + t[3]) - 4.0 * x1[3]);
            }
            const double m01 = max_drop_nan(fabs(r[0]), fabs(r[1])), m23 = max_drop_nan(fabs(r[2]), fabs(r[3]));
            mxp = max_drop_nan(mxp, max_drop_nan(m01, m23));
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) px[q] = x1[q];  // row k-1 unrelaxed, the next iteration's S
    // ---- red half-sweep of row j = k-1 (as step_w)
    {
        const int j = k - 1;
        if (j >= G.r0 - 2 && j >= 0 && j < G.ny) {
            const double* b = w.b[s1];
            constexpr int qa = P1, qb = qa + 2;
            const double Wa = qa == 0 ? redW : x1[0], Ea = x1[qa + 1];
            const double Wb = x1[qb - 1], Eb = qb == 3 ? redE : x1[3];
            double va = ((((Wa + Ea) + x2[qa]) + t[qa]) - b[qa]) * 0.25;
            double vb = ((((Wb + Eb) + x2[qb]) + t[qb]) - b[qb]) * 0.25;
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                va = L.red[qa] ? gs_exact(Wa, Ea, x2[qa], t[qa], b[qa], L.dc[qa] + dr) : x1[qa];
                vb = L.red[qb] ? gs_exact(Wb, Eb, x2[qb], t[qb], b[qb], L.dc[qb] + dr) : x1[qb];
            }
            if (!L.frozen) x1[qa] = va, x1[qb] = vb;
        }
    }
    // ---- black half-sweep of row j = k-2
    {
        const int j = k - 2;
        if (j >= G.r0 - 1 && j >= 0 && j < G.ny) {
            const double* b = w.b[s2];
            constexpr int qa = P1, qb = qa + 2;
            const double Wa = qa == 0 ? blkW : x2[0], Ea = x2[qa + 1];
            const double Wb = x2[qb - 1], Eb = qb == 3 ? blkE : x2[3];
            double va = ((((Wa + Ea) + x3[qa]) + x1[qa]) - b[qa]) * 0.25;
            double vb = ((((Wb + Eb) + x3[qb]) + x1[qb]) - b[qb]) * 0.25;
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                va = L.blk[qa] ? gs_exact(Wa, Ea, x3[qa], x1[qa], b[qa], L.dc[qa] + dr) : x2[qa];
                vb = L.blk[qb] ? gs_exact(Wb, Eb, x3[qb], x1[qb], b[qb], L.dc[qb] + dr) : x2[qb];
            }
            if (!L.frozen) x2[qa] = va, x2[qb] = vb;
        }
    }
    // ---- residual of row j = k-3 and store (as step_w)
    {
        const int j = k - 3;
        if (j >= G.r0 && j < G.r1 && L.owned) {
            const double* b = w.b[s3];
            double r[4];
            if ((j == 0) || (j == G.ny - 1) || L.spec) {
                const double dr = row_part(G, j);
                r[0] = b[0] - ((((resW + x3[1]) + x4[0]) + x2[0]) - (L.dc[0] + dr) * x3[0]);
                r[1] = b[1] - ((((x3[0] + x3[2]) + x4[1]) + x2[1]) - (L.dc[1] + dr) * x3[1]);
                r[2] = b[2] - ((((x3[1] + x3[3]) + x4[2]) + x2[2]) - (L.dc[2] + dr) * x3[2]);
                r[3] = b[3] - ((((x3[2] + resE) + x4[3]) + x2[3]) - (L.dc[3] + dr) * x3[3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) r[q] = L.dom[q] ? r[q] : 0.0;
            } else {
                r[0] = b[0] - ((((resW + x3[1]) + x4[0]) + x2[0]) - 4.0 * x3[0]);
                r[1] = b[1] - ((((x3[0] + x3[2]) + x4[1]) + x2[1]) - 4.0 * x3[1]);
                r[2] = b[2] - ((((x3[1] + x3[3]) + x4[2]) + x2[2]) - 4.0 * x3[2]);
                r[3] = b[3] - ((((x3[2] + resE) + x4[3]) + x2[3]) - 4.0 * x3[3]);
            }
            const double m01 = max_drop_nan(fabs(r[0]), fabs(r[1])), m23 = max_drop_nan(fabs(r[2]), fabs(r[3]));
            A.mx = max_drop_nan(A.mx, max_drop_nan(m01, m23));
            A.sx = A.sx + ((x3[0] + x3[1]) + (x3[2] + x3[3]));
            A.tacc = A.tacc + ((r[0] + r[1]) + (r[2] + r[3]));
            put_row(G, L, j, x3);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) w.x[s0][q] = t[q];
}

// the fused pass's epilogue: warp_epilogue with a fourth partial (max |rp|); multi-GPU:
// into this rank's pack slot (scalar 5) for mp_unpack_kernel, which decides
template <bool MP>
__device__ __forceinline__ void fused_epilogue(const Params& P, double mx, double sx, double cm, int nan,
                                               double mp, const Ctl& st) {
    const int nb = gridDim.x * gridDim.y;
    const int bid = blockIdx.y * gridDim.x + blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int ng = (nb + 31) >> 5, grp = bid >> 5;
    double* gpart = P.part + 4 * nb;
    mx = warp_max(mx);
    sx = warp_sum_down(sx);
    cm = warp_max(cm);
    mp = warp_max(mp);
    const int anynan = __any_sync(kFull, nan);
    unsigned last = 0;
    if (lane == 0) {
        P.part[4 * bid] = mx, P.part[4 * bid + 1] = sx, P.part[4 * bid + 2] = cm, P.part[4 * bid + 3] = mp;
        if (anynan) P.ctl->nan_seen = 1;
        const unsigned gsize = unsigned(min(32, nb - 32 * grp));
        last = atom_add_release(&P.ticket[1 + grp], 1u) == gsize - 1;
    }
    if (!__shfl_sync(kFull, last, 0)) return;
    __threadfence();
    {
        const int k = 32 * grp + lane;
        double m = 0.0, s = 0.0, c = 0.0, p = 0.0;
        if (k < nb)
            m = __ldcg(&P.part[4 * k]), s = __ldcg(&P.part[4 * k + 1]), c = __ldcg(&P.part[4 * k + 2]),
            p = __ldcg(&P.part[4 * k + 3]);
        m = warp_max(m);
        s = warp_sum_down(s);
        c = warp_max(c);
        p = warp_max(p);
        last = 0;
        if (lane == 0) {
            gpart[4 * grp] = m, gpart[4 * grp + 1] = s, gpart[4 * grp + 2] = c, gpart[4 * grp + 3] = p;
            P.ticket[1 + grp] = 0u;
            __threadfence();
            last = atomicAdd(P.ticket, 1u) == unsigned(ng - 1);
        }
    }
    if (!__shfl_sync(kFull, last, 0)) return;
    __threadfence();
    double m = 0.0, s = 0.0, c = 0.0, p = 0.0;
    for (int k = lane; k < ng; k += 32) {
        m = fmax(m, __ldcg(&gpart[4 * k]));
        s += __ldcg(&gpart[4 * k + 1]);
        c = fmax(c, __ldcg(&gpart[4 * k + 2]));
        p = fmax(p, __ldcg(&gpart[4 * k + 3]));
    }
    m = warp_max(m);
    s = warp_sum_down(s);
    c = warp_max(c);
    p = warp_max(p);
    if (lane == 0) {
        if constexpr (MP) {
            const int pp = int(st.mp_seq & 1ull);
            double* mine = P.xch[P.rank] + (int64_t(pp) * P.nranks + P.rank) * P.pack_len;
            mine[0] = m, mine[1] = c, mine[2] = 1.0, mine[3] = double(kFused), mine[4] = s, mine[5] = p;
            fence_release_sys();
            for (int q = 0; q < P.nranks; ++q) atomicExch(P.xflag[q] + P.rank, st.mp_seq + 1ull);
        } else {
            fine_decide_fused(P, p, m, s, c);
            publish_phase(P, P.ctl->phase);
        }
        *P.ticket = 0u;
        __threadfence();
    }
}

template <bool MP>
__device__ __forceinline__ void fused_w(SmemW& sm, const Params& P, const Ctl& st, int nq) {
    const int W = 4 * nq;
    const int a = blockIdx.x * W;
    const Lane L(P, a, nq);
    Geo G;
    G.r0 = P.row0 + blockIdx.y * P.H, G.r1 = min(G.r0 + P.H, P.row1), G.ny = P.ny;
    G.c = st.has_shift ? st.shift : -0.0;
    G.fwS = face_weight(P.bc.k[ISMG_SIDE_SOUTH]), G.fwN = face_weight(P.bc.k[ISMG_SIDE_NORTH]);
    G.outp = st.buf[st.cur ^ 1] + L.c0;
    G.pitch = P.pitch;
    const double cN = st.fshift;
    const int tmask = P.tile - 1, lg = ilog2(P.tile);
    const uint32_t bytes = uint32_t(((min(a + W + 4, P.nx + 5) - (a - 4)) + 1) & ~1) * 8u;
    const double* xin = st.buf[st.cur];
    const double* brow0 = st.b + (a - 4);
    const int kfirst = G.r0 - 3, klast = G.r1 + 2;
    const int mpp = int(st.mp_seq & 1ull);  // multi-GPU: this pass's pack parity
    double* mpk = MP ? my_pack(P, mpp) : nullptr;
    auto xsrc = [&](int k) {  // x row k (multi-GPU: the neighbours' rows from the gathered packs)
        return MP ? row_src(P, xin, k, a - 4, mpp ^ 1) : xin + int64_t(k) * G.pitch + (a - 4);
    };
    // the lane's column weights and coarse pair (TileAxis::locate_cell of its columns)
    ProW pw;
    pw.i0 = pw.i1 = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        pw.ar[q] = pw.sr[q] = 0.0;
        if (L.dom[q]) {
            const int col = L.c0 + q;
            const double sq = P.ax.t[col], dxq = P.ax.dk[col], idx = pow2_recip(dxq);
            pw.ar[q] = (dxq - sq) * idx, pw.sr[q] = sq * idx;
            if (q == 0) pw.i0 = P.ax.k0[col], pw.i1 = P.ax.k1[col];
        }
    }
    // the chunk's rows of the y-axis tables, scaled: (dy - t) / dy, t / dy
    __shared__ double s_w0[kFuRows], s_tt[kFuRows];
    __shared__ int s_j0[kFuRows], s_j1[kFuRows];
    for (int i = int(threadIdx.x & 31); i < klast - kfirst + 1; i += 32) {
        const int k = kfirst + i;
        const bool in = k >= 0 && k < G.ny;
        const double t = in ? P.ay.t[k] : 0.0, dk = in ? P.ay.dk[k] : 1.0, idk = pow2_recip(dk);
        s_w0[i] = (dk - t) * idk, s_tt[i] = t * idk;
        s_j0[i] = in ? P.ay.k0[k] : 0, s_j1[i] = in ? P.ay.k1[k] : 0;
    }
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < kRingW; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    for (int s = 0; s < kRingW && kfirst + s <= klast; ++s)
        issue_row_w(sm, xsrc(kfirst + s), brow0 + int64_t(kfirst + s) * G.pitch, s, bytes);
    Win w;
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) w.x[s][q] = w.b[s][q] = 0.0;
    Acc A;
    double px[4] = {0.0, 0.0, 0.0, 0.0}, mxp = 0.0;
    int cJ0 = -1, cJ1 = -1;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    const uint32_t bar0 = su32(&sm.bar[0]);
    int slot = 0;
    uint32_t phase = 0;
    auto row = [&](auto u, int k) {
        constexpr int U = decltype(u)::value;
        const int i = k - kfirst;
        const double w0 = s_w0[i], tt = s_tt[i];
        const int J0 = s_j0[i], J1 = s_j1[i];
        if (L.dom[0] && (J0 != cJ0 || J1 != cJ1)) {
            c00 = P.ce.at(pw.i0, J0), c01 = P.ce.at(pw.i0, J1), c10 = P.ce.at(pw.i1, J0), c11 = P.ce.at(pw.i1, J1);
            cJ0 = J0, cJ1 = J1;
        }
        const double ca = w0 * c00 + tt * c01, cb = w0 * c10 + tt * c11;
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), phase);
        step_f<U, (U & 1)>(sm, slot, L, G, w, A, k, pw, cN, ca, cb, px, mxp);
        const int j = k - 3;
        if (j >= G.r0 && j < G.r1 && ((j & tmask) == tmask || j == P.ny - 1)) tile_flush_w<MP>(P, L, j, lg, A, mpk);
        __syncwarp();
        if (k + kRingW <= klast) issue_row_w(sm, xsrc(k + kRingW), brow0 + int64_t(k + kRingW) * G.pitch, slot, bytes);
        if (++slot == kRingW) slot = 0, phase ^= 1u;
    };
    for (int kb = kfirst; kb <= klast; kb += 4) {
        row(std::integral_constant<int, 0>{}, kb);
        if (kb + 1 <= klast) row(std::integral_constant<int, 1>{}, kb + 1);
        if (kb + 2 <= klast) row(std::integral_constant<int, 2>{}, kb + 2);
        if (kb + 3 <= klast) row(std::integral_constant<int, 3>{}, kb + 3);
    }
    if (MP) {  // output rows for the next pass; input rows for a rollback's redo (h_off[2], [3])
        mp_push(P, L, G, mpp, G.outp);
        mp_push(P, L, G, mpp, xin + L.c0, 2);
    }
    fused_epilogue<MP>(P, A.mx, A.sx, A.cm, A.nan, mxp, st);
}

// kProlong -> kFused: the anchor of the prolonged field from the coarse correction,
// sum(P ce) = sum ce(I, J) pax[I] pay[J], a fixed-order sum (blocks, then the last
// block over the block partials by ticket). The field before the prolongation is
// anchored (its mean is zero up to rounding), so c' = -sum(P ce) / cells.
__global__ void __launch_bounds__(256) prolong_sum_kernel(Params P) {
    Ctl* st = P.ctl;
    if (!P.fuse || st->phase != kProlong || st->no_fuse) return;
    __shared__ double red[8];
    __shared__ int last;
    const int ncx = P.ncx;
    const int64_t n = int64_t(ncx) * P.ncy;
    double v = 0.0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int J = int(k / ncx), I = int(k - int64_t(J) * ncx);
        v += (P.ce.at(I, J) * P.pax[I]) * P.pay[J];
    }
    v = warp_sum_down(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
        P.part[blockIdx.x] = s;
        __threadfence();
        last = atomicAdd(P.ticket, 1u) == gridDim.x - 1;
        if (last) {
            __threadfence();
            double S = 0.0;
            for (int b = 0; b < int(gridDim.x); ++b) S += __ldcg(&P.part[b]);
            st->fshift = P.singular ? -(S / P.ncells) : -0.0;
            st->phase = kFused;
            *P.ticket = 0u;
            __threadfence();
        }
    }
}

// PH selects the phases a kernel serves: 0 all, 1 the sweep only, 2 the
// prolongation / residual pass (prolong_w2). A single-GPU graph slot launches
// PH 2 then PH 0; a multi-GPU slot PH 2, its exchange, PH 1, its exchange (the
// all-phases multi-GPU kernel needs > 128 registers: 8 warps per SM). The kernel whose
// phase it is not exits at once. The PH 0 kernel is the sweep kernel, compiled as it
// was before the split: the sweep sits at the 128-register cap and its speed
// follows the whole kernel's register allocation (measured: a sweep-only
// instantiation, or any growth of the inlined prolongation, ran 142-144 against
// 125 us per 4096^2 pass).
template <bool MP, int PH>
__global__ void __launch_bounds__(32, PH == 2 ? ISMG_FINE_MINB_PR
                                              : (PH == 3 ? ISMG_FINE_MINB_FU
                                                         : (MP ? (PH == 1 ? ISMG_FINE_MINB_MP_SW : ISMG_FINE_MINB_MP)
                                                               : ISMG_FINE_MINB)))
    fine_pass_w_kernel(Params P, int nq) {
    __shared__ __align__(128) SmemW sm;
    {  // not this kernel's phase: exit on one load (the snapshot below copies the whole Ctl
       // through local memory; a no-op launch of 29k CTAs cost ~30 us with it, ncu launch list)
        const int ph = *reinterpret_cast<const volatile int*>(&P.ctl->phase);
        const bool mine = PH == 3   ? ph == kFused
                          : PH == 2 ? (ph == kProlong || ph == kResid)
                          : PH == 1 ? ph == kFine
                                    : (ph == kFine || ph == kProlong || ph == kResid);
        if (!mine) return;
    }
    const Ctl st = *P.ctl;  // snapshot (written only by the previous kernel)
#ifdef ISMG_MP_TRACE
    if (MP && threadIdx.x == 0 && (st.phase == kFine || st.phase == kProlong || st.phase == kResid))
        atomicMin(&P.ctl->mp_t0, (unsigned long long)gtimer());
#endif
    if (PH == 3) {
        if (st.phase == kFused) fused_w<MP>(sm, P, st, nq);
    } else if (PH == 2) {
        if (st.phase == kProlong) prolong_w2<MP>(sm, P, st, nq, true);
        else if (st.phase == kResid) prolong_w2<MP>(sm, P, st, nq, false);
    } else if (PH == 1) {
        if (st.phase == kFine) sweep_w<MP>(sm, P, st, nq);
    } else {
        if (st.phase == kFine) sweep_w<MP>(sm, P, st, nq);
        else if (st.phase == kProlong) prolong_w<MP>(sm, P, st, nq, true);
        else if (st.phase == kResid) prolong_w<MP>(sm, P, st, nq, false);
    }
}

}  // namespace

// owned quads per warp: the most tile-aligned quads that fit 30 lanes
int fine_pass_w_quads(int tile) {
    const int g = tile / 4;
    return (30 / g) * g;
}
int fine_pass_w_resident(bool mp, int device) {
    int per_sm = 0, sms = 0;
    // multi-GPU: the sweep-only kernel the passes launch (the all-phases kernel is an A/B hook);
    // sized on it, 4 GPUs at 16384^2 take 64-row chunks: 226.9 G against 222.1 G with 96
    if (mp) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fine_pass_w_kernel<true, 1>, 32, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fine_pass_w_kernel<false, 0>, 32, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return std::max(1, per_sm) * std::max(1, sms);
}
size_t fine_pass_w_smem() { return 0; }  // static shared memory
void set_fine_pass_w_smem() {}
dim3 fine_pass_w_grid(const Params& P) {
    const int W = 4 * fine_pass_w_quads(P.tile);
    return dim3((P.nx + W - 1) / W, P.nchunks);
}
// multi-GPU fused slot pieces (each followed by the caller's exchange where it moves data)
void launch_prolong_sum(const Params& P, cudaStream_t st) { prolong_sum_kernel<<<148, 256, 0, st>>>(P); }
void launch_fused_mp(const Params& P, dim3 grid, cudaStream_t st) {
    fine_pass_w_kernel<true, 3><<<grid, 32, 0, st>>>(P, fine_pass_w_quads(P.tile));
}
int launch_fine_pass_w(const Params& P, dim3 grid, cudaStream_t st, bool sweep_only, bool ph2_only) {
    const int nq = fine_pass_w_quads(P.tile);
    if (P.mp) {  // one kernel per call; the caller follows each with the exchange (fused_host.cu)
        if (getenv("ISMG_MP_ALLPHASE")) fine_pass_w_kernel<true, 0><<<grid, 32, 0, st>>>(P, nq);  // A/B hook
        else if (ph2_only) fine_pass_w_kernel<true, 2><<<grid, 32, 0, st>>>(P, nq);
        else fine_pass_w_kernel<true, 1><<<grid, 32, 0, st>>>(P, nq);
        return 1;
    }
    if (P.fuse && !sweep_only && !ph2_only) {  // [anchor of P ce, PH 2 (rollback), fused pass, sweep]
        prolong_sum_kernel<<<148, 256, 0, st>>>(P);
        fine_pass_w_kernel<false, 2><<<grid, 32, 0, st>>>(P, nq);
        fine_pass_w_kernel<false, 3><<<grid, 32, 0, st>>>(P, nq);
        fine_pass_w_kernel<false, 0><<<grid, 32, 0, st>>>(P, nq);
        return 4;
    }
    if (!sweep_only) fine_pass_w_kernel<false, 2><<<grid, 32, 0, st>>>(P, nq);
    if (ph2_only) return 1;
    fine_pass_w_kernel<false, 0><<<grid, 32, 0, st>>>(P, nq);
    return sweep_only ? 1 : 2;
}

}  // namespace fz
}  // namespace ismgb

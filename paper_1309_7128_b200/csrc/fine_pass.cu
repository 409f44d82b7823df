// fine_pass.cu — the hot path: device-resident solve_two_level (cycles.hpp:101-165).
//
// One fine iteration = ONE HBM pass (24 B/cell: read x, b; write x):
//   x' = x + c (pending anchor, smoother.hpp:145-148)  -> red half-sweep ->
//   black half-sweep (smoother.hpp:101-117) -> residual (smoother.hpp:121-141)
//   -> 16h/32h tile sums of the residual (restrict_sum, coarsening.hpp:471-480)
//   -> sum of x (next anchor) and max|r|.
// Rows are streamed through a shared-memory ring by TMA bulk copies
// (cp.async.bulk + mbarrier); each CTA owns a 256-column strip x H-row chunk
// and recomputes a 3-cell halo, so the red, black and residual stages run in
// one pass with 2 CTA barriers per row. Each thread owns a column pair and
// keeps its vertical window in registers; horizontal neighbours come from
// shared memory. A tile row of 32 (16) cells maps to 16 (8) lanes whose
// partial sums are folded by warp shuffles.
//
// Control flow never leaves the device: the last CTA of every kernel applies
// the reference's branch logic to the reduced scalars and writes the next
// phase into a device state block. The host replays a CUDA graph of
// [coarse-visit, fine-pass] slots; kernels whose phase is not current exit at
// once. The host only polls the phase once per graph launch.
#include "fused_impl.cuh"

namespace ismgb {
namespace fz {

// ---- SWEEP body: anchor-shift, red, black, residual, restriction ------------
// ---- per-thread column geometry -------------------------------------------
// Threads 0..kPairs-1 own the column pairs (a + 2t, a + 2t + 1) of the strip;
// thread kPairs holds the left halo pair (a-2, a-1), kPairs+1 the right halo
// pair (a+W, a+W+1). The last lane of the halo warp issues the TMA copies.
struct ColGeom {
    int t, c0, sidx;
    bool owned, active, in0, in1, inL, inR;
    double dc0, dc1;  // column part of the diagonal (W + E faces)
    __device__ __forceinline__ ColGeom(const Params& P, int a) {
        t = threadIdx.x;
        owned = t < kPairs;
        const bool halo = (t == kPairs) || (t == kPairs + 1);
        active = owned || halo;
        c0 = owned ? a + 2 * t : (t == kPairs ? a - 2 : a + kW);
        sidx = c0 - (a - 4);
        in0 = active && c0 >= 0 && c0 < P.nx;
        in1 = active && c0 + 1 >= 0 && c0 + 1 < P.nx;
        inL = active && c0 - 1 >= 0 && c0 - 1 < P.nx;
        inR = active && c0 + 2 >= 0 && c0 + 2 < P.nx;
        dc0 = col_diag(P, c0);
        dc1 = col_diag(P, c0 + 1);
    }
};

constexpr int kProducer = kThreads - 1;  // TMA issuer (idle lane of the halo warp)

// ---- SWEEP body: anchor-shift, red, black, residual, restriction ------------
// Iteration k: load row k, red half-sweep of row k-1, black half-sweep of row
// k-2, residual + store of row k-3 (each stage reads only rows the previous
// stages have finished; see the file comment).
__device__ __forceinline__ void sweep_body(Smem& sm, const Params& P, const Ctl& st) {
    const int a = blockIdx.x * kW;
    const int r0 = blockIdx.y * P.H, r1 = min(r0 + P.H, P.ny);
    const double* xin = st.buf[st.cur];
    double* xout = st.buf[st.cur ^ 1];
    const double* b = st.b;
    const bool shift_on = st.has_shift != 0;
    const double c = st.shift;
    const ColGeom cg(P, a);
    const int t = cg.t, sidx = cg.sidx, c0 = cg.c0;
    const uint32_t bar0 = su32(&sm.bar[0]);
    const double fwS = face_weight(P.bc.k[ISMG_SIDE_SOUTH]), fwN = face_weight(P.bc.k[ISMG_SIDE_NORTH]);
    const uint32_t ncopy = uint32_t(((min(a + kW + 4, P.nx + 5) - (a - 4)) + 1) & ~1);
    const int tmask = P.tile - 1;  // power-of-two tile (fused_supported)

    if (t == kProducer) {
        for (int s = 0; s < kRing; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int kfirst = r0 - 3, klast = r1 + 2;
    if (t == kProducer)
        for (int k = kfirst; k <= min(klast, kfirst + kAheadSweep - 1); ++k) issue_row(sm, P, xin, b, k, a, ncopy);

    // vertical register window: x{d}, b{d}, dr{d} = row k-d of this column pair
    double x0a = 0, x0b = 0, x1a = 0, x1b = 0, x2a = 0, x2b = 0, x3a = 0, x3b = 0, x4a = 0, x4b = 0;
    double b0a = 0, b0b = 0, b1a = 0, b1b = 0, b2a = 0, b2b = 0, b3a = 0, b3b = 0;
    double dr0 = 0, dr1 = 0, dr2 = 0, dr3 = 0;
    double mx = 0.0, sx = 0.0, tacc = 0.0, cm = 0.0;
    int nan = 0;
    const int g = P.tile >> 1;

    for (int k = kfirst; k <= klast; ++k) {
        const int slot = k & (kRing - 1);
        const uint32_t parity = (uint32_t(k - kfirst) >> 3) & 1u;  // fill count of this slot, mod 2
        // -- load row k (raw + pending anchor shift), masked outside the domain
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), parity);
        const bool rk = k >= 0 && k < P.ny;
        dr0 = ((k > 0) ? 1.0 : fwS) + ((k < P.ny - 1) ? 1.0 : fwN);  // row part of smoother.hpp:60-61
        if (cg.active) {
            const double2 xv = *reinterpret_cast<const double2*>(&sm.x[slot][sidx]);
            const double2 bv = *reinterpret_cast<const double2*>(&sm.b[slot][sidx]);
            x0a = (rk && cg.in0) ? (shift_on ? xv.x + c : xv.x) : 0.0;
            x0b = (rk && cg.in1) ? (shift_on ? xv.y + c : xv.y) : 0.0;
            b0a = bv.x;
            b0b = bv.y;
        }
        // -- stage 1: red half-sweep of row j = k-1 (smoother.hpp:111-113)
        {
            const int j = k - 1;
            if (cg.active && j >= r0 - 2 && j >= 0 && j < P.ny) {
                double* row = sm.x[j & (kRing - 1)];
                if ((j & 1) == 0) {  // red cell is c0
                    if (cg.in0) {
                        double W = 0.0;
                        if (cg.inL) W = shift_on ? row[sidx - 1] + c : row[sidx - 1];
                        const double s = W + x1b + x2a + x0a;
                        x1a = div_by_diag(s - b1a, cg.dc0 + dr1);
                        row[sidx] = x1a;
                    }
                } else {  // red cell is c1
                    if (cg.in1) {
                        double E = 0.0;
                        if (cg.inR) E = shift_on ? row[sidx + 2] + c : row[sidx + 2];
                        const double s = x1a + E + x2b + x0b;
                        x1b = div_by_diag(s - b1b, cg.dc1 + dr1);
                        row[sidx + 1] = x1b;
                    }
                }
            }
        }
        // (no barrier: stage 2 reads red cells of row k-2 written one iteration
        // ago; its N/S neighbours are this thread's own registers)
        // -- stage 2: black half-sweep of row j = k-2
        {
            const int j = k - 2;
            if (cg.active && j >= r0 - 1 && j >= 0 && j < P.ny) {
                double* row = sm.x[j & (kRing - 1)];
                if ((j & 1) == 0) {  // black cell is c1
                    if (cg.in1) {
                        const double E = cg.inR ? row[sidx + 2] : 0.0;
                        const double s = x2a + E + x3b + x1b;
                        x2b = div_by_diag(s - b2b, cg.dc1 + dr2);
                        row[sidx + 1] = x2b;
                    }
                } else {  // black cell is c0
                    if (cg.in0) {
                        const double W = cg.inL ? row[sidx - 1] : 0.0;
                        const double s = W + x2b + x3a + x1a;
                        x2a = div_by_diag(s - b2a, cg.dc0 + dr2);
                        row[sidx] = x2a;
                    }
                }
            }
        }
        // -- stage 3: residual of row j = k-3 (smoother.hpp:134-137), tile sums, store
        // (its horizontal neighbours were final one iteration ago)
        {
            const int j = k - 3;
            if (j >= r0 && j < r1) {
                if (cg.owned) {
                    const double* row = sm.x[j & (kRing - 1)];
                    double ra = 0.0, rb = 0.0;
                    if (cg.in0) {
                        const double W = cg.inL ? row[sidx - 1] : 0.0;
                        const double ax = W + x3b + x4a + x2a - (cg.dc0 + dr3) * x3a;
                        ra = b3a - ax;
                        mx = fmax(mx, fabs(ra));  // fmax drops NaN, as std::max(rmax, |r|) does
                        sx = sx + x3a;
                    }
                    if (cg.in1) {
                        const double E = cg.inR ? row[sidx + 2] : 0.0;
                        const double ax = x3a + E + x4b + x2b - (cg.dc1 + dr3) * x3b;
                        rb = b3b - ax;
                        mx = fmax(mx, fabs(rb));
                        sx = sx + x3b;
                    }
                    double* dst = xout + int64_t(j) * P.pitch + c0;
                    if (cg.in0 && cg.in1) *reinterpret_cast<double2*>(dst) = make_double2(x3a, x3b);
                    else if (cg.in0) dst[0] = x3a;
                    tacc = tacc + (ra + rb);
                }
                if ((j & tmask) == tmask || j == P.ny - 1) {  // tile row-block complete
                    if (t < kPairs) {
                        const double tsum = group_sum(tacc, g);
                        if ((t & (g - 1)) == 0 && cg.in0) {
                            P.cb.at(c0 / P.tile, j / P.tile) = tsum;
                            cm = max_drop_nan(cm, fabs(tsum));
                            nan |= (tsum != tsum);  // a NaN residual poisons its tile sum
                        }
                    }
                    tacc = 0.0;
                }
            }
        }
        // rotate the register window
        x4a = x3a, x4b = x3b, x3a = x2a, x3b = x2b, x2a = x1a, x2b = x1b, x1a = x0a, x1b = x0b;
        b3a = b2a, b3b = b2b, b2a = b1a, b2b = b1b, b1a = b0a, b1b = b0b;
        dr3 = dr2, dr2 = dr1, dr1 = dr0;
        // one barrier per row: iteration k+1 reads what iteration k wrote, and
        // rows <= k-3 are free, so the slot of row k + kAheadSweep can refill
        __syncthreads();
        if (t == kProducer && k + kAheadSweep <= klast) issue_row(sm, P, xin, b, k + kAheadSweep, a, ncopy);
    }
    pass_epilogue(sm, P, kFine, mx, sx, cm, nan);
}

// ---- PROLONG / RESID body: x' = x + c + P ce, residual, restriction ---------
__device__ __forceinline__ void prolong_body(Smem& sm, const Params& P, const Ctl& st, bool prolong) {
    const int a = blockIdx.x * kW;
    const int r0 = blockIdx.y * P.H, r1 = min(r0 + P.H, P.ny);
    const double* xin = st.buf[st.cur];
    double* xout = st.buf[st.cur ^ 1];
    const double* b = st.b;
    const bool shift_on = st.has_shift != 0;
    const double c = st.shift;
    const ColGeom cg(P, a);
    const int t = cg.t, sidx = cg.sidx, c0 = cg.c0;
    const uint32_t bar0 = su32(&sm.bar[0]);
    const double fwS = face_weight(P.bc.k[ISMG_SIDE_SOUTH]), fwN = face_weight(P.bc.k[ISMG_SIDE_NORTH]);
    const uint32_t ncopy = uint32_t(((min(a + kW + 4, P.nx + 5) - (a - 4)) + 1) & ~1);
    const int tmask = P.tile - 1;
    // prolongation geometry of this thread's columns (TileAxis::locate_cell)
    int I0a = 0, I1a = 0, I0b = 0, I1b = 0;
    double sa = 0, dxa = 1, sb = 0, dxb = 1;
    if (prolong) {
        if (cg.in0) I0a = P.ax.k0[c0], I1a = P.ax.k1[c0], sa = P.ax.t[c0], dxa = P.ax.dk[c0];
        if (cg.in1) I0b = P.ax.k0[c0 + 1], I1b = P.ax.k1[c0 + 1], sb = P.ax.t[c0 + 1], dxb = P.ax.dk[c0 + 1];
    }

    if (t == kProducer) {
        for (int s = 0; s < kRing; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int kfirst = r0 - 1, klast = r1;
    if (t == kProducer)
        for (int k = kfirst; k <= min(klast, kfirst + kAheadRes - 1); ++k) issue_row(sm, P, xin, b, k, a, ncopy);

    double x0a = 0, x0b = 0, x1a = 0, x1b = 0, x2a = 0, x2b = 0, b0a = 0, b0b = 0, b1a = 0, b1b = 0;
    double dr0 = 0, dr1 = 0;
    double mx = 0.0, sx = 0.0, tacc = 0.0, cm = 0.0;
    int nan = 0;
    const int g = P.tile >> 1;
    for (int k = kfirst; k <= klast; ++k) {
        const int slot = k & (kRing - 1);
        const uint32_t parity = (uint32_t(k - kfirst) >> 3) & 1u;  // fill count of this slot, mod 2
        mbar_wait_addr(bar0 + 8u * uint32_t(slot), parity);
        const bool rk = k >= 0 && k < P.ny;
        dr0 = ((k > 0) ? 1.0 : fwS) + ((k < P.ny - 1) ? 1.0 : fwN);  // row part of smoother.hpp:60-61
        if (cg.active) {
            const double2 xv = *reinterpret_cast<const double2*>(&sm.x[slot][sidx]);
            const double2 bv = *reinterpret_cast<const double2*>(&sm.b[slot][sidx]);
            double va = (rk && cg.in0) ? (shift_on ? xv.x + c : xv.x) : 0.0;
            double vb = (rk && cg.in1) ? (shift_on ? xv.y + c : xv.y) : 0.0;
            if (prolong && rk) {  // coarsening.hpp:495-500
                const double tt = P.ay.t[k], dy = P.ay.dk[k];
                const int J0 = P.ay.k0[k], J1 = P.ay.k1[k];
                if (cg.in0)
                    va += ((dxa - sa) * ((dy - tt) * P.ce.at(I0a, J0) + tt * P.ce.at(I0a, J1)) +
                           sa * ((dy - tt) * P.ce.at(I1a, J0) + tt * P.ce.at(I1a, J1))) /
                          (dxa * dy);
                if (cg.in1)
                    vb += ((dxb - sb) * ((dy - tt) * P.ce.at(I0b, J0) + tt * P.ce.at(I0b, J1)) +
                           sb * ((dy - tt) * P.ce.at(I1b, J0) + tt * P.ce.at(I1b, J1))) /
                          (dxb * dy);
            }
            x0a = va, x0b = vb;
            b0a = bv.x, b0b = bv.y;
            *reinterpret_cast<double2*>(&sm.x[slot][sidx]) = make_double2(va, vb);
        }
        __syncthreads();
        if (t == kProducer && k + kAheadRes <= klast) issue_row(sm, P, xin, b, k + kAheadRes, a, ncopy);
        const int j = k - 1;
        if (j >= r0 && j < r1) {
            if (cg.owned) {
                const double* row = sm.x[j & (kRing - 1)];
                double ra = 0.0, rb = 0.0;
                if (cg.in0) {
                    const double W = cg.inL ? row[sidx - 1] : 0.0;
                    const double ax = W + x1b + x2a + x0a - (cg.dc0 + dr1) * x1a;
                    ra = b1a - ax;
                    mx = fmax(mx, fabs(ra));  // fmax drops NaN, as std::max(rmax, |r|) does
                    sx = sx + x1a;
                }
                if (cg.in1) {
                    const double E = cg.inR ? row[sidx + 2] : 0.0;
                    const double ax = x1a + E + x2b + x0b - (cg.dc1 + dr1) * x1b;
                    rb = b1b - ax;
                    mx = fmax(mx, fabs(rb));
                    sx = sx + x1b;
                }
                if (prolong) {
                    double* dst = xout + int64_t(j) * P.pitch + c0;
                    if (cg.in0 && cg.in1) *reinterpret_cast<double2*>(dst) = make_double2(x1a, x1b);
                    else if (cg.in0) dst[0] = x1a;
                }
                tacc = tacc + (ra + rb);
            }
            if ((j & tmask) == tmask || j == P.ny - 1) {
                if (t < kPairs) {
                    const double tsum = group_sum(tacc, g);
                    if ((t & (g - 1)) == 0 && cg.in0) {
                        P.cb.at(c0 / P.tile, j / P.tile) = tsum;
                        cm = max_drop_nan(cm, fabs(tsum));
                        nan |= (tsum != tsum);  // a NaN residual poisons its tile sum
                    }
                }
                tacc = 0.0;
            }
        }
        x2a = x1a, x2b = x1b, x1a = x0a, x1b = x0b, b1a = b0a, b1b = b0b;
        dr1 = dr0;
    }
    pass_epilogue(sm, P, prolong ? kProlong : kResid, mx, sx, cm, nan);
}

__global__ void __launch_bounds__(kThreads) fine_pass_kernel(Params P) {
    __shared__ __align__(128) Smem sm;  // static: every ring access is an LDS/STS
    const Ctl st = *P.ctl;              // snapshot (written only by the previous kernel)
    if (st.phase == kFine) sweep_body(sm, P, st);
    else if (st.phase == kProlong) prolong_body(sm, P, st, true);
    else if (st.phase == kResid) prolong_body(sm, P, st, false);
}

// final anchor + copy into the caller's field: x = buf[cur] + c (the rank's rows)
__global__ void finalize_kernel(Params P, View xuser) {
    const Ctl* s = P.ctl;
    const double* src = s->buf[s->cur];
    const bool sh = s->has_shift != 0;
    const double c = s->shift;
    if (s->cur == 0 && !sh) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = P.row0 + int(blockIdx.y);
    if (i >= P.nx) return;
    const double v = src[int64_t(j) * P.pitch + i];
    xuser.at(i, j) = sh ? v + c : v;
}

void launch_fine_pass(const Params& P, dim3 grid, size_t, cudaStream_t st) { fine_pass_kernel<<<grid, kThreads, 0, st>>>(P); }
size_t fine_pass_smem() { return 0; }  // static shared memory (sizeof(Smem) < 48 KB)
void set_fine_pass_smem(size_t) {}
void launch_finalize(const Params& P, View xuser, cudaStream_t st) {
    finalize_kernel<<<dim3((P.nx + 255) / 256, P.row1 - P.row0), 256, 0, st>>>(P, xuser);
}

// multi-GPU, after the allgather of every rank's pack: reduce the pass partials
// in rank order (max|r|, max|tile sum| by MAX; sum x by a fixed-order SUM, so
// every rank decides on identical values), assemble the coarse rhs from the
// ranks' coarse rows, and apply the reference's branch logic. The next pass
// reads its halo rows straight from the gathered packs.
// The exchange after a multi-GPU fine pass, on every rank: wait for every
// rank's flag of this pass, pull every rank's coarse-rhs rows from its pack slot
// (peer memory over NVLink) into cb, then (the last CTA, by ticket) reduce the
// pass partials in rank order (identical bits on every rank) and decide. The
// copy is spread over kUnpackCtas CTAs: one CTA pulling the 2 MB of a 512^2
// coarse rhs took ~125 us per pass (latency-bound NVLink loads).
constexpr int kUnpackCtas = 32;
__global__ void mp_unpack_kernel(Params P) {
    __shared__ int s_pass;
    __shared__ unsigned s_last;
    Ctl* st = P.ctl;
#ifdef ISMG_MP_TRACE
    const long long tu0 = gtimer();
#endif
    const unsigned long long want = st->mp_seq + 1ull;  // flag value of this slot's pass (mp_seq changes only
                                                         // after every CTA has passed the ticket below)
    if (threadIdx.x == 0) {
        const volatile unsigned long long* f = P.xflag[P.rank];
        int pass = f[P.rank] >= want;  // a fine pass ran in this slot (on every rank alike)
        if (pass) {
            const long long t0 = gtimer();
            for (int q = 0; q < P.nranks && pass; ++q)
                while (f[q] < want)
                    if (gtimer() - t0 > 4000000000ll) {  // a peer is gone: stop instead of hanging
                        st->mp_error = 1, pass = 0;
                        break;
                    }
            __threadfence_system();
        }
        s_pass = pass;
    }
    __syncthreads();
    if (!s_pass) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && st->mp_error == 1) st->phase = kDone;
        return;
    }
    const int L = P.pack_len;
    const int64_t po = int64_t((want - 1ull) & 1ull) * P.nranks * L;  // this pass's parity
    // coarse rhs rows of every rank -> cb (used by the next coarse visit)
    const int nthr = int(gridDim.x * blockDim.x), tid = int(blockIdx.x * blockDim.x + threadIdx.x);
    for (int r = 0; r < P.nranks; ++r) {
        int f0, f1;
        strip_of(P.ny, P.tile, P.nranks, r, &f0, &f1);
        const int c0 = f0 / P.tile, c1 = (f1 + P.tile - 1) / P.tile;
        const double* src = P.xch[r] + po + int64_t(r) * L + 8;
        const int n = (c1 - c0) * P.ncx;
        for (int k0 = tid; k0 < n; k0 += 4 * nthr) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // four loads in flight per thread
                const int k = k0 + u * nthr;
                const int jj = k / P.ncx, I = k - jj * P.ncx;
                v[u] = k < n ? __ldcv(src + int64_t(jj) * P.cb.pitch + I) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + u * nthr;
                const int jj = k / P.ncx, I = k - jj * P.ncx;
                if (k < n) P.cb.at(I, c0 + jj) = v[u];
            }
        }
    }
    __syncthreads();
    unsigned* ticket = P.ticket + 1 + (P.nstrips * P.nchunks + 31) / 32;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) {  // pass partials reduced in rank order: identical bits on every rank
        *ticket = 0u;
        __threadfence();
        if (st->mp_error == 1) {
            st->phase = kDone;
            return;
        }
        double m = 0.0, c = 0.0, sx = 0.0;
        for (int r = 0; r < P.nranks; ++r) {
            const double* v = P.xch[r] + po + int64_t(r) * L;
            m = fmax(m, __ldcv(v + 0));
            c = fmax(c, __ldcv(v + 1));
            sx += __ldcv(v + 4);
        }
        const double* g = P.xch[0] + po;
        st->mp_seq = want;
        const int mode = int(__ldcv(g + 3));
        if (mode == kFused) {  // the fused pass: its prolongation residual too (pack scalar 5)
            double rp = 0.0;
            for (int r = 0; r < P.nranks; ++r) rp = fmax(rp, __ldcv(P.xch[r] + po + int64_t(r) * L + 5));
            fine_decide_fused(P, rp, m, sx, c);
            publish_phase(P, st->phase);
        } else {
            fine_decide(P, mode, m, sx, c);
        }
#ifdef ISMG_MP_TRACE
        const long long tu1 = gtimer();
        if (want % 64 == 0)
            printf("MPTRACE rank %d seq %llu fine %lld gap %lld unpack %lld\n", P.rank, want,
                   (long long)(st->mp_t1 - st->mp_t0), (long long)(tu0 - (long long)st->mp_t1), tu1 - tu0);
        st->mp_t0 = ~0ull;
#endif
    }
}
void launch_mp_unpack(const Params& P, cudaStream_t st) { mp_unpack_kernel<<<kUnpackCtas, 512, 0, st>>>(P); }

}  // namespace fz
}  // namespace ismgb

// fused_impl.cuh — shared definitions of the fused hot path (fine_pass.cu,
// coarse.cu, fused_host.cu): phases, the device-resident solve state, kernel
// parameters and the mbarrier / TMA bulk-copy helpers.
#pragma once

#include "kernels.cuh"
#include "solver.h"

namespace ismgb {
namespace fz {

constexpr int kW = 256;                 // owned columns per CTA strip
constexpr int kPairs = kW / 2;          // owned column pairs (one per thread)
constexpr int kThreads = kPairs + 32;   // + one warp for the two halo pairs
constexpr int kRing = 8;                // smem row ring
constexpr int kRowCap = kW + 8;         // smem row: columns [a-4, a+W+4)
constexpr int kAheadSweep = kRing - 3;  // rows in flight ahead of the sweep (slot of row k-3 is free)
constexpr int kAheadRes = kRing - 2;    // rows prefetched ahead (prolong/residual)
constexpr int kCoarseThreads = 1024;
constexpr int kCoarseSmemThreads = 512;

enum Phase : int { kFine = 0, kCoarse = 1, kProlong = 2, kResid = 3, kDone = 4, kFused = 5 };
// kFused: the prolongation and the first sweep after it in ONE fine pass (single GPU,
// uniform power-of-two tiles; fine_pass_w.cu fused_w); prolong_sum_kernel turns a
// kProlong phase into kFused after computing the anchor of the prolonged field.

// Device-resident solve state (one per solver).
constexpr int kMaxRanks = 8;  // multi-GPU: ranks of one node

struct Ctl {
    int phase;
    int converged;
    int cur;        // fine iterate lives in buf[cur]; buf[0] is the caller's x
    int has_shift;  // singular: a pending anchor shift applies to buf[cur]
    int nan_seen;
    int nvisits;
    int hold;  // benchmark hook: passes leave the phase unchanged
    int pred;  // predicted coarse-visit length (sweeps of the previous visit)
    long long total, fine, coarse, restrictions, prolongations;
    long long passes, coarse_launches;
    long long coarse_ns, coarse_steps;  // device-timed coarse visits (globaltimer) and their wavefront steps
    long long coarse_group_ns;          // ... of which inside the wavefront groups
    double r, prev, shift, rc;
    double* buf[2];
    const double* b;
    unsigned long long mp_seq;  // multi-GPU: fine passes exchanged so far (all solves)
    int mp_error;               // multi-GPU: a peer's pack never arrived
    unsigned long long mp_t0, mp_t1;  // ISMG_MP_TRACE: first CTA start / last CTA end of the pass
    // coarse visit handed from the one-SM kernel to the cluster kernel at a group
    // boundary (iterate in ce): next group size, sweeps done, residual
    int cl_hand, cl_hand_G;
    long long cl_hand_done;
    double cl_hand_rc;
    double fshift;  // kFused: anchor shift of the prolonged field, -(sum of P ce) / cells
    int no_fuse;    // the fused pass rolled back (its prolongation ended the solve): run PH 2 alone
};

struct Params {
    int nx, ny;
    int64_t pitch;  // shared by every fine field of this grid
    int tile, ncx, ncy, H, nstrips, nchunks;
    PBC bc;
    int singular, nslots;
    double tol_fine, tol_coarse, stall;
    long long max_total;
    double ncells;
    Ctl* ctl;
    View cb, ce;  // coarse rhs / correction
    const double* w;
    AxisDev ax, ay;
    double* part;  // 3 per CTA: max|r|, sum x, max|tile sum|
    unsigned* ticket;
    int* visit_log;  // (coarse sweeps, fine sweeps) per coarse visit
    int visit_cap;
    double* coarse_scratch;  // reduction scratch for the coarse kernel
    // strip decomposition (multi-GPU): this rank relaxes fine rows [row0, row1);
    // rows row0-3..row0-1 / row1..row1+2 are the neighbours' and arrive with
    // their packs. A pack (pack_len doubles) = [8 scalars: max|r|, max|tile
    // sum|, pass flag, mode, sum x | the rank's coarse-rhs rows (pitched) | its
    // first 3 rows | its last 3 rows (pitched, column origin kXOff)].
    // Exchange by peer stores (NVLink): every rank owns an exchange buffer
    // [2 parities][nranks][pack_len], mapped into every rank (xch[q]). Pass s
    // (Ctl::mp_seq) writes its pack into slot [s & 1][rank] of every rank's
    // buffer while it computes, then raises xflag[q][rank] to s + 1 on every
    // rank; mp_unpack_kernel waits for all ranks' flags and decides. The
    // parities keep pass s's writes off the halo rows pass s reads (s - 1).
    int row0, row1, mp;
    int rank, nranks, pack_len, pack_cb_rows;
    double* xch[kMaxRanks];
    unsigned long long* xflag[kMaxRanks];
    int64_t cb_off, cb_pitch;  // pack offset of coarse cell (I, J): cb_off + J * cb_pitch + I
    int64_t h_off[4];          // pack offsets of the first / last 3 rows; [2], [3]: a fused pass's INPUT rows (its rollback)
    View cbw;                  // single GPU: where the fused pass writes its tile sums (= cb)
    // conditional CUDA graph of the single-GPU solve (fused_host.cu): WHILE(phase
    // != done) { SWITCH(phase) { fine pass | coarse visit | prolong | resid } };
    // the kernel that decides the next phase sets both conditions
    int cond;
    cudaGraphConditionalHandle h_while, h_switch;
    // fused prolongation + sweep pass (single GPU, uniform power-of-two tiles):
    // pax[I] / pay[J] = the prolongation weights of coarse column I / row J summed
    // over the fine columns / rows, so sum(P ce) = sum ce(I, J) pax[I] pay[J]
    int fuse;
    const double* pax;
    const double* pay;
};

// the next phase to the solve's conditional graph (no-op outside it). Built only
// with -DISMG_WITH_COND_GRAPH (tools/build_variant.sh): ncu refuses to profile
// the kernel nodes of any graph whose kernels can set conditionals, and the
// conditional graph measured slower than the slot graphs (fused_host.cu).
__device__ __forceinline__ void publish_phase(const Params& P, int phase) {
#ifdef ISMG_WITH_COND_GRAPH
    if (P.cond) {
        cudaGraphSetConditional(P.h_switch, unsigned(phase));
        cudaGraphSetConditional(P.h_while, phase != kDone ? 1u : 0u);
    }
#else
    (void)P, (void)phase;
#endif
}

// x-row source of the fused passes: the rank's own rows from the field, the
// neighbours' rows from their packs of the previous pass (parity hp)
__device__ __forceinline__ const double* row_src(const Params& P, const double* xin, int k, int col, int hp,
                                                 bool alt = false) {
    if (P.mp) {  // alt: the rows a fused pass read (its rollback redoes the prolongation on them)
        const double* x = P.xch[P.rank] + int64_t(hp) * P.nranks * P.pack_len;
        if (k < P.row0 && P.row0 > 0)
            return x + int64_t(P.rank - 1) * P.pack_len + P.h_off[alt ? 3 : 1] + int64_t(k - (P.row0 - 3)) * P.pitch +
                   kXOff + col;
        if (k >= P.row1 && P.row1 < P.ny)
            return x + int64_t(P.rank + 1) * P.pack_len + P.h_off[alt ? 2 : 0] + int64_t(k - P.row1) * P.pitch + kXOff +
                   col;
    }
    return xin + int64_t(k) * P.pitch + col;
}

// multi-GPU: one pack word of pass parity p into every rank's exchange buffer
__device__ __forceinline__ void mp_put(const Params& P, int p, int64_t off, double v) {
    const int64_t o = (int64_t(p) * P.nranks + P.rank) * P.pack_len + off;
    for (int q = 0; q < P.nranks; ++q) P.xch[q][o] = v;
}
__device__ __forceinline__ void mp_put2(const Params& P, int p, int64_t off, double a, double b) {
    const int64_t o = (int64_t(p) * P.nranks + P.rank) * P.pack_len + off;
    for (int q = 0; q < P.nranks; ++q) *reinterpret_cast<double2*>(P.xch[q] + o) = make_double2(a, b);
}

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- PTX helpers: mbarrier + TMA bulk copy ----------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_wait_addr(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITA_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITA_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

struct Smem {
    double x[kRing][kRowCap];
    double b[kRing][kRowCap];
    uint64_t bar[kRing];
    double red[3][32];
    int last;
};

// Issue the TMA bulk copies of fine row `row` (x and b) into ring slot.
__device__ __forceinline__ void issue_row(Smem& sm, const Params& P, const double* xin, const double* b, int row,
                                          int a, uint32_t ncopy) {
    const int slot = (row + 2 * kRing) % kRing;  // row may be -3
#ifdef ISMG_PROXY_FENCE
    fence_proxy_async();
#endif
    mbar_expect_tx(&sm.bar[slot], 2u * ncopy * 8u);
    const int64_t off = int64_t(row) * P.pitch + (a - 4);
    bulk_load(sm.x[slot], xin + off, ncopy * 8u, &sm.bar[slot]);
    bulk_load(sm.b[slot], b + off, ncopy * 8u, &sm.bar[slot]);
}

__device__ __forceinline__ double row_diag(const Params& P, int j) {
    return ((j > 0) ? 1.0 : face_weight(P.bc.k[ISMG_SIDE_SOUTH])) +
           ((j < P.ny - 1) ? 1.0 : face_weight(P.bc.k[ISMG_SIDE_NORTH]));
}
__device__ __forceinline__ double col_diag(const Params& P, int i) {
    return ((i > 0) ? 1.0 : face_weight(P.bc.k[ISMG_SIDE_WEST])) +
           ((i < P.nx - 1) ? 1.0 : face_weight(P.bc.k[ISMG_SIDE_EAST]));
}

// Tile-sum fold over the g = tile/2 lanes of one coarse cell (g divides 32).
__device__ __forceinline__ double group_sum(double v, int g) {
    for (int o = g >> 1; o > 0; o >>= 1) v = v + __shfl_down_sync(kFull, v, o);
    return v;
}

// ---- per-CTA epilogue + control flow (last CTA) ------------------------------
__device__ __forceinline__ void fine_decide_(const Params& P, int mode, double r, double sum, double rc0);
// cycles.hpp:111-161 on the pass's reductions; then the next phase to the graph
__device__ __forceinline__ void fine_decide(const Params& P, int mode, double r, double sum, double rc0) {
    fine_decide_(P, mode, r, sum, rc0);
    publish_phase(P, P.ctl->phase);
}
__device__ __forceinline__ void fine_decide_(const Params& P, int mode, double r, double sum, double rc0) {
    Ctl* s = P.ctl;
    s->passes += 1;
    s->r = r;
    if (P.singular) {  // anchor after every residual check (field.hpp:49,53-59)
        s->shift = -(sum / P.ncells);
        s->has_shift = 1;
    }
    if (mode != kResid) s->cur ^= 1;
    if (s->hold) return;  // ismg_bench_fine_pass: repeat the same pass kind
    auto to_coarse = [&]() {
        s->restrictions += 1;
        if (s->nvisits < P.visit_cap) {
            P.visit_log[2 * s->nvisits] = 0;
            P.visit_log[2 * s->nvisits + 1] = 0;
        }
        s->nvisits += 1;
        s->rc = rc0;
        if (rc0 > P.tol_coarse) {
            s->phase = kCoarse;
        } else {  // zero-sweep visit: no prolongation, relax again (cycles.hpp:125,138,146)
            s->prev = r;
            s->phase = kFine;
        }
    };
    if (mode == kFine) {  // cycles.hpp:147-161
        s->total += 1;
        s->fine += 1;
        if (s->nvisits > 0 && s->nvisits <= P.visit_cap) P.visit_log[2 * (s->nvisits - 1) + 1] += 1;
        if (r <= P.tol_fine) {
            s->phase = kDone, s->converged = 1;
        } else if (s->total >= P.max_total) {
            s->phase = kDone, s->converged = 0;
        } else if (r > P.stall * s->prev) {
            to_coarse();
        } else {
            s->prev = r;
            s->phase = kFine;
        }
    } else if (mode == kProlong) {  // cycles.hpp:138-146
        s->no_fuse = 0;
        s->prolongations += 1;
        if (r <= P.tol_fine) {
            s->phase = kDone, s->converged = 1;
        } else {
            s->prev = r;
            if (s->total >= P.max_total) s->phase = kDone, s->converged = 0;
            else s->phase = kFine;
        }
    } else {  // initial residual, cycles.hpp:111-118
        if (r <= P.tol_fine) {
            s->phase = kDone, s->converged = 1;
        } else if (s->total >= P.max_total) {
            s->phase = kDone, s->converged = 0;
        } else {
            to_coarse();
        }
    }
}

// The fused pass (kFused): the prolongation's decision (cycles.hpp:138-146) on rp,
// then the first sweep's (cycles.hpp:147-161) on r with prev = rp. Where the
// prolongation itself ends the solve (rp <= tol, or the sweep budget is spent) the
// pass's sweep must not count: roll back (buf[cur] still holds the input; PH 2
// redoes the prolongation alone and decides).
__device__ __forceinline__ void fine_decide_fused(const Params& P, double rp, double r, double sum, double rc0) {
    Ctl* s = P.ctl;
    s->passes += 1;
    if (rp <= P.tol_fine || s->total >= P.max_total) {
        s->no_fuse = 1;
        s->phase = kProlong;
        return;
    }
    s->prolongations += 1;
    s->cur ^= 1;
    s->prev = rp;
    s->r = r;
    if (P.singular) {
        s->shift = -(sum / P.ncells);
        s->has_shift = 1;
    }
    s->total += 1;
    s->fine += 1;
    if (s->nvisits > 0 && s->nvisits <= P.visit_cap) P.visit_log[2 * (s->nvisits - 1) + 1] += 1;
    if (r <= P.tol_fine) {
        s->phase = kDone, s->converged = 1;
    } else if (s->total >= P.max_total) {
        s->phase = kDone, s->converged = 0;
    } else if (r > P.stall * s->prev) {
        s->restrictions += 1;
        if (s->nvisits < P.visit_cap) {
            P.visit_log[2 * s->nvisits] = 0;
            P.visit_log[2 * s->nvisits + 1] = 0;
        }
        s->nvisits += 1;
        s->rc = rc0;
        if (rc0 > P.tol_coarse) {
            s->phase = kCoarse;
        } else {
            s->prev = r;
            s->phase = kFine;
        }
    } else {
        s->prev = r;
        s->phase = kFine;
    }
}

// cm = max |tile sum| this CTA wrote to cb: the coarse entry residual
// coarse_residual(ce = 0, cb) = max|cb| (cycles.hpp:122-123) is complete when
// the pass ends, so a visit that needs no coarse sweep is decided here.
template <class S>
__device__ __noinline__ void pass_epilogue(S& sm, const Params& P, int mode, double mx, double sx, double cm, int nan) {
    const int nb = gridDim.x * gridDim.y;
    const int bid = blockIdx.y * gridDim.x + blockIdx.x;
    double bm = block_max(mx, sm.red[0]);
    double bs = block_sum(sx, sm.red[1]);
    double bc = block_max(cm, sm.red[2]);
    int anynan = __syncthreads_or(nan);
    if (threadIdx.x == 0) {
        P.part[3 * bid] = bm;
        P.part[3 * bid + 1] = bs;
        P.part[3 * bid + 2] = bc;
        if (anynan) P.ctl->nan_seen = 1;
        __threadfence();
        const unsigned t = atomicAdd(P.ticket, 1u);
        sm.last = (t == unsigned(nb - 1));
    }
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    double m = 0.0, s = 0.0, c = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        m = fmax(m, __ldcg(&P.part[3 * k]));
        s += __ldcg(&P.part[3 * k + 1]);
        c = fmax(c, __ldcg(&P.part[3 * k + 2]));
    }
    m = block_max(m, sm.red[0]);
    s = block_sum(s, sm.red[1]);
    c = block_max(c, sm.red[2]);
    if (threadIdx.x == 0) {
        fine_decide(P, mode, m, s, c);
        *P.ticket = 0u;
        __threadfence();
    }
}


// launchers (each in the translation unit of its kernel)
void launch_fine_pass(const Params& P, dim3 grid, size_t smem, cudaStream_t st);
size_t fine_pass_smem();
void set_fine_pass_smem(size_t bytes);
// independent warp strips (fine_pass_w.cu; tiles >= 4)
int fine_pass_w_quads(int tile);
int fine_pass_w_resident(bool mp, int device);  // resident one-warp CTAs on the device
size_t fine_pass_w_smem();
void set_fine_pass_w_smem();
dim3 fine_pass_w_grid(const Params& P);
// kernels launched: single-GPU, the prolongation kernel then the sweep kernel (sweep_only: the sweep)
// (sweep_only: the sweep kernel alone; ph2_only: the prolongation / residual kernel alone)
int launch_fine_pass_w(const Params& P, dim3 grid, cudaStream_t st, bool sweep_only = false, bool ph2_only = false);
void launch_finalize(const Params& P, View xuser, cudaStream_t st);
void launch_mp_unpack(const Params& P, cudaStream_t st);
void launch_prolong_sum(const Params& P, cudaStream_t st);
void launch_fused_mp(const Params& P, dim3 grid, cudaStream_t st);
void launch_coarse_global(const Params& P, cudaStream_t st);
void launch_coarse_smem(const Params& P, double* backup, size_t smem, cudaStream_t st);
void set_coarse_smem(size_t bytes);

// TMEM-resident coarse visit (coarse.cu): geometry of the diagonal layout.
struct TmGeom {
    int ncx, ncy;
    int PP;     // diagonal slots per row (period of the skew)
    int pitch;  // smem row pitch = PP + 6 (3 mirrored slots each side), = 1 mod 16
    int ring;
    int ncls;     // distinct boundary-ring stencils (class table rows)
    int fastdiv;  // ring divisions by Markstein's correction (host-verified) instead of DDIV
    int kind;   // interior stencil: 0 generic (stdw), 1 ISMG (-3, 1/2, 1/4), 2 five-point (-4, 1)
    bool five;
    double stdw[9];
};
// Cluster coarse visit (coarse_cl.cu): row bands over the CTAs of one cluster.
struct ClGeom {
    int ncx, ncy;
    int pitch, bpitch;  // shared-memory row pitches (3 mod 16 doubles)
    int csize, band;    // cluster size (CTAs), rows per CTA band
    int bsmem;          // rhs: 1 shared memory, 2 Tensor Memory, 0 read through L1
    int ring, ncls, fastdiv, kind;
    int role;  // 0: whole visits; 1: one-SM kernel, hands groups above 4 sweeps on; 2: cluster kernel, resumes them
    bool five;
    double stdw[9];  // interior weights (slot order C, E, W, N, S, NE, NW, SE, SW)
    double stdy;     // RN(1 / stdw[0]): Markstein's reciprocal (fastdiv)
};
// Stencil classes of a non-periodic coarse operator (coarse_cl.cu)
struct StencilClasses {
    int ncls = 0, ring = 0, kind = 0, fastdiv = 0;
    bool five = false;
    double stdw[9] = {};      // interior weights
    std::vector<double> spec;  // [ncls + 1][10] (w0..w8, RN(1 / w0); interior last), then ring class ids (int)
};
bool stencil_classes(const CoarseOpH& op, StencilClasses& S);
bool cl_coarse_plan(const CoarseOpH& op, ClGeom& T, std::vector<double>& spec, size_t& smem, int band_min = 0);
size_t cl_backup_doubles(const ClGeom& T);
void launch_coarse_cl(const Params& P, const ClGeom& T, const double* spec, double* backup, size_t smem,
                      cudaStream_t st);
void set_coarse_cl_smem(size_t bytes);

// Register-wavefront coarse visit over many SMs (coarse_rw.cu); nullptr when
// the operator does not fit it (then a cluster / TMEM / smem / global engine).
struct RwEngine;
RwEngine* rw_try_create(const CoarseOpH& op, int device);
void rw_destroy(RwEngine* e);
void launch_coarse_rw(const Params& P, const RwEngine& e, cudaStream_t st);
std::vector<double> rw_trace_take();

// Sweep pipeline over the SMs (coarse_sp.cu): one CTA per sweep; nullptr when
// the operator does not fit it.
struct SpEngine;
SpEngine* sp_try_create(const CoarseOpH& op, int device);
void sp_destroy(SpEngine* e);
void launch_coarse_sp(const Params& P, const SpEngine& e, cudaStream_t st);
// ... several 32-row blocks per warp, up to 32 blocks (coarse_sp2.cu)
struct Sp2Engine;
Sp2Engine* sp2_try_create(const CoarseOpH& op, int device);
void sp2_destroy(Sp2Engine* e);
void launch_coarse_sp2(const Params& P, const Sp2Engine& e, cudaStream_t st);

bool tmem_coarse_plan(const CoarseOpH& op, TmGeom& T, std::vector<double>& spec, size_t& smem);
void launch_coarse_tmem(const Params& P, const TmGeom& T, const double* spec, double* backup, size_t smem,
                        cudaStream_t st);
void set_coarse_tmem_smem(size_t bytes);

}  // namespace fz
}  // namespace ismgb

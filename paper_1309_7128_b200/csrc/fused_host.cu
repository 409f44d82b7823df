// fused_host.cu — host side of the fused hot path: engine setup, CUDA-graph
// capture of [coarse-visit, fine-pass] slots, and the solve driver that polls
// the device-resident phase once per graph launch.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fused_impl.cuh"

namespace ismgb {
using namespace fz;

struct FusedEngine {
    Solver* s = nullptr;
    Params P{};
    Ctl* d_ctl = nullptr;
    Ctl* h_ctl = nullptr;  // pinned
    DevBuf scratch;        // second ping-pong buffer
    int* d_log = nullptr;
    std::vector<int> h_log;
    cudaGraphExec_t graphs[4] = {nullptr, nullptr, nullptr, nullptr};  // 8, 16, 32, 64 slots, captured once
    // single GPU: one conditional graph per solve, WHILE(phase != done) { SWITCH(phase) }
    // (state 0 not built yet, 1 built, -1 unavailable: the slot graphs above)
    cudaGraphExec_t cond_exec = nullptr;
    int cond_state = 0;
    int fine_launches = 1;  // kernels per fine slot (single-GPU one-warp pass: prolongation + sweep)
    double* coarse_backup = nullptr;
    size_t coarse_smem = 0;  // dynamic shared memory of the coarse-visit kernel
    int coarse_kind = 0;     // 0 global wavefront, 1 shared-memory iterate, 2 + TMEM rhs, 3 cluster bands,
                             // 4 register wavefront over many SMs, 5 sweep pipeline over the SMs,
                             // 6 sweep pipeline with several blocks per warp (> 16 blocks)
    RwEngine* rw = nullptr;
    SpEngine* sp = nullptr;
    Sp2Engine* sp2 = nullptr;
    TmGeom tm{};
    ClGeom cl{};
    // hybrid coarse visits: a one-SM kernel (cl1, role 1) runs groups of <= 4
    // sweeps and hands larger ones to the cluster kernel (cl, role 2)
    bool cl_hybrid = false;
    ClGeom cl1{};
    size_t coarse_smem1 = 0;
    double* coarse_backup1 = nullptr;
    double* tm_spec = nullptr;
    size_t smem = 0;
    int fine_kind = 0;  // 0 column pairs (256-column CTA strips), 2 one-warp strips of column quads
    dim3 grid;
    cudaEvent_t ev = nullptr;
    // multi-GPU strip decomposition (P.mp): this rank's exchange buffer, the
    // peers' buffers mapped through CUDA IPC, the pass counter across solves
    char* xbuf = nullptr;
    void* peer_map[kMaxRanks] = {};
    double* bar_scratch = nullptr;
    unsigned long long mp_seq = 0;
    std::vector<std::pair<int, int>> fine_rows, coarse_rows;  // per rank
};

bool fused_supported(const Solver& s) {
    if (s.cfg.scheme != ISMG_SCHEME_ISMG && s.cfg.scheme != ISMG_SCHEME_GMG) return false;
    if (s.bc.px() || s.bc.py()) return false;
    const int tile = s.g.tile;
    if (tile < 2 || tile > 64 || (tile & (tile - 1)) != 0) return false;  // tile | 256, lanes fold in a warp
    if (s.levels.empty()) return false;
    const CoarseOpH& h = s.levels.front().h;
    for (size_t k = 0; k < size_t(h.ncx) * h.ncy; ++k)
        if (h.w[k] == 0.0) return false;  // singular coarse row: op-level path raises
    return true;
}

// returns the kernels launched (the single-GPU one-warp pass is two kernels, by phase)
static int launch_fine(const FusedEngine& e, cudaStream_t st, bool sweep_only = false) {
    if (e.fine_kind == 2) return launch_fine_pass_w(e.P, e.grid, st, sweep_only);
    launch_fine_pass(e.P, e.grid, e.smem, st);
    return 1;
}

// the coarse-visit kernel(s) of this engine with parameters P
static void launch_coarse(const FusedEngine& e, const Params& P, cudaStream_t st) {
    if (e.coarse_kind == 6) {
        launch_coarse_sp2(P, *e.sp2, st);
    } else if (e.coarse_kind == 5) {
        launch_coarse_sp(P, *e.sp, st);
    } else if (e.coarse_kind == 4) {
        launch_coarse_rw(P, *e.rw, st);
    } else if (e.coarse_kind == 3) {
        if (e.cl_hybrid) launch_coarse_cl(P, e.cl1, e.tm_spec, e.coarse_backup1, e.coarse_smem1, st);
        launch_coarse_cl(P, e.cl, e.tm_spec, e.coarse_backup, e.coarse_smem, st);
    } else if (e.coarse_kind == 2) {
        launch_coarse_tmem(P, e.tm, e.tm_spec, e.coarse_backup, e.coarse_smem, st);
    } else if (e.coarse_kind == 1) {
        launch_coarse_smem(P, e.coarse_backup, e.coarse_smem, st);
    } else {
        launch_coarse_global(P, st);
    }
}

// The single-GPU solve as ONE conditional graph: WHILE (phase != done) {
// SWITCH (phase) { kFine: sweep pass | kCoarse: coarse visit | kProlong,
// kResid: prolongation / residual pass } }. The kernel that decides the next
// phase sets both conditions (publish_phase), so every launch does work and
// the host waits once per solve. Returns false where conditional nodes are
// unavailable (the slot graphs then run the solve).
[[maybe_unused]] static bool build_cond_graph(FusedEngine& e) {
    Ctx& c = *e.s->ctx;
    cudaGraph_t g = nullptr;
    bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
    cudaGraphConditionalHandle hw = 0, hs = 0;
    ok = ok && cudaGraphConditionalHandleCreate(&hw, g, 1u, cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wn = nullptr, sn = nullptr;
    ok = ok && cudaGraphAddNode(&wn, g, nullptr, 0, &wp) == cudaSuccess;
    cudaGraph_t body = ok ? wp.conditional.phGraph_out[0] : nullptr;
    ok = ok && cudaGraphConditionalHandleCreate(&hs, body, unsigned(kResid), cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNodeParams sp = {};
    sp.type = cudaGraphNodeTypeConditional;
    sp.conditional.handle = hs;
    sp.conditional.type = cudaGraphCondTypeSwitch;
    sp.conditional.size = 4;  // kFine, kCoarse, kProlong, kResid; kDone runs no body
    ok = ok && cudaGraphAddNode(&sn, body, nullptr, 0, &sp) == cudaSuccess;
    if (ok) {
        Params Pc = e.P;
        Pc.cond = 1, Pc.h_while = hw, Pc.h_switch = hs;
        for (int ph = 0; ph < 4 && ok; ++ph) {
            ok = cudaStreamBeginCaptureToGraph(c.stream, sp.conditional.phGraph_out[ph], nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (!ok) break;
            if (ph == kCoarse) {
                launch_coarse(e, Pc, c.stream);
            } else if (e.fine_kind == 2) {
                launch_fine_pass_w(Pc, e.grid, c.stream, ph == kFine, ph != kFine);
            } else {
                launch_fine_pass(Pc, e.grid, e.smem, c.stream);
            }
            cudaGraph_t tmp = nullptr;
            ok = cudaStreamEndCapture(c.stream, &tmp) == cudaSuccess;
        }
    }
    ok = ok && cudaGraphInstantiate(&e.cond_exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();  // a refused node type leaves no sticky error
    return ok;
}

// multi-GPU, after every fine-pass slot: the fine pass has stored its pack into
// every rank's exchange buffer (NVLink peer stores) and raised its flags;
// mp_unpack_kernel waits for all ranks' flags, reduces the pass partials in rank
// order, assembles the coarse rhs and applies the branch logic. No NCCL call.
static void mp_exchange(FusedEngine& e, Ctx& c) {
    (void)c;
    launch_mp_unpack(e.P, c.stream);
}

static int slot_index(int slots) { return slots <= 8 ? 0 : (slots <= 16 ? 1 : (slots <= 32 ? 2 : 3)); }

// The graph of `slots` [coarse-visit, fine-pass (+ exchange)] slots, captured on
// first use and kept for the engine's lifetime (capturing NCCL calls is costly).
static cudaGraphExec_t graph_for(FusedEngine& e, int slots) {
    cudaGraphExec_t& ge = e.graphs[slot_index(slots)];
    if (ge) return ge;
    Ctx& c = *e.s->ctx;
    cudaGraph_t g;
    ISMG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < slots; ++k) {
        launch_coarse(e, e.P, c.stream);
        if (e.P.mp && e.fine_kind == 2 && !getenv("ISMG_MP_ALLPHASE")) {
            // multi-GPU: [(anchor of P ce,) prolongation / residual pass, exchange, (fused pass,
            // exchange,) sweep pass, exchange]; the exchange after a pass that did not run (not
            // its phase) returns at once
            if (e.P.fuse) launch_prolong_sum(e.P, c.stream);
            launch_fine_pass_w(e.P, e.grid, c.stream, false, true);
            mp_exchange(e, c);
            if (e.P.fuse) {
                launch_fused_mp(e.P, e.grid, c.stream);
                mp_exchange(e, c);
            }
            launch_fine_pass_w(e.P, e.grid, c.stream, true, false);
            mp_exchange(e, c);
            e.fine_launches = e.P.fuse ? 5 : 3;  // (+1 exchange counted by the caller)
            continue;
        }
        e.fine_launches = launch_fine(e, c.stream);
        if (e.P.mp) mp_exchange(e, c);
    }
    ISMG_CUDA(cudaStreamEndCapture(c.stream, &g));
    ISMG_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    return ge;
}

// The coarse-visit kernel of level h: the sweep pipeline where it plans (coarse
// grids up to 16 blocks of 32 rows, every zero weight facing a ghost), else the
// cluster engine (up to 16 x 32-row bands), the register wavefront (config 4's
// 512 x 1024 level), then TMEM-resident rhs, shared-memory iterate, global
// wavefront. P.ncx / P.ncy must be set.
static void plan_coarse(FusedEngine& ee, const CoarseOpH& h, int device) {
    FusedEngine* e = &ee;
    Params& P = e->P;
    std::vector<double> spec;
    const char* force = getenv("ISMG_COARSE_KERNEL");  // test hook: "sp" | "sp2" | "rw" | "cl" | "tmem" | "smem" | "global"
    const bool allow_sp = !force || std::string(force) == "sp";
    const bool allow_sp2 = !force || std::string(force) == "sp2";
    if (allow_sp && (e->sp = sp_try_create(h, device)) != nullptr) {
        e->coarse_kind = 5;
        return;
    }
    if (allow_sp2 && (e->sp2 = sp2_try_create(h, device)) != nullptr) {
        e->coarse_kind = 6;
        return;
    }
    const bool allow_rw = !force || std::string(force) == "rw";
    const bool allow_cl = !force || std::string(force) == "cl";
    const bool allow_tmem = !force || std::string(force) == "tmem";
    const bool allow_smem = !force || std::string(force) == "smem" || std::string(force) == "tmem";
    const bool force_rw = force && std::string(force) == "rw";
    if (!force_rw && allow_cl && cl_coarse_plan(h, e->cl, spec, e->coarse_smem)) {
        e->coarse_kind = 3;
        ISMG_CUDA(cudaMalloc(&e->tm_spec, sizeof(double) * spec.size()));
        ISMG_H2D(e->tm_spec, spec.data(), sizeof(double) * spec.size());
        ISMG_CUDA(cudaMalloc(&e->coarse_backup, sizeof(double) * cl_backup_doubles(e->cl)));
        size_t smax = e->coarse_smem;
        // hybrid when the grid also fits one SM and the cluster is 2 SMs: a 2048^2
        // step 1 takes 170 ms with it against 181 without; at 4096^2 (4 SMs) the
        // one-SM kernel's shorter small groups are eaten by the extra launch per
        // slot (494 against 487 ms). ISMG_CL_HYBRID=0 / 1 forces it off / on.
        const char* hy = getenv("ISMG_CL_HYBRID");
        const bool want = hy ? std::string(hy) != "0" : e->cl.csize == 2;
        std::vector<double> spec1;
        if (e->cl.csize > 1 && want &&
            cl_coarse_plan(h, e->cl1, spec1, e->coarse_smem1, 128) && e->cl1.csize == 1 && spec1 == spec) {
            e->cl_hybrid = true;
            e->cl1.role = 1, e->cl.role = 2;
            ISMG_CUDA(cudaMalloc(&e->coarse_backup1, sizeof(double) * cl_backup_doubles(e->cl1)));
            smax = std::max(smax, e->coarse_smem1);
        }
        set_coarse_cl_smem(smax);
    } else if (allow_rw && (e->rw = rw_try_create(h, device)) != nullptr) {
        e->coarse_kind = 4;
    } else if (allow_tmem && tmem_coarse_plan(h, e->tm, spec, e->coarse_smem)) {
        e->coarse_kind = 2;
        ISMG_CUDA(cudaMalloc(&e->tm_spec, sizeof(double) * spec.size()));
        ISMG_H2D(e->tm_spec, spec.data(), sizeof(double) * spec.size());
        ISMG_CUDA(cudaMalloc(&e->coarse_backup, sizeof(double) * size_t(P.ncy + 2) * e->tm.pitch));
        set_coarse_tmem_smem(e->coarse_smem);
    } else if (allow_smem && size_t(P.ncx + 2) * (P.ncy + 2) * sizeof(double) <= 200 * 1024) {
        e->coarse_kind = 1;
        e->coarse_smem = size_t(P.ncx + 2) * (P.ncy + 2) * sizeof(double);
        ISMG_CUDA(cudaMalloc(&e->coarse_backup, e->coarse_smem));
        set_coarse_smem(e->coarse_smem);
    }
}

// A coarse-visit engine alone, for level L of a solver (the ACM hierarchy's
// coarsest level, cycles.hpp:222-235): the same kernels as the fused path's
// coarse phase, on L's rhs / iterate, one launch and one wait per visit.
FusedEngine* make_coarse_engine(Solver& s, LevelDev& L) {
    auto* e = new FusedEngine();
    e->s = &s;
    Params& P = e->P;
    P.ncx = L.h.ncx, P.ncy = L.h.ncy, P.tile = 1;
    P.singular = L.h.singular ? 1 : 0;
    P.nslots = L.h.stencil_points();
    P.tol_fine = s.cfg.tol_fine, P.tol_coarse = s.cfg.tol_coarse, P.stall = s.cfg.stall_factor;
    P.max_total = s.cfg.max_total_sweeps;
    P.cb = L.b->view();
    P.ce = L.x->view();
    P.cbw = P.cb;
    P.w = L.d_w;
    P.visit_cap = 1;
    ISMG_CUDA(cudaMalloc(&e->d_log, sizeof(int) * 2));
    P.visit_log = e->d_log;
    ISMG_CUDA(cudaMalloc(&e->d_ctl, sizeof(Ctl)));
    ISMG_CUDA(cudaMallocHost(&e->h_ctl, sizeof(Ctl)));
    P.ctl = e->d_ctl;
    ISMG_CUDA(cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming));
    plan_coarse(*e, L.h, s.ctx->device);
    return e;
}

// One visit: GS sweeps of the level until its residual is <= tol_coarse or the
// budget (max_total_sweeps - total) is spent, from x = 0, anchored once when
// singular; rc0 = the entry residual max|b|. Returns the sweeps; *rc the residual.
long long coarse_engine_visit(FusedEngine& e, long long total, double rc0, int pred, double* rc) {
    Ctx& c = *e.s->ctx;
    Ctl init{};
    init.phase = kCoarse;
    init.rc = rc0;
    init.pred = pred;
    init.total = total;
    init.nvisits = 1;
    *e.h_ctl = init;
    ISMG_CUDA(cudaMemcpyAsync(e.d_ctl, e.h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, c.stream));
    launch_coarse(e, e.P, c.stream);
    c.launches += e.cl_hybrid ? 2 : 1;
    ISMG_CUDA(cudaMemcpyAsync(e.h_ctl, e.d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
    ISMG_CUDA(cudaEventRecord(e.ev, c.stream));
    ISMG_CUDA(cudaEventSynchronize(e.ev));
    if (e.h_ctl->mp_error == 2) fail(ISMG_ERR_INTERNAL, "coarse visit: watchdog (mailbox / barrier timeout)");
    *rc = e.h_ctl->rc;
    return e.h_ctl->coarse;
}

FusedEngine* make_fused(Solver& s) {
    auto* e = new FusedEngine();
    e->s = &s;
    Ctx& c = *s.ctx;
    LevelDev& L = s.levels.front();
    e->scratch.alloc(s.g.nx + 1, s.g.ny + 1);
    Params& P = e->P;
    P.nx = s.g.nx, P.ny = s.g.ny, P.pitch = e->scratch.pitch;
    P.tile = s.g.tile, P.ncx = L.h.ncx, P.ncy = L.h.ncy;
    // fine kernel: one-warp strips of column quads when a tile spans >= 4 columns
    // (test hook ISMG_FINE_KERNEL=pair forces the column-pair kernel)
    const char* fk = getenv("ISMG_FINE_KERNEL");
    e->fine_kind = (P.tile >= 4) ? 2 : 0;
    if (fk && std::string(fk) == "pair") e->fine_kind = 0;
    const int width = e->fine_kind == 2 ? 4 * fine_pass_w_quads(P.tile) : kW;
    // strip decomposition over the context's NCCL ranks (one-warp kernel only)
    P.row0 = 0, P.row1 = P.ny, P.mp = 0;
    if (c.comm && c.comm->nranks > 1 && e->fine_kind == 2) {
        const int R = c.comm->nranks;
        for (int r = 0; r < R; ++r) {
            int a = 0, b = 0;
            strip_rows(P.ny, P.tile, R, r, &a, &b);
            e->fine_rows.emplace_back(a, b);
            e->coarse_rows.emplace_back(a / P.tile, (b + P.tile - 1) / P.tile);
        }
        P.row0 = e->fine_rows[size_t(c.comm->rank)].first, P.row1 = e->fine_rows[size_t(c.comm->rank)].second;
        P.mp = 1;
        P.nranks = R;
        // pack = [8 scalars | this rank's coarse rows (pitched) | 3 first rows | 3 last rows]
        const int rank = c.comm->rank;
        if (R > kMaxRanks) fail(ISMG_ERR_INVALID_ARGUMENT, "multi-GPU: more ranks than supported");
        const int64_t cpitch = L.b->view().pitch;
        int maxc = 0;
        for (auto& cr : e->coarse_rows) maxc = std::max(maxc, cr.second - cr.first);
        P.pack_cb_rows = maxc;
        const int64_t cbr = int64_t(maxc) * cpitch;
        int64_t len = 8 + cbr + 12 * P.pitch;  // + a fused pass's 3 + 3 input rows
        len = (len + 15) / 16 * 16;
        P.pack_len = int(len);
        P.rank = rank;
        P.nranks = R;
        const int cr0 = e->coarse_rows[size_t(rank)].first;
        P.cb_off = 8 - int64_t(cr0) * cpitch, P.cb_pitch = cpitch;
        P.h_off[0] = 8 + cbr, P.h_off[1] = 8 + cbr + 3 * P.pitch;
        P.h_off[2] = 8 + cbr + 6 * P.pitch, P.h_off[3] = 8 + cbr + 9 * P.pitch;
        // exchange buffer [2][R][len] doubles + R flags, shared with the peers by CUDA IPC
        const size_t data = sizeof(double) * size_t(2) * size_t(R) * size_t(len);
        const size_t bytes = data + 256;
        ISMG_CUDA(cudaMalloc(&e->xbuf, bytes));
        ISMG_ZERO(e->xbuf, bytes);
        ISMG_CUDA(cudaMalloc(&e->bar_scratch, sizeof(double) * 8 * size_t(R)));
        cudaIpcMemHandle_t h;
        ISMG_CUDA(cudaIpcGetMemHandle(&h, e->xbuf));
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        ISMG_H2D(e->bar_scratch + 8 * rank, &h, 64);
        std::vector<double> all(size_t(8) * size_t(R));
        double* d_all = nullptr;
        ISMG_CUDA(cudaMalloc(&d_all, sizeof(double) * all.size()));
        comm_allgather(*c.comm, e->bar_scratch + 8 * rank, d_all, 8, c.stream);
        ISMG_CUDA(cudaMemcpyAsync(all.data(), d_all, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        cudaFree(d_all);
        for (int q = 0; q < R; ++q) {
            char* base = e->xbuf;
            if (q != rank) {
                cudaIpcMemHandle_t hq;
                std::memcpy(&hq, all.data() + 8 * q, 64);
                void* ptr = nullptr;
                ISMG_CUDA(cudaIpcOpenMemHandle(&ptr, hq, cudaIpcMemLazyEnablePeerAccess));
                e->peer_map[q] = ptr;
                base = static_cast<char*>(ptr);
            }
            P.xch[q] = reinterpret_cast<double*>(base);
            P.xflag[q] = reinterpret_cast<unsigned long long*>(base + data);
        }
    }
    P.nstrips = (P.nx + width - 1) / width;
    // rows per CTA chunk. Short chunks keep the SMs full to the end of a pass; long
    // ones re-read fewer halo rows (3 per chunk). One-warp strips take the longest
    // chunk (<= 96 rows) that still gives >= 4 waves of resident warps, measured
    // (tools/probe_fine.py, B200): 4096^2 32 rows (2.7 waves) 125 us against 150 at
    // 64; 8192^2 64 rows 350 us against 368 at 32, 377 at 96; 16384^2 96 rows
    // 1159 us against 1320 at 32, 1191 at 64, 1163 at 128.
    if (e->fine_kind == 2) {
        const int slots = fine_pass_w_resident(P.mp != 0, c.device);
        P.H = std::max(P.tile, 32);
        for (int h = 96; h > 32; h -= 32) {
            const int hh = std::max(P.tile, h / P.tile * P.tile);
            const long ctas = long(P.nstrips) * ((P.row1 - P.row0 + hh - 1) / hh);
            if (ctas >= 4L * slots) {
                P.H = hh;
                break;
            }
        }
    } else {
        P.H = std::max(P.tile, 128 / P.tile * P.tile);
    }
    if (const char* h = getenv("ISMG_FINE_H")) {  // tuning hook: rows per CTA chunk (rounded to tiles)
        const int v = atoi(h);
        if (v > 0) P.H = std::max(P.tile, v / P.tile * P.tile);
    }
    P.nchunks = std::max(1, (P.row1 - P.row0 + P.H - 1) / P.H);
    P.bc = s.bc;
    P.singular = s.singular ? 1 : 0;
    P.nslots = L.h.stencil_points();
    P.tol_fine = s.cfg.tol_fine, P.tol_coarse = s.cfg.tol_coarse, P.stall = s.cfg.stall_factor;
    P.max_total = s.cfg.max_total_sweeps;
    P.ncells = double(int64_t(P.nx) * P.ny);
    P.cb = L.b->view();
    P.ce = L.x->view();
    if (!P.mp) P.cbw = P.cb;
    P.w = L.d_w;
    P.ax = L.ax, P.ay = L.ay;
    const int nb = P.nstrips * P.nchunks;
    // per-CTA partials + per-32-CTA group partials; tickets: [all, per group, exchange (multi-GPU)]
    const int ngrp = (nb + 31) / 32;
    // (4 per CTA / group: the fused pass adds max |rp|; >= 148 for prolong_sum_kernel's partials)
    ISMG_CUDA(cudaMalloc(&P.part, sizeof(double) * std::max<size_t>(148, 4 * size_t(nb + ngrp))));
    ISMG_CUDA(cudaMalloc(&P.ticket, sizeof(unsigned) * size_t(2 + ngrp)));
    ISMG_ZERO(P.ticket, sizeof(unsigned) * size_t(2 + ngrp));
    P.visit_cap = int(std::min<long long>(P.max_total + 2, 1 << 22));
    ISMG_CUDA(cudaMalloc(&e->d_log, sizeof(int) * 2 * P.visit_cap));
    P.visit_log = e->d_log;
    ISMG_CUDA(cudaMalloc(&e->d_ctl, sizeof(Ctl)));
    ISMG_CUDA(cudaMallocHost(&e->h_ctl, sizeof(Ctl)));
    P.ctl = e->d_ctl;
    e->grid = dim3(P.nstrips, P.nchunks);
    if (e->fine_kind == 2) {
        e->grid = fine_pass_w_grid(P);
        e->smem = fine_pass_w_smem();
        set_fine_pass_w_smem();
    } else {
        e->smem = fine_pass_smem();
        set_fine_pass_smem(e->smem);
    }
    ISMG_CUDA(cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming));
    plan_coarse(*e, L.h, c.device);
    // the fused prolongation + sweep pass (fine_pass_w.cu fused_w): single GPU, one-warp
    // strips, chunks of <= 96 rows, and uniform power-of-two tiles: every fine column /
    // row extent a power of two and every column quad inside one coarse pair (what the
    // pass's exact weight scaling assumes). ISMG_FUSE=0 turns it off (A/B hook).
    {
        const TileAxisH& ax = L.h.ax;
        const TileAxisH& ay = L.h.ay;
        auto pow2 = [](double d) {
            uint64_t u;
            std::memcpy(&u, &d, 8);
            return d > 0.0 && (u & 0x000FFFFFFFFFFFFFull) == 0;
        };
        bool ok = e->fine_kind == 2 && P.H + 7 <= 104 && e->cond_state != 1;
        if (P.mp && getenv("ISMG_MP_ALLPHASE")) ok = false;  // that A/B path has no fused slot
        if (const char* f = getenv("ISMG_FUSE")) ok = ok && f[0] != '0';
        if (const char* g = getenv("ISMG_COND_GRAPH")) ok = ok && g[0] != '1';  // its SWITCH has no fused case
        for (int i = 0; ok && i < P.nx; ++i) {
            ok = pow2(ax.dk[size_t(i)]);
            if (ok && (i & 3) != 0) ok = ax.k0[size_t(i)] == ax.k0[size_t(i - 1)] && ax.k1[size_t(i)] == ax.k1[size_t(i - 1)];
        }
        for (int j = 0; ok && j < P.ny; ++j) ok = pow2(ay.dk[size_t(j)]);
        if (ok) {
            // pax[I] = sum over fine columns i of the weight of coarse column I in P (the
            // pass's ar = (dx - s) / dx on k0, sr = s / dx on k1); pay likewise
            auto sums = [](const TileAxisH& a, int nc) {
                std::vector<double> v(size_t(nc), 0.0);
                for (int i = 0; i < a.n; ++i) {
                    const double d = a.dk[size_t(i)], t = a.t[size_t(i)];
                    v[size_t(a.k0[size_t(i)])] += (d - t) / d;
                    v[size_t(a.k1[size_t(i)])] += t / d;
                }
                return v;
            };
            const std::vector<double> hx = sums(ax, L.h.ncx), hy = sums(ay, L.h.ncy);
            double* d = nullptr;
            ISMG_CUDA(cudaMalloc(&d, sizeof(double) * (hx.size() + hy.size())));
            ISMG_H2D(d, hx.data(), sizeof(double) * hx.size());
            ISMG_H2D(d + hx.size(), hy.data(), sizeof(double) * hy.size());
            P.pax = d, P.pay = d + hx.size();
            P.fuse = 1;
        }
    }
    (void)c;
    return e;
}

void destroy_fused(FusedEngine* e) {
    if (!e) return;
    for (auto& ge : e->graphs)
        if (ge) cudaGraphExecDestroy(ge);
    if (e->cond_exec) cudaGraphExecDestroy(e->cond_exec);
    e->scratch.free();
    cudaFree(e->P.part);
    if (e->P.pax) cudaFree(const_cast<double*>(e->P.pax));
    cudaFree(e->P.ticket);
    cudaFree(e->d_log);
    cudaFree(e->coarse_backup);
    cudaFree(e->tm_spec);
    cudaFree(e->coarse_backup1);
    rw_destroy(e->rw);
    sp_destroy(e->sp);
    sp2_destroy(e->sp2);
    for (void* p : e->peer_map)
        if (p) cudaIpcCloseMemHandle(p);
    cudaFree(e->xbuf);
    cudaFree(e->bar_scratch);
    cudaFree(e->d_ctl);
    cudaFreeHost(e->h_ctl);
    if (e->ev) cudaEventDestroy(e->ev);
    delete e;
}

// Benchmark hook: `iters` fused sweep passes (red, black, residual, tile sums,
// anchor sum) back to back on (x, b), each bracketed by CUDA events on the
// context stream. Returns the mean event time per pass in ms. x is relaxed in
// place (ping-pong through the scratch buffer).
double fused_bench_fine_pass(Solver& s, Field& x, const Field& b, int iters) {
    FusedEngine& e = *s.fused;
    Ctx& c = *s.ctx;
    if (x.buf.pitch != e.P.pitch || b.buf.pitch != e.P.pitch)
        fail(ISMG_ERR_INTERNAL, "fused path: field pitch mismatch");
    if (e.P.mp) fail(ISMG_ERR_INVALID_ARGUMENT, "bench_fine_pass: single-GPU contexts only");
    k_zero_ghosts(c, x.view());
    Ctl init{};
    init.phase = kFine;
    init.hold = 1;
    init.buf[0] = x.buf.origin();
    init.buf[1] = e.scratch.origin();
    init.b = b.buf.origin();
    *e.h_ctl = init;
    ISMG_CUDA(cudaMemcpyAsync(e.d_ctl, e.h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, c.stream));
    std::vector<cudaEvent_t> ev(size_t(iters) + 1);
    for (auto& v : ev) ISMG_CUDA(cudaEventCreate(&v));
    ISMG_CUDA(cudaEventRecord(ev[0], c.stream));
    for (int k = 0; k < iters; ++k) {
        c.launches += launch_fine(e, c.stream, true);
        ISMG_CUDA(cudaEventRecord(ev[size_t(k) + 1], c.stream));
    }
    ISMG_CUDA(cudaMemcpyAsync(e.h_ctl, e.d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    double total = 0.0;
    for (int k = 0; k < iters; ++k) {
        float ms = 0.f;
        ISMG_CUDA(cudaEventElapsedTime(&ms, ev[size_t(k)], ev[size_t(k) + 1]));
        total += ms;
    }
    for (auto& v : ev) cudaEventDestroy(v);
    if (e.h_ctl->cur != 0) {  // leave the relaxed iterate in the caller's field
        ISMG_CUDA(cudaMemcpyAsync(x.buf.base, e.scratch.base, x.buf.bytes, cudaMemcpyDeviceToDevice, c.stream));
        c.sync();
    }
    return total / iters;
}

// Measurement / parity hook: ONE coarse visit of this engine's coarse-visit
// kernel on rhs cb from ce = 0, at most `budget` sweeps, first group `first`
// sweeps; ce receives the iterate. Returns the kernel's CUDA-event time (ms).
double fused_bench_coarse_visit(Solver& s, const Field& cb, Field& ce, long long budget, int first,
                                long long* sweeps, double* rc) {
    FusedEngine& e = *s.fused;
    Ctx& c = *s.ctx;
    LevelDev& L = s.levels.front();
    if (cb.nx != L.h.ncx || cb.ny != L.h.ncy || ce.nx != L.h.ncx || ce.ny != L.h.ncy)
        fail(ISMG_ERR_INVALID_ARGUMENT, "bench_coarse_visit: fields must have the coarse extent");
    if (budget < 1 || first < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "bench_coarse_visit: budget, first >= 1");
    const size_t w = sizeof(double) * size_t(L.h.ncx);
    ISMG_CUDA(cudaMemcpy2DAsync(L.b->buf.origin(), sizeof(double) * L.b->buf.pitch, cb.buf.origin(),
                                sizeof(double) * cb.buf.pitch, w, size_t(L.h.ncy), cudaMemcpyDeviceToDevice,
                                c.stream));
    std::vector<double> h(size_t(L.h.ncx) * L.h.ncy);
    ISMG_CUDA(cudaMemcpy2DAsync(h.data(), w, cb.buf.origin(), sizeof(double) * cb.buf.pitch, w, size_t(L.h.ncy),
                                cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    double rc0 = 0.0;
    for (double v : h) rc0 = (rc0 < std::abs(v)) ? std::abs(v) : rc0;  // coarse_residual(ce = 0)
    Ctl init{};
    init.phase = kCoarse;
    init.rc = rc0;
    init.pred = first;
    init.total = e.P.max_total - budget;
    init.nvisits = 1;
    *e.h_ctl = init;
    ISMG_CUDA(cudaMemcpyAsync(e.d_ctl, e.h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, c.stream));
    cudaEvent_t e0, e1;
    ISMG_CUDA(cudaEventCreate(&e0));
    ISMG_CUDA(cudaEventCreate(&e1));
    ISMG_CUDA(cudaEventRecord(e0, c.stream));
    launch_coarse(e, e.P, c.stream);
    ISMG_CUDA(cudaEventRecord(e1, c.stream));
    ISMG_CUDA(cudaMemcpyAsync(e.h_ctl, e.d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
    ISMG_CUDA(cudaMemcpy2DAsync(ce.buf.origin(), sizeof(double) * ce.buf.pitch, L.x->buf.origin(),
                                sizeof(double) * L.x->buf.pitch, w, size_t(L.h.ncy), cudaMemcpyDeviceToDevice,
                                c.stream));
    c.sync();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e.h_ctl->mp_error == 2) fail(ISMG_ERR_INTERNAL, "coarse visit: watchdog (mailbox / barrier timeout)");
    if (e.coarse_kind == 4 && getenv("ISMG_RW_TRACE")) {  // debug: per-group residual maxima to stderr
        const std::vector<double> t = rw_trace_take();
        for (double v : t)
            fprintf(stderr, v == -1.0 ? "\nRWTRACE" : (v == -2.0 ? "\nRWSLOW" : (v == -3.0 ? "\nRWCYC" : " %.17g")), v);
        fprintf(stderr, "\n");
    }
    *sweeps = e.h_ctl->coarse;
    *rc = e.h_ctl->rc;
    s.last.coarse_engine = e.coarse_kind;
    return ms;
}

void fused_solve(Solver& s, Field& x, const Field& b, ismg_report& rep, Metrics& M, bool, double**) {
    FusedEngine& e = *s.fused;
    Ctx& c = *s.ctx;
    if (x.buf.pitch != e.P.pitch || b.buf.pitch != e.P.pitch)
        fail(ISMG_ERR_INTERNAL, "fused path: field pitch mismatch");
    k_zero_ghosts(c, x.view());  // cycles.hpp:106
    Ctl init{};
    init.phase = kResid;
    init.converged = 1;
    init.cur = 0;
    init.buf[0] = x.buf.origin();
    init.buf[1] = e.scratch.origin();
    init.b = b.buf.origin();
    init.mp_seq = e.mp_seq;
    *e.h_ctl = init;
    ISMG_CUDA(cudaMemcpyAsync(e.d_ctl, e.h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, c.stream));
    if (e.P.mp) {  // first halo rows: this rank's boundary rows of x into every rank's
                   // slot of the parity the solve's first pass reads (that of pass mp_seq - 1)
        const size_t rows3 = size_t(3) * size_t(e.P.pitch);
        const double* row0 = x.buf.origin() - kXOff;  // start of logical row 0
        const int R = e.P.nranks, p = int((e.mp_seq + 1ull) & 1ull);
        for (int q = 0; q < R; ++q) {
            double* slot = e.P.xch[q] + (int64_t(p) * R + e.P.rank) * e.P.pack_len;
            if (e.P.row0 > 0)
                ISMG_CUDA(cudaMemcpyAsync(slot + e.P.h_off[0], row0 + int64_t(e.P.row0) * e.P.pitch,
                                          rows3 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
            if (e.P.row1 < e.P.ny)
                ISMG_CUDA(cudaMemcpyAsync(slot + e.P.h_off[1], row0 + int64_t(e.P.row1 - 3) * e.P.pitch,
                                          rows3 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
        }
        // every rank's copies done before any rank's first pass reads them
        comm_reduce_scalars(*c.comm, e.bar_scratch, 1, 0, c.stream);
        c.comm->collectives += 1;
    }
    if (!e.P.mp && e.cond_state == 0) {
        // ISMG_COND_GRAPH=1: the conditional graph. Off by default: measured A/B on one
        // box (tools/visit_hist.py), the slot graphs' no-op launches cost less than the
        // conditional nodes' per-iteration overhead: 4096^2 steps 1-3 449 / 239 / 251 ms
        // against 456 / 245 / 257; 16384^2 3235 / 2385 / 3057 against 3321 / 2391 / 3062.
        const char* cg = getenv("ISMG_COND_GRAPH");
#ifdef ISMG_WITH_COND_GRAPH
        e.cond_state = (cg && cg[0] == '1') ? (build_cond_graph(e) ? 1 : -1) : -1;
#else
        (void)cg;
        e.cond_state = -1;
#endif
    }
    long long launched_slots = 0;
    if (e.cond_state == 1) {  // the whole solve: one graph launch, one wait
        ISMG_CUDA(cudaGraphLaunch(e.cond_exec, c.stream));
        ISMG_CUDA(cudaMemcpyAsync(e.h_ctl, e.d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
        ISMG_CUDA(cudaEventRecord(e.ev, c.stream));
        ISMG_CUDA(cudaEventSynchronize(e.ev));
        s.last.host_syncs += 1;
        if (e.h_ctl->phase != kDone) fail(ISMG_ERR_INTERNAL, "fused solve: conditional graph ended before the solve");
        c.launches += e.h_ctl->passes + e.h_ctl->coarse_launches * (e.cl_hybrid ? 2 : 1);
    }
    // else: batches of [coarse-visit, fine-pass] slots until the phase is done
    int slots = 8;
    int since_poll = 0;
    for (; e.cond_state != 1;) {
        ISMG_CUDA(cudaGraphLaunch(graph_for(e, slots), c.stream));
        c.launches += (1 + e.fine_launches + (e.P.mp ? 1 : 0)) * slots + (e.cl_hybrid ? slots : 0);
        launched_slots += slots;
        ISMG_CUDA(cudaMemcpyAsync(e.h_ctl, e.d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
        ISMG_CUDA(cudaEventRecord(e.ev, c.stream));
        ISMG_CUDA(cudaEventSynchronize(e.ev));
        s.last.host_syncs += 1;
        ++since_poll;
        if (e.h_ctl->phase == kDone) break;
        if (launched_slots > 4 * (s.cfg.max_total_sweeps + 8)) fail(ISMG_ERR_INTERNAL, "fused solve did not terminate");
        slots = std::min(64, slots * 2);
    }
    (void)since_poll;
    launch_finalize(e.P, x.view(), c.stream);
    c.launches += 1;
    if (e.P.mp) {  // every rank's strip of the solution to every rank
        comm_gather_rows(*c.comm, x.buf.origin() - kXOff, e.P.pitch, e.fine_rows, c.stream);
        c.comm->collectives += c.comm->nranks;
    }
    ISMG_CUDA(cudaGetLastError());
    const Ctl& st = *e.h_ctl;
    e.mp_seq = st.mp_seq;
    if (st.mp_error == 2) fail(ISMG_ERR_INTERNAL, "coarse visit: a mailbox word or grid barrier timed out (watchdog)");
    if (st.mp_error) fail(ISMG_ERR_INTERNAL, "multi-GPU: a peer's pack did not arrive (exchange timed out)");
    // replay the sweep sequence into the metrics (lap_equiv order, metrics.hpp:46-56)
    const int nv = std::min(st.nvisits, e.P.visit_cap);
    e.h_log.resize(size_t(2) * std::max(nv, 1));
    if (nv > 0)
        ISMG_CUDA(cudaMemcpyAsync(e.h_log.data(), e.d_log, sizeof(int) * 2 * nv, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    s.visit_log.assign(e.h_log.begin(), e.h_log.begin() + 2 * nv);
    const int64_t cells = int64_t(s.g.nx) * s.g.ny;
    const LevelDev& L = s.levels.front();
    const int64_t ccells = int64_t(L.h.ncx) * L.h.ncy;
    for (int v = 0; v < nv; ++v) {
        M.restriction();
        for (int k = 0; k < e.h_log[2 * v]; ++k) M.sweep(false, L.h.stencil_points(), ccells);
        for (int k = 0; k < e.h_log[2 * v + 1]; ++k) M.sweep(true, 5, cells);
    }
    for (long long k = 0; k < st.prolongations; ++k) M.prolongation();
    rep.converged = st.converged;
    rep.nan_seen = st.nan_seen;
    rep.fine_sweeps = st.fine;
    rep.coarse_sweeps = st.coarse;
    rep.residual = st.r;
    s.last.fine_passes = st.fine;
    s.last.prolong_passes = st.prolongations;
    s.last.coarse_visits = st.coarse_launches;
    s.last.coarse_ms = double(st.coarse_ns) * 1e-6;
    s.last.coarse_steps = st.coarse_steps;
    s.last.coarse_engine = e.coarse_kind;
    s.last.collectives = c.comm ? c.comm->collectives : 0;
    s.last.fine_pass_ms = 0.0;  // not separated on the fused path (coarse_ms is device-timed)
    s.last.kernel_launches = e.cond_state == 1 ? st.passes + st.coarse_launches * (e.cl_hybrid ? 2 : 1) + 2
                                               : ((e.P.mp ? 3 : 1 + e.fine_launches) + (e.cl_hybrid ? 1 : 0)) * launched_slots + 2;
}

}  // namespace ismgb

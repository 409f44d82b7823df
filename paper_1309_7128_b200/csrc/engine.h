// engine.h — device-resident objects behind the C-ABI handles and the kernel
// launchers (ops.cu: op-level + projection kernels; fused.cu: the hot path).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <utility>
#include <vector>

#include "common.h"

namespace ismgb {

// Per-context scratch for reductions and scalar hand-back.
struct Scratch {
    double* part = nullptr;     // per-block partials (kMaxPartials)
    double* scal = nullptr;     // device scalars (kScalars)
    double* host = nullptr;     // pinned host mirror of scal
    unsigned* ticket = nullptr; // last-block tickets
    static constexpr int kMaxPartials = 65536;
    static constexpr int kScalars = 64;
};

// multi-GPU (comm.cpp): NCCL communicator of the strip decomposition
struct Comm {
    void* nccl = nullptr;  // ncclComm_t
    int rank = 0, nranks = 1;
    long long collectives = 0;  // NCCL calls issued (stats)
};
Comm* make_comm(int device, const void* unique_id, int rank, int nranks);
void destroy_comm(Comm* c);
void nccl_unique_id(void* out128);
void strip_rows(int ny, int tile, int nranks, int rank, int* r0, int* r1);
void comm_reduce_scalars(Comm& c, double* v, int nmax, int nsum, cudaStream_t st);
void comm_gather_rows(Comm& c, double* origin, int64_t pitch, const std::vector<std::pair<int, int>>& rows,
                      cudaStream_t st);
void comm_halo(Comm& c, double* const send[2], double* const recv[2], size_t count, cudaStream_t st);
void comm_allgather(Comm& c, const double* pack, double* gathered, size_t count, cudaStream_t st);

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sms = 148;
    long long launches = 0;  // kernels launched through this context (stream order)
    Scratch s;
    Comm* comm = nullptr;
    Ctx(int device, cudaStream_t stream);
    ~Ctx();
    void sync();
};

struct Field {
    Ctx* ctx;
    int nx, ny;
    DevBuf buf;
    Field(Ctx* c, int nx, int ny);
    ~Field() { buf.free(); }
    View view() const { return View{buf.origin(), buf.pitch, nx, ny}; }
};

struct Velocity {
    Ctx* ctx;
    int nx, ny;
    DevBuf u, v;
    Velocity(Ctx* c, int nx, int ny);
    ~Velocity() {
        u.free();
        v.free();
    }
    View uv() const { return View{u.origin(), u.pitch, nx + 1, ny}; }  // u(i,j), i in [-1, nx+1]
    View vv() const { return View{v.origin(), v.pitch, nx, ny + 1}; }  // v(i,j), j in [-1, ny+1]
};

// ---- op-level launchers (ops.cu) -------------------------------------------
// Whole logical field (interior + ghost ring) of extent (nx+2)x(ny+2).
void k_fill(Ctx& c, View f, double v);
void k_zero_ghosts(Ctx& c, View f);
void k_refresh_periodic(Ctx& c, View f, bool px, bool py);
void k_rbgs_half(Ctx& c, View x, View b, PBC bc, int color);
// r = b - A x; out may have p == nullptr; writes max|r| (NaN dropped) to *d_rmax
// and the NaN count to *d_nan (may be null).
void k_fine_residual(Ctx& c, View x, View b, View out, PBC bc, double* d_rmax, double* d_nan);
// interior sum (deterministic tree) -> d_out[0]; d_out[1] = -(sum / (nx*ny))
void k_mean_shift(Ctx& c, View x, double* d_out);
void k_shift_interior(Ctx& c, View x, const double* d_shift);
void k_restrict_exact(Ctx& c, View fine, View coarse, int tile_x, int tile_y, int ncx, int ncy);
void k_prolong_bilinear(Ctx& c, View coarse, View fine, const AxisDev& ax, const AxisDev& ay);
void k_prolong_constant(Ctx& c, View coarse, View fine, int tile_x, int tile_y);
void k_coarse_residual(Ctx& c, View x, View b, View out, const double* w, int ncx, int ncy, bool px, bool py,
                       int nslots, double* d_rmax);
void k_gs_lex(Ctx& c, View x, View b, const double* w, int ncx, int ncy, bool px, bool py, int nslots);
void k_rbgs_op(Ctx& c, View x, View b, const double* w, int ncx, int ncy, bool px, bool py, int color);
void k_copy_field(Ctx& c, View dst, View src, int w, int h);  // logical [-1, w) x [-1, h)

// ---- projection launchers (ops.cu) ----------------------------------------
void k_scalar_bc(Ctx& c, View f, PBC bc);
void k_velocity_bc(Ctx& c, Velocity& vel, const ismg_grid_spec& g);
void k_divergence(Ctx& c, const Velocity& vel, View out, double invh, double scale, bool do_scale);
void k_correct(Ctx& c, Velocity& vel, View dp, double cdt);
void k_predictor(Ctx& c, const Velocity& vel, View p, double dt, double nu, double invh, double invh2, bool px,
                 bool py, Velocity& out);
void k_add_interior(Ctx& c, View dst, View src);

}  // namespace ismgb

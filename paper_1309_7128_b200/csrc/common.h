// common.h — internal definitions shared by the host C++ and the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ismg_b200.h"

namespace ismgb {

// ---------------------------------------------------------------------------
// Errors: thrown inside the library, mapped to status codes at the C-ABI.
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Status(code, msg); }

#define ISMG_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            ::ismgb::fail(ISMG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Zero freshly allocated device memory and wait for it. cudaMemset runs on the
// legacy default stream, which does NOT order against the context's non-blocking
// stream: without the wait, a later upload or kernel on that stream could run
// before the memset and have its data zeroed (seen as a rare solve that read
// b = 0 and "converged" with residual 0).
#define ISMG_ZERO(ptr, bytes)                                         \
    do {                                                              \
        ISMG_CUDA(cudaMemset((ptr), 0, (bytes)));      \
        ISMG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));           \
    } while (0)
// A blocking host-to-device copy of setup data (tables, weights), complete before
// anything on a non-blocking stream can read it (a pageable cudaMemcpy may return
// before its DMA lands).
#define ISMG_H2D(dst, src, bytes)                                                \
    do {                                                                         \
        ISMG_CUDA(cudaMemcpy((dst), (src), (bytes), cudaMemcpyHostToDevice));    \
        ISMG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));                      \
    } while (0)

// ---------------------------------------------------------------------------
// Device field layout: the reference's logical ghosted
// layout embedded in a padded, pitched allocation. Logical (i, j) lives at
// base[(j + kYOff) * pitch + (i + kXOff)]: interior column 0 is 128-byte
// aligned (pitch is a multiple of 16 doubles) and there are >= 3 padding
// cells beyond every ghost so halo loads of the fused kernels never leave the
// allocation. View::p points at logical (0, 0).
constexpr int kXOff = 16;
constexpr int kYOff = 4;
constexpr int kPadRight = 4;  // logical columns [w, w + 4) addressable beyond the extent
constexpr int kPadTop = 4;

struct View {
    double* p = nullptr;
    int64_t pitch = 0;  // doubles
    int nx = 0, ny = 0; // interior extent of the logical field
    __host__ __device__ double& at(int i, int j) const { return p[int64_t(j) * pitch + i]; }
    __host__ __device__ double* row(int j) const { return p + int64_t(j) * pitch; }
};

// Pitched padded buffer covering logical columns [-kXOff, w + kPadRight) and
// rows [-kYOff, h + kPadTop), where (w, h) is the logical extent counted from
// index 0 to the last ghost inclusive (e.g. nx + 1, ny + 1 for a scalar field).
struct DevBuf {
    double* base = nullptr;
    int64_t pitch = 0;
    int64_t rows = 0;
    size_t bytes = 0;
    void alloc(int w, int h);
    void free();
    double* origin() const { return base + int64_t(kYOff) * pitch + kXOff; }
};

// Pressure closures per side (grid.hpp:119-141) as kernel parameters.
struct PBC {
    int k[4];  // ISMG_PBC_* indexed by ISMG_SIDE_*
    __host__ __device__ bool px() const { return k[ISMG_SIDE_WEST] == ISMG_PBC_PERIODIC; }
    __host__ __device__ bool py() const { return k[ISMG_SIDE_SOUTH] == ISMG_PBC_PERIODIC; }
};

// Per-axis TileAxis tables (coarsening.hpp:42-105) uploaded once per solver.
struct AxisDev {
    int n = 0, tile = 1, nc = 0, periodic = 0;
    int* k0 = nullptr;     // locate_cell(i).k0
    int* k1 = nullptr;
    double* t = nullptr;   // offset from center[k0]
    double* dk = nullptr;  // rectangle extent
};

// ---------------------------------------------------------------------------
// Host-side geometry (geometry.cpp): restated from the reference headers.
struct TileAxisH {
    int n = 0, tile = 1, nc = 0;
    bool periodic = false;
    std::vector<int> start, width;
    std::vector<double> center, rect;
    double rect_wrap = 0.0;
    std::vector<int> k0, k1;
    std::vector<double> t, dk;
    TileAxisH() = default;
    TileAxisH(int n, int tile, bool periodic);
};

// Strip decomposition (multi-GPU): rows [r0, r1) of `rank` are whole tiles, as
// even as possible (the first ntiles % nranks ranks take one more tile).
__host__ __device__ inline void strip_of(int ny, int tile, int nranks, int rank, int* r0, int* r1) {
    const int ntiles = (ny + tile - 1) / tile;
    const int base = ntiles / nranks, extra = ntiles % nranks;
    const int t0 = rank * base + (rank < extra ? rank : extra);
    const int t1 = t0 + base + (rank < extra ? 1 : 0);
    *r0 = t0 * tile < ny ? t0 * tile : ny;
    *r1 = t1 * tile < ny ? t1 * tile : ny;
}

struct CoarseOpH {
    int ncx = 0, ncy = 0;
    TileAxisH ax, ay;
    bool px = false, py = false, five_point = false, singular = false;
    std::vector<double> w;  // 9 planes, plane-major, slot order C,E,W,N,S,NE,NW,SE,SW
    double& at(int slot, int I, int J) { return w[size_t(slot) * ncx * ncy + size_t(J) * ncx + I]; }
    double at(int slot, int I, int J) const { return w[size_t(slot) * ncx * ncy + size_t(J) * ncx + I]; }
    int stencil_points() const { return five_point ? 5 : 9; }
};

void grid_validate(const ismg_grid_spec& g);
void cycle_validate(const ismg_cycle_config& c);
PBC pressure_bc(const ismg_grid_spec& g, bool* singular = nullptr);
void check_fine_stage(const ismg_grid_spec& g);  // domain_error on an empty stencil
CoarseOpH build_ismg_operator(const ismg_grid_spec& g);
CoarseOpH build_gmg_operator(const ismg_grid_spec& g);
std::vector<CoarseOpH> build_acm_hierarchy(const ismg_grid_spec& g, int depth);

}  // namespace ismgb

// objects.cu — context, device fields and velocity pairs.
#include <algorithm>
#include <cstring>

#include "engine.h"

namespace ismgb {

void DevBuf::alloc(int w, int h) {
    // logical columns [-kXOff, w + kPadRight), rows [-kYOff, h + kPadTop)
    const int64_t cols = int64_t(kXOff) + w + kPadRight;
    pitch = (cols + 15) / 16 * 16;
    rows = int64_t(kYOff) + h + kPadTop;
    bytes = size_t(pitch) * size_t(rows) * sizeof(double);
    ISMG_CUDA(cudaMalloc(&base, bytes));
    ISMG_ZERO(base, bytes);
}

void DevBuf::free() {
    if (base) cudaFree(base);
    base = nullptr;
}

Ctx::Ctx(int dev, cudaStream_t st) : device(dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(ISMG_ERR_NO_DEVICE, "no CUDA device available");
    }
    if (dev < 0 || dev >= n) fail(ISMG_ERR_INVALID_ARGUMENT, "device index out of range");
    ISMG_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop;
    ISMG_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
        fail(ISMG_ERR_NO_DEVICE, std::string("sm_100a build needs a Blackwell device, found ") + prop.name);
    sms = prop.multiProcessorCount;
    if (st) {
        stream = st;
    } else {
        ISMG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        own_stream = true;
    }
    ISMG_CUDA(cudaMalloc(&s.part, sizeof(double) * Scratch::kMaxPartials));
    ISMG_CUDA(cudaMalloc(&s.scal, sizeof(double) * Scratch::kScalars));
    ISMG_ZERO(s.scal, sizeof(double) * Scratch::kScalars);
    ISMG_CUDA(cudaMalloc(&s.ticket, sizeof(unsigned) * 64));
    ISMG_ZERO(s.ticket, sizeof(unsigned) * 64);
    ISMG_CUDA(cudaMallocHost(&s.host, sizeof(double) * Scratch::kScalars));
}

Ctx::~Ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    destroy_comm(comm);
    cudaFree(s.part);
    cudaFree(s.scal);
    cudaFree(s.ticket);
    cudaFreeHost(s.host);
    if (own_stream) cudaStreamDestroy(stream);
}

void Ctx::sync() { ISMG_CUDA(cudaStreamSynchronize(stream)); }

Field::Field(Ctx* c, int nx_, int ny_) : ctx(c), nx(nx_), ny(ny_) {
    if (nx < 1 || ny < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "field: nx, ny must be >= 1");
    ISMG_CUDA(cudaSetDevice(c->device));
    buf.alloc(nx + 1, ny + 1);
}

Velocity::Velocity(Ctx* c, int nx_, int ny_) : ctx(c), nx(nx_), ny(ny_) {
    if (nx < 1 || ny < 1) fail(ISMG_ERR_INVALID_ARGUMENT, "velocity: nx, ny must be >= 1");
    ISMG_CUDA(cudaSetDevice(c->device));
    u.alloc(nx + 2, ny + 1);  // u(i,j): i in [-1, nx+1], j in [-1, ny]
    v.alloc(nx + 1, ny + 2);  // v(i,j): i in [-1, nx],   j in [-1, ny+1]
}

}  // namespace ismgb

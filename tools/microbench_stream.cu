// Streaming microbenchmark for the fine-pass access pattern: every warp walks
// H rows of a pitched fp64 field pair (x, b), reading a window of C doubles
// per row per array, and writes C-8 doubles of x back. Variants:
//   tma  : lane 0 issues cp.async.bulk row copies into a per-warp ring of R
//          slots (mbarrier-tracked), all lanes consume from shared memory;
//   ldg  : every lane reads its 2 x 16 B of x and b with LDG.128, D rows ahead
//          in registers (software pipeline).
// Reports the algorithmic bandwidth (16 B read + 8 B written per owned cell).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(bar)),
                 "r"(ph) : "memory");
}

template <int C, int R>
__global__ void tma_stream(const double* x, const double* b, double* out, int64_t pitch, int nstrip, int ny, int H) {
    extern __shared__ __align__(128) unsigned char raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* sx = reinterpret_cast<double*>(raw) + size_t(warp) * R * 2 * C;
    double* sb = sx + R * C;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(raw) + size_t(nw) * R * 2 * C) + warp * R;
    const int strip = blockIdx.x * nw + warp;
    if (strip >= nstrip) return;
    const int a = strip * (C - 8) + 8;
    const int r0 = blockIdx.y * H, r1 = min(r0 + H, ny);
    if (lane == 0) {
        for (int s = 0; s < R; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int row, int s) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        expect_tx(&bars[s], 2u * C * 8u);
        bulk(sx + s * C, x + row * pitch + a - 4, C * 8u, &bars[s]);
        bulk(sb + s * C, b + row * pitch + a - 4, C * 8u, &bars[s]);
    };
    if (lane == 0)
        for (int k = 0; k < R && r0 + k < r1; ++k) issue(r0 + k, k);
    double acc = 0.0;
    int s = 0, ph = 0;
    for (int k = r0; k < r1; ++k) {
        wait(&bars[s], ph);
        for (int c = lane * 2; c < C - 8; c += 64) {
            const double2 v = *reinterpret_cast<const double2*>(sx + s * C + 4 + c);
            const double2 w = *reinterpret_cast<const double2*>(sb + s * C + 4 + c);
            *reinterpret_cast<double2*>(out + k * pitch + a + c) = make_double2(v.x + w.x, v.y + w.y);
        }
        __syncwarp();
        if (lane == 0 && k + R < r1) issue(k + R, s);
        if (++s == R) s = 0, ph ^= 1;
    }
    (void)acc;
}

template <int D>
__global__ void ldg_stream(const double* x, const double* b, double* out, int64_t pitch, int nstrip, int ny, int H, int C) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int strip = blockIdx.x * nw + warp;
    if (strip >= nstrip) return;
    const int a = strip * (C - 8) + 8;
    const int r0 = blockIdx.y * H, r1 = min(r0 + H, ny);
    const int c = a - 4 + 4 * lane;  // 4 doubles per lane (C = 128)
    double4 px[D], pb[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int row = min(r0 + d, r1 - 1);
        const double2 u0 = __ldg(reinterpret_cast<const double2*>(x + row * pitch + c));
        const double2 u1 = __ldg(reinterpret_cast<const double2*>(x + row * pitch + c + 2));
        const double2 w0 = __ldg(reinterpret_cast<const double2*>(b + row * pitch + c));
        const double2 w1 = __ldg(reinterpret_cast<const double2*>(b + row * pitch + c + 2));
        px[d] = make_double4(u0.x, u0.y, u1.x, u1.y);
        pb[d] = make_double4(w0.x, w0.y, w1.x, w1.y);
    }
    for (int k = r0; k < r1; k += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if (k + d < r1 && lane >= 1 && lane <= 30) {
                double* o = out + (k + d) * pitch + c;
                reinterpret_cast<double2*>(o)[0] = make_double2(px[d].x + pb[d].x, px[d].y + pb[d].y);
                reinterpret_cast<double2*>(o)[1] = make_double2(px[d].z + pb[d].z, px[d].w + pb[d].w);
            }
            const int row = min(k + d + D, r1 - 1);
            const double2 u0 = __ldg(reinterpret_cast<const double2*>(x + row * pitch + c));
            const double2 u1 = __ldg(reinterpret_cast<const double2*>(x + row * pitch + c + 2));
            const double2 w0 = __ldg(reinterpret_cast<const double2*>(b + row * pitch + c));
            const double2 w1 = __ldg(reinterpret_cast<const double2*>(b + row * pitch + c + 2));
            px[d] = make_double4(u0.x, u0.y, u1.x, u1.y);
            pb[d] = make_double4(w0.x, w0.y, w1.x, w1.y);
        }
    }
}

template <int C, int R>
int run_tma(const double* x, const double* b, double* out, int64_t pitch, int n, int H, int warps, cudaEvent_t e0,
            cudaEvent_t e1) {
    const int nstrip = (n + (C - 8) - 1) / (C - 8);
    const size_t smem = size_t(warps) * (R * 2 * C * 8 + R * 8);
    CK(cudaFuncSetAttribute(tma_stream<C, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 grid((nstrip + warps - 1) / warps, (n + H - 1) / H);
    tma_stream<C, R><<<grid, 32 * warps, smem>>>(x, b, out, pitch, nstrip, n, H);
    CK(cudaEventRecord(e0));
    const int it = 10;
    for (int i = 0; i < it; ++i) tma_stream<C, R><<<grid, 32 * warps, smem>>>(x, b, out, pitch, nstrip, n, H);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_stream<C, R>, 32 * warps, smem);
    printf("tma C=%4d R=%d warps=%d H=%4d occ=%d: %7.1f us  %6.0f GB/s\n", C, R, warps, H, occ, ms * 1e3 / it,
           24.0 * n * double(n) / (ms * 1e-3 / it) / 1e9);
    return 0;
}

template <int D>
int run_ldg(const double* x, const double* b, double* out, int64_t pitch, int n, int H, int warps, cudaEvent_t e0,
            cudaEvent_t e1) {
    const int C = 128;
    const int nstrip = (n + (C - 8) - 1) / (C - 8);
    dim3 grid((nstrip + warps - 1) / warps, (n + H - 1) / H);
    ldg_stream<D><<<grid, 32 * warps>>>(x, b, out, pitch, nstrip, n, H, C);
    CK(cudaEventRecord(e0));
    const int it = 10;
    for (int i = 0; i < it; ++i) ldg_stream<D><<<grid, 32 * warps>>>(x, b, out, pitch, nstrip, n, H, C);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("ldg D=%d warps=%d H=%4d: %7.1f us  %6.0f GB/s\n", D, warps, H, ms * 1e3 / it,
           24.0 * n * double(n) / (ms * 1e-3 / it) / 1e9);
    return 0;
}

int main() {
    const int n = 4096;
    const int64_t pitch = 4096 + 64;
    const size_t bytes = size_t(pitch) * (n + 16) * 8;
    double *x, *b, *o;
    CK(cudaMalloc(&x, bytes));
    CK(cudaMalloc(&b, bytes));
    CK(cudaMalloc(&o, bytes));
    cudaMemset(x, 0, bytes), cudaMemset(b, 0, bytes), cudaMemset(o, 0, bytes);
    double* xo = x + 8 * pitch;
    double* bo = b + 8 * pitch;
    double* oo = o + 8 * pitch;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    for (int H : {64, 128, 256}) {
        run_tma<128, 4>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_tma<128, 6>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_tma<128, 8>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_tma<128, 12>(xo, bo, oo, pitch, n, H, 2, e0, e1);
        run_tma<264, 8>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_tma<520, 4>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_tma<520, 8>(xo, bo, oo, pitch, n, H, 2, e0, e1);
        run_ldg<2>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_ldg<4>(xo, bo, oo, pitch, n, H, 4, e0, e1);
        run_ldg<8>(xo, bo, oo, pitch, n, H, 4, e0, e1);
    }
    // cudaMemcpy D2D reference
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 10; ++i) cudaMemcpyAsync(o, x, bytes, cudaMemcpyDeviceToDevice);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("memcpy D2D %.1f MB: %.0f GB/s (read+write)\n", bytes / 1e6, 2.0 * bytes / (ms * 1e-3 / 10) / 1e9);
    return 0;
}

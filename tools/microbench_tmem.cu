// microbench_tmem.cu — dependent-load latency of tcgen05.ld vs ld.shared on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_tmem.cu && /tmp/mb
#include <cstdio>
#include <cstdint>

__global__ void lat(long long* out, int n) {
    __shared__ uint32_t tbase;
    __shared__ double sm[1024];
    const int warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) sm[k] = 0.0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            uint32_t(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = tbase + (uint32_t(32 * (warp & 3)) << 16);
    if (warp == 0) {
        for (int c = 0; c < 512; c += 2) asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(tq + c), "r"(0), "r"(0));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        // dependent TMEM load chain
        uint32_t col = 0, lo, hi;
        long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(tq + col));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            col = (col + 2 + lo) & 511;
        }
        long long t1 = clock64();
        // dependent smem load chain
        int idx = threadIdx.x;
        double acc = 0;
        long long t2 = clock64();
        for (int i = 0; i < n; ++i) {
            double v = sm[idx];
            acc += v;
            idx = (idx + 32 + int(v)) & 1023;
        }
        long long t3 = clock64();
        // dependent DDIV chain
        double x = 1.0 + acc;
        long long t4 = clock64();
        for (int i = 0; i < n; ++i) x = (x + 1.0) / -3.0;
        long long t5 = clock64();
        if (threadIdx.x == 0) {
            out[0] = (t1 - t0) / n;
            out[1] = (t3 - t2) / n;
            out[2] = (t5 - t4) / n;
            out[3] = (long long)(x * 1e-300) + col;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

__global__ void bar_lat(long long* out, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
}

int main() {
    long long* d;
    long long h[4];
    cudaMalloc(&d, 64);
    lat<<<1, 128>>>(d, 1000);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: tcgen05.ld+wait %lld, ld.shared %lld, fp64 add+div %lld\n", h[0], h[1], h[2]);
    for (int t : {128, 512, 1024}) {
        bar_lat<<<1, t>>>(d, 1000);
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads with %d threads: %lld cycles\n", t, h[0]);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

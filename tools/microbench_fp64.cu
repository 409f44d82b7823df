// Dependent-latency microbenchmarks (one warp): DADD, DMUL, DFMA, FADD, LDS.64, BAR.SYNC.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 0.5;
    __syncthreads();
    double x = a, y = b;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) { x = x * y; x = x * y; x = x * y; x = x * y; }
    long long t2 = clock64();
    float f = float(a), g = float(b);
    for (int i = 0; i < n; ++i) { f = f + g; f = f + g; f = f + g; f = f + g; }
    long long t3 = clock64();
    int idx = threadIdx.x & 7;
    for (int i = 0; i < n; ++i) { idx = int(sm[idx]) & 7; idx = int(sm[idx]) & 7; idx = int(sm[idx]) & 7; idx = int(sm[idx]) & 7; }
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
    long long t5 = clock64();
    // independent DADD throughput, 8 chains
    double c0 = a, c1 = a, c2 = a, c3 = a, c4 = a, c5 = a, c6 = a, c7 = a;
    for (int i = 0; i < n; ++i) { c0 += y; c1 += y; c2 += y; c3 += y; c4 += y; c5 += y; c6 += y; c7 += y; }
    long long t6 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    }
    out[threadIdx.x] = x + f + idx + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
    const int n = 4096;
    for (int th : {32, 128, 160, 320}) {
        lat<<<1, th>>>(out, cyc, 1.0, 1e-9, n);
        cudaDeviceSynchronize();
        printf("threads %d: DADD %.1f  DMUL %.1f  FADD %.1f  LDS->cvt chain %.1f  BAR %.1f  DADDx8 indep %.2f cyc/op\n", th,
               cyc[0] / (4.0 * n), cyc[1] / (4.0 * n), cyc[2] / (4.0 * n), cyc[3] / (4.0 * n), cyc[4] / (4.0 * n),
               cyc[5] / (8.0 * n));
    }
    // many warps per SM: throughput of the 8-chain loop
    lat<<<148, 1024>>>(out, cyc, 1.0, 1e-9, n);
    cudaDeviceSynchronize();
    printf("1024 thr/SM: DADDx8 indep %.2f cyc/op per warp\n", cyc[5] / (8.0 * n));
    return 0;
}

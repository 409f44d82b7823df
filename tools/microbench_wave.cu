// Wavefront-step latency microbenchmark: one CTA, `act` active warps each doing
// one coarse cell pair (9-point update + residual from shared memory) per step,
// then a CTA barrier. Prints cycles per step for a few variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/microbench_wave.cu -o tools/mb_wave
#include <cstdio>
#include <cuda_runtime.h>

constexpr int P = 131;  // row pitch (3 mod 16)

__device__ __forceinline__ double div_m3(double a) {
    constexpr double y = -1.0 / 3.0;
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, -3.0, a);
    return __fma_rn(r, y, q);
}

template <int MODE>
__global__ void wave(double* out, long long* cyc, int steps, int act) {
    extern __shared__ double xs[];
    for (int i = threadIdx.x; i < 130 * P; i += blockDim.x) xs[i] = 0.001 * (i % 97);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int J = 1 + 32 * (warp & 3) + lane;
    const int rowo = J * P + 1;
    const bool on = warp < act;
    double lmax = 0.0;
    const long long t0 = clock64();
    for (int tau = 0; tau < steps; ++tau) {
        if (on) {
            const int Iu = ((tau - 2 * J) & 127) | 1, Ir = ((tau - 4 - 2 * J) & 127) | 1;
            const double* pu = xs + rowo + Iu;
            const double* pr = xs + rowo + Ir;
            if (MODE == 0) {  // update + residual, interleaved
                const double e = pu[1], w = pu[-1], n = pu[P], s = pu[-P], ne = pu[P + 1], nw = pu[P - 1],
                             se = pu[1 - P], sw = pu[-1 - P];
                const double rc = pr[0], re = pr[1], rw = pr[-1], rn = pr[P], rs = pr[-P], rne = pr[P + 1],
                             rnw = pr[P - 1], rse = pr[1 - P], rsw = pr[-1 - P];
                double acc = 0.0;
                acc += 0.5 * e; acc += 0.5 * w; acc += 0.5 * n; acc += 0.5 * s;
                acc += 0.25 * ne; acc += 0.25 * nw; acc += 0.25 * se; acc += 0.25 * sw;
                double ra = -3.0 * rc;
                ra += 0.5 * re; ra += 0.5 * rw; ra += 0.5 * rn; ra += 0.5 * rs;
                ra += 0.25 * rne; ra += 0.25 * rnw; ra += 0.25 * rse; ra += 0.25 * rsw;
                xs[rowo + Iu] = div_m3(0.1 - acc);
                lmax = fmax(lmax, fabs(0.1 - ra));
            } else if (MODE == 2 || MODE == 3) {  // pair with per-lane weights from shared memory
                int off = 129 * P + 1;  // class table row (10 doubles, 16-byte aligned)
                if (MODE == 3 && lane == 0) off += 10 * (int(xs[128 * P + (Iu & 7)]) & 1);
                const double2* wp = reinterpret_cast<const double2*>(xs + off);
                const double2 w01 = wp[0], w23 = wp[1], w45 = wp[2], w67 = wp[3], w89 = wp[4];
                const double e = pu[1], w = pu[-1], n = pu[P], s = pu[-P], ne = pu[P + 1], nw = pu[P - 1],
                             se = pu[1 - P], sw = pu[-1 - P];
                const double rc = pr[0], re = pr[1], rw = pr[-1], rn = pr[P], rs = pr[-P], rne = pr[P + 1],
                             rnw = pr[P - 1], rse = pr[1 - P], rsw = pr[-1 - P];
                const double2* wq = reinterpret_cast<const double2*>(xs + off + 20);
                const double2 v01 = wq[0], v23 = wq[1], v45 = wq[2], v67 = wq[3], v89 = wq[4];
                double acc = 0.0;
                acc += w01.y * e; acc += w23.x * w; acc += w23.y * n; acc += w45.x * s;
                acc += w45.y * ne; acc += w67.x * nw; acc += w67.y * se; acc += w89.x * sw;
                double ra = v01.x * rc;
                ra += v01.y * re; ra += v23.x * rw; ra += v23.y * rn; ra += v45.x * rs;
                ra += v45.y * rne; ra += v67.x * rnw; ra += v67.y * rse; ra += v89.x * rsw;
                const double num = 0.1 - acc;
                const double q = __dmul_rn(num, w89.y);
                const double r = __fma_rn(-q, w01.x, num);
                xs[rowo + Iu] = __fma_rn(r, w89.y, q);
                lmax = fmax(lmax, fabs(0.1 - ra));
            } else {  // update only
                const double e = pu[1], w = pu[-1], n = pu[P], s = pu[-P], ne = pu[P + 1], nw = pu[P - 1],
                             se = pu[1 - P], sw = pu[-1 - P];
                double acc = 0.0;
                acc += 0.5 * e; acc += 0.5 * w; acc += 0.5 * n; acc += 0.5 * s;
                acc += 0.25 * ne; acc += 0.25 * nw; acc += 0.25 * se; acc += 0.25 * sw;
                xs[rowo + Iu] = div_m3(0.1 - acc);
            }
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = lmax;
}

__global__ void barrier_only(long long* cyc, int steps) {
    const long long t0 = clock64();
    for (int tau = 0; tau < steps; ++tau) __syncthreads();
    if (threadIdx.x == 0) cyc[0] = clock64() - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    const int steps = 4000;
    const size_t smem = 130 * P * sizeof(double);
    cudaFuncSetAttribute(wave<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(wave<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(wave<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(wave<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int threads : {512}) {
        barrier_only<<<1, threads>>>(cyc, steps);
        cudaDeviceSynchronize();
        printf("threads %d barrier only: %.1f cycles/step\n", threads, double(cyc[0]) / steps);
        for (int act : {1, 4, 8, 16}) {
            wave<0><<<1, threads, smem>>>(out, cyc, steps, act);
            cudaDeviceSynchronize();
            const double c0 = double(cyc[0]) / steps;
            wave<1><<<1, threads, smem>>>(out, cyc, steps, act);
            cudaDeviceSynchronize();
            const double c1 = double(cyc[0]) / steps;
            wave<2><<<1, threads, smem>>>(out, cyc, steps, act);
            cudaDeviceSynchronize();
            const double c2 = double(cyc[0]) / steps;
            wave<3><<<1, threads, smem>>>(out, cyc, steps, act);
            cudaDeviceSynchronize();
            printf("threads %d active warps %2d: pair %.1f  update-only %.1f  smem-weights %.1f  +class %.1f\n", threads,
                   act, c0, c1, c2, double(cyc[0]) / steps);
        }
    }
    return 0;
}

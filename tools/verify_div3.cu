// verify_div3.cu — check that Markstein's correction reproduces IEEE division by
// a constant bit for bit: y = RN(1/b); q = RN(a y); r = RN(a - b q) (exact, FMA);
// q' = RN(q + r y). Compares against __ddiv_rn on random doubles (random
// significands over a wide exponent range, plus random bit patterns).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/vd tools/verify_div3.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double div_const(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    return __fma_rn(r, y, q);
}

__device__ __forceinline__ uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void check(double b, double y, long long per_thread, unsigned long long* bad, double* example, int mode) {
    uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 0x1234567ull + 77 + mode;
    unsigned long long nb = 0;
    for (long long k = 0; k < per_thread; ++k) {
        uint64_t u = splitmix(s);
        double a;
        if (mode == 0) {  // significand random, exponent in [-200, 200]
            const uint64_t e = uint64_t(1023 - 200 + (splitmix(s) % 401));
            u = (u & 0x800FFFFFFFFFFFFFull) | (e << 52);
            a = __longlong_as_double((long long)u);
        } else {  // raw bit patterns (skip NaN / inf / subnormal ranges)
            const uint64_t e = (u >> 52) & 0x7FF;
            if (e < 60 || e > 2000) continue;
            a = __longlong_as_double((long long)u);
        }
        const double want = __ddiv_rn(a, b);
        const double got = div_const(a, b, y);
        if (__double_as_longlong(want) != __double_as_longlong(got)) {
            ++nb;
            example[0] = a;
        }
    }
    atomicAdd(bad, nb);
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMalloc(&bad, 8);
    cudaMalloc(&ex, 8);
    const double divisors[] = {-3.0, 3.0, 5.0, 6.0, 7.0, -4.0, -6.0, -5.0, -7.0, -12.0};
    for (double b : divisors) {
        for (int mode = 0; mode < 2; ++mode) {
            cudaMemset(bad, 0, 8);
            const double y = 1.0 / b;  // host RN(1/b)
            check<<<148 * 8, 256>>>(b, y, 2000, bad, ex, mode);
            unsigned long long h = 0;
            double e = 0;
            cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&e, ex, 8, cudaMemcpyDeviceToHost);
            printf("b=%g mode=%d samples=%.2e mismatches=%llu%s\n", b, mode, 148.0 * 8 * 256 * 2000, h,
                   h ? " (counterexample found)" : "");
            if (h) printf("   e.g. a=%.17g\n", e);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

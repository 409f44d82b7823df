// L2 hop latency between SMs: two CTAs (on different SMs) ping-pong a 16-byte
// LL word (4-byte data + 4-byte tag per 8 bytes, as coarse_rw.cu's mailboxes)
// `n` times; prints ns per one-way hop for each store / load flavour.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_l2hop tools/microbench_l2hop.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kSt, int kLd>
__device__ __forceinline__ void st4(uint4* p, unsigned v, unsigned t) {
    if (kSt == 0) asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v), "r"(t), "r"(v), "r"(t) : "memory");
    else if (kSt == 1) asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v), "r"(t), "r"(v), "r"(t) : "memory");
    else asm volatile("st.release.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v), "r"(t), "r"(v), "r"(t) : "memory");
}
template <int kLd>
__device__ __forceinline__ uint4 ld4(const uint4* p) {
    uint4 u;
    if (kLd == 0) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p) : "memory");
    else if (kLd == 1) asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p) : "memory");
    return u;
}

template <int kSt, int kLd>
__global__ void pingpong(uint4* box, int n, long long* out) {
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x, other = 1 - me;
    long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (unsigned k = 1; k <= unsigned(n); ++k) {
        if (me == 0) {
            st4<kSt, kLd>(box + other, k, k);
            uint4 u;
            do u = ld4<kLd>(box + me); while (u.y != k || u.w != k);
        } else {
            uint4 u;
            do u = ld4<kLd>(box + me); while (u.y != k || u.w != k);
            st4<kSt, kLd>(box + other, k, k);
        }
    }
    long long t1 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (me == 0) out[0] = t1 - t0;
}

template <int kSt, int kLd>
void run(const char* name, uint4* box, long long* d_out, int n) {
    cudaMemset(box, 0, 2 * sizeof(uint4) * 64);
    pingpong<kSt, kLd><<<2, 32>>>(box, n, d_out);
    long long ns = 0;
    cudaMemcpy(&ns, d_out, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f ns per hop\n", name, double(ns) / (2.0 * n));
}

int main() {
    uint4* box;
    long long* out;
    cudaMalloc(&box, 2 * sizeof(uint4) * 64);
    cudaMalloc(&out, sizeof(long long));
    const int n = 20000;
    run<0, 0>("st.volatile / ld.volatile", box, out, n);
    run<1, 1>("st.relaxed / ld.relaxed", box, out, n);
    run<2, 2>("st.release / ld.acquire", box, out, n);
    run<0, 0>("st.volatile / ld.volatile", box, out, n);
    return 0;
}

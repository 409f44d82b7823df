// Cluster step-synchronisation microbenchmark: a cluster of C CTAs x 512 threads
// runs `steps` empty steps ended by
//   0: cg cluster.sync()
//   1: split barrier.cluster arrive.release / wait.acquire
//   2: __syncthreads + thread 0 arrives on both neighbours' mbarriers (one per
//      neighbour and step parity), all threads wait on their own
//   3: __syncthreads + release-store flags into the neighbours, thread 0 polls
//      (acquire), __syncthreads
// Prints cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench_clsync.cu -o tools/mb_clsync
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void clsync(long long* cyc, int steps) {
    __shared__ __align__(8) unsigned long long bar[2][2];  // [neighbour: 0 south, 1 north][parity]
    __shared__ unsigned flag[2];
    cg::cluster_group cl = cg::this_cluster();
    const int c = int(cl.block_rank()), C = int(cl.num_blocks());
    const bool has_s = c > 0, has_n = c + 1 < C;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i)
            for (int p = 0; p < 2; ++p)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i][p])));
        flag[0] = flag[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    cl.sync();
    // remote addresses: my arrival for the south neighbour goes to its "north" barrier, etc.
    uint32_t rs[2] = {0, 0}, rn[2] = {0, 0};
    for (int p = 0; p < 2; ++p) {
        if (has_s) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rs[p]) : "r"(smem_u32(&bar[1][p])), "r"(c - 1));
        if (has_n) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rn[p]) : "r"(smem_u32(&bar[0][p])), "r"(c + 1));
    }
    unsigned* fs = has_s ? cl.map_shared_rank(&flag[1], c - 1) : nullptr;
    unsigned* fn = has_n ? cl.map_shared_rank(&flag[0], c + 1) : nullptr;
    const long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        if (MODE == 0) {
            cl.sync();
        } else if (MODE == 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else if (MODE == 2) {
            const int p = s & 1;
            const uint32_t ph = uint32_t((s >> 1) & 1);
            __syncthreads();
            if (threadIdx.x == 0) {
                if (has_s) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rs[p]) : "memory");
                if (has_n) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rn[p]) : "memory");
            }
            for (int i = 0; i < 2; ++i) {
                if ((i == 0 && !has_s) || (i == 1 && !has_n)) continue;
                uint32_t done = 0;
                while (!done)
                    asm volatile(
                        "{ .reg .pred q; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                        : "=r"(done)
                        : "r"(smem_u32(&bar[i][p])), "r"(ph)
                        : "memory");
            }
        } else {
            const unsigned n = unsigned(s + 1);
            __syncthreads();
            if (threadIdx.x == 0) {
                if (fs) asm volatile("st.release.cluster.u32 [%0], %1;" ::"l"(fs), "r"(n) : "memory");
                if (fn) asm volatile("st.release.cluster.u32 [%0], %1;" ::"l"(fn), "r"(n) : "memory");
                unsigned a = 0, b = 0;
                do {
                    if (has_s) asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(a) : "l"(&flag[0]) : "memory");
                    else a = n;
                    if (has_n) asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(b) : "l"(&flag[1]) : "memory");
                    else b = n;
                } while (a < n || b < n);
            }
            __syncthreads();
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0 && c == 0) cyc[0] = t1 - t0;
    cl.sync();
}

template <int MODE>
double run(long long* cyc, int C, int steps) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(clsync<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, clsync<MODE>, cyc, steps);
    if (e != cudaSuccess) return -1;
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    return double(cyc[0]) / steps;
}

int main() {
    long long* cyc;
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    const int steps = 4000;
    for (int C : {2, 4, 8, 16})
        printf("C=%2d  cluster.sync %.0f  split %.0f  mbarrier %.0f  flags %.0f cycles/step\n", C, run<0>(cyc, C, steps),
               run<1>(cyc, C, steps), run<2>(cyc, C, steps), run<3>(cyc, C, steps));
    return 0;
}

// Barrier latency microbenchmark: __syncthreads and cluster.sync() per step,
// for 1024-thread CTAs in clusters of 1..16 (one CTA per SM).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void cl_sync(long long* out, int n, int mode) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double s[1024];
    s[threadIdx.x] = threadIdx.x;
    cl.sync();
    long long t0 = clock64();
    double acc = 0;
    for (int i = 0; i < n; ++i) {
        if (mode == 0) __syncthreads();
        else if (mode == 1) cl.sync();
        else {  // cluster barrier + one DSMEM read from the neighbour
            double* peer = cl.map_shared_rank(s, (cl.block_rank() + 1) % cl.num_blocks());
            acc += peer[threadIdx.x];
            cl.sync();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (acc == -1) out[1] = 1;
}

int main() {
    long long* out;
    cudaMallocManaged(&out, 16);
    const int n = 20000;
    for (int C : {1, 2, 4, 8, 16}) {
        cudaFuncSetAttribute(cl_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int threads : {256, 1024}) {
            for (int mode = 0; mode < 3; ++mode) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(C);
                cfg.blockDim = dim3(threads);
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeClusterDimension;
                a[0].val.clusterDim.x = C, a[0].val.clusterDim.y = 1, a[0].val.clusterDim.z = 1;
                cfg.attrs = a, cfg.numAttrs = 1;
                cudaError_t e = cudaLaunchKernelEx(&cfg, cl_sync, out, n, mode);
                cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("C=%d err %s\n", C, cudaGetErrorString(e)); continue; }
                printf("C=%2d threads=%4d %-22s %7.1f cycles/step\n", C, threads,
                       mode == 0 ? "__syncthreads" : (mode == 1 ? "cluster.sync" : "dsmem load + cluster.sync"),
                       double(out[0]) / n);
            }
        }
    }
    return 0;
}

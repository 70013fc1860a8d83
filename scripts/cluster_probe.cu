// Cost of a thread-block-cluster barrier (cg::this_cluster().sync()) and of a
// DSMEM read after it, per iteration, on one B200 (256-thread CTAs, 1 CTA/SM).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k(int iters, int mode, double* out) {
    __shared__ double buf[2][256];
    cg::cluster_group cl = cg::this_cluster();
    const int r = cl.block_rank(), n = cl.num_blocks();
    double acc = 0;
    buf[0][threadIdx.x] = buf[1][threadIdx.x] = r + threadIdx.x;
    cl.sync();
    for (int it = 0; it < iters; ++it) {
        buf[it & 1][threadIdx.x] += 1.0;
        if (mode == 0) __syncthreads();
        else cl.sync();
        if (mode == 2) {
            for (int p = 0; p < n; ++p) acc += cl.map_shared_rank(&buf[it & 1][0], p)[threadIdx.x];
        }
    }
    cl.sync();
    if (acc == -1.0) out[0] = acc;
}
int main() {
    double* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int C : {1, 2, 4, 8}) for (int mode = 0; mode < 3; ++mode) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(C * 16); cfg.blockDim = dim3(256); cfg.attrs = at; cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, k, iters, mode, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("cluster %d %-26s %.3f us per iteration\n", C,
                            mode == 0 ? "__syncthreads" : mode == 1 ? "cluster.sync" : "cluster.sync + DSMEM read",
                            ms * 1e3 / iters);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}

// Microbenchmark (not product code): do DMMA (FP64 tensor pipe) and DFMA
// (FP64 vector pipe) issue concurrently on B200?  Runs warps of each kind
// alone and mixed in one CTA per SM and reports both rates.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void probe(double* out, int iters, int dmma_warps, int dfma_warps) {
    const int warp = threadIdx.x >> 5;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    double s = 0;
    if (warp < dmma_warps) {
        double c0[8], c1[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) { c0[k] = k; c1[k] = -k; }
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) dmma(c0[k], c1[k], a, b);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += c0[k] + c1[k];
    } else if (warp < dmma_warps + dfma_warps) {
        double c[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k] = k;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 16; ++k) c[k] = fma(c[k], b, a);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) s += c[k];
    }
    if (s == 12345.0) out[0] = s;
}

int main() {
    double* out; cudaMalloc(&out, 16);
    const int iters = 4096;
    int cfg[][2] = {{8, 0}, {16, 0}, {0, 8}, {0, 16}, {8, 8}, {16, 16}, {8, 16}};
    for (auto& c : cfg) {
        int threads = 32 * (c[0] + c[1]);
        probe<<<148, threads>>>(out, 16, c[0], c[1]);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<148, threads>>>(out, iters, c[0], c[1]);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double dm = 148.0 * c[0] * iters * 8 * 512, df = 148.0 * c[1] * iters * 16 * 32 * 2;
        printf("dmma warps %2d dfma warps %2d: %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n", c[0], c[1], ms,
               dm / ms / 1e9, df / ms / 1e9, (dm + df) / ms / 1e9);
    }
    return 0;
}

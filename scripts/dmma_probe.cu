// Microbenchmark (not product code): DMMA.8x8x4 throughput vs independent
// accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void probe(double* out, int iters) {
    double c0[CH], c1[CH];
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
#pragma unroll
    for (int k = 0; k < CH; ++k) { c0[k] = k; c1[k] = -k; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < CH; ++k) dmma(c0[k], c1[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += c0[k] + c1[k];
    if (s == 12345.0) out[0] = s;
}

template <int CH>
void run(int warps_per_sm, double* out) {
    const int iters = 2048;
    int threads = 32 * warps_per_sm;
    int blocks = 148;
    if (threads > 1024) { blocks = 148 * (threads / 1024); threads = 1024; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    probe<CH><<<blocks, threads>>>(out, 16);
    cudaEventRecord(a);
    probe<CH><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double dmmas = (double)blocks * threads / 32 * iters * CH;
    double tflops = dmmas * 512 / (ms * 1e-3) / 1e12;
    printf("chains=%2d warps/SM=%2d: %.2f TFLOP/s fp64 (%.3f DMMA/clk/SM @1.965GHz)\n", CH, warps_per_sm,
           tflops, dmmas / 148 / (ms * 1e-3 * 1.965e9));
}

int main() {
    double* out; cudaMalloc(&out, 16);
    for (int w : {1, 2, 4, 8, 16}) { run<1>(w, out); run<4>(w, out); run<8>(w, out); run<12>(w, out); run<16>(w, out); }
    return 0;
}

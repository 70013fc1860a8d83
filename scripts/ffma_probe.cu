// FP32 FMA throughput on one B200: scalar FFMA vs packed FFMA2 (fma.rn.f32x2),
// 8 independent chains per thread, 1024 threads/SM worth of blocks.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    unsigned long long a, b, c, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(d0), "f"(d1));
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(r));
}
template <bool PACKED>
__global__ void k(float* out, int iters, float a, float b) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-7f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (PACKED) ffma2(x[i], x[i + 1], x[i], x[i + 1], a, b);
            else { x[i] = fmaf(x[i], a, b); x[i + 1] = fmaf(x[i + 1], a, b); }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.f) out[0] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, 4);
    const int iters = 20000, threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int packed = 0; packed < 2; ++packed) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (packed) k<true><<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f);
            else k<false><<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 16 * iters * (double)threads * blocks;
            if (rep) printf("%s: %.1f TFLOP/s fp32 (%.3f ms)\n", packed ? "FFMA2" : "FFMA", flops / ms / 1e9, ms);
        }
    }
    return 0;
}

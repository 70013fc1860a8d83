// Microbenchmark (not product code): dependent-chain latency of FP64 and
// warp ops on B200, one warp, clock64 around N dependent ops.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    double x = a, y = b;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) y = y + x;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // SHFL (double) chain
    double z = x + y;
    t0 = clock64();
    for (int i = 0; i < n; ++i) z = __shfl_xor_sync(0xffffffffu, z, 1) + 1.0;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // rcp.approx.f64 chain
    double r = z;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double q; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(r)); r = q; }
    t1 = clock64();
    cyc[3] = t1 - t0;
    // LDS chain (pointer chasing in smem)
    __shared__ int sm[256];
    for (int i = threadIdx.x; i < 256; i += 32) sm[i] = (i + 1) & 255;
    __syncwarp();
    int p = threadIdx.x & 7;
    t0 = clock64();
    for (int i = 0; i < n; ++i) p = sm[p];
    t1 = clock64();
    cyc[4] = t1 - t0;
    // exact f64 division chain
    double d = r + 3.0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) d = 1.5 / d + 1.0;
    t1 = clock64();
    cyc[5] = t1 - t0;
    out[threadIdx.x] = x + y + z + r + p + d;
}

int main() {
    double* out; long long* cyc; cudaMalloc(&out, 256); cudaMallocManaged(&cyc, 64);
    const int n = 1024;
    k<<<1, 32>>>(out, cyc, 0.5, 0.999, n);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(out, cyc, 0.5, 0.999, n);
    cudaDeviceSynchronize();
    const char* nm[] = {"DFMA", "DADD", "SHFL.f64+DADD", "MUFU.RCP64H", "LDS (chase)", "f64 div + DADD"};
    for (int i = 0; i < 6; ++i) printf("%-16s %.1f cycles/op\n", nm[i], (double)cyc[i] / n);
    return 0;
}

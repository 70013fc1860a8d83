// Microbenchmark (not product code): HBM read rate for the cost build's access
// pattern — rows of E (2400 B) selected by a sorted row list.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void read_flush(const double4* __restrict__ p, size_t n, double* out) {
    double acc = 0.0;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        double4 v = p[k]; acc += v.x + v.w;
    }
    if (acc == 12345.678) out[1] = acc;
}

__global__ void read_rows(const double2* __restrict__ E, int ld2, const int* __restrict__ rows, int nrows,
                          int row2, double* out) {
    double acc = 0.0;
    const int warps = gridDim.x * (blockDim.x / 32);
    const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    for (int r = w; r < nrows; r += warps) {
        const double2* e = E + (size_t)rows[r] * ld2;
#pragma unroll 5
        for (int p = lane; p < row2; p += 32) { double2 v = __ldg(e + p); acc += v.x + v.y; }
    }
    if (acc == 12345.678) out[0] = acc;
}

int main() {
    const int V = 100000, dim = 300;
    double* E; cudaMalloc(&E, (size_t)V * dim * 8);
    cudaMemset(E, 0, (size_t)V * dim * 8);
    std::vector<int> rows;
    std::mt19937 g(1);
    for (int i = 0; i < V; ++i) if (g() % 100 < 36) rows.push_back(i);
    int* d_rows; cudaMalloc(&d_rows, rows.size() * 4);
    cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
    std::vector<int> all(V); for (int i = 0; i < V; ++i) all[i] = i;
    int* d_all; cudaMalloc(&d_all, V * 4); cudaMemcpy(d_all, all.data(), V * 4, cudaMemcpyHostToDevice);
    double* out; cudaMalloc(&out, 8);
    char* flush; cudaMalloc(&flush, 256 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode)
    for (int cfg = 0; cfg < 2; ++cfg) {
        const int* rl = cfg ? d_all : d_rows; int n = cfg ? V : (int)rows.size();
        for (int bs : {128, 256}) for (int bpsm : {2, 4, 8, 16}) {
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                if (mode == 0) cudaMemset(flush, it, 256 << 20);
                else read_flush<<<148 * 8, 256>>>((const double4*)flush, (256u << 20) / 32, out);
                cudaEventRecord(a);
                read_rows<<<148 * bpsm, bs>>>((const double2*)E, dim / 2, rl, n, dim / 2, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
            }
            double bytes = (double)n * dim * 8;
            printf("flush=%s %s rows=%d block=%d blocks/SM=%d: %.1f us  %.0f GB/s\n", mode ? "read" : "write", cfg ? "all" : "present", n, bs, bpsm, best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}

// L2 bandwidth probe (B200): streaming 128-bit reads of an L2-resident buffer
// and random row gathers (row = 160 B or 2 KB) from an L2-resident table.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/l2_probe scripts/l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stream_read(const double2* __restrict__ p, int64_t n, int reps, double* sink) {
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(p + i);
            acc += v.x + v.y;
        }
    if (acc == 12345.678) *sink = acc;
}

// each warp gathers rows of `row_bytes` at pseudo-random row ids
__global__ void gather_rows(const double2* __restrict__ t, int64_t n_rows, int row_v16, int64_t n_gathers,
                            double* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0;
    uint32_t x = 2463534242u ^ (uint32_t)warp;
    for (int64_t g = warp; g < n_gathers; g += nwarps) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        const int64_t row = x % n_rows;
        for (int v = lane; v < row_v16; v += 32) {
            double2 d = __ldg(t + row * row_v16 + v);
            acc += d.x + d.y;
        }
    }
    if (acc == 12345.678) *sink = acc;
}

// the c2 solve's access pattern: lane pair g of a warp gathers its own 160 B
// row, lane h of the pair the interleaved 16-byte chunks h, h+2, ..; U rows
// per lane pair in flight (16 U rows per warp)
template <int U>
__global__ void gather_pairs(const double2* __restrict__ t, int64_t n_rows, int64_t n_gathers,
                             double* sink) {
    const int lane = threadIdx.x & 31, g = lane >> 1, h = lane & 1;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0;
    uint32_t x = 2463534242u ^ (uint32_t)(warp * 32 + g);
    for (int64_t base = warp * 16 * U; base < n_gathers; base += nwarps * 16 * U) {
        double2 v[U][5];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            const double2* row = t + (int64_t)(x % n_rows) * 10 + h;
#pragma unroll
            for (int k = 0; k < 5; ++k) v[u][k] = __ldg(row + 2 * k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 5; ++k) acc += v[u][k].x + v[u][k].y;
    }
    if (acc == 12345.678) *sink = acc;
}

// best-case 160 B row gather: 10 consecutive lanes read one row's ten 16-byte
// chunks in one instruction (5 full sectors), 3 rows per warp-instruction,
// U instructions in flight
template <int U>
__global__ void gather_rows10(const double2* __restrict__ t, int64_t n_rows, int64_t n_gathers,
                              double* sink) {
    const int lane = threadIdx.x & 31, grp = lane / 10, c = lane % 10;
    const bool on = lane < 30;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0;
    uint32_t x = 2463534242u ^ (uint32_t)(warp * 4 + grp);
    for (int64_t base = warp * 3 * U; base < n_gathers; base += nwarps * 3 * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            v[u] = on ? __ldg(t + (int64_t)(x % n_rows) * 10 + c) : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 12345.678) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int64_t mb : {16, 32, 48, 64, 96}) {
        const int64_t bytes = mb << 20;
        double2* p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 0, bytes);
        const int64_t n = bytes / 16;
        const int reps = 20;
        for (int bpsm : {4, 8}) {
            stream_read<<<sms * bpsm, 256>>>(p, n, 2, sink);
            cudaEventRecord(a);
            stream_read<<<sms * bpsm, 256>>>(p, n, reps, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("stream  %3lld MB  %d blk/SM: %.1f TB/s\n", (long long)mb, bpsm,
                   (double)bytes * reps / (ms * 1e-3) / 1e12);
        }
        cudaFree(p);
    }
    for (int row_bytes : {160, 2048}) {
        for (int64_t mb : {16, 64, 400}) {
            const int64_t bytes = mb << 20;
            double2* t;
            cudaMalloc(&t, bytes);
            cudaMemset(t, 0, bytes);
            const int rv = row_bytes / 16;
            const int64_t n_rows = bytes / row_bytes;
            const int64_t ng = (int64_t)4 << 20;
            gather_rows<<<sms * 8, 256>>>(t, n_rows, rv, ng / 4, sink);
            cudaEventRecord(a);
            gather_rows<<<sms * 8, 256>>>(t, n_rows, rv, ng, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("gather  row %4d B  table %3lld MB: %.1f TB/s\n", row_bytes, (long long)mb,
                   (double)ng * row_bytes / (ms * 1e-3) / 1e12);
            cudaFree(t);
        }
    }
    // the c2 K-row pattern: 160 B rows, lane pairs, 16 x U rows per warp in flight
    for (int64_t mb : {16, 64}) {
        const int64_t bytes = mb << 20;
        double2* t;
        cudaMalloc(&t, bytes);
        cudaMemset(t, 0, bytes);
        const int64_t n_rows = bytes / 160;
        const int64_t ng = (int64_t)16 << 20;
        for (int wps : {16, 32, 64}) {
            for (int U : {1, 2, 4}) {
                auto run = [&](int64_t n) {
                    if (U == 1) gather_pairs<1><<<sms * wps / 8, 256>>>(t, n_rows, n, sink);
                    else if (U == 2) gather_pairs<2><<<sms * wps / 8, 256>>>(t, n_rows, n, sink);
                    else gather_pairs<4><<<sms * wps / 8, 256>>>(t, n_rows, n, sink);
                };
                run(ng / 4);
                cudaEventRecord(a);
                run(ng);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("pairs   row  160 B  table %3lld MB  warps/SM %2d  rows/pair %d: %.1f TB/s\n",
                       (long long)mb, wps, U, (double)ng * 160 / (ms * 1e-3) / 1e12);
            }
        }
        for (int wps : {16, 32, 64}) {
            for (int U : {2, 4, 8}) {
                auto run = [&](int64_t n) {
                    if (U == 2) gather_rows10<2><<<sms * wps / 8, 256>>>(t, n_rows, n, sink);
                    else if (U == 4) gather_rows10<4><<<sms * wps / 8, 256>>>(t, n_rows, n, sink);
                    else gather_rows10<8><<<sms * wps / 8, 256>>>(t, n_rows, n, sink);
                };
                run(ng / 4);
                cudaEventRecord(a);
                run(ng);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("rows10  row  160 B  table %3lld MB  warps/SM %2d  in flight %d: %.1f TB/s\n",
                       (long long)mb, wps, U, (double)ng * 160 / (ms * 1e-3) / 1e12);
            }
        }
        cudaFree(t);
    }
    return 0;
}

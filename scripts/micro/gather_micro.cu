// Random row gather bandwidth: 200-B rows (stride 50 floats) vs 256-B padded
// rows (stride 64 floats), rows visited in a random order, one warp per 32
// rows, lanes read float2 (25 lanes busy).  Prints ms and effective GB/s.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void gather(const float* __restrict__ x, uint32_t ld, const uint32_t* __restrict__ order,
                       uint64_t n, uint32_t D, double* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    double a0 = 0, a1 = 0;
    for (uint64_t r0 = w * 32; r0 < n; r0 += nw * 32) {
        const uint32_t my = r0 + lane < n ? order[r0 + lane] : 0;
        float2 v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t row = __shfl_sync(0xffffffffu, my, j);
            v[j] = (2 * lane < D) ? *reinterpret_cast<const float2*>(x + (uint64_t)row * ld + 2 * lane)
                                  : make_float2(0, 0);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) { a0 += v[j].x; a1 += v[j].y; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
}

int main() {
    const uint64_t n = 10000000;
    const uint32_t D = 50;
    std::vector<uint32_t> ord(n);
    for (uint64_t i = 0; i < n; ++i) ord[i] = (uint32_t)i;
    std::mt19937_64 g(1);
    std::shuffle(ord.begin(), ord.end(), g);
    uint32_t* d_ord; float* x; double* out;
    cudaMalloc(&d_ord, n * 4);
    cudaMalloc(&x, n * 64 * 4 + 4096);
    cudaMalloc(&out, 148 * 16 * 256 * 8);
    cudaMemset(x, 0, n * 64 * 4);
    for (int mode = 0; mode < 4; ++mode) {
        // 0: random order, stride 50; 1: random, stride 64; 2: sequential 50; 3: seq 64
        if (mode == 2) { for (uint64_t i = 0; i < n; ++i) ord[i] = (uint32_t)i; }
        cudaMemcpy(d_ord, ord.data(), n * 4, cudaMemcpyHostToDevice);
        const uint32_t ld = (mode & 1) ? 64 : 50;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
            gather<<<grid, 256>>>(x, ld, d_ord, n, D, out);
            cudaEventRecord(a);
            for (int it = 0; it < 5; ++it) gather<<<grid, 256>>>(x, ld, d_ord, n, D, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
            printf("mode %d (%s, ld %u) grid %d: %.3f ms, useful %.0f GB/s\n", mode,
                   mode < 2 ? "random" : "seq", ld, grid, ms, n * D * 4 / ms / 1e6);
        }
    }
    return 0;
}

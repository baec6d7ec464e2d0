// Random 200-B row gather over a large array: is the c4 K2 gather TLB-bound?
// 1e7 rows picked from N_total rows (sorted pick = a rho selection), visited
// (a) in a random global order, (b) random within windows of 131072 picks,
// (c) in pick order.  Same warp structure as gather_micro.cu.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void gather(const float* __restrict__ x, const uint64_t* __restrict__ order, uint64_t n,
                       uint32_t D, double* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    double a0 = 0, a1 = 0;
    for (uint64_t r0 = w * 32; r0 < n; r0 += nw * 32) {
        const uint64_t my = r0 + lane < n ? order[r0 + lane] : 0;
        float2 v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint64_t row = __shfl_sync(0xffffffffu, my, j);
            v[j] = (2 * lane < D) ? *reinterpret_cast<const float2*>(x + row * D + 2 * lane)
                                  : make_float2(0, 0);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) { a0 += v[j].x; a1 += v[j].y; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
}

int main() {
    const uint32_t D = 50;
    const uint64_t m = 10000000;
    std::mt19937_64 g(1);
    for (uint64_t total : {10000000ull, 100000000ull}) {
        float* x; uint64_t* d_ord; double* out;
        cudaMalloc(&x, total * D * 4 + 4096);
        cudaMemset(x, 0, total * D * 4);
        cudaMalloc(&d_ord, m * 8);
        cudaMalloc(&out, 148 * 8 * 256 * 8);
        std::vector<uint64_t> pick(m);
        if (total == m) { for (uint64_t i = 0; i < m; ++i) pick[i] = i; }
        else { for (uint64_t i = 0; i < m; ++i) pick[i] = i * (total / m) + (g() % (total / m)); }
        for (int mode = 0; mode < 3; ++mode) {
            std::vector<uint64_t> ord = pick;
            if (mode == 0) std::shuffle(ord.begin(), ord.end(), g);
            if (mode == 1)
                for (uint64_t c = 0; c < m; c += 131072)
                    std::shuffle(ord.begin() + c, ord.begin() + std::min(m, c + 131072), g);
            cudaMemcpy(d_ord, ord.data(), m * 8, cudaMemcpyHostToDevice);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            gather<<<148 * 8, 256>>>(x, d_ord, m, D, out);
            cudaEventRecord(a);
            for (int it = 0; it < 5; ++it) gather<<<148 * 8, 256>>>(x, d_ord, m, D, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
            printf("array %llu rows, %s: %.3f ms (%.0f GB/s useful)\n", (unsigned long long)total,
                   mode == 0 ? "random global" : mode == 1 ? "random in 131k windows" : "pick order",
                   ms, m * D * 4 / ms / 1e6);
        }
        cudaFree(x); cudaFree(d_ord); cudaFree(out);
    }
    return 0;
}

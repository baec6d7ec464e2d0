// Microbenchmark of K1 epilogue instruction mixes (register data, no TMEM):
// cycles per value per SM for each top-2 variant.  Diagnostics only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float r; asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}

template <int V>
__global__ void __launch_bounds__(256) kern(const uint32_t* in, float* out, int iters, uint32_t one, uint32_t neg1) {
    uint32_t r[32];
    for (int k = 0; k < 32; ++k) r[k] = in[(threadIdx.x + k * 37) & 1023];
    uint32_t mask; asm volatile("mov.b32 %0, 0xFFFFFF00;" : "=r"(mask));
    float b1[4], b2[4]; uint32_t b1k[4];
    for (int s = 0; s < 4; ++s) { b1[s] = 1e30f; b2[s] = 1e30f; b1k[s] = 0x7F000000u; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int s = m & 3;
            uint32_t a = r[2 * m] ^ it, b = r[2 * m + 1] ^ it;  // defeat hoisting
            if (V == 0 || V == 1 || V == 3) {
                asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(a) : "r"(a), "r"((uint32_t)(2 * m)), "r"(mask));
                asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(b) : "r"(b), "r"((uint32_t)(2 * m + 1)), "r"(mask));
            }
            if (V == 0 || V == 2) {  // IMAD variant
                const uint32_t hi = __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b)));
                const uint32_t lo = a * one + b + hi * neg1;
                const uint32_t tt = __float_as_uint(fmaxf(__uint_as_float(b1k[s]), __uint_as_float(lo)));
                b1k[s] = b1k[s] * one + lo + tt * neg1;
                b2[s] = fmin3f(b2[s], __uint_as_float(tt), __uint_as_float(hi));
            } else if (V == 1) {  // all ALU
                const float fa = __uint_as_float(a), fb = __uint_as_float(b);
                const float hi = fmaxf(fa, fb), lo = fminf(fa, fb);
                const float tt = fmaxf(b1[s], lo);
                b1[s] = fminf(b1[s], lo);
                b2[s] = fmin3f(b2[s], tt, hi);
            } else if (V == 3) {  // min only (lower bound)
                b1[s] = fmin3f(b1[s], __uint_as_float(a), __uint_as_float(b));
            } else if (V == 4) {  // pass-2 style: count/idx of values <= lim
                const float lim = b2[0];
                if (__uint_as_float(a) <= lim) { b1k[1] = 2 * m; b1k[2] += one; }
                if (__uint_as_float(b) <= lim) { b1k[1] = 2 * m + 1; b1k[2] += one; }
            }
        }
    }
    long long t1 = clock64();
    float acc = 0;
    for (int s = 0; s < 4; ++s) acc += b1[s] + b2[s] + __uint_as_float(b1k[s]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}

int main() {
    uint32_t* in; float* out;
    cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, (1 << 20) * 4 + 64);
    uint32_t h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 0x3F800000u + i * 7919u % 100000u;
    cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
    const int iters = 2000;
    for (int warps = 2; warps <= 2; warps *= 2) {
        const int threads = warps * 32 * 4;  // warps per SMSP x 4 SMSPs
        if (threads > 1024) break;
        for (int v = 0; v < 5; ++v) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto k = v == 0 ? kern<0> : v == 1 ? kern<1> : v == 2 ? kern<2> : v == 3 ? kern<3> : kern<4>;
            k<<<148, threads>>>(in, out, 10, 1u, 0xFFFFFFFFu);
            cudaEventRecord(e0);
            k<<<148, threads>>>(in, out, iters, 1u, 0xFFFFFFFFu);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            float cyc; cudaMemcpy(&cyc, out + (1 << 20), 4, cudaMemcpyDeviceToHost);
            const int wps = threads / 4 / 32;
            printf("warps/SMSP=%d variant=%d: %.2f SMSP cycles per warp-pair (2 values x 32 lanes), %.3f ms\n",
                   wps, v, cyc / ((double)iters * 16 * wps), ms);
        }
    }
    return 0;
}

// k_guard.cu — the accumulation-term guard of the reference, exactly.
//
// The reference quantises every term of an epoch (accumulate,
// trainer.hpp:318-336; quantize_term, accum.hpp:34-38) and throws
// "numerical fault: accumulation term out of range (|term| >= 2^22)" when
//     |h[b][j]|  >= 2^22        (add_h)   or
//     |fl(fl(eta h[b][j]) fl(x_ik - w_jk))| >= 2^22   (add_u)
// for any row i (BMU b) of the selection, node j and feature k.  The engine
// never forms those N K d terms.  It checks, on the device:
//   1. a cheap bound: |eta| max|h| (max||x|| + max||w||) < 2^22 and
//      max|h| < 2^22 — true for any sane data, and then nothing else runs;
//   2. only when the bound fails, the exact test: per BMU node b and feature
//      k the smallest and largest x_ik over its rows (one pass over the
//      rows), then for every (b, j, k) the reference's term at both extremes.
//      Every operation is monotone in x (IEEE rounding is), so the largest
//      |term| over a node's rows is attained at one of them: the test fires
//      exactly when the reference would throw, and for h only over the rows
//      b some row maps to.
// The codebook is the epoch's own (before apply_update), like the reference's.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace cg = cooperative_groups;

namespace tsom {

namespace {

constexpr double kTermLimit = 4194304.0;  // 2^22, accum.hpp:30

// float -> uint32 whose unsigned order is the float order
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// the cheap bound, with max|h| folded from the kHmaxParts block maxima
// (every block of the caller evaluates it identically)
__device__ __forceinline__ bool cheap_bound_over(const float* x2max, const float* w2max,
                                                 const double* hpart, double eta) {
    __shared__ double s_h[32];
    double h = 0.0;
    for (unsigned k = threadIdx.x; k < kHmaxParts; k += blockDim.x) {
        const double v = hpart[k];
        h = v > h || v != v ? v : h;
    }
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, h, o);
        h = v > h || v != v ? v : h;
    }
    if ((threadIdx.x & 31) == 0) s_h[threadIdx.x >> 5] = h;
    __syncthreads();
    h = 0.0;
    for (unsigned w = 0; w < (blockDim.x + 31) / 32; ++w) h = s_h[w] > h || s_h[w] != s_h[w] ? s_h[w] : h;
    __syncthreads();
    const double bound = fabs(eta) * h * (sqrt((double)*x2max) + sqrt((double)*w2max));
    return !(h < kTermLimit && bound < kTermLimit);  // NaN anywhere: over
}

__global__ void __launch_bounds__(256) k_infl_absmax(const double* __restrict__ infl, size_t n,
                                                     double* __restrict__ hpart) {
    double m = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double a = fabs(infl[i]);
        m = a > m || a != a ? a : m;  // NaN wins (it fails every comparison the guard makes)
    }
    block_max_to(m, hpart);
}

// The flags carry the invocation's tag (a counter the host passes) instead of
// a boolean, so nothing is spent clearing them: flag[0] == tag: the cheap
// bound failed this time; flag[1] == tag: a term the reference would reject.
// mn / mx / seen are all zero between invocations (phase 3 restores that
// after a use).  One cooperative launch: every block evaluates the cheap
// bound first and, in the common case, returns at once (uniformly, so the
// grid barriers are never reached).
__global__ void __launch_bounds__(256) k_term_guard(
    const float* __restrict__ x, uint32_t ldx, const uint32_t* __restrict__ sel, uint64_t n,
    const uint32_t* __restrict__ bmu, const float* __restrict__ w,
    const double* __restrict__ infl, uint32_t P, uint32_t D, double eta,
    const float* __restrict__ x2max, const float* __restrict__ w2max,
    const double* __restrict__ hmax, uint32_t tag, uint32_t* __restrict__ flag,
    uint32_t* __restrict__ mn, uint32_t* __restrict__ mx, uint32_t* __restrict__ seen,
    int* __restrict__ dead, uint32_t epoch) {
    if (!cheap_bound_over(x2max, w2max, hmax, eta)) return;
    cg::grid_group grid = cg::this_grid();
    const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t ts = (uint64_t)gridDim.x * blockDim.x;
    if (t0 == 0) flag[0] = tag;
    bool bad_all = false;
    if (!x) {
        bad_all = true;  // no resident rows (streamed): the bound decides alone
    } else {
        // phase 1: per BMU node and feature, the extremes of the rows
        for (uint64_t e = t0; e < n * D; e += ts) {
            const uint64_t i = e / D;
            const uint32_t k = (uint32_t)(e - i * D);
            const uint32_t b = bmu[i];
            const float v = x[(sel ? (uint64_t)sel[i] : i) * ldx + k];
            // min as the max of the complemented order key (both start at 0)
            atomicMax(mx + (size_t)b * D + k, f2ord(v));
            atomicMax(mn + (size_t)b * D + k, ~f2ord(v));
            if (k == 0) seen[b] = 1u;
        }
        grid.sync();
        // phase 2: the reference's term at both extremes, every (b, j, k)
        for (uint64_t e = t0; e < (uint64_t)P * P; e += ts) {
            const uint32_t b = (uint32_t)(e / P), j = (uint32_t)(e - (uint64_t)b * P);
            if (!seen[b]) continue;
            const double h = infl[(size_t)b * P + j];
            bool bad = !(fabs(h) < kTermLimit);
            const double eh = __dmul_rn(eta, h);
            for (uint32_t k = 0; k < D && !bad; ++k) {
                const double wk = (double)w[(size_t)j * D + k];
                const double t1 = __dmul_rn(eh, __dsub_rn((double)ord2f(mx[(size_t)b * D + k]), wk));
                const double t2 = __dmul_rn(eh, __dsub_rn((double)ord2f(~mn[(size_t)b * D + k]), wk));
                bad = !(fabs(t1) < kTermLimit) || !(fabs(t2) < kTermLimit);
            }
            if (bad) flag[1] = tag;
        }
        grid.sync();
        // phase 3: back to all-zero extremes
        for (uint64_t e = t0; e < (uint64_t)P * D; e += ts) {
            mn[e] = 0u;
            mx[e] = 0u;
            if (e < P) seen[e] = 0u;
        }
    }
    if (bad_all && t0 == 0) flag[1] = tag;
    // a violation of this epoch fails a multi-epoch run before its update
    if (dead && t0 == 0) {
        __threadfence();
        if (dead[0] == 0 && (bad_all || flag[1] == tag)) {
            dead[0] = (int)epoch + 1;
            dead[1] = 2;
        }
    }
}

}  // namespace

void launch_infl_absmax(const double* infl, size_t n, double* hpart, cudaStream_t st) {
    TSOM_LAUNCH(k_infl_absmax<<<kHmaxParts, 256, 0, st>>>(infl, n, hpart));
}

cudaError_t launch_term_guard(const float* x, uint32_t ldx, const uint32_t* sel, uint64_t n,
                       const uint32_t* bmu, const float* w, const double* infl, uint32_t P,
                       uint32_t D, double eta, const float* x2max, const float* w2max,
                       const double* hmax, uint32_t tag, GuardScratch g, int sm_count,
                       cudaStream_t st, int* dead, uint32_t epoch) {
    void* args[] = {(void*)&x,     (void*)&ldx,   (void*)&sel,   (void*)&n,    (void*)&bmu,
                    (void*)&w,     (void*)&infl,  (void*)&P,     (void*)&D,    (void*)&eta,
                    (void*)&x2max, (void*)&w2max, (void*)&hmax,  (void*)&tag,  (void*)&g.flag,
                    (void*)&g.mn,  (void*)&g.mx,  (void*)&g.seen, (void*)&dead, (void*)&epoch};
    ++g_launches;
    return cudaLaunchCooperativeKernel((const void*)k_term_guard, dim3((unsigned)sm_count * 2),
                                       dim3(256), args, 0, st);
}

size_t guard_scratch_words(uint32_t P, uint32_t D) { return 2 + (size_t)P + 2 * (size_t)P * D; }

GuardScratch guard_scratch(uint32_t* base, uint32_t P, uint32_t D) {
    GuardScratch g;
    g.flag = base;
    g.seen = base + 2;
    g.mn = g.seen + P;
    g.mx = g.mn + (size_t)P * D;
    return g;
}

}  // namespace tsom

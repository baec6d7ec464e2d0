// k_smooth.cu — K3 neighbourhood smoothing + update, influence, synthetic data.
//
//   U_j = eta * ( sum_b h[b][j] S_b  -  w_j * sum_b h[b][j] c_b )
//   H_j = sum_b h[b][j] c_b
// (trainer.hpp:318-336 regrouped by BMU; h[b][j] = influence row b, :326),
// then apply_update (trainer.hpp:341-369).  All in FP64: the GEMM is
// P x P x (d+1) = 1.07e8 flop per epoch at P=1024, d=50 — noise next to K1.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <climits>
#include <cstdint>

#include "engine.h"

namespace tsom {

// H_j = sum_b infl[b][j] c_b: block = 32 nodes x 8 b-slices, fixed-order fold.
// Two values per node:
//   Hx[j] — in FP64, the denominator's exact value, for U's  - w_j H_j  term;
//   H[j]  — the reference's H: every term h[b][j] is quantised to the 2^-40
//           grid (quantize_term, accum.hpp:34-38) and the c_b copies of it are
//           summed exactly, H = (double)(sum_b c_b llrint(h 2^40)) 2^-40
//           (dequantize, accum.hpp:40-42): bit-identical to the reference,
//           so its H < 1e-12 freeze rule (trainer.hpp:350) fires on the same
//           nodes (terms below 2^-41 vanish there too).
constexpr int kDenSlices = 32;  // b-slices per block (32 nodes x 32 slices = 1024 threads)
__global__ void __launch_bounds__(1024) k_smooth_den(const double* __restrict__ infl,
                                                     const double* __restrict__ sums, uint32_t P,
                                                     uint32_t D, double* __restrict__ H,
                                                     double* __restrict__ Hx) {
    __shared__ double part[kDenSlices][33];
    __shared__ __int128 qpart[kDenSlices][33];
    const uint32_t tj = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const uint32_t j = blockIdx.x * 32 + tj;
    const double* c = sums + (size_t)P * D;
    double acc = 0.0;
    __int128 qacc = 0;
    if (j < P)
        for (uint32_t b = sl; b < P; b += kDenSlices) {
            const double h = infl[(size_t)b * P + j];
            acc = fma(h, c[b], acc);
            const long long q = __double2ll_rn(h * 1099511627776.0);  // llrint(h 2^40)
            qacc += (__int128)q * (__int128)(unsigned long long)c[b];
        }
    part[sl][tj] = acc;
    qpart[sl][tj] = qacc;
    __syncthreads();
    if (sl == 0 && j < P) {
        double v = 0.0;
        __int128 qv = 0;
        for (int k = 0; k < kDenSlices; ++k) {
            v += part[k][tj];
            qv += qpart[k][tj];
        }
        Hx[j] = v;
        H[j] = (double)qv * (1.0 / 1099511627776.0);
    }
}

// partial[z][j][k] = sum_{b in slice z} infl[b][j] * S_b[k], k < d (S = the
// first P d entries of the sums buffer, read in place).
// Block: 32 nodes j x 64 columns k x one of SM_SPLIT b-slices (fills the GPU).
constexpr int SM_TJ = 32, SM_TB = 32, SM_KG = 8, SM_KC = SM_KG * 8, SM_SPLIT = 8;
__global__ void __launch_bounds__(256) k_smooth_gemm(const double* __restrict__ infl,
                                                     const double* __restrict__ sums, uint32_t P,
                                                     uint32_t D, double* __restrict__ partial) {
    __shared__ double hs[SM_TB * SM_TJ];
    __shared__ double ss[SM_TB * SM_KC];
    const int tj = threadIdx.x % SM_TJ, kg = threadIdx.x / SM_TJ;
    const uint32_t j0 = blockIdx.x * SM_TJ, j = j0 + tj;
    const uint32_t k0 = blockIdx.y * SM_KC;
    const uint32_t span = (P + SM_SPLIT - 1) / SM_SPLIT;
    const uint32_t bz0 = blockIdx.z * span, bz1 = min(P, bz0 + span);
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (uint32_t b0 = bz0; b0 < bz1; b0 += SM_TB) {
        __syncthreads();
        for (int e = threadIdx.x; e < SM_TB * SM_TJ; e += 256) {
            const uint32_t bb = b0 + e / SM_TJ, jj = j0 + e % SM_TJ;
            hs[e] = (bb < bz1 && jj < P) ? infl[(size_t)bb * P + jj] : 0.0;
        }
        for (int e = threadIdx.x; e < SM_TB * SM_KC; e += 256) {
            const uint32_t bb = b0 + e / SM_KC, kk = k0 + e % SM_KC;
            ss[e] = (bb < bz1 && kk < D) ? sums[(size_t)bb * D + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int bb = 0; bb < SM_TB; ++bb) {
            const double hv = hs[bb * SM_TJ + tj];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = fma(hv, ss[bb * SM_KC + kg + q * SM_KG], acc[q]);
        }
    }
    if (j >= P) return;
    double* out = partial + (size_t)blockIdx.z * P * D;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t k = k0 + kg + q * SM_KG;
        if (k < D) out[(size_t)j * D + k] = acc[q];
    }
}

// U = eta * (sum_z partial[z] - w * Hx), fixed slice order (deterministic)
__global__ void k_smooth_finish(const double* __restrict__ partial, const float* __restrict__ w,
                                const double* __restrict__ H, uint32_t P, uint32_t D, double eta,
                                double* __restrict__ U, int* __restrict__ status) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (status && e == 0) *status = INT_MAX;  // apply_update's fault slot (k_status_reset)
    if (e >= (size_t)P * D) return;
    double s = 0.0;
    for (int z = 0; z < SM_SPLIT; ++z) s += partial[(size_t)z * P * D + e];
    U[e] = eta * (s - (double)w[e] * H[e / D]);
}

void launch_smooth(const double* infl, const double* sums, const float* w, uint32_t P, uint32_t D,
                   double eta, double* U, double* H, double* scratch, cudaStream_t st,
                   int* status) {
    // scratch: P*(d+1) (unused) + SM_SPLIT*P*d (slice partials) + P (Hx) doubles
    double* partial = scratch + (size_t)P * (D + 1);
    double* Hx = partial + (size_t)SM_SPLIT * P * D;
    TSOM_LAUNCH(k_smooth_den<<<(P + 31) / 32, 32 * kDenSlices, 0, st>>>(infl, sums, P, D, H, Hx));
    dim3 grid((P + SM_TJ - 1) / SM_TJ, (D + SM_KC - 1) / SM_KC, SM_SPLIT);
    TSOM_LAUNCH(k_smooth_gemm<<<grid, 256, 0, st>>>(infl, sums, P, D, partial));
    const size_t pd = (size_t)P * D;
    TSOM_LAUNCH(k_smooth_finish<<<(unsigned)((pd + 255) / 256), 256, 0, st>>>(partial, w, Hx, P,
                                                                            D, eta, U, status));
}

size_t smooth_scratch_doubles(uint32_t P, uint32_t D) {
    return (size_t)P * (D + 1) + (size_t)SM_SPLIT * P * D + P;
}

// apply_update (trainer.hpp:341-369): H < 1e-12 → node frozen (momentum memory
// zeroed); else delta = U/H (+ beta*prev); non-finite → numerical fault.
__global__ void k_apply_update(float* __restrict__ w, float* __restrict__ prev, uint32_t P,
                               uint32_t D, const double* __restrict__ U,
                               const double* __restrict__ H, int use_momentum, double momentum,
                               int* __restrict__ status, const int* __restrict__ dead) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (e >= (size_t)P * D) return;
    if (dead && *dead) return;  // an earlier epoch of this multi-epoch run failed
    const uint32_t j = (uint32_t)(e / D);
    const double h = H[j];
    if (h < 1e-12) {
        if (use_momentum) prev[e] = 0.0f;
        return;
    }
    double delta = U[e] / h;
    if (use_momentum) delta += momentum * (double)prev[e];
    const double updated = (double)w[e] + delta;
    if (!isfinite(delta) || !isfinite(updated)) {
        atomicMin(status, (int)j);  // lowest failing node, like the reference's loop
        return;
    }
    w[e] = (float)updated;
    if (use_momentum) prev[e] = (float)delta;
}

void launch_apply_update(float* w, float* prev, uint32_t P, uint32_t D, const double* U,
                         const double* H, bool use_momentum, double momentum, int* status,
                         cudaStream_t st) {
    const size_t n = (size_t)P * D;
    TSOM_LAUNCH(k_apply_update<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, prev, P, D, U, H,
                                                                use_momentum ? 1 : 0, momentum,
                                                                status, nullptr));
}

void launch_apply_update_guarded(float* w, float* prev, uint32_t P, uint32_t D, const double* U,
                                 const double* H, bool use_momentum, double momentum, int* status,
                                 const int* dead, cudaStream_t st) {
    const size_t n = (size_t)P * D;
    TSOM_LAUNCH(k_apply_update<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, prev, P, D, U, H,
                                                                use_momentum ? 1 : 0, momentum,
                                                                status, dead));
}

// the host checks of tsom_train_epoch (non-finite update; |term| bound of
// accum.hpp:35: |eta| max_h (||x|| + ||w||) < 2^22), evaluated on the device
__global__ void k_epoch_guard(const int* __restrict__ status, uint32_t epoch,
                              int* __restrict__ dead) {
    if (dead[0]) return;
    if (*status != INT_MAX) {
        dead[0] = (int)epoch + 1;
        dead[1] = 1;
        dead[2] = *status;
    }
}

void launch_epoch_guard(const int* status, uint32_t epoch, int* dead, cudaStream_t st) {
    TSOM_LAUNCH(k_epoch_guard<<<1, 1, 0, st>>>(status, epoch, dead));
}

__global__ void k_status_reset(int* status) { *status = INT_MAX; }

void launch_status_reset(int* status, cudaStream_t st) {
    TSOM_LAUNCH(k_status_reset<<<1, 1, 0, st>>>(status));
}

// influence_matrix (topology.hpp:342-364): z = (d*d)*inv, h = z > 57.6 ? 0 : exp(-z)
// (also the per-block maxima of |h| the term guard reduces: hpart[kHmaxParts])
__global__ void __launch_bounds__(256) k_influence(const double* __restrict__ dist, size_t n,
                                                   double inv, double* __restrict__ out,
                                                   double* __restrict__ hpart) {
    double m = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double d = dist[i];
        const double z = __dmul_rn(__dmul_rn(d, d), inv);
        const double h = z > 57.6 ? 0.0 : exp(-z);
        out[i] = h;
        m = h > m || h != h ? h : m;
    }
    block_max_to(m, hpart);
}

void launch_influence(const double* dist, size_t n, double inv_two_sigma_sq, double* out,
                      cudaStream_t st, double* hpart) {
    TSOM_LAUNCH(k_influence<<<kHmaxParts, 256, 0, st>>>(dist, n, inv_two_sigma_sq, out, hpart));
}

// Synthetic Gaussian mixture: component and unit normal noise
// from a counter-based hash (splitmix64 of (seed, row, k)) + Box-Muller.
__device__ __forceinline__ uint64_t smix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void k_synth_gmm(float* __restrict__ x, uint64_t n, uint32_t D, uint32_t ldx,
                            const float* __restrict__ centres, uint32_t n_comp, uint64_t seed,
                            uint64_t row_offset) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t g = row_offset + i;
    const uint64_t base = smix(seed ^ smix(g));
    const uint32_t m = (uint32_t)(base % n_comp);
    float* row = x + i * ldx;
    for (uint32_t k = D; k < ldx; ++k) row[k] = 0.0f;  // padded rows: zero tail
    for (uint32_t k = 0; k < D; k += 2) {
        const uint64_t h = smix(base + k);
        const float u1 = 1.0f - (float)(h >> 40) * 0x1.0p-24f;  // (0, 1]
        const float u2 = (float)(h & 0xFFFFFFu) * 0x1.0p-24f;
        const float r = sqrtf(-2.0f * logf(u1));
        float s, c;
        sincospif(2.0f * u2, &s, &c);
        row[k] = centres[m * D + k] + r * c;
        if (k + 1 < D) row[k + 1] = centres[m * D + k + 1] + r * s;
    }
}

void launch_synth_gmm(float* x, uint64_t n, uint32_t D, const float* centres, uint32_t n_comp,
                      uint64_t seed, uint64_t row_offset, cudaStream_t st, uint32_t ldx) {
    if (n == 0) return;
    TSOM_LAUNCH(k_synth_gmm<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        x, n, D, ldx ? ldx : D, centres, n_comp, seed, row_offset));
}

}  // namespace tsom

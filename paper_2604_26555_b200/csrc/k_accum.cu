// k_accum.cu — K2: per-BMU accumulation (the data pass of accumulate,
// trainer.hpp:318-336) and the exact BMU distances (find_bmus distances,
// trainer.hpp:306; mean_bmu_distance :377-398).
//
// Algebra: the reference folds eta*h[b][j]*(x - w_j) for
// every sample and every node.  Grouping the samples by BMU b gives
//   U_j = eta * sum_b h[b][j] * (S_b - c_b w_j),   H_j = sum_b h[b][j] c_b
// with S_b = sum_{i: b_i = b} x_i and c_b = #{i: b_i = b}.  This kernel builds
// (R_b = sum (x_i - w_b), c_b) — residuals keep FP32 partial sums well
// conditioned — in shared memory per CTA, then flushes each CTA's partials to
// its own FP64 slot (no global atomics, deterministic final reduce).  The
// smoothing GEMM (k_smooth.cu) forms S_b = R_b + c_b w_b in FP64.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace tsom {

constexpr int ACC_THREADS = 1024;
constexpr int ACC_WARPS = ACC_THREADS / 32;
constexpr uint64_t kMaxRowsPerSlotPass = 1u << 16;  // FP32 partials cover <= 65536 rows

// Shared-memory privatised variant: smem = R[P*D] f32 + c[P] u32.
__global__ void __launch_bounds__(ACC_THREADS, 1) k_accumulate_smem(
    const float* __restrict__ x, const uint32_t* __restrict__ sel, uint64_t n, uint32_t D,
    const float* __restrict__ w, uint32_t P, const uint32_t* __restrict__ bmu,
    double* __restrict__ dist_out, double* __restrict__ slots, uint64_t rows_per_cta,
    int accumulate, int first_pass) {
    extern __shared__ float smem[];
    float* R = smem;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + (size_t)P * D);
    __shared__ double red[ACC_WARPS];
    const size_t slot_len = (size_t)P * D + P + 2;
    double* slot = slots + (size_t)blockIdx.x * slot_len;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (accumulate) {
        for (size_t e = threadIdx.x; e < (size_t)P * D; e += ACC_THREADS) R[e] = 0.0f;
        for (uint32_t e = threadIdx.x; e < P; e += ACC_THREADS) cnt[e] = 0u;
    }
    __syncthreads();

    const uint64_t r0 = (uint64_t)blockIdx.x * rows_per_cta;
    uint64_t r1 = r0 + rows_per_cta;
    if (r1 > n) r1 = n;
    double dsum = 0.0;
    for (uint64_t pos = r0 + warp; pos < r1; pos += ACC_WARPS) {
        const uint64_t row = sel ? (uint64_t)sel[pos] : pos;
        const uint32_t b = bmu[pos];
        const float* xr = x + row * D;
        const float* wb = w + (size_t)b * D;
        double d2 = 0.0;
        for (uint32_t k = lane; k < D; k += 32) {
            const float xv = xr[k], wv = wb[k];
            const double diff = (double)xv - (double)wv;
            d2 = fma(diff, diff, d2);
            if (accumulate) atomicAdd(&R[(size_t)b * D + k], xv - wv);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
        const double dist = sqrt(d2 > 0.0 ? d2 : 0.0);
        if (lane == 0) {
            if (accumulate) atomicAdd(&cnt[b], 1u);
            if (dist_out) dist_out[pos] = dist;
        }
        dsum += dist;
    }
    // the warp's lanes hold identical dsum; one per warp
    if (lane == 0) red[warp] = dsum;
    __syncthreads();
    if (warp == 0) {
        double v = lane < ACC_WARPS ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
            const double rows = r1 > r0 ? (double)(r1 - r0) : 0.0;
            if (first_pass) {
                slot[(size_t)P * D + P] = v;
                slot[(size_t)P * D + P + 1] = rows;
            } else {
                slot[(size_t)P * D + P] += v;
                slot[(size_t)P * D + P + 1] += rows;
            }
        }
    }
    if (!accumulate) return;
    // flush FP32 partials into this CTA's FP64 slot (exclusive owner: no atomics)
    for (size_t e = threadIdx.x; e < (size_t)P * D; e += ACC_THREADS) {
        const double v = (double)R[e];
        slot[e] = first_pass ? v : slot[e] + v;
    }
    for (uint32_t e = threadIdx.x; e < P; e += ACC_THREADS) {
        const double v = (double)cnt[e];
        slot[(size_t)P * D + e] = first_pass ? v : slot[(size_t)P * D + e] + v;
    }
}

// Fallback for codebooks whose partials exceed shared memory: FP64 atomics
// straight into slot 0 (correct, slower; P*D > ~51k).
__global__ void __launch_bounds__(256) k_accumulate_global(
    const float* __restrict__ x, const uint32_t* __restrict__ sel, uint64_t n, uint32_t D,
    const float* __restrict__ w, uint32_t P, const uint32_t* __restrict__ bmu,
    double* __restrict__ dist_out, double* __restrict__ slot, int accumulate) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double dsum = 0.0, rows = 0.0;
    for (uint64_t pos = wid; pos < n; pos += nw) {
        rows += 1.0;
        const uint64_t row = sel ? (uint64_t)sel[pos] : pos;
        const uint32_t b = bmu[pos];
        const float* xr = x + row * D;
        const float* wb = w + (size_t)b * D;
        double d2 = 0.0;
        for (uint32_t k = lane; k < D; k += 32) {
            const float xv = xr[k], wv = wb[k];
            const double diff = (double)xv - (double)wv;
            d2 = fma(diff, diff, d2);
            if (accumulate) atomicAdd(&slot[(size_t)b * D + k], (double)(xv - wv));
        }
        for (int o = 16; o; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
        const double dist = sqrt(d2 > 0.0 ? d2 : 0.0);
        if (lane == 0) {
            if (accumulate) atomicAdd(&slot[(size_t)P * D + b], 1.0);
            if (dist_out) dist_out[pos] = dist;
        }
        dsum += dist;
    }
    if (lane == 0 && rows > 0.0) {
        atomicAdd(&slot[(size_t)P * D + P], dsum);
        atomicAdd(&slot[(size_t)P * D + P + 1], rows);
    }
}

int accumulate_slots(uint32_t P, uint32_t D, size_t smem_optin, int sm_count) {
    const size_t need = ((size_t)P * D + P) * 4;
    if (need + 1024 > smem_optin) return 1;  // global fallback uses one slot
    return sm_count;
}

void launch_accumulate(const float* x, const uint32_t* sel, uint64_t n, uint32_t D,
                       const float* w, uint32_t P, const uint32_t* bmu, double* dist_out,
                       double* slots, int nslots, bool accumulate, bool first_pass,
                       size_t smem_optin, cudaStream_t st) {
    const size_t slot_len = (size_t)P * D + P + 2;
    const size_t need = ((size_t)P * D + P) * 4;
    if (need + 1024 > smem_optin) {
        if (first_pass) cudaMemsetAsync(slots, 0, slot_len * sizeof(double), st);
        if (n == 0) return;
        uint64_t blocks = (n * 32 + 255) / 256;
        if (blocks > 148 * 64) blocks = 148 * 64;
        TSOM_LAUNCH(k_accumulate_global<<<(unsigned)blocks, 256, 0, st>>>(x, sel, n, D, w, P, bmu, dist_out,
                                                             slots, accumulate ? 1 : 0));
        return;
    }
    static size_t attr_bytes = 0;
    if (attr_bytes < need) {
        cudaFuncSetAttribute(k_accumulate_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(smem_optin - 1024));
        attr_bytes = smem_optin;
    }
    // rows are split over nslots CTAs per pass; each pass covers <= nslots*64k rows
    const uint64_t pass_rows = (uint64_t)nslots * kMaxRowsPerSlotPass;
    bool first = first_pass;
    uint64_t done = 0;
    if (n == 0) {
        TSOM_LAUNCH(k_accumulate_smem<<<nslots, ACC_THREADS, accumulate ? need : 16, st>>>(
            x, sel, 0, D, w, P, bmu, dist_out, slots, 1, accumulate ? 1 : 0, first ? 1 : 0));
        return;
    }
    while (done < n) {
        const uint64_t chunk = (n - done) < pass_rows ? (n - done) : pass_rows;
        const uint64_t per_cta = (chunk + nslots - 1) / nslots;
        // with a selection the row ids are read through sel; without one the
        // rows of this pass are contiguous from `done`
        TSOM_LAUNCH(k_accumulate_smem<<<nslots, ACC_THREADS, accumulate ? need : 16, st>>>(
            sel ? x : x + done * D, sel ? sel + done : nullptr, chunk, D, w, P, bmu + done,
            dist_out ? dist_out + done : nullptr, slots, per_cta, accumulate ? 1 : 0,
            first ? 1 : 0));
        first = false;
        done += chunk;
    }
}

__global__ void k_reduce_slots(const double* __restrict__ slots, int nslots, size_t len,
                               double* __restrict__ sums) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (e >= len) return;
    double s = 0.0;
    for (int c = 0; c < nslots; ++c) s += slots[(size_t)c * len + e];  // fixed order
    sums[e] = s;
}

void launch_reduce_slots(const double* slots, int nslots, size_t len, double* sums,
                         cudaStream_t st) {
    TSOM_LAUNCH(k_reduce_slots<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(slots, nslots, len, sums));
}

}  // namespace tsom

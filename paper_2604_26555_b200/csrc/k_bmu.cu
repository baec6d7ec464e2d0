// k_bmu.cu — BMU search support kernels (SIMT path, exact re-check, codebook prep).
//
// Reference semantics (trainer.hpp:282-308 find_bmus): for each row,
//   best_j = argmin_j  sum_k (double(x_k) - w_jk)^2   (strict <, ties -> lowest j)
// computed in FP64.  The GPU evaluates the Gram form ||w_j||^2 - 2 x.w_j in
// FP32 (SIMT here, 3xTF32 tcgen05 in k1_bmu_tc.cu), keeps the best and
// second-best value per row, and re-scans in exact FP64 — with the reference's
// loop order and no FMA contraction — every row whose top-2 gap is within the
// FP32 error bound tau * (max||x||^2 + max||w||^2).  Rows outside that window
// have a unique FP64 argmin equal to the FP32 one, so BMU indices are
// bit-identical to the reference for every row.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "engine.h"

namespace tsom {

// ---------------------------------------------------------------------------
// Codebook prep (once per codebook change)
// ---------------------------------------------------------------------------

// SIMT operand wt ((d+1) x Ppad: -2 w^T and the ||w||^2 row), FP64 norms w2
// and max ||w||^2 (the error window).
__global__ void k_prep_codebook(const float* __restrict__ w, uint32_t P, uint32_t D,
                                double* __restrict__ w2, float* __restrict__ w2max,
                                float* __restrict__ wt, uint32_t Ppad) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Ppad) return;
    if (j >= P) {  // padding node: never wins
        for (uint32_t k = 0; k < D; ++k) wt[(size_t)k * Ppad + j] = 0.0f;
        wt[(size_t)D * Ppad + j] = CUDART_INF_F;
        return;
    }
    const float* wj = w + (size_t)j * D;
    double s = 0.0;
    for (uint32_t k = 0; k < D; ++k) s = __dadd_rn(s, __dmul_rn((double)wj[k], (double)wj[k]));
    w2[j] = s;
    atomicMax(reinterpret_cast<int*>(w2max), __float_as_int((float)s * 1.0000003f));
    for (uint32_t k = 0; k < D; ++k) wt[(size_t)k * Ppad + j] = -2.0f * wj[k];
    wt[(size_t)D * Ppad + j] = (float)s;
}

void launch_prep_codebook(const float* w, uint32_t P, uint32_t D, double* w2, float* w2max,
                          float* wt, uint32_t Ppad, cudaStream_t st) {
    // (one block reducing the maximum itself instead: 21 us vs 4.5 + 1.6 us)
    cudaMemsetAsync(w2max, 0, sizeof(float), st);
    TSOM_LAUNCH(k_prep_codebook<<<(Ppad + 127) / 128, 128, 0, st>>>(w, P, D, w2, w2max, wt, Ppad));
}

// ---------------------------------------------------------------------------
// max ||x||^2 (bound once per dataset)
// ---------------------------------------------------------------------------

__global__ void k_row_norm_max(const float* __restrict__ x, uint64_t n, uint32_t D, uint32_t ldx,
                               float* __restrict__ out) {
    float best = 0.0f;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const float* r = x + i * ldx;
        double s = 0.0;
        for (uint32_t k = 0; k < D; ++k) s += (double)r[k] * (double)r[k];
        best = fmaxf(best, (float)s * 1.0000002f);
    }
    for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(best));
}

void launch_row_norm_max(const float* x, uint64_t n, uint32_t D, float* out, cudaStream_t st,
                         bool reset, uint32_t ldx) {
    if (reset) cudaMemsetAsync(out, 0, sizeof(float), st);
    if (n == 0) return;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    TSOM_LAUNCH(k_row_norm_max<<<(unsigned)blocks, 256, 0, st>>>(x, n, D, ldx ? ldx : D, out));
}

__global__ void k_fold_max(float* a) { a[0] = fmaxf(a[0], a[1]); }

void launch_fold_max(float* a, cudaStream_t st) { TSOM_LAUNCH(k_fold_max<<<1, 1, 0, st>>>(a)); }

// ---------------------------------------------------------------------------
// K1 (SIMT): FP32 Gram distances, per-row top-2 over all nodes, flag near-ties
// ---------------------------------------------------------------------------
//
// Block = 256 threads = 16 (node lanes, tx) x 16 (row lanes, ty); tile = 128
// rows x 64-node chunks.  Thread (tx, ty) owns rows ty*8..+7 and nodes
// tx*4..+3 of each chunk: 32 FP32 accumulators, 3 LDS.128 per 32 FFMA.

constexpr int SIMT_TM = 128;
constexpr int SIMT_TN = 64;
constexpr int SIMT_XS = SIMT_TM + 4;  // padded row stride of the transposed x tile

__device__ __forceinline__ void top2_merge(float& b1, uint32_t& i1, float& b2, float ob1,
                                           uint32_t oi1, float ob2) {
    if (ob1 < b1 || (ob1 == b1 && oi1 < i1)) {
        b2 = fminf(b1, ob2);
        b1 = ob1;
        i1 = oi1;
    } else {
        b2 = fminf(b2, ob1);
    }
}

__global__ void __launch_bounds__(256) k1_bmu_simt(
    const float* __restrict__ x, uint32_t ldx, const uint32_t* __restrict__ sel, uint64_t n, uint32_t D,
    const float* __restrict__ wt, uint32_t P, uint32_t Ppad, const float* __restrict__ x2max,
    const float* __restrict__ w2max, float tau, uint32_t* __restrict__ bmu,
    uint32_t* __restrict__ flags) {
    extern __shared__ __align__(16) float sm[];
    const uint32_t Dp = D + 1;
    float* xs = sm;                        // [Dp][SIMT_XS]
    float* ws = sm + (size_t)Dp * SIMT_XS; // [Dp][SIMT_TN]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const float thr = tau * (__ldg(x2max) + __ldg(w2max));

    for (uint64_t tile = blockIdx.x; tile * SIMT_TM < n; tile += gridDim.x) {
        const uint64_t row0 = tile * SIMT_TM;
        __syncthreads();
        // transposed x tile; column Dp-1 = 1 (multiplies the ||w||^2 row)
        for (uint32_t e = tid; e < SIMT_TM * D; e += 256) {
            const uint32_t r = e / D, k = e - r * D;
            const uint64_t pos = row0 + r;
            float v = 0.0f;
            if (pos < n) {
                const uint64_t row = sel ? (uint64_t)sel[pos] : pos;
                v = x[row * ldx + k];
            }
            xs[k * SIMT_XS + r] = v;
        }
        for (int r = tid; r < SIMT_TM; r += 256) xs[D * SIMT_XS + r] = 1.0f;

        float b1[8], b2[8];
        uint32_t i1[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            b1[s] = CUDART_INF_F;
            b2[s] = CUDART_INF_F;
            i1[s] = 0;
        }
        for (uint32_t c0 = 0; c0 < Ppad; c0 += SIMT_TN) {
            __syncthreads();
            for (uint32_t e = tid; e < Dp * SIMT_TN; e += 256) {
                const uint32_t k = e / SIMT_TN, nn = e % SIMT_TN;
                ws[k * SIMT_TN + nn] = wt[(size_t)k * Ppad + c0 + nn];
            }
            __syncthreads();
            float acc[8][4];
#pragma unroll
            for (int s = 0; s < 8; ++s)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[s][q] = 0.0f;
            for (uint32_t k = 0; k < Dp; ++k) {
                const float4 xa = *reinterpret_cast<const float4*>(&xs[k * SIMT_XS + ty * 8]);
                const float4 xb = *reinterpret_cast<const float4*>(&xs[k * SIMT_XS + ty * 8 + 4]);
                const float4 wv = *reinterpret_cast<const float4*>(&ws[k * SIMT_TN + tx * 4]);
                const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
                const float wr[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                for (int s = 0; s < 8; ++s)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[s][q] = fmaf(xr[s], wr[q], acc[s][q]);
            }
#pragma unroll
            for (int s = 0; s < 8; ++s)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float v = acc[s][q];
                    if (v < b2[s]) {
                        if (v < b1[s]) {
                            b2[s] = b1[s];
                            b1[s] = v;
                            i1[s] = c0 + tx * 4 + q;
                        } else {
                            b2[s] = v;
                        }
                    }
                }
        }
        // merge the 16 node lanes of each row group (lanes differ in tx only)
#pragma unroll
        for (int s = 0; s < 8; ++s) {
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const float ob1 = __shfl_xor_sync(0xffffffffu, b1[s], o);
                const uint32_t oi1 = __shfl_xor_sync(0xffffffffu, i1[s], o);
                const float ob2 = __shfl_xor_sync(0xffffffffu, b2[s], o);
                top2_merge(b1[s], i1[s], b2[s], ob1, oi1, ob2);
            }
        }
        if (tx == 0) {
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const uint64_t pos = row0 + ty * 8 + s;
                if (pos < n) {
                    bmu[pos] = i1[s];
                    if (!(b2[s] - b1[s] > thr)) {
                        const uint32_t slot = atomicAdd(&flags[0], 1u);
                        flags[2 + slot] = (uint32_t)pos;
                    }
                }
            }
        }
    }
}

void launch_bmu_simt(const float* x, uint32_t ldx, const uint32_t* sel, uint64_t n, uint32_t D,
                     const float* wt, uint32_t P, uint32_t Ppad, const float* x2max,
                     const float* w2max, float tau, uint32_t* bmu, uint32_t* flags, int sm_count,
                     cudaStream_t st) {
    if (n == 0) return;
    const size_t smem = (size_t)(D + 1) * (SIMT_XS + SIMT_TN) * sizeof(float);
    ensure_smem_attr((const void*)k1_bmu_simt, 200 * 1024);
    uint64_t tiles = (n + SIMT_TM - 1) / SIMT_TM;
    uint64_t grid = (uint64_t)sm_count * 8;
    if (grid > tiles) grid = tiles;
    TSOM_LAUNCH(k1_bmu_simt<<<(unsigned)grid, 256, smem, st>>>(x, ldx, sel, n, D, wt, P, Ppad, x2max, w2max, tau, bmu,
                                                   flags));
}

// ---------------------------------------------------------------------------
// Merge per-group top-2 partials of the tcgen05 kernel
// ---------------------------------------------------------------------------

__device__ __forceinline__ double exact_d2(const float* __restrict__ x,
                                           const float* __restrict__ wj, uint32_t D) {
    // the reference's loop (trainer.hpp:295-299): FP64, sequential k, no contraction
    double acc = 0.0;
    for (uint32_t k = 0; k < D; ++k) {
        const double diff = __dsub_rn((double)x[k], (double)wj[k]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// exact_d2 for d even, d <= 64 and 8-byte aligned rows: all loads of both rows
// are issued before the first add (the scalar loop waits on a load per
// feature); the arithmetic and its order are exact_d2's
__device__ __forceinline__ double exact_d2_v2(const float* __restrict__ x,
                                              const float* __restrict__ wj, uint32_t D) {
    double acc = 0.0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {  // four chunks of 16 features: 32 data registers
        float2 xv[8], wv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (2u * (8 * h + q) < D) {
                xv[q] = __ldg(reinterpret_cast<const float2*>(x) + 8 * h + q);
                wv[q] = __ldg(reinterpret_cast<const float2*>(wj) + 8 * h + q);
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (2u * (8 * h + q) < D) {
                const double d0 = __dsub_rn((double)xv[q].x, (double)wv[q].x);
                acc = __dadd_rn(acc, __dmul_rn(d0, d0));
                const double d1 = __dsub_rn((double)xv[q].y, (double)wv[q].y);
                acc = __dadd_rn(acc, __dmul_rn(d1, d1));
            }
        }
    }
    return acc;
}

// Main-pass merge.  part[sg] = [B1 | code] per row and sub-group sg = g * sets
// + h, the group's chunks [h nch / sets, (h+1) nch / sets) (k1_bmu_tc merges
// its two epilogue sets in the CTA and passes sets = 1): the sub-group's raw minimum
// and, when it is the only node of the sub-group within the error window of
// that minimum, its id relative to the sub-group (else 0xFFFFFFFF).  A row is
// clear when its best sub-group has a unique in-window node and every other
// sub-group's minimum lies outside the window; it then gets its BMU here.
// Otherwise its position joins `ties` ([0] = count, positions from [1]) for the
// enumerate pass, with the bitmask of codebook groups inside the window.  If the
// FP16 codebook operand overflowed (scale[2] != 0) every row goes to the full
// exact re-scan.
__global__ void __launch_bounds__(256, 8) k_merge_fast(
    const float* __restrict__ part, uint64_t n, uint32_t groups, uint32_t sets, uint32_t gn,
    const float* __restrict__ xn2, const float* __restrict__ w2max,
    const float* __restrict__ scale, TieWin win, uint32_t* __restrict__ bmu,
    uint32_t* __restrict__ ties, uint32_t* __restrict__ tmask, uint32_t* __restrict__ flags) {
    constexpr uint32_t kCache = 8;  // sub-group minima kept in registers (K <= 2048 at sets 1)
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nsub = groups * sets, nch = gn / 32;
    bool need_tie = false;
    uint32_t mask = 0;
    if (valid) {
        float bc[kCache];
        float B1 = CUDART_INF_F;
        uint32_t smin = 0;
#pragma unroll
        for (uint32_t sg = 0; sg < kCache; ++sg) {  // strict <: lowest node ids on equal minima
            bc[sg] = sg < nsub ? __ldg(part + (size_t)sg * 2 * n + i) : CUDART_INF_F;
            if (bc[sg] < B1) {
                B1 = bc[sg];
                smin = sg;
            }
        }
        for (uint32_t sg = kCache; sg < nsub; ++sg) {
            const float b = __ldg(part + (size_t)sg * 2 * n + i);
            if (b < B1) {
                B1 = b;
                smin = sg;
            }
        }
        const uint32_t code = __float_as_uint(__ldg(part + (size_t)smin * 2 * n + n + i));
        const uint32_t gmin = smin / sets, hmin = smin % sets;
        bmu[i] = gmin * gn + (hmin * nch / sets) * 32 + (code == 0xFFFFFFFFu ? 0u : code);
        if (__float_as_uint(__ldg(scale + 2)) != 0u) {
            const uint32_t slot = atomicAdd(&flags[0], 1u);
            flags[2 + slot] = (uint32_t)i;
        } else {
            const float thr = __ldg(xn2 + i) + tie_wpart(__ldg(w2max), __ldg(scale + 1), win);
            const float lim = B1 + thr;
            bool clear = code != 0xFFFFFFFFu;
#pragma unroll
            for (uint32_t sg = 0; sg < kCache; ++sg) {
                const bool in = sg < nsub && bc[sg] <= lim;
                const uint32_t g = sg / sets;
                if (in) mask |= (g < 32 ? 1u << g : 0u);
                if (in && sg != smin) clear = false;
            }
            for (uint32_t sg = kCache; sg < nsub; ++sg) {
                const bool in = __ldg(part + (size_t)sg * 2 * n + i) <= lim;
                const uint32_t g = sg / sets;
                if (in) mask |= (g < 32 ? 1u << g : 0u);
                if (in && sg != smin) clear = false;
            }
            need_tie = !clear;
        }
    }
    // warp-aggregated append to the near-tie list (one atomic per warp)
    const uint32_t ballot = __ballot_sync(0xffffffffu, need_tie);
    if (ballot) {
        uint32_t base = 0;
        if (lane == (uint32_t)(__ffs(ballot) - 1)) base = atomicAdd(&ties[0], (uint32_t)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, __ffs(ballot) - 1);
        if (need_tie) {
            const uint32_t slot = base + __popc(ballot & ((1u << lane) - 1u));
            ties[1 + slot] = (uint32_t)i;
            tmask[slot] = groups <= 32 ? mask : 0xFFFFFFFFu;
        }
    }
}

// The same merge, four consecutive rows per thread (one sub-group record per
// codebook group, groups <= 8, n % 4 == 0): every load of a thread — the
// minima and codes of all groups and the row windows, 16 B each — is
// independent and issued at once, so a warp pays one memory latency instead of
// the two of the per-row kernel (the code of the winning group is read
// without knowing the winner).  BMUs, the near-tie rows and their masks are
// those of k_merge_fast; the list is appended to once per block (its order,
// which no result depends on, is by block).
template <int kG>
__global__ void __launch_bounds__(256) k_merge_fast4(
    const float* __restrict__ part, uint64_t n, uint32_t gn, const float* __restrict__ xn2,
    const float* __restrict__ w2max, const float* __restrict__ scale, TieWin win,
    uint32_t* __restrict__ bmu, uint32_t* __restrict__ ties, uint32_t* __restrict__ tmask,
    uint32_t* __restrict__ flags, uint32_t* __restrict__ cls, uint32_t* __restrict__ tile_mask) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;  // row quad
    const uint64_t i0 = q * 4;
    const bool valid = i0 < n;
    const uint32_t lane = threadIdx.x & 31;
    float4 mn[kG];
    uint4 cd[kG];
    float4 xw = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
#pragma unroll
        for (int g = 0; g < kG; ++g) {
            mn[g] = __ldg(reinterpret_cast<const float4*>(part + (size_t)g * 2 * n + i0));
            cd[g] = __ldg(reinterpret_cast<const uint4*>(part + (size_t)g * 2 * n + n + i0));
        }
        xw = __ldg(reinterpret_cast<const float4*>(xn2 + i0));
    }
    const bool overflow = __float_as_uint(__ldg(scale + 2)) != 0u;
    const float wpart = tie_wpart(__ldg(w2max), __ldg(scale + 1), win);
    uint32_t out[4], masks[4], ballots[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        float b[kG];
        uint32_t c[kG];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
            b[g] = r == 0 ? mn[g].x : r == 1 ? mn[g].y : r == 2 ? mn[g].z : mn[g].w;
            c[g] = r == 0 ? cd[g].x : r == 1 ? cd[g].y : r == 2 ? cd[g].z : cd[g].w;
        }
        float B1 = CUDART_INF_F;
        uint32_t gmin = 0, code = 0;
#pragma unroll
        for (int g = 0; g < kG; ++g)  // strict <: lowest node ids on equal minima
            if (b[g] < B1) {
                B1 = b[g];
                gmin = g;
                code = c[g];
            }
        out[r] = gmin * gn + (code == 0xFFFFFFFFu ? 0u : code);
        bool need_tie = false;
        uint32_t mask = 0;
        if (valid) {
            if (overflow) {
                const uint32_t slot = atomicAdd(&flags[0], 1u);
                flags[2 + slot] = (uint32_t)(i0 + r);
            } else {
                const float x2 = r == 0 ? xw.x : r == 1 ? xw.y : r == 2 ? xw.z : xw.w;
                const float lim = B1 + (x2 + wpart);
                bool clear = code != 0xFFFFFFFFu;
#pragma unroll
                for (int g = 0; g < kG; ++g) {
                    const bool in = b[g] <= lim;
                    if (in) mask |= 1u << g;
                    if (in && (uint32_t)g != gmin) clear = false;
                }
                need_tie = !clear;
            }
        }
        masks[r] = mask;
        ballots[r] = __ballot_sync(0xffffffffu, need_tie);
    }
    // block-aggregated append to the near-tie list: one atomic per block of
    // 1024 rows (a per-warp atomic on the one counter serialises ~2e5 atomics
    // per epoch at a 3 % near-tie rate); slots within the block in (warp, r,
    // lane) order
    __shared__ uint32_t wtot[8], blk_base, ccount[kTieClasses];
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t wcount = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) wcount += __popc(ballots[r]);
    if (lane == 0) wtot[warp] = wcount;
    if (cls && threadIdx.x < kTieClasses) ccount[threadIdx.x] = 0u;
    // k_tie_classes' tile masks start at zero (this block: 1024 list slots)
    if (tile_mask && threadIdx.x < 1024u / kTcTileM)
        tile_mask[blockIdx.x * (1024u / kTcTileM) + threadIdx.x] = 0u;
    __syncthreads();
    if (cls) {  // the near-tie rows' group classes (k_tie_classes), counted here
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if ((ballots[r] >> lane) & 1u) {
                const uint32_t c = tie_class(masks[r]);
                atomicAdd(&ccount[c], 1u);
            }
    }
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t k = 0; k < blockDim.x / 32; ++k) {
            const uint32_t v = wtot[k];
            wtot[k] = t;
            t += v;
        }
        blk_base = t ? atomicAdd(&ties[0], t) : 0u;
    }
    __syncthreads();
    if (cls && threadIdx.x < kTieClasses && ccount[threadIdx.x])
        atomicAdd(&cls[threadIdx.x], ccount[threadIdx.x]);
    uint32_t base = blk_base + wtot[warp];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if ((ballots[r] >> lane) & 1u) {
            const uint32_t slot = base + __popc(ballots[r] & ((1u << lane) - 1u));
            ties[1 + slot] = (uint32_t)(i0 + r);
            tmask[slot] = masks[r];
        }
        base += __popc(ballots[r]);
    }
    if (valid) *reinterpret_cast<uint4*>(bmu + i0) = make_uint4(out[0], out[1], out[2], out[3]);
}

bool launch_merge_fast(const float* part, uint64_t n, uint32_t groups, uint32_t sets, uint32_t gn,
                       const float* xn2, const float* w2max, const float* scale, TieWin win,
                       uint32_t* bmu, uint32_t* ties, uint32_t* tmask, uint32_t* flags,
                       cudaStream_t st, uint32_t* cls, uint32_t* tile_mask) {
    if (n == 0) return false;
    if (sets == 1 && n % 4 == 0 && groups <= 8 && !g_merge_v1) {
        const unsigned blocks = (unsigned)((n / 4 + 255) / 256);
#define TSOM_MERGE4(G)                                                                       \
    case G:                                                                                  \
        TSOM_LAUNCH(k_merge_fast4<G><<<blocks, 256, 0, st>>>(part, n, gn, xn2, w2max, scale, \
                                                             win, bmu, ties, tmask, flags,   \
                                                             cls, tile_mask));               \
        return cls != nullptr;
        switch (groups) {
            TSOM_MERGE4(1) TSOM_MERGE4(2) TSOM_MERGE4(3) TSOM_MERGE4(4)
            TSOM_MERGE4(5) TSOM_MERGE4(6) TSOM_MERGE4(7) TSOM_MERGE4(8)
        }
#undef TSOM_MERGE4
    }
    TSOM_LAUNCH(k_merge_fast<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        part, n, groups, sets, gn, xn2, w2max, scale, win, bmu, ties, tmask, flags));
    return false;  // (no group classes counted: the near-tie list stays as it is)
}

int g_merge_v1 = 0;  // diagnostics (TSOM option 96): 1 = the per-row merge


// Near-tie rows by the codebook groups they need enumerated (their window
// mask from k_merge_fast4): class g < kTieClasses - 1 = group g alone, the
// last class = several (or a group past the classes).  The list is re-ordered
// class by class, so the enumerate pass's 128-row tiles are (nearly all) of one
// class, and tile_mask[t] = OR of the tile's row masks tells the CTAs of group
// g which tiles hold any row of theirs: most near-ties need one group, which
// then does all their enumerate work instead of every group.
// In: the class counts cls[0, kTieClasses) and the zeroed tile masks (both from
// k_merge_fast4).  Out: ties_s = [count | positions], tmask_s, tile_mask.  The
// order within a class is arbitrary (no result depends on the list order).
// cls[kTieClasses, 2 kTieClasses) = fill counters (zeroed by k_set_scale).
__global__ void k_tie_classes(const uint32_t* __restrict__ ties, const uint32_t* __restrict__ tmask,
                              uint32_t* __restrict__ cls, uint32_t* __restrict__ ties_s,
                              uint32_t* __restrict__ tmask_s, uint32_t* __restrict__ tile_mask) {
    const uint32_t count = ties[0];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t off[kTieClasses];
    uint32_t run = 0;
#pragma unroll
    for (int c = 0; c < (int)kTieClasses; ++c) {
        off[c] = run;
        run += cls[c];
    }
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < count; i0 += stride) {
        const uint32_t i = i0 + threadIdx.x;
        const bool in = i < count;
        const uint32_t m = in ? tmask[i] : 0u;
        const uint32_t c = tie_class(m);
        const uint32_t peers = __match_any_sync(0xffffffffu, in ? c : 0xFFFFFFFFu);
        const uint32_t leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (in && lane == leader) base = atomicAdd(&cls[kTieClasses + c], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        // the class group's slots are consecutive: its leader ORs the group's
        // masks into the (at most two) tiles they fall in
        uint32_t mor = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
            const uint32_t v = __shfl_sync(0xffffffffu, m, l);
            if ((peers >> l) & 1u) mor |= v;
        }
        if (in) {
            const uint32_t idx = off[c] + base + __popc(peers & ((1u << lane) - 1u));
            ties_s[1 + idx] = ties[1 + i];
            tmask_s[idx] = m;
            if (lane == leader) {
                const uint32_t first = off[c] + base, last = first + __popc(peers) - 1;
                atomicOr(&tile_mask[first / kTcTileM], mor);
                if (last / kTcTileM != first / kTcTileM) atomicOr(&tile_mask[last / kTcTileM], mor);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ties_s[0] = count;
}

void launch_tie_classes(const uint32_t* ties, const uint32_t* tmask, uint64_t n_max, uint32_t* cls,
                        uint32_t* ties_s, uint32_t* tmask_s, uint32_t* tile_mask, cudaStream_t st) {
    const unsigned blocks = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((n_max + 255) / 256, 148ull * 8));
    TSOM_LAUNCH(k_tie_classes<<<blocks, 256, 0, st>>>(ties, tmask, cls, ties_s, tmask_s,
                                                      tile_mask));
}

// Enumerate-pass merge over the near-tie rows f < n (position ties[f]).
// part[g] = [raw b1 | ids 0-3 | ids 4-7 | count] (k1_bmu_tc<.., true>, 8-bit
// local ids, count 0 = group not enumerated).  One candidate -> bmu; several
// -> exact FP64 distances of just those nodes in ascending node order with
// strict < (lowest index wins), as find_bmus (trainer.hpp:293-304); > 8
// candidates in a group (or > kMaxCand in all) -> full exact re-scan list.
//
// A warp takes 32 near-tie rows (lane = row) and flattens their (row,
// candidate) pairs into a warp-private shared-memory list, so each exact
// distance — 50 dependent FP64 adds in the reference's feature order — runs on
// its own lane instead of one row's candidates running one after another on
// the row's lane; then every row picks its best pair in ascending node order.
// The re-check count is added once per warp (a per-row atomic on the one
// counter serialises ~3e5 atomics per epoch).
constexpr uint32_t kMaxCand = 16;  // candidates per row evaluated here
constexpr int kMpWarps = 8;

__global__ void __launch_bounds__(kMpWarps * 32, 3) k_merge_partials(
    const float* __restrict__ part, const uint32_t* __restrict__ ties,
    const uint32_t* __restrict__ dev_count, uint64_t cap, uint32_t groups, uint32_t gn,
    const float* __restrict__ xn2, const float* __restrict__ w2max,
    const float* __restrict__ scale, TieWin win, const float* __restrict__ x, uint32_t ldx,
    const uint32_t* __restrict__ sel, const float* __restrict__ w, uint32_t D,
    uint32_t* __restrict__ bmu, uint32_t* __restrict__ flags, const uint32_t* __restrict__ rmask) {
    __shared__ uint16_t pj[kMpWarps][32 * kMaxCand];  // candidate node of pair p
    __shared__ uint8_t prow[kMpWarps][32 * kMaxCand]; // owning lane of pair p
    __shared__ double pd[kMpWarps][32 * kMaxCand];    // exact squared distance
    __shared__ const float* xrow[kMpWarps][32];
    // the near-tie list length is read on the device (no host round trip);
    // rows past the enumerate capacity fall back to the full exact re-scan
    const uint64_t count = *dev_count;
    const uint64_t n = count < cap ? count : cap;
    const float S = __ldg(scale + 1);
    const uint32_t lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const uint64_t wstride = (uint64_t)gridDim.x * kMpWarps * 32;
    // 8-byte rows (d even): both rows loaded up front, one latency per pair
    const bool pairs_v2 = (D % 2) == 0 && D <= 64 && (ldx % 2) == 0 &&
                          ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 7u) == 0;
    for (uint64_t f0 = (blockIdx.x * (uint64_t)kMpWarps + wp) * 32; f0 < count; f0 += wstride) {
        const uint64_t f = f0 + lane;
        uint32_t pos = 0, ncand = 0, only = 0, gm = 0;
        bool rescan = false;
        float lim = 0.0f;
        if (f < count) {
            pos = ties[f];
            if (f >= cap) {
                rescan = true;
            } else {
                // the row's lines start towards L2 now (a DRAM round trip, hidden
                // behind the candidate records) for the distance pass below
                const float* xr = x + (sel ? (uint64_t)sel[pos] : (uint64_t)pos) * ldx;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(xr));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + D - 1));
                const float thr = __ldg(xn2 + f) + tie_wpart(__ldg(w2max), S, win);
                // groups enumerated for this row (the others' records are not
                // written when their CTAs skip the row's tile)
                gm = rmask ? rmask[f] : 0xFFFFFFFFu;
                float B1 = CUDART_INF_F;
                for (uint32_t g = 0; g < groups; ++g)
                    if ((gm >> (g & 31)) & 1u) B1 = fminf(B1, part[(size_t)g * 4 * n + f]);
                lim = B1 + thr;
                bool overflow = false;
                for (uint32_t g = 0; g < groups; ++g) {
                    const float* pg = part + (size_t)g * 4 * n;
                    if (!((gm >> (g & 31)) & 1u) || !(pg[f] <= lim)) continue;
                    const uint32_t cnt = __float_as_uint(pg[3 * n + f]);
                    if (cnt == 0) continue;
                    if (cnt > 8) overflow = true;
                    ncand += cnt;
                    only = g * gn + (__float_as_uint(pg[n + f]) & 0xFFu);
                }
                if (overflow || ncand == 0 || ncand > kMaxCand) rescan = true;
                else if (ncand == 1) bmu[pos] = only;
            }
        }
        if (rescan) {
            const uint32_t slot = atomicAdd(&flags[0], 1u);
            flags[2 + slot] = pos;
            bmu[pos] = only;
        }
        const bool multi = !rescan && ncand >= 2;
        const uint32_t mball = __ballot_sync(0xffffffffu, multi);
        if (!mball) continue;
        if (lane == 0) atomicAdd(&flags[1], (uint32_t)__popc(mball));
        // exclusive scan of the pair counts over the warp
        uint32_t mine = multi ? ncand : 0u, off = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, off, o);
            if ((int)lane >= o) off += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
        off -= mine;
        if (multi) {
            xrow[wp][lane] = x + (sel ? (uint64_t)sel[pos] : (uint64_t)pos) * ldx;
            uint32_t c = 0;
            for (uint32_t g = 0; g < groups; ++g) {
                const float* pg = part + (size_t)g * 4 * n;
                if (!((gm >> (g & 31)) & 1u) || !(pg[f] <= lim)) continue;
                const uint32_t cnt = __float_as_uint(pg[3 * n + f]);
                const uint32_t pk0 = __float_as_uint(pg[n + f]), pk1 = __float_as_uint(pg[2 * n + f]);
                for (uint32_t k = 0; k < cnt; ++k, ++c) {
                    const uint32_t pk = k < 4 ? pk0 : pk1;
                    pj[wp][off + c] = (uint16_t)(g * gn + ((pk >> (8 * (k & 3))) & 0xFFu));
                    prow[wp][off + c] = (uint8_t)lane;
                }
            }
        }
        __syncwarp();
        for (uint32_t p = lane; p < total; p += 32) {
            const uint32_t j = pj[wp][p];
            const float* xr = xrow[wp][prow[wp][p]];
            const float* wj = w + (size_t)j * D;
            pd[wp][p] = pairs_v2 ? exact_d2_v2(xr, wj, D) : exact_d2(xr, wj, D);
        }
        __syncwarp();
        if (multi) {
            double best = CUDART_INF;
            uint32_t best_j = 0;
            for (uint32_t c = 0; c < ncand; ++c) {  // ascending node order, strict <
                const double d2 = pd[wp][off + c];
                if (d2 < best) {
                    best = d2;
                    best_j = pj[wp][off + c];
                }
            }
            bmu[pos] = best_j;
        }
        __syncwarp();  // pair lists rewritten by the next round
    }
}

void launch_merge_partials(const float* part, const uint32_t* ties, const uint32_t* dev_count,
                           uint64_t cap, uint64_t n_max, uint32_t groups, uint32_t gn,
                           const float* xn2, const float* w2max, const float* scale, TieWin win,
                           const float* x, uint32_t ldx, const uint32_t* sel, const float* w,
                           uint32_t D, uint32_t* bmu, uint32_t* flags, cudaStream_t st,
                           const uint32_t* rmask) {
    if (n_max == 0) return;
    // grid-strides over the device count; sized for the enumerate capacity
    uint64_t blocks = (std::min(cap, n_max) + kMpWarps * 32 - 1) / (kMpWarps * 32);
    blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, 148ull * 8));
    TSOM_LAUNCH(k_merge_partials<<<(unsigned)blocks, kMpWarps * 32, 0, st>>>(
        part, ties, dev_count, cap, groups, gn, xn2, w2max, scale, win, x, ldx, sel, w, D, bmu,
        flags, rmask));
}

// ---------------------------------------------------------------------------
// Exact re-scan of flagged rows, reference order and rounding
// ---------------------------------------------------------------------------

// A block takes 32 flagged rows; the codebook streams through shared memory in
// chunks of 64 nodes, so each node row is read once per 32 rows.  Thread
// (r, q) = (tid / 8, tid % 8) evaluates row r against nodes q, q + 8, ... of a
// chunk in FP64 with the reference's operation order (sub, mul, add per
// feature, strict < over ascending j), then the 8 threads of a row reduce
// with ties to the lowest j.
constexpr int kRescanRows = 32, kRescanNodes = 64;

__global__ void __launch_bounds__(256) k_rescan(const float* __restrict__ x, uint32_t ldx,
                                                const uint32_t* __restrict__ sel,
                                                const float* __restrict__ w, uint32_t P,
                                                uint32_t D, const uint32_t* __restrict__ flags,
                                                uint32_t* __restrict__ bmu) {
    extern __shared__ float rs_smem[];
    float* xs = rs_smem;                          // [32][D]
    float* ws = rs_smem + kRescanRows * D;        // [64][D + 1]
    const uint32_t ldw = D + 1;
    const uint32_t count = flags[0];
    const uint32_t t = threadIdx.x, r = t >> 3, q = t & 7;
    for (uint32_t f0 = blockIdx.x * kRescanRows; f0 < count; f0 += gridDim.x * kRescanRows) {
        const uint32_t nr = min((uint32_t)kRescanRows, count - f0);
        __syncthreads();  // previous rows' shared data consumed
        for (uint32_t e = t; e < nr * D; e += blockDim.x) {
            const uint32_t rr = e / D, k = e - rr * D;
            const uint32_t pos = flags[2 + f0 + rr];
            const uint64_t row = sel ? (uint64_t)sel[pos] : pos;
            xs[rr * D + k] = x[row * ldx + k];
        }
        double best = CUDART_INF;
        uint32_t best_j = 0xFFFFFFFFu;
        const float* xr = xs + r * D;
        for (uint32_t c0 = 0; c0 < P; c0 += kRescanNodes) {
            const uint32_t nc = min((uint32_t)kRescanNodes, P - c0);
            __syncthreads();  // (first chunk: x rows staged; later: chunk consumed)
            for (uint32_t e = t; e < nc * D; e += blockDim.x) {
                const uint32_t jj = e / D, k = e - jj * D;
                ws[jj * ldw + k] = w[(size_t)(c0 + jj) * D + k];
            }
            __syncthreads();
            if (r < nr) {
                for (uint32_t jj = q; jj < nc; jj += 8) {
                    const float* wj = ws + jj * ldw;
                    double acc = 0.0;
                    for (uint32_t k = 0; k < D; ++k) {
                        const double diff = __dsub_rn((double)xr[k], (double)wj[k]);
                        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                    }
                    if (acc < best) {  // ascending j per thread: strict < keeps the lowest
                        best = acc;
                        best_j = c0 + jj;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) {  // the row's 8 threads (lanes 8r' .. 8r' + 7)
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, best_j, o);
            if (ob < best || (ob == best && oj < best_j)) {
                best = ob;
                best_j = oj;
            }
        }
        if (q == 0 && r < nr) bmu[flags[2 + f0 + r]] = best_j == 0xFFFFFFFFu ? 0u : best_j;
    }
}

void launch_rescan(const float* x, uint32_t ldx, const uint32_t* sel, const float* w, uint32_t P,
                   uint32_t D, const uint32_t* flags, uint64_t n, uint32_t* bmu, cudaStream_t st) {
    if (n == 0) return;
    // flagged rows are usually few: the kernel grid-strides over the device count
    const size_t smem = ((size_t)kRescanRows * D + (size_t)kRescanNodes * (D + 1)) * sizeof(float);
    ensure_smem_attr((const void*)k_rescan, smem);
    TSOM_LAUNCH(k_rescan<<<148 * 2, 256, smem, st>>>(x, ldx, sel, w, P, D, flags, bmu));
}

}  // namespace tsom

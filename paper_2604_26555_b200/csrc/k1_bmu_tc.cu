// k1_bmu_tc.cu — K1: BMU search as a tcgen05 tile GEMM with split-precision
// operands and a fused top-2 epilogue (the samples x codebook distance matrix
// never reaches HBM).  Reference: find_bmus, trainer.hpp:282-308.
//
// For row x and node j the kernel evaluates one augmented dot product whose
// value is (up to FP32 rounding and a power-of-two scale S = s^2)
//     v_j = ||x||^2 + ||w_j||^2 - 2 x.w_j  = d^2(x, w_j).
// Two operand encodings (TcKind), both "3-split" so FP32-level accuracy holds:
//   * kTcTf32 (3xTF32, kind::tf32): x' = [x, 1, 1, ||x||^2, 0..] and
//     w' = [-2w, p1+p2, p3, 1, 0..] (K = 56 = 7 k-steps of 8), split into
//     hi/lo halves; per k-step  xh.wh + xl.wh + xh.wl  (21 MMAs per tile).
//   * kTcF16 (3xFP16, kind::f16, 2x the TF32 rate): the three products are
//     concatenated along K instead of issued separately,
//         A = [xh | xl | xh | n_hi, n_lo, 1, 1, 1]   (x scaled by s)
//         B = [wh | wh | wl | 1,    1,    p1, p2, p3] (w' = -2 w s)
//     so one K = 16*ceil((3d+5)/16) pass (10 MMAs of K=16 at d = 50) yields
//     xh.wh + xl.wh + xh.wl + ||x s||^2 + ||w s||^2.  s = 2^e is chosen from
//     max ||x||^2 so every |x s| <= 16 (FP16 range; k_set_scale).
// Rows whose best/second-best gap falls inside the error window (tie_thr) are
// re-checked exactly in FP64 (k_bmu.cu), so BMU indices are bit-identical to
// the reference.
//
// Epilogue: thread = row (TMEM lane), 256 node values per group, two passes
// over TMEM: the row minimum b (3-input FMNMX), then for every value the
// window test c = sat(big (b + thr - v)) and a += c (j + 256) on the FMA pipe:
// a in [256, 512) means the minimum is the only node within the error window
// thr, and gives its id.  No per-value index bookkeeping on the ALU pipe.
//
// Work split: the codebook is cut into groups of gn <= 256 nodes.  A CTA keeps
// one group resident in shared memory for its whole life and streams 128-row
// sample tiles through a cp.async.bulk pipeline.  Warp roles (384 threads):
//   warp 0      : producer — bulk copies (mbarrier complete_tx)
//   warp 1      : MMA issuer — one elected thread
//   warp 2      : TMEM allocator (2 accumulator buffers x gn columns)
//   warps 4..11 : two sets of 4 epilogue warps; both drain every tile, set h
//                 taking node columns [128h, 128h + 128) (warp q of a set owns
//                 TMEM lanes 32q.., i.e. tile rows 32q..32q+31)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "engine.h"
#include "tc_ptx.cuh"

namespace tsom {

using namespace ptx;

namespace {

// epilogue warp sets (4 warps each, one per TMEM lane quarter); each set keeps
// its column slice of a tile in registers
template <int kKind>
struct EpiCfg {
    static constexpr int kSets = (int)kTcEpiSets;
    static constexpr int kThreads = 128 + kSets * 128;  // 4 role warps + the sets
    static constexpr int kCPS = 8 / kSets;              // 32-column chunks per set (gn = 256)
};
constexpr int kMaxStages = 4;

__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

}  // namespace

// diagnostics (option 99 bit 5): CTA 0 timestamps [tile][8] (clock64)
__device__ unsigned long long g_k1_trace[512 * 8];
// diagnostics (option 99 bit 7): every raw main-pass value v[row][group * gn + col]
// (scaled units) to this buffer, to measure the split-product error against
// the window (scripts/k1_window_error.py)
__device__ float* g_k1_dump = nullptr;
#define TSOM_TRACE(slot_, it_)                                                       \
    do {                                                                              \
        if (!kEnum && (dbg & 32u) && blockIdx.x == 0 && (it_) < 512u)                        \
            g_k1_trace[(it_) * 8 + (slot_)] = (unsigned long long)clock64();          \
    } while (0)

// ---------------------------------------------------------------------------
// Geometry of the two operand encodings
// ---------------------------------------------------------------------------

size_t tc_wsplit_bytes(int kind, uint32_t P, uint32_t D) {
    const uint32_t gn = tc_group_width(P);
    const uint32_t groups = (P + gn - 1) / gn;
    const TcGeom g = tc_geom(kind, D);
    return (size_t)groups * gn * g.row_bytes;
}

bool tc_supported(int kind, uint32_t P, uint32_t D) {
    if (P < 1) return false;
    if (kind == kTcTf32) return D + 3 <= (uint32_t)kTcKPad;
    if (kind == kTcF16) return 3u * D + 5u <= kTcF16MaxK;
    return false;
}

// ---------------------------------------------------------------------------
// Scale (kTcF16) and codebook operand
// ---------------------------------------------------------------------------

// scale[0] = s, scale[1] = s^2, scale[2] = overflow flag (bits), from max ||x||^2:
// the largest power of two with max||x|| * s <= 16 (so |x_k s| <= 16 and
// ||x s||^2 <= 256 fit FP16 with a 256x margin for ||w s||^2).
__global__ void k_set_scale(int kind, const float* __restrict__ x2max, float* __restrict__ scale,
                            uint32_t* __restrict__ zero, uint32_t nzero, uint32_t* __restrict__ zero2,
                            uint32_t* __restrict__ zero3, uint32_t nzero3) {
    // the pass's counters start at zero (no separate memset launches)
    for (uint32_t k = 0; k < nzero; ++k) zero[k] = 0u;
    if (zero2) *zero2 = 0u;
    for (uint32_t k = 0; k < nzero3; ++k) zero3[k] = 0u;
    float s = 1.0f;
    if (kind == kTcF16) {
        const float m = *x2max;
        if (m > 0.0f && isfinite(m)) {
            int e = ilogbf(16.0f / sqrtf(m));
            e = max(-100, min(60, e));
            s = ldexpf(1.0f, e);
            while (m * s * s > 256.0f) s *= 0.5f;
        }
    }
    scale[0] = s;
    scale[1] = s * s;
    scale[2] = 0.0f;
}

void launch_set_scale(int kind, const float* x2max, float* scale, cudaStream_t st, uint32_t* zero,
                      uint32_t nzero, uint32_t* zero2, uint32_t* zero3, uint32_t nzero3) {
    TSOM_LAUNCH(k_set_scale<<<1, 1, 0, st>>>(kind, x2max, scale, zero, nzero, zero2, zero3,
                                             zero3 ? nzero3 : 0u));
}

__device__ __forceinline__ float tf32_trunc(float v) {
    return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
}

// One thread per (node, 16-byte K core).  Group g = j / gn holds gn nodes in
// UMMA K-major core-matrix order: node r, core c at byte ((c * gn) + r) * 16
// (kTcTf32: hi half then lo half; kTcF16: one concatenated operand).
template <int kKind>
__global__ void k_prep_wsplit(const float* __restrict__ w, uint32_t P, uint32_t D, uint32_t gn,
                              uint32_t groups, const float* __restrict__ scale,
                              uint8_t* __restrict__ wsplit) {
    const uint32_t cores = kKind == kTcTf32 ? kTcKPad / 4 : tc_geom(kKind, D).kpad / 8;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t total = (uint64_t)groups * gn * cores;
    if (tid >= total) return;
    const uint32_t j = (uint32_t)(tid / cores), c = (uint32_t)(tid % cores);
    const uint32_t g = j / gn, r = j % gn;
    const bool pad = j >= P;
    const float* wj = w + (size_t)(pad ? 0 : j) * D;
    if (kKind == kTcTf32) {
        // w' = [-2w | p1 (hi) + p2 (lo) | p3 | 1 | 0..]; padding: 3e38 norm
        double s2 = 0.0;
        if (!pad)
            for (uint32_t k = 0; k < D; ++k)
                s2 = __dadd_rn(s2, __dmul_rn((double)wj[k], (double)wj[k]));
        const float p1 = tf32_trunc((float)s2);
        const float p2 = tf32_trunc((float)(s2 - (double)p1));
        const float p3 = tf32_trunc((float)(s2 - (double)p1 - (double)p2));
        float hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t k = c * 4 + q;
            float h = 0.0f, l = 0.0f;
            if (pad) {
                if (k == D) h = tf32_trunc(3.0e38f);
            } else if (k < D) {
                const float v = -2.0f * wj[k];
                h = tf32_trunc(v);
                l = v - h;
            } else if (k == D) {
                h = p1;
                l = p2;
            } else if (k == D + 1) {
                h = p3;
            } else if (k == D + 2) {
                h = 1.0f;
            }
            hi[q] = h;
            lo[q] = l;
        }
        float* base = reinterpret_cast<float*>(wsplit) + (size_t)g * 2 * gn * kTcKPad;
        const size_t off = ((size_t)c * gn + r) * 4;
        *reinterpret_cast<float4*>(base + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(base + (size_t)gn * kTcKPad + off) =
            make_float4(lo[0], lo[1], lo[2], lo[3]);
    } else {
        // B = [wh | wh | wl | 1, 1, p1, p2, p3 | 0..], w' = -2 w s; padding:
        // p1 = p2 = p3 = 65504 (never wins: real values are < 2^17)
        const float s = scale[0];
        double n2 = 0.0;
        if (!pad)
            for (uint32_t k = 0; k < D; ++k) {
                const double v = (double)(wj[k] * s);
                n2 += v * v;
            }
        const __half q1 = __double2half(n2);
        const __half q2 = __double2half(n2 - (double)__half2float(q1));
        const __half q3 =
            __double2half(n2 - (double)__half2float(q1) - (double)__half2float(q2));
        if (!pad && c == 0 && !(n2 < 60000.0))
            atomicOr(reinterpret_cast<unsigned*>(const_cast<float*>(scale)) + 2, 1u);
        __align__(16) __half h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t k = c * 8 + q;
            __half v = __float2half(0.0f);
            if (pad) {
                if (k >= 3 * D + 2 && k < 3 * D + 5) v = __float2half(65504.0f);
            } else if (k < 3 * D) {
                const uint32_t kk = k % D;
                const float wv = -2.0f * (wj[kk] * s);
                const __half whi = __float2half_rn(wv);
                v = k < 2 * D ? whi : __float2half_rn(wv - __half2float(whi));
            } else if (k == 3 * D || k == 3 * D + 1) {
                v = __float2half(1.0f);
            } else if (k == 3 * D + 2) {
                v = q1;
            } else if (k == 3 * D + 3) {
                v = q2;
            } else if (k == 3 * D + 4) {
                v = q3;
            }
            h[q] = v;
        }
        uint8_t* base = wsplit + (size_t)g * gn * cores * 16;
        *reinterpret_cast<uint4*>(base + ((size_t)c * gn + r) * 16) = *reinterpret_cast<uint4*>(h);
    }
}

void launch_prep_wsplit(int kind, const float* w, uint32_t P, uint32_t D, const float* scale,
                        void* wsplit, cudaStream_t st) {
    const uint32_t gn = tc_group_width(P);
    const uint32_t groups = (P + gn - 1) / gn;
    const uint32_t cores = kind == kTcTf32 ? kTcKPad / 4 : tc_geom(kind, D).kpad / 8;
    const uint64_t total = (uint64_t)groups * gn * cores;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    if (kind == kTcTf32)
        TSOM_LAUNCH(k_prep_wsplit<kTcTf32><<<blocks, 256, 0, st>>>(
            w, P, D, gn, groups, scale, static_cast<uint8_t*>(wsplit)));
    else
        TSOM_LAUNCH(k_prep_wsplit<kTcF16><<<blocks, 256, 0, st>>>(
            w, P, D, gn, groups, scale, static_cast<uint8_t*>(wsplit)));
}

// ---------------------------------------------------------------------------
// Split (optionally gathered) rows into A-operand tiles
// ---------------------------------------------------------------------------
//
// Tile t (rows 128t..128t+127), row r, 16-byte K core c at byte
// (c * 128 + r) * 16 (kTcTf32: hi half then lo half).  Rows past n are zero
// (their results are ignored).  xn2[f] = ||x||^2 rounded up (unscaled): the
// row's own error window (tie_thr).

// One block (256 threads) per 128-row tile: the tile's rows are gathered into
// shared memory with coalesced loads (consecutive threads read consecutive
// floats of a row), row norms come from shared memory, and every 16-byte K
// core of the tile is written by one thread (consecutive threads = consecutive
// rows of a core: coalesced stores).
constexpr int kSplitThreads = 256;

template <int kKind>
__global__ void __launch_bounds__(kSplitThreads) k_split_rows(
    const float* __restrict__ x, uint32_t ldx, const uint32_t* __restrict__ sel,
    const uint32_t* __restrict__ idx, const uint32_t* __restrict__ dev_n, uint64_t n_host,
    uint32_t D, const float* __restrict__ scale, TieWin win, uint8_t* __restrict__ tiles,
    float* __restrict__ xn2) {
    extern __shared__ float srow[];                 // [128][D + 1]
    __shared__ uint64_t rbase[kTcTileM];            // row offsets (floats)
    __shared__ float snorm[kTcTileM];
    const uint64_t n = dev_n ? min((uint64_t)*dev_n, n_host) : n_host;
    const uint64_t ntiles = (n + kTcTileM - 1) / kTcTileM;
    const TcGeom geo = tc_geom(kKind, D);
    const float s = kKind == kTcF16 ? scale[0] : 1.0f;
    const float S = kKind == kTcF16 ? scale[1] : 1.0f;
    const uint32_t ld = D + 1;
    const int t = threadIdx.x;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t f0 = tile * kTcTileM;
        const uint32_t rows = (uint32_t)(n - f0 < (uint64_t)kTcTileM ? n - f0 : (uint64_t)kTcTileM);
        __syncthreads();  // previous tile's shared memory fully consumed
        if (t < kTcTileM && (uint32_t)t < rows) {
            const uint64_t pos = idx ? (uint64_t)idx[f0 + t] : f0 + t;
            rbase[t] = (sel ? (uint64_t)sel[pos] : pos) * ldx;
        }
        __syncthreads();
        {
            // one warp per row (rows w, w+8, ...), lanes along K (D <= 64):
            // all of a warp's loads are issued before its stores so the
            // gathered rows' latencies overlap
            const uint32_t w = t >> 5, lane = t & 31;
            constexpr int kRowsPerWarp = kTcTileM / (kSplitThreads / 32);
            float v[kRowsPerWarp][2];
#pragma unroll
            for (int i = 0; i < kRowsPerWarp; ++i) {
                const uint32_t r = w + 8u * i;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t k = lane + 32u * h;
                    v[i][h] = (r < rows && k < D) ? __ldg(x + rbase[r] + k) : 0.0f;
                }
            }
#pragma unroll
            for (int i = 0; i < kRowsPerWarp; ++i) {
                const uint32_t r = w + 8u * i;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t k = lane + 32u * h;
                    if (r < rows && k < D) srow[r * ld + k] = v[i][h];
                }
            }
        }
        __syncthreads();
        if (t < kTcTileM) {
            double nrm = 0.0;
            if ((uint32_t)t < rows)
                for (uint32_t k = 0; k < D; ++k) {
                    const double v = (double)srow[t * ld + k];
                    nrm += v * v;
                }
            snorm[t] = (float)nrm;
            if (xn2 && (uint32_t)t < rows)
                xn2[f0 + t] = tie_xpart((float)nrm * 1.0000003f, S, win);
        }
        __syncthreads();
        uint8_t* base = tiles + tile * geo.tile_bytes;
        if (kKind == kTcTf32) {
            // x' = [x | 1 | 1 | ||x||^2 | 0..], hi half then lo half
            float* fb = reinterpret_cast<float*>(base);
            for (uint32_t e = t; e < (uint32_t)(kTcKPad / 4) * kTcTileM; e += kSplitThreads) {
                const uint32_t kc = e / kTcTileM, r = e % kTcTileM;
                const bool valid = r < rows;
                float hi[4], lo[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t k = kc * 4 + q;
                    float val = 0.0f;
                    if (valid) {
                        if (k < D) val = srow[r * ld + k];
                        else if (k == D || k == D + 1) val = 1.0f;
                        else if (k == D + 2) val = snorm[r];
                    }
                    hi[q] = tf32_trunc(val);
                    lo[q] = val - hi[q];
                }
                const size_t off = ((size_t)kc * kTcTileM + r) * 4;
                *reinterpret_cast<float4*>(fb + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4*>(fb + (size_t)kTcTileM * kTcKPad + off) =
                    make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
        } else {
            // A = [xh | xl | xh | n_hi, n_lo, 1, 1, 1 | 0..], x scaled by s
            for (uint32_t e = t; e < (geo.kpad / 8) * kTcTileM; e += kSplitThreads) {
                const uint32_t kc = e / kTcTileM, r = e % kTcTileM;
                const bool valid = r < rows;
                __align__(16) __half h[8];
                __half nh = __float2half(0.0f), nl = nh;
                if (valid && kc * 8 + 8 > 3 * D) {
                    const double ns = (double)snorm[r] * (double)s * (double)s;
                    nh = __double2half(ns);
                    nl = __double2half(ns - (double)__half2float(nh));
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t k = kc * 8 + q;
                    __half v = __float2half(0.0f);
                    if (valid) {
                        if (k < 3 * D) {
                            const uint32_t kk = k < D ? k : (k < 2 * D ? k - D : k - 2 * D);
                            const float xv = srow[r * ld + kk] * s;
                            const __half xh = __float2half_rn(xv);
                            v = (k >= D && k < 2 * D) ? __float2half_rn(xv - __half2float(xh)) : xh;
                        } else if (k == 3 * D) {
                            v = nh;
                        } else if (k == 3 * D + 1) {
                            v = nl;
                        } else if (k < 3 * D + 5) {
                            v = __float2half(1.0f);
                        }
                    }
                    h[q] = v;
                }
                *reinterpret_cast<uint4*>(base + ((size_t)kc * kTcTileM + r) * 16) =
                    *reinterpret_cast<uint4*>(h);
            }
        }
    }
}

// 3xFP16 split, warp-synchronous: a warp owns 16 consecutive tile rows (an
// eighth of a tile) and no block-wide barrier is involved.
//   1. row loads are coalesced (lanes along K, 16 rows in flight);
//   2. lane k converts element k of each row once (xh, xl) and stores the
//      halves at K positions k, D + k, 2D + k of the row in the warp's
//      half-precision row image (consecutive lanes -> consecutive halves);
//   3. the FP64 row norms are reduced across lanes with a transposing
//      butterfly (16 rows in 16 double shuffles), lane 2r ends with row r's
//      norm and writes the row's augmented columns and its window term;
//   4. lanes copy the image out in 16-byte cores (lanes 0-15: rows 0-15 of
//      the first half of the cores, lanes 16-31: the second half), 256
//      contiguous bytes per half-warp store.  The image's row stride is an odd
//      number of 16-byte units, so those reads are bank-conflict free.
// Matches k_split_rows<kTcF16> except for the summation order of the FP64 norm
// (enters only the approximate distances and the error window, whose 1.0000003
// factor covers it; decisions inside the window are re-checked in FP64).
constexpr int kSplitWarpRows = 16;

// img_w > 0: the rows go to a row-major image instead (row r at tiles + r *
// img_w halves, cores [0, kpad / 8) of it; launch_split_image).
//
// kTma (gathered rows: a selection or the near-tie list, d even <= 64, rows
// 8-byte aligned): the rows are not loaded through registers but staged by
// TMA — lane l < 16 bulk-copies row l's 16-byte window into the warp's
// staging buffer — double-buffered, so the next chunk's 16 rows are in flight
// while this one is converted (the register loads keep only one chunk in
// flight per warp at the 64 registers of 4 blocks per SM).
template <bool kTma>
__global__ void __launch_bounds__(kSplitThreads, kTma ? 2 : 4) k_split_rows_f16(
    const float* __restrict__ x, uint32_t ldx, const uint32_t* __restrict__ sel,
    const uint32_t* __restrict__ idx, const uint32_t* __restrict__ dev_n, uint64_t n_host,
    uint32_t D, const float* __restrict__ scale, TieWin win, uint8_t* __restrict__ tiles,
    float* __restrict__ xn2, uint32_t img_w = 0, int prefetch = 0) {
    extern __shared__ __align__(16) uint8_t split_wsm[];
    __shared__ __align__(8) uint64_t sbars[kTma ? kSplitThreads / 32 : 1][2];
    const uint64_t n = dev_n ? min((uint64_t)*dev_n, n_host) : n_host;
    constexpr uint32_t kChunksPerTile = kTcTileM / kSplitWarpRows;
    const uint64_t nchunks = (n + kTcTileM - 1) / kTcTileM * kChunksPerTile;
    const TcGeom geo = tc_geom(kTcF16, D);
    const uint32_t hs = geo.kpad + 8;  // halves per image row: odd number of 16-byte units
    const uint32_t ncores = geo.kpad / 8;
    const float s = scale[0];
    const float S = scale[1];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __half* img = reinterpret_cast<__half*>(split_wsm) + (size_t)w * kSplitWarpRows * hs;
    const __half one = __float2half(1.0f), zero = __float2half(0.0f);
    const uint64_t nwarps = (uint64_t)gridDim.x * (kSplitThreads / 32);
    // kTma: staging buffers [2][16 rows][slot] after the 8 warps' images
    const uint32_t slot = (D * 4 + 8 + 15) / 16 * 16;
    uint8_t* stage = split_wsm + (size_t)(kSplitThreads / 32) * kSplitWarpRows * hs * sizeof(__half) +
                     (size_t)w * 2 * kSplitWarpRows * slot;
    uint32_t phase = 0;
    // issue chunk cc into buffer b: lane l < 16 copies row l's window; returns
    // the row's byte offset in the buffer (lane l)
    auto stage_issue = [&](uint64_t cc, int b) -> uint32_t {
        const uint64_t q0 = cc * kSplitWarpRows;
        const bool mine = lane < (uint32_t)kSplitWarpRows && cc < nchunks && q0 + lane < n;
        uint64_t a = 0;
        uint32_t len = 0;
        if (mine) {
            const uint64_t pos = idx ? (uint64_t)idx[q0 + lane] : q0 + lane;
            a = reinterpret_cast<uint64_t>(x + (sel ? (uint64_t)sel[pos] : pos) * ldx);
            len = (uint32_t)(((a + D * 4u + 15) & ~15ull) - (a & ~15ull));
        }
        const uint32_t total = __reduce_add_sync(0xffffffffu, len);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) ptx::mbar_expect_tx(&sbars[w][b], total);
        __syncwarp();
        if (mine)
            ptx::bulk_g2s(stage + ((size_t)b * kSplitWarpRows + lane) * slot,
                          reinterpret_cast<const void*>(a & ~15ull), len, &sbars[w][b]);
        return ((size_t)b * kSplitWarpRows + (lane & 15u)) * slot + (uint32_t)(a & 15);
    };
    uint32_t soff[2] = {0u, 0u};
    const uint64_t cfirst = blockIdx.x * (uint64_t)(kSplitThreads / 32) + w;
    if (kTma) {
        if (lane == 0) {
            ptx::mbar_init(&sbars[w][0], 1);
            ptx::mbar_init(&sbars[w][1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        soff[0] = stage_issue(cfirst, 0);
    }
    int sb = 0;
    for (uint64_t c = cfirst; c < nchunks; c += nwarps, sb ^= 1) {
        const uint64_t r0 = c * kSplitWarpRows;
        const uint32_t rows =
            r0 >= n ? 0u : (n - r0 < (uint64_t)kSplitWarpRows ? (uint32_t)(n - r0) : kSplitWarpRows);
        uint64_t myrow = 0;
        if (!kTma && lane < rows) {
            const uint64_t pos = idx ? (uint64_t)idx[r0 + lane] : r0 + lane;
            myrow = sel ? (uint64_t)sel[pos] : pos;
        }
        if (kTma) {
            soff[sb ^ 1] = stage_issue(c + nwarps, sb ^ 1);
            ptx::mbar_wait(&sbars[w][sb], (phase >> sb) & 1u);
            phase ^= 1u << sb;
        }
        if (!kTma && (sel || idx) && prefetch) {
            // gathered rows: the warp's chunk `prefetch` iterations ahead into
            // L2 while this one is loaded and converted (lane l < 16: row l,
            // lane l + 16: its second 128-B line), raising the rows in flight
            const uint64_t cn = c + (uint64_t)prefetch * nwarps, rn = cn * kSplitWarpRows + (lane & 15u);
            if (rn < n && rn < nchunks * kSplitWarpRows) {
                const uint64_t pos = idx ? (uint64_t)idx[rn] : rn;
                const float* a = x + (sel ? (uint64_t)sel[pos] : pos) * ldx + (lane >> 4) * 32u;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
            }
        }
        double p[kSplitWarpRows];
        if (kTma) {
            // lane l: the adjacent elements 2l, 2l + 1 (d even): one packed
            // conversion per half pair (F2FP) and 4-byte image stores; the
            // halves are those of the element-wise path (both round to nearest)
            const uint32_t so = soff[sb];
            const bool on = 2u * lane < D;
#pragma unroll
            for (int i = 0; i < kSplitWarpRows; ++i) {
                const uint8_t* rs = stage + __shfl_sync(0xffffffffu, so, i);
                const float2 v = ((uint32_t)i < rows && on)
                                     ? *reinterpret_cast<const float2*>(rs + 8u * lane)
                                     : make_float2(0.0f, 0.0f);
                if (on) {
                    __half* row = img + i * hs;
                    const float x0 = v.x * s, x1 = v.y * s;
                    const __half2 hh = __floats2half2_rn(x0, x1);
                    const float2 hf = __half22float2(hh);
                    const __half2 hl = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
                    *reinterpret_cast<__half2*>(row + 2u * lane) = hh;
                    *reinterpret_cast<__half2*>(row + D + 2u * lane) = hl;
                    *reinterpret_cast<__half2*>(row + 2u * D + 2u * lane) = hh;
                }
                p[i] = (double)v.x * (double)v.x + (double)v.y * (double)v.y;
            }
        } else {
            float v[kSplitWarpRows][2];
#pragma unroll
            for (int i = 0; i < kSplitWarpRows; ++i) {
                const uint64_t rb = __shfl_sync(0xffffffffu, myrow, i) * ldx;
                v[i][0] = ((uint32_t)i < rows && lane < D) ? __ldg(x + rb + lane) : 0.0f;
                v[i][1] = ((uint32_t)i < rows && lane + 32u < D) ? __ldg(x + rb + lane + 32u) : 0.0f;
            }
#pragma unroll
            for (int i = 0; i < kSplitWarpRows; ++i) {
                __half* row = img + i * hs;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t k = lane + 32u * h;
                    if (k < D) {
                        const float xv = v[i][h] * s;
                        const __half xh = __float2half_rn(xv);
                        row[k] = xh;
                        row[D + k] = __float2half_rn(xv - __half2float(xh));
                        row[2 * D + k] = xh;
                    }
                }
                p[i] = (double)v[i][0] * (double)v[i][0] + (double)v[i][1] * (double)v[i][1];
            }
        }
        // transposing butterfly: after the level with offset o, lanes with bit
        // o set hold the upper half of the remaining rows
#pragma unroll
        for (int lvl = 0; lvl < 4; ++lvl) {
            const int half = 8 >> lvl;
            const uint32_t o = 16u >> lvl;
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < half; ++i) {
                const double keep = up ? p[i + half] : p[i];
                const double send = up ? p[i] : p[i + half];
                p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        p[0] += __shfl_xor_sync(0xffffffffu, p[0], 1);
        const uint32_t rr = (lane >> 1) & 15u;  // the row whose norm this lane holds
        const uint32_t ka = 3 * D + (lane & 1u) * 16u;
        {
            // lanes 2r, 2r+1 write row r's augmented columns [3D, kpad)
            const bool valid = rr < rows;
            const float nf = (float)p[0];
            const double ns = (double)nf * (double)s * (double)s;
            const __half nh = __double2half(ns);
            const __half nl = __double2half(ns - (double)__half2float(nh));
            __half* row = img + rr * hs;
            for (uint32_t k = ka; k < geo.kpad && k < ka + 16u; ++k) {
                const uint32_t a = k - 3 * D;
                row[k] = !valid ? zero : a == 0 ? nh : a == 1 ? nl : a < 5 ? one : zero;
            }
            if (!(lane & 1u) && valid && xn2) xn2[r0 + rr] = tie_xpart(nf * 1.0000003f, S, win);
        }
        __syncwarp();
        if (img_w) {
            // row-major image: consecutive lanes store consecutive 16-B cores
            // of a row (the warp's 16 rows x ncores cores in order)
            for (uint32_t e = lane; e < rows * ncores; e += 32) {
                const uint32_t r = e / ncores, kc = e - r * ncores;
                *reinterpret_cast<uint4*>(tiles + ((r0 + r) * img_w + kc * 8) * sizeof(__half)) =
                    *reinterpret_cast<const uint4*>(img + r * hs + kc * 8);
            }
            __syncwarp();  // image reused by the next chunk
            continue;
        }
        const uint32_t lr = lane & 15u, kc0 = (lane >> 4) * (ncores / 2);
        uint8_t* out = tiles + (c / kChunksPerTile) * (uint64_t)geo.tile_bytes +
                       (size_t)((c % kChunksPerTile) * kSplitWarpRows + lr) * 16;
        const __half* src = img + lr * hs;
        const bool valid = lr < rows;
        for (uint32_t q = 0; q < ncores / 2; ++q) {
            const uint32_t kc = kc0 + q;
            uint4 val = valid ? *reinterpret_cast<const uint4*>(src + kc * 8) : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(out + (size_t)kc * kTcTileM * 16) = val;
        }
        __syncwarp();  // image reused by the next chunk
    }
}

int g_split_v1 = 0;  // debug: the element-wise split (TSOM option 98)
int g_split_prefetch = 1;  // gathered split: L2 prefetch distance in chunks (option 92; 0 off)
int g_split_tma = 1;       // gathered split: rows staged by TMA (option 91; 0 = register loads)

void launch_split_rows(int kind, const float* x, const uint32_t* sel, const uint32_t* idx,
                       uint64_t n, uint32_t D, const float* scale, TieWin win, void* tiles,
                       float* xn2, cudaStream_t st, const uint32_t* dev_n, uint32_t ldx) {
    if (n == 0) return;
    if (ldx == 0) ldx = D;
    uint64_t tiles_n = (n + kTcTileM - 1) / kTcTileM;
    if (tiles_n > 148ull * 16) tiles_n = 148ull * 16;
    uint8_t* t = static_cast<uint8_t*>(tiles);
    const size_t smem = (size_t)kTcTileM * (D + 1) * sizeof(float);
    if (kind == kTcTf32)
        TSOM_LAUNCH(k_split_rows<kTcTf32><<<(unsigned)tiles_n, kSplitThreads, smem, st>>>(
            x, ldx, sel, idx, dev_n, n, D, scale, win, t, xn2));
    else if (g_split_v1)
        TSOM_LAUNCH(k_split_rows<kTcF16><<<(unsigned)tiles_n, kSplitThreads, smem, st>>>(
            x, ldx, sel, idx, dev_n, n, D, scale, win, t, xn2));
    else {
        const size_t wsmem = (size_t)(kSplitThreads / 32) * kSplitWarpRows *
                             (tc_geom(kTcF16, D).kpad + 8) * sizeof(__half);
        uint64_t blocks = (n + kTcTileM - 1) / kTcTileM;  // 8 warps x 16 rows per tile
        // gathered rows staged by TMA (needs d even <= 64, 8-byte aligned rows)
        const bool tma = (sel || idx) && g_split_tma && D % 2 == 0 && D <= 64 && ldx % 2 == 0 &&
                         (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
        if (tma) {
            const size_t tsmem = wsmem + (size_t)(kSplitThreads / 32) * 2 * kSplitWarpRows *
                                             ((D * 4 + 8 + 15) / 16 * 16);
            ensure_smem_attr((const void*)k_split_rows_f16<true>, tsmem);
            if (blocks > 148ull * 2) blocks = 148ull * 2;
            TSOM_LAUNCH(k_split_rows_f16<true><<<(unsigned)blocks, kSplitThreads, tsmem, st>>>(
                x, ldx, sel, idx, dev_n, n, D, scale, win, t, xn2, 0u, 0));
            return;
        }
        bool first = false;
        ensure_smem_attr((const void*)k_split_rows_f16<false>,
                         (kSplitThreads / 32) * kSplitWarpRows * (kTcF16MaxK + 8) * sizeof(__half),
                         &first);
        if (first)
            cudaFuncSetAttribute(k_split_rows_f16<false>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (blocks > 148ull * 8) blocks = 148ull * 8;
        TSOM_LAUNCH(k_split_rows_f16<false><<<(unsigned)blocks, kSplitThreads, wsmem, st>>>(
            x, ldx, sel, idx, dev_n, n, D, scale, win, t, xn2, 0u, g_split_prefetch));
    }
}

void launch_split_image(const float* x, uint32_t ldx, uint64_t n, uint32_t D, const float* scale,
                        TieWin win, void* img, uint32_t img_w, float* xn2, cudaStream_t st) {
    if (n == 0) return;
    if (ldx == 0) ldx = D;
    const size_t wsmem = (size_t)(kSplitThreads / 32) * kSplitWarpRows *
                         (tc_geom(kTcF16, D).kpad + 8) * sizeof(__half);
    bool first = false;
    ensure_smem_attr((const void*)k_split_rows_f16<false>,
                     (kSplitThreads / 32) * kSplitWarpRows * (kTcF16MaxK + 8) * sizeof(__half),
                     &first);
    if (first)
        cudaFuncSetAttribute(k_split_rows_f16<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             100);
    uint64_t blocks = (n + kTcTileM - 1) / kTcTileM;
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    TSOM_LAUNCH(k_split_rows_f16<false><<<(unsigned)blocks, kSplitThreads, wsmem, st>>>(
        x, ldx, nullptr, nullptr, nullptr, n, D, scale, win, static_cast<uint8_t*>(img), xn2,
        img_w));
}

// ---------------------------------------------------------------------------
// K1
// ---------------------------------------------------------------------------

// kEnum = false (main pass): per (row, group) the packed top-2 -> [B1 | i1 | B2]
//   (B1, B2 with the 8 id bits cleared).
// kEnum = true (near-tie rows only, see k_merge_fast): per (row, group) the raw
// best value plus up to 8 local candidate ids within tie_thr of it (count 15 =
// overflow, 0 = group not relevant for the row (rmask)).
// dev_n (optional): row count read on the device (the near-tie list length).
// kDump (diagnostics, option 99 bit 7): the main pass also stores every raw value
// kSkip (main pass over rows in BMU order): pass 2 skips the 32-column chunks
//   no row of the warp needs (see below).
// kGather (3xFP16, rows picked by id: selections, near-tie rows): instead of
//   pre-split tiles, the producer warp gathers each tile's 128 rows straight
//   from the row-major split image (one TMA tile::gather4 per 4 rows and
//   64-column atom, 128-B swizzled; tensor map tmap, row ids grow[pos]), and
//   the MMAs read the A operand through SWIZZLE_128B descriptors.
template <int kKind, bool kEnum, bool kDump = false, bool kSkip = false, bool kGather = false>
__global__ void __launch_bounds__(EpiCfg<kKind>::kThreads, 1)
    k1_bmu_tc(const uint8_t* __restrict__ tiles, uint64_t n_host, const uint32_t* __restrict__ dev_n,
              uint32_t groups, uint32_t gn, uint32_t D, uint32_t stages,
              const uint8_t* __restrict__ wsplit, const float* __restrict__ xn2,
              const float* __restrict__ w2max, const float* __restrict__ scale, TieWin win,
              const uint32_t* __restrict__ rmask, float* __restrict__ part, uint32_t dbg,
              uint32_t mc, const uint32_t* __restrict__ tile_mask,
              const __grid_constant__ CUtensorMap tmap, const uint32_t* __restrict__ grow,
              uint32_t natoms) {
    // mc > 1: the CTAs of a cluster are the mc codebook groups of the same tile
    // sequence; each loads 1/mc of every A tile and multicasts it to all, so the
    // tile crosses L2 -> SM once per cluster instead of once per group.
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kSets = EpiCfg<kKind>::kSets, kCPS = EpiCfg<kKind>::kCPS;
    const TcGeom geo = tc_geom(kKind, D);
    const uint64_t n = dev_n ? min((uint64_t)*dev_n, n_host) : n_host;
    if (n == 0) return;  // an empty near-tie pass (uniform over the grid and its clusters)
    const uint32_t ntiles = (uint32_t)((n + kTcTileM - 1) / kTcTileM);
    const uint32_t w_bytes = gn * geo.row_bytes;  // this CTA's group (both halves for tf32)
    // one A stage: a pre-split tile, or natoms 128-row x 128-B swizzle atoms
    const uint32_t tbytes = kGather ? natoms * (kTcTileM * 128u) : geo.tile_bytes;
    uint8_t* sW = smem;
    uint8_t* sX = smem + ((w_bytes + 1023u) & ~1023u);
    if (kGather && (smem_u32(sX) & 1023u)) __trap();  // swizzle atoms need 1024-B alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + stages * tbytes);
    uint64_t* full_bar = bars;                    // [stages] X tile landed
    uint64_t* empty_bar = bars + kMaxStages;      // [stages] MMAs done with X tile
    uint64_t* tfull_bar = bars + 2 * kMaxStages;  // [2] accumulator ready
    uint64_t* tempty_bar = tfull_bar + 2;         // [2] accumulator drained
    uint64_t* w_bar = tfull_bar + 4;              // codebook group landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_bar + 1);
    // [2 tiles][128 rows] (b, code) of epilogue set 1, merged into set 0's
    float* xch_b = reinterpret_cast<float*>(bars + 16);
    uint32_t* xch_c = reinterpret_cast<uint32_t*>(xch_b + 2 * kTcTileM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g = blockIdx.x % groups;
    const uint32_t cta_in_group = blockIdx.x / groups;
    const uint32_t ctas_per_group = gridDim.x / groups;
    const uint32_t acc_cols = gn <= 32 ? 32 : (gn <= 64 ? 64 : (gn <= 128 ? 128 : 256));

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], mc);  // one MMA-completion arrival per CTA of the cluster
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull_bar[a], 1);
            mbar_init(&tempty_bar[a], 4u * kSets);  // one arrival per epilogue warp
        }
        mbar_init(w_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(2 * acc_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    if (mc > 1) cluster_sync();  // every CTA's barriers initialised before remote arrivals
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint16_t mc_mask = (uint16_t)((1u << mc) - 1u);

    if (kGather && warp == 0) {
        if (ntiles > cta_in_group) {
            if (lane == 0) {  // resident codebook group, in <= 64 KB bulk copies
                mbar_expect_tx(w_bar, w_bytes);
                const uint8_t* wg = wsplit + (size_t)g * w_bytes;
                for (uint32_t off = 0; off < w_bytes; off += 65536u)
                    bulk_g2s(sW + off, wg + off, min(65536u, w_bytes - off), w_bar);
            }
            uint32_t stage = 0, phase = 0;
            // mc > 1: the cluster's CTAs (the codebook groups, same tile
            // sequence) each gather 128 / mc rows of the tile and multicast
            // them to all, so every row is fetched once per cluster
            const uint32_t rpc = kTcTileM / mc;
            const uint32_t row = (mc > 1 ? (g % mc) * rpc : 0u) + 4u * lane;
            for (uint32_t t = cta_in_group; t < ntiles; t += ctas_per_group) {
                if (kEnum && tile_mask && !((tile_mask[t] >> (g & 31)) & 1u)) continue;
                mbar_wait(&empty_bar[stage], phase ^ 1);
                if (lane == 0) mbar_expect_tx(&full_bar[stage], tbytes);
                __syncwarp();
                // lane l gathers rows row..row+3 of the tile (rows past n repeat a
                // valid id; their results are never read) into every atom
                if (4u * lane < rpc) {
                    const uint64_t p0 = (uint64_t)t * kTcTileM + row;
                    int id[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        id[j] = (int)__ldg(grow + (p0 + j < n ? p0 + j : n - 1));
                    uint8_t* dst = sX + stage * tbytes + row * 128u;
                    for (uint32_t a = 0; a < natoms; ++a) {
                        if (mc > 1)
                            tma_gather4_mc(dst + a * (kTcTileM * 128u), &tmap, (int)(a * 64u), id[0],
                                           id[1], id[2], id[3], &full_bar[stage], mc_mask);
                        else
                            tma_gather4(dst + a * (kTcTileM * 128u), &tmap, (int)(a * 64u), id[0],
                                        id[1], id[2], id[3], &full_bar[stage]);
                    }
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 0) {
        if (lane == 0 && ntiles > cta_in_group) {
            // resident codebook group, in <= 64 KB bulk copies
            mbar_expect_tx(w_bar, w_bytes);
            const uint8_t* wg = wsplit + (size_t)g * w_bytes;
            for (uint32_t off = 0; off < w_bytes; off += 65536u)
                bulk_g2s(sW + off, wg + off, min(65536u, w_bytes - off), w_bar);
            uint32_t stage = 0, phase = 0;
            for (uint32_t t = cta_in_group; t < ntiles; t += ctas_per_group) {
                if (kEnum && tile_mask && !((tile_mask[t] >> (g & 31)) & 1u)) continue;
                mbar_wait(&empty_bar[stage], phase ^ 1);
                if (dbg & 4u) {
                    mbar_arrive(&full_bar[stage]);
                } else if (mc > 1) {
                    // this CTA's slice of the tile, to the same stage of every CTA
                    const uint32_t slice = geo.tile_bytes / mc, off = (g % mc) * slice;
                    mbar_expect_tx(&full_bar[stage], geo.tile_bytes);
                    bulk_g2s_mc(sX + stage * geo.tile_bytes + off,
                                tiles + (size_t)t * geo.tile_bytes + off, slice, &full_bar[stage],
                                mc_mask);
                } else {
                    mbar_expect_tx(&full_bar[stage], geo.tile_bytes);
                    bulk_g2s(sX + stage * geo.tile_bytes, tiles + (size_t)t * geo.tile_bytes,
                             geo.tile_bytes, &full_bar[stage]);
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && ntiles > cta_in_group) {
            const uint32_t idesc = kKind == kTcTf32 ? idesc_tf32(kTcTileM, gn)
                                                    : idesc_f16(kTcTileM, gn);
            const uint32_t w_lbo = gn * 16u;
            const uint32_t sw = smem_u32(sW);
            mbar_wait(w_bar, 0);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            for (uint32_t t = cta_in_group; t < ntiles; t += ctas_per_group) {
                if (kEnum && tile_mask && !((tile_mask[t] >> (g & 31)) & 1u)) continue;
                const uint32_t it_ = (t - cta_in_group) / ctas_per_group;
                mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                mbar_wait(&full_bar[stage], phase);
                TSOM_TRACE(0, it_);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * acc_cols;
                const uint32_t sx = smem_u32(sX + stage * tbytes);
                if (dbg & 2u) {
                } else if (kGather) {
                    // k-step k: atom k / 4, 32 B into its (swizzled) rows
                    for (uint32_t k = 0; k < geo.ksteps; ++k)
                        mma_f16(d, umma_desc_sw128(sx + (k >> 2) * (kTcTileM * 128u) + (k & 3u) * 32u),
                                umma_desc(sw + k * 2u * w_lbo, w_lbo, 128u), idesc,
                                k > 0 ? 1u : 0u);
                } else if (kKind == kTcTf32) {
                    const uint32_t sx_lo = sx + geo.tile_bytes / 2;
                    const uint32_t sw_lo = sw + w_bytes / 2;
#pragma unroll
                    for (int k = 0; k < kTcKPad / 8; ++k) {
                        const uint64_t ah = umma_desc(sx + k * 4096u, 2048u, 128u);
                        const uint64_t al = umma_desc(sx_lo + k * 4096u, 2048u, 128u);
                        const uint64_t bh = umma_desc(sw + k * 2u * w_lbo, w_lbo, 128u);
                        const uint64_t bl = umma_desc(sw_lo + k * 2u * w_lbo, w_lbo, 128u);
                        mma_tf32(d, ah, bh, idesc, k > 0 ? 1u : 0u);
                        mma_tf32(d, al, bh, idesc, 1u);
                        mma_tf32(d, ah, bl, idesc, 1u);
                    }
                } else {
                    for (uint32_t k = 0; k < geo.ksteps; ++k)
                        mma_f16(d, umma_desc(sx + k * 4096u, 2048u, 128u),
                                umma_desc(sw + k * 2u * w_lbo, w_lbo, 128u), idesc,
                                k > 0 ? 1u : 0u);
                }
                TSOM_TRACE(1, it_);
                if (mc > 1)
                    mma_commit_mc(&empty_bar[stage], mc_mask);  // stage free in every CTA's view
                else
                    mma_commit(&empty_bar[stage]);  // X stage free once these MMAs retire
                mma_commit(&tfull_bar[acc]);    // accumulator ready for the epilogue
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // Epilogue.  Warp (set, q) owns TMEM lanes 32q..32q+31 (= tile rows).
        const uint32_t q = warp & 3, set = (warp - 4) >> 2;
        const uint32_t row = q * 32 + lane;
        const uint32_t nch = gn / 32;  // gn is a multiple of 32 (tc_group_width)
        const float S = scale[1];
        const float wpart = tie_wpart(__ldg(w2max), S, win);  // codebook part of the window
        if (!kEnum) {
            // Main pass: both sets drain every tile, set h taking chunks
            // [h nch / kSets, (h+1) nch / kSets).  Per row and set:
            //   pass 1: b = min v (3-input FMNMX, 0.5 ALU op per value);
            //   pass 2: over the same columns, c = sat(big (lim - v)) is 1 for
            //     every v <= lim = b + thr and 0 otherwise (one FFMA.SAT), and
            //     a += c (j + 256) (one FFMA): a = 256 count + sum of ids, so
            //     a in [256, 512) <=> exactly one node (the minimum) lies in
            //     the window, and then id = a - 256.  Two FMA-pipe ops per
            //     value, no ALU op, no index bookkeeping.
            // The set's slice is loaded into registers once (the accumulator
            // is released right after), and the set writes [b | id within the
            // slice, or 0xFFFFFFFF when several nodes lie in the window] as
            // sub-group g * kSets + set for k_merge_fast.
            const uint32_t c_begin = set * nch / kSets;
            const uint32_t c_count = (dbg & 1u) ? 0u : (set + 1) * nch / kSets - c_begin;
            uint32_t acc = 0, acc_phase = 0;
            const uint32_t t0 = cta_in_group, tstep = ctas_per_group;
            // ||x||^2 of the row, prefetched one tile ahead (hides the load latency)
            uint64_t pos_next = (uint64_t)t0 * kTcTileM + row;
            float x2_next = pos_next < n ? __ldg(xn2 + pos_next) : 0.0f;
            for (uint32_t t = t0; t < ntiles; t += tstep) {
                const uint64_t pos = (uint64_t)t * kTcTileM + row;
                const float x2 = x2_next;
                pos_next = pos + (uint64_t)tstep * kTcTileM;
                x2_next = pos_next < n ? __ldg(xn2 + pos_next) : 0.0f;
                mbar_wait(&tfull_bar[acc], acc_phase);
                const uint32_t it_ = (t - cta_in_group) / ctas_per_group;
                if (lane == 0 && q == 0) TSOM_TRACE(2 + 3 * (set & 1), it_);
                tc_fence_after();
                const uint32_t taddr =
                    tmem_base + ((q * 32u) << 16) + acc * acc_cols + c_begin * 32;
                // this set's (<= 4) chunks are loaded once into registers (one
                // TMEM round trip) and both passes run on the registers
                uint32_t r[kCPS][32];
                const bool full = c_count == (uint32_t)kCPS;  // the common case: no guards
                if (full) {
#pragma unroll
                    for (int c = 0; c < kCPS; ++c) TSOM_TMEM_LD32(taddr + c * 32, r[c]);
                } else {
#pragma unroll
                    for (int c = 0; c < kCPS; ++c)
                        if ((uint32_t)c < c_count) TSOM_TMEM_LD32(taddr + c * 32, r[c]);
                }
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[acc]);  // warp done with the accumulator
                if (kDump && pos < n) {
                    float* dp = g_k1_dump + pos * (uint64_t)(groups * gn) + g * gn + c_begin * 32;
#pragma unroll
                    for (int c = 0; c < kCPS; ++c)
                        if ((uint32_t)c < c_count)
#pragma unroll
                            for (int k = 0; k < 32; ++k) dp[c * 32 + k] = __uint_as_float(r[c][k]);
                }
                // pass 1 keeps one minimum per 32-column chunk (two chains
                // each).  kSkip: pass 2 then skips every chunk whose minimum
                // lies outside the window for all 32 rows of the warp — such
                // a chunk adds exactly 0 to a (sat(big (lim - v)) = 0 for v >=
                // lim), so the skip changes no result.  Rows whose values
                // cluster (the BMU-ordered resident rows) need
                // pass 2 on ~40 % of the chunks; on rows in random order the
                // vote costs more than it saves, hence the template switch.
                float mc[kCPS][2];
#pragma unroll
                for (int c = 0; c < kCPS; ++c) mc[c][0] = mc[c][1] = CUDART_INF_F;
#define TSOM_PASS1(c)                                                                       \
    _Pragma("unroll") for (int m = 0; m < 16; ++m) mc[c][m & 1] =                          \
        fmin3f(mc[c][m & 1], __uint_as_float(r[c][2 * m]), __uint_as_float(r[c][2 * m + 1]))
#define TSOM_PASS2(c)                                                                       \
    if (!kSkip || __any_sync(0xffffffffu, cmin[c] < lim))                                  \
    _Pragma("unroll") for (int k = 0; k < 32; ++k) a[k & 7] =                              \
        fmaf(__saturatef(fmaf(__uint_as_float(r[c][k]), nb, lb)), (float)((c) * 32 + k + 256), \
             a[k & 7])
#define TSOM_ALL(P)                                                                         \
    do {                                                                                    \
        if (full) {                                                                         \
            _Pragma("unroll") for (int c = 0; c < kCPS; ++c) P(c);                          \
        } else {                                                                            \
            _Pragma("unroll") for (int c = 0; c < kCPS; ++c) if ((uint32_t)c < c_count)     \
                P(c);                                                                       \
        }                                                                                   \
    } while (0)
                TSOM_ALL(TSOM_PASS1);
                if (lane == 0 && q == 0) TSOM_TRACE(3 + 3 * (set & 1), it_);
                float cmin[kCPS];
#pragma unroll
                for (int c = 0; c < kCPS; ++c) cmin[c] = fminf(mc[c][0], mc[c][1]);
                float b = cmin[0];
#pragma unroll
                for (int c = 1; c < kCPS; ++c) b = fminf(b, cmin[c]);
                if (dbg & 512u) {  // diagnostics: pass-2 chunks run / chunks, trace slots 4094-4095
                    const float l0 = b + (x2 + wpart);
                    const float l1 = l0 + fabsf(l0) * 2.4e-7f;
                    uint32_t run = 0;
#pragma unroll
                    for (int c = 0; c < kCPS; ++c)
                        run += ((uint32_t)c < c_count) && __any_sync(0xffffffffu, cmin[c] < l1);
                    if (lane == 0) {
                        atomicAdd(&g_k1_trace[4094], (unsigned long long)run);
                        atomicAdd(&g_k1_trace[4095], (unsigned long long)c_count);
                    }
                }
                const float thr = x2 + wpart;
                // window limit, nudged up so a value exactly at b + thr counts
                const float lim0 = b + thr;
                const float lim = lim0 + fabsf(lim0) * 2.4e-7f;
                // big = 2^(60 - e(lim)): big * lim ~ 2^60, far from FP32 overflow
                const int ef = (int)((__float_as_uint(lim) >> 23) & 0xFFu);
                const float big = __int_as_float(max(67, min(247, 314 - ef)) << 23);
                const float lb = lim * big, nb = -big;
                float a[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
                TSOM_ALL(TSOM_PASS2);
#undef TSOM_ALL
#undef TSOM_PASS1
#undef TSOM_PASS2
                if (lane == 0 && q == 0) TSOM_TRACE(4 + 3 * (set & 1), it_);
                // a = 256 count + sum(local ids); decode: exactly one -> global id
                const float asum = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
                uint32_t code = 0xFFFFFFFFu;  // id relative to the set's first column
                if (asum >= 256.0f && asum < 512.0f && asum == floorf(asum))
                    code = (uint32_t)asum - 256u;
                // the sets' results for the group are merged here, exactly as
                // k_merge_fast would merge them (set 0 wins equal minima; the
                // group's id is ambiguous when the other set's minimum lies in
                // the window of the group's), so one record per (row, group)
                // leaves the CTA
                static_assert(kSets == 2, "set merge assumes two epilogue sets");
                if (set == 1) {
                    xch_b[acc * kTcTileM + row] = b;
                    xch_c[acc * kTcTileM + row] = code;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kSets * 128) : "memory");
                if (set == 0 && pos < n) {
                    const float b1 = xch_b[acc * kTcTileM + row];
                    const uint32_t c1 = xch_c[acc * kTcTileM + row];
                    float bg = b, other = b1;
                    uint32_t cg = code;
                    if (b1 < b) {
                        bg = b1;
                        other = b;
                        cg = c1 == 0xFFFFFFFFu ? c1 : c1 + (nch / kSets) * 32u;
                    }
                    if (other <= bg + thr) cg = 0xFFFFFFFFu;
                    float* pg = part + (size_t)g * 2 * n;
                    pg[pos] = bg;
                    pg[n + pos] = __uint_as_float(cg);
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        } else {
            // Enumerate pass (near-tie rows only), laid out like the main pass:
            // both sets drain every tile, set h loading its chunks [h nch /
            // kSets, (h+1) nch / kSets) into registers with one TMEM round trip
            // (the accumulator is released at once).  The sets swap their
            // minima through shared memory, so each enumerates its columns
            // against the group's raw minimum B1: a 32-bit mask of v <= B1 +
            // thr per chunk, then the set bits in ascending order.  Set 1
            // hands its candidates to set 0, which appends them after its own
            // (set 1's ids are the higher ones: ascending node order) and
            // writes [B1 | ids 0-3 | ids 4-7 | count] (count 0: group not
            // relevant for the row, kCandOverflow: > 8 candidates).
            static_assert(kSets == 2, "set exchange assumes two epilogue sets");
            // single-buffered: a set rewrites its slots for the next tile only
            // after the second barrier of this one, which the reader has passed
            float* xmin = xch_b;                                                  // [2 set][128]
            uint32_t* xlist = reinterpret_cast<uint32_t*>(xch_b + 2 * kTcTileM);  // [3][128]
            const uint32_t c_begin = set * nch / kSets;
            const uint32_t c_count = (set + 1) * nch / kSets - c_begin;
            uint32_t acc = 0, acc_phase = 0;
            for (uint32_t t = cta_in_group; t < ntiles; t += ctas_per_group) {
                // (tiles without a row needing this group are skipped by all
                // three roles alike; the merge ignores their records)
                if (tile_mask && !((tile_mask[t] >> (g & 31)) & 1u)) continue;
                const uint64_t pos = (uint64_t)t * kTcTileM + row;
                const bool need = pos < n && ((__ldg(rmask + pos) >> (g & 31)) & 1u);
                const float thr = need ? __ldg(xn2 + pos) + wpart : 0.0f;
                mbar_wait(&tfull_bar[acc], acc_phase);
                tc_fence_after();
                const uint32_t taddr =
                    tmem_base + ((q * 32u) << 16) + acc * acc_cols + c_begin * 32;
                uint32_t r[kCPS][32];
#pragma unroll
                for (int c = 0; c < kCPS; ++c)
                    if ((uint32_t)c < c_count) TSOM_TMEM_LD32(taddr + c * 32, r[c]);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[acc]);  // warp done with the accumulator
                float mn[2] = {CUDART_INF_F, CUDART_INF_F};
#pragma unroll
                for (int c = 0; c < kCPS; ++c)
                    if ((uint32_t)c < c_count) {
#pragma unroll
                        for (int m = 0; m < 16; ++m)
                            mn[m & 1] = fmin3f(mn[m & 1], __uint_as_float(r[c][2 * m]),
                                               __uint_as_float(r[c][2 * m + 1]));
                    }
                const float bs = fminf(mn[0], mn[1]);
                xmin[set * kTcTileM + row] = bs;
                asm volatile("bar.sync 1, %0;" ::"n"(kSets * 128) : "memory");
                const float B1 = fminf(bs, xmin[(set ^ 1) * kTcTileM + row]);
                const float lim = B1 + thr;
                uint32_t pk0 = 0, pk1 = 0, nc = 0;
                if (__any_sync(0xffffffffu, need)) {
#pragma unroll
                    for (int c = 0; c < kCPS; ++c)
                        if ((uint32_t)c < c_count) {
                            uint32_t m = 0;
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                m |= (__uint_as_float(r[c][k]) <= lim ? 1u : 0u) << k;
                            if (!need) m = 0;
                            while (m && nc <= 8) {
                                const uint32_t id = (c_begin + c) * 32u + (__ffs(m) - 1);
                                m &= m - 1;
                                if (nc < 4) pk0 |= id << (8 * nc);
                                else if (nc < 8) pk1 |= id << (8 * (nc - 4));
                                ++nc;
                            }
                        }
                }
                if (set == 1) {
                    uint32_t* xl = xlist;
                    xl[row] = nc;
                    xl[kTcTileM + row] = pk0;
                    xl[2 * kTcTileM + row] = pk1;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kSets * 128) : "memory");
                if (set == 0 && pos < n) {
                    const uint32_t* xl = xlist;
                    const uint32_t n1 = xl[row];
                    uint32_t cnt = nc + n1;
                    if (need && nc <= 8 && cnt <= 8) {
                        const uint32_t q0 = xl[kTcTileM + row], q1 = xl[2 * kTcTileM + row];
                        for (uint32_t i = 0; i < n1; ++i) {
                            const uint32_t id = ((i < 4 ? q0 : q1) >> (8 * (i & 3))) & 0xFFu;
                            const uint32_t p = nc + i;
                            if (p < 4) pk0 |= id << (8 * p);
                            else pk1 |= id << (8 * (p - 4));
                        }
                    } else if (need) {
                        cnt = kCandOverflow;
                    }
                    float* pg = part + (size_t)g * 4 * n;
                    pg[pos] = B1;
                    pg[n + pos] = __uint_as_float(pk0);
                    pg[2 * n + pos] = __uint_as_float(pk1);
                    pg[3 * n + pos] = __uint_as_float(!need ? 0u : cnt);
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (mc > 1) cluster_sync();  // no CTA leaves while a peer may still signal it
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(2 * acc_cols));
    }
}

// diagnostics only (option 99): bit0 skips the epilogue math, bit1 the MMAs,
// bit2 the A-tile loads, so the stages can be timed in isolation; bit5 traces
// CTA 0; bit6 multicasts A tiles over clusters of all group CTAs; bit7 dumps
// every raw main-pass value; bit8 turns the chunk skip off; bit9 counts the
// pass-2 chunks run; bit10 unicasts the gather4 path; bit12 turns the
// default cluster-of-2 multicast off
uint32_t g_k1_debug = 0;

int k1_set_dump(float* d_buf) {
    return cudaMemcpyToSymbol(g_k1_dump, &d_buf, sizeof(d_buf)) == cudaSuccess ? 0 : 4;
}

int k1_trace_copy(unsigned long long* out, uint32_t n) {
    return cudaMemcpyFromSymbol(out, g_k1_trace, (n < 4096u ? n : 4096u) * 8) == cudaSuccess ? 0
                                                                                             : 4;
}

cudaError_t launch_bmu_tc(int kind, const void* tiles, uint64_t n, const uint32_t* dev_n,
                          bool enumerate, uint32_t P, uint32_t D, const void* wsplit,
                          const float* xn2, const float* w2max, const float* scale, TieWin win,
                          const uint32_t* rmask, float* part, int sm_count, size_t smem_optin,
                          cudaStream_t st, const uint32_t* tile_mask, bool skip,
                          const CUtensorMap* tmap, const uint32_t* grow) {
    if (n == 0) return cudaSuccess;
    skip = skip && !enumerate && !(g_k1_debug & (128u | 256u));  // (bit 8: A/B of the skip)
    const bool gather = tmap != nullptr;
    if (gather && kind != kTcF16) return cudaErrorInvalidValue;
    const TcGeom geo = tc_geom(kind, D);
    const uint32_t natoms = (geo.kpad + 63u) / 64u;
    const uint32_t tbytes = gather ? natoms * (kTcTileM * 128u) : geo.tile_bytes;
    const uint32_t gn = tc_group_width(P);
    const uint32_t groups = (P + gn - 1) / gn;
    const uint32_t ntiles = (uint32_t)((n + kTcTileM - 1) / kTcTileM);  // upper bound
    uint32_t per_group = (uint32_t)sm_count / groups;
    if (per_group < 1) per_group = 1;
    if (per_group > ntiles) per_group = ntiles;
    const uint32_t grid = per_group * groups;
    const uint32_t w_bytes = gn * geo.row_bytes;
    const size_t fixed = ((w_bytes + 1023u) & ~1023u) + 128 + 2 * kTcTileM * 10;  // + set exchange
    uint32_t stages = 2;
    while (stages < 3 && fixed + (size_t)(stages + 1) * tbytes <= smem_optin) ++stages;
    const size_t smem = fixed + (size_t)stages * tbytes;
    if (smem > smem_optin) return cudaErrorInvalidConfiguration;
    using KernT = void (*)(const uint8_t*, uint64_t, const uint32_t*, uint32_t, uint32_t, uint32_t,
                           uint32_t, const uint8_t*, const float*, const float*, const float*,
                           TieWin, const uint32_t*, float*, uint32_t, uint32_t, const uint32_t*,
                           const CUtensorMap, const uint32_t*, uint32_t);
    KernT kern;
    if (gather) {
        kern = enumerate ? k1_bmu_tc<kTcF16, true, false, false, true>
                         : (skip ? k1_bmu_tc<kTcF16, false, false, true, true>
                                 : k1_bmu_tc<kTcF16, false, false, false, true>);
    } else if (kind == kTcTf32) {
        kern = enumerate ? k1_bmu_tc<kTcTf32, true>
                         : ((g_k1_debug & 128u) ? k1_bmu_tc<kTcTf32, false, true>
                                                : (skip ? k1_bmu_tc<kTcTf32, false, false, true>
                                                        : k1_bmu_tc<kTcTf32, false>));
    } else {
        kern = enumerate ? k1_bmu_tc<kTcF16, true>
                         : ((g_k1_debug & 128u) ? k1_bmu_tc<kTcF16, false, true>
                                                : (skip ? k1_bmu_tc<kTcF16, false, false, true>
                                                        : k1_bmu_tc<kTcF16, false>));
    }
    {
        const cudaError_t e = ensure_smem_attr((const void*)kern, smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = kind == kTcF16 ? EpiCfg<kTcF16>::kThreads : EpiCfg<kTcTf32>::kThreads;
    // cluster of the `groups` CTAs that share each A tile (multicast loads);
    // as many clusters as can be co-resident (one CTA per SM)
    uint32_t mc = 1;
    // (measured neutral at K = 1024 on B200, so off unless option 99 bit 6 asks)
    if (!gather && (g_k1_debug & 64u) && groups >= 2 && groups <= 8 &&
        geo.tile_bytes % (16u * groups) == 0)
        mc = groups;
    // main pass: clusters of 2 group CTAs share each A tile (each CTA loads half
    // and multicasts it), so a tile leaves HBM/L2 twice instead of four times at
    // K = 1024: less DRAM power under the cap, K1 2.37 -> 2.30 ms (bench A/B,
    // scripts/ab_mc2.sh; all four groups per cluster packs fewer clusters onto
    // the GPCs and was slower).  Option 99 bit 12 turns it off.
    if (!gather && !enumerate && mc == 1 && !(g_k1_debug & 4096u) && groups % 2 == 0 &&
        geo.tile_bytes % 32u == 0)
        mc = 2;
    // gathered rows: each row fetched once per cluster of the group CTAs
    // (the per-CTA gather4 rate bounds the kernel otherwise; option 99 bit 10 off)
    if (gather && groups >= 2 && groups <= 8 && kTcTileM % (4u * groups) == 0 &&
        !(g_k1_debug & 1024u))
        mc = groups;
    uint32_t clusters = per_group;
    if (mc > 1) {
        // max co-resident clusters, per (kernel, device, cluster size)
        static std::mutex mu;
        static std::map<std::tuple<const void*, int, uint32_t>, int> max_clusters;
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        auto it = max_clusters.find({(const void*)kern, dev, mc});
        if (it == max_clusters.end()) {
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(mc * per_group);
            qc.blockDim = dim3(threads);
            qc.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = mc;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            qc.attrs = qa;
            qc.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, kern, &qc) != cudaSuccess) {
                cudaGetLastError();
                nc = 0;
            }
            it = max_clusters.emplace(std::make_tuple((const void*)kern, dev, mc), nc).first;
        }
        if (it->second < 1) mc = 1;
        else clusters = std::min<uint32_t>(per_group, (uint32_t)it->second);
    }
    const uint32_t grid_x = clusters * groups;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_x);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeClusterDimension;
    attr1[0].val.clusterDim.x = mc;
    attr1[0].val.clusterDim.y = 1;
    attr1[0].val.clusterDim.z = 1;
    cfg.attrs = attr1;
    cfg.numAttrs = 1;
    ++g_launches;
    const cudaError_t e = cudaLaunchKernelEx(
        &cfg, kern, static_cast<const uint8_t*>(tiles), n, dev_n, groups, gn, D, stages,
        static_cast<const uint8_t*>(wsplit), xn2, w2max, scale, win, rmask, part, g_k1_debug, mc,
        (enumerate && mc == 1) ? tile_mask : nullptr,  // (multicast loads need every tile)
        gather ? *tmap : CUtensorMap{}, grow, natoms);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace tsom

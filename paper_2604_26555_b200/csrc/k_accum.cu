// k_accum.cu — K2: per-BMU accumulation (the data pass of accumulate,
// trainer.hpp:318-336) and the exact BMU distances (find_bmus distances,
// trainer.hpp:306; mean_bmu_distance :377-398).
//
// Algebra: the reference folds eta*h[b][j]*(x - w_j) for
// every sample and every node.  Grouping the samples by BMU b gives
//   U_j = eta * sum_b h[b][j] * (S_b - c_b w_j),   H_j = sum_b h[b][j] c_b
// with S_b = sum_{i: b_i = b} x_i and c_b = #{i: b_i = b}.  K2 produces S_b
// (FP64 register sums of exact FP64 terms, no float atomics) and c_b.
//
// Pipeline (all deterministic, no floating-point atomics):
//   k_hist      block-local BMU histograms            [nblk][P]
//   k_colscan   per-node exclusive scan over blocks   (in place) + node totals
//   k_nodescan  node starts, counts c_b, piece table  (one block)
//   k_scatter   stable counting sort of row positions by BMU
//   k_gather_tma  one warp per piece (<= 256 rows of one node): 32-row
//               batches staged by TMA bulk copies (one per run of consecutive
//               rows), FP64 register accumulation, optional exact distances;
//               one partial row per piece (k_gather_async / k_gather_any: the
//               cp.async and register-load variants for other shapes)
//   k_piece_reduce  sums the pieces of every node in order -> sums buffer
// HBM traffic per row: ~4 B x 3 (bmu passes) + 8 B (sorted position) + the
// 200 B row => ~212 B/row (204 B algorithmic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "engine.h"
#include "tc_ptx.cuh"

namespace tsom {

constexpr uint32_t kHistRows = 16384;   // rows per histogram / scatter block
constexpr int kScatterWarps = 8;        // sub-chunks of 2048 rows
constexpr uint32_t kPieceRows = 256;    // rows per gather task (one warp)
constexpr int kGatherBatch = 16;

uint64_t accum_pieces_max(uint64_t n, uint32_t P) { return n / kPieceRows + P + 1; }
uint64_t accum_blocks(uint64_t n) { return (n + kHistRows - 1) / kHistRows; }

// ---------------------------------------------------------------------------
// counting sort by BMU
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(512) k_hist(const uint32_t* __restrict__ bmu, uint64_t n,
                                              uint32_t P, uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t hist[];
    for (uint32_t b = threadIdx.x; b < P; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint64_t r0 = (uint64_t)blockIdx.x * kHistRows;
    const uint64_t r1 = r0 + kHistRows < n ? r0 + kHistRows : n;
    for (uint64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) atomicAdd(&hist[bmu[i]], 1u);
    __syncthreads();
    uint32_t* out = counts + (size_t)blockIdx.x * P;
    for (uint32_t b = threadIdx.x; b < P; b += blockDim.x) out[b] = hist[b];
}

// counts[blk][b] -> exclusive prefix over blk (per node b); totals[b].
// Block = 32 nodes x 8 block-segments: segment sums, scan over segments, rewrite.
__global__ void __launch_bounds__(256) k_colscan(uint32_t* __restrict__ counts, uint32_t nblk,
                                                 uint32_t P, uint32_t* __restrict__ totals) {
    __shared__ uint32_t seg[8][33];
    const uint32_t tn = threadIdx.x & 31, sg = threadIdx.x >> 5;
    const uint32_t b = blockIdx.x * 32 + tn;
    const uint32_t per = (nblk + 7) / 8;
    const uint32_t s0 = sg * per, s1 = min(nblk, s0 + per);
    uint32_t sum = 0;
    if (b < P) {
        uint32_t k = s0;
        for (; k + 8 <= s1; k += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = counts[(size_t)(k + u) * P + b];
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += v[u];
        }
        for (; k < s1; ++k) sum += counts[(size_t)k * P + b];
    }
    seg[sg][tn] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t q = 0; q < sg; ++q) run += seg[q][tn];
    if (b < P) {
        if (sg == 7) totals[b] = run + sum;
        uint32_t k = s0;
        for (; k + 8 <= s1; k += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = counts[(size_t)(k + u) * P + b];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                counts[(size_t)(k + u) * P + b] = run;
                run += v[u];
            }
        }
        for (; k < s1; ++k) {
            const uint32_t v = counts[(size_t)k * P + b];
            counts[(size_t)k * P + b] = run;
            run += v;
        }
    }
}

// node_start[b] (exclusive scan of totals), piece_start[b], piece_node[], and
// the counts c_b into the sums buffer.  One block of 1024 threads.
__global__ void __launch_bounds__(1024) k_nodescan(const uint32_t* __restrict__ totals, uint32_t P,
                                                   uint32_t D, uint32_t* __restrict__ node_start,
                                                   uint32_t* __restrict__ piece_start,
                                                   uint32_t* __restrict__ piece_node,
                                                   double* __restrict__ sums, int add_counts,
                                                   int zero_dsum) {
    __shared__ uint32_t s_rows[1024], s_pcs[1024];
    __shared__ uint32_t carry_rows, carry_pcs;
    if (threadIdx.x == 0) {
        carry_rows = 0;
        carry_pcs = 0;
        if (zero_dsum) sums[(size_t)P * D + P] = 0.0;  // no distances this pass
    }
    __syncthreads();
    for (uint32_t base = 0; base < P; base += 1024) {
        const uint32_t b = base + threadIdx.x;
        const uint32_t t = b < P ? totals[b] : 0u;
        const uint32_t pc = (t + kPieceRows - 1) / kPieceRows;
        s_rows[threadIdx.x] = t;
        s_pcs[threadIdx.x] = pc;
        __syncthreads();
        for (uint32_t off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
            uint32_t a = 0, c = 0;
            if (threadIdx.x >= off) {
                a = s_rows[threadIdx.x - off];
                c = s_pcs[threadIdx.x - off];
            }
            __syncthreads();
            s_rows[threadIdx.x] += a;
            s_pcs[threadIdx.x] += c;
            __syncthreads();
        }
        const uint32_t ns = carry_rows + s_rows[threadIdx.x] - t;
        const uint32_t ps = carry_pcs + s_pcs[threadIdx.x] - pc;
        if (b < P) {
            node_start[b] = ns;
            piece_start[b] = ps;
            double* cb = sums + (size_t)P * D + b;
            *cb = add_counts ? *cb + (double)t : (double)t;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry_rows += s_rows[1023];
            carry_pcs += s_pcs[1023];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        node_start[P] = carry_rows;
        piece_start[P] = carry_pcs;
    }
}

// piece -> node table: thread per piece, binary search in piece_start (a node
// with many rows would otherwise write its hundreds of entries serially)
__global__ void k_piece_nodes(const uint32_t* __restrict__ piece_start, uint32_t P,
                              uint32_t max_pieces, uint32_t* __restrict__ piece_node) {
    const uint32_t np = piece_start[P];
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < np && p < max_pieces;
         p += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = P;  // last b with piece_start[b] <= p
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (piece_start[mid] <= p) lo = mid;
            else hi = mid;
        }
        piece_node[p] = lo;
    }
}

// Stable scatter of positions into BMU order (ties in position order).
// Each lane loads its 64 BMUs of the warp's 2048-row sub-chunk once, up front
// (one memory latency instead of one per 32-row step), counts them into the
// warp's shared-memory histogram, and after the block's prefix places them
// with __match_any_sync ranks from the same registers.
// (Measured and reverted: ordering a block's 16384 positions by node in shared
// memory first and writing node runs out whole — 125 us vs 79 us at 1e7 rows:
// the larger block footprint halves the resident blocks.)
constexpr int kScatterPer = kHistRows / kScatterWarps / 32;  // BMUs per lane (64)
__global__ void __launch_bounds__(kScatterWarps * 32) k_scatter(
    const uint32_t* __restrict__ bmu, uint64_t n, uint32_t P, const uint32_t* __restrict__ offs,
    const uint32_t* __restrict__ node_start, uint32_t* __restrict__ sorted) {
    // only the per-warp histograms live in shared memory (32 KB at P = 1024),
    // so ~7 blocks fit an SM and the whole grid runs in one wave
    extern __shared__ uint32_t whist[];  // [kScatterWarps][P]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t r0 = (uint64_t)blockIdx.x * kHistRows;
    for (uint32_t e = threadIdx.x; e < kScatterWarps * P; e += blockDim.x) whist[e] = 0;
    const uint32_t sub = kHistRows / kScatterWarps;
    const uint64_t w0 = r0 + (uint64_t)warp * sub;
    uint32_t v[kScatterPer];
#pragma unroll
    for (int m = 0; m < kScatterPer; ++m) {
        const uint64_t i = w0 + 32u * m + lane;
        v[m] = i < n ? __ldg(bmu + i) : 0xFFFFFFFFu;
    }
    __syncthreads();
    uint32_t* mine = whist + (size_t)warp * P;
#pragma unroll
    for (int m = 0; m < kScatterPer; ++m)
        if (v[m] != 0xFFFFFFFFu) atomicAdd(&mine[v[m]], 1u);
    __syncthreads();
    const uint32_t* boff = offs + (size_t)blockIdx.x * P;
    for (uint32_t b = threadIdx.x; b < P; b += blockDim.x) {
        uint32_t run = node_start[b] + boff[b];
        for (int w = 0; w < kScatterWarps; ++w) {
            const uint32_t c = whist[(size_t)w * P + b];
            whist[(size_t)w * P + b] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < kScatterPer; ++m) {
        const uint32_t b = v[m];
        const bool valid = b != 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, b);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        if (valid) sorted[mine[b] + rank] = (uint32_t)(w0 + 32u * m + lane);
        __syncwarp();
        if (valid && rank == 0) mine[b] += __popc(peers);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// gather + FP64 accumulation per piece
// ---------------------------------------------------------------------------

// Generic gather (any d <= 256): lane l owns features l, l+32, ... (NQ slots),
// rows loaded through registers in batches of 8.  partial[p][k] (k < D) =
// sum over the piece's rows of x_k in FP64; partial[p][D] = sum of exact
// distances (when requested).
template <int NQ>
__global__ void __launch_bounds__(256) k_gather_any(
    const float* __restrict__ x, const uint32_t* __restrict__ sel, const float* __restrict__ w,
    uint32_t P, uint32_t D, const uint32_t* __restrict__ sorted,
    const uint32_t* __restrict__ node_start, const uint32_t* __restrict__ piece_start,
    const uint32_t* __restrict__ piece_node, double* __restrict__ partial,
    double* __restrict__ dist_out, int want_dist, int accumulate) {
    constexpr int B = 8;
    const int lane = threadIdx.x & 31;
    const uint32_t npieces = piece_start[P];
    const uint32_t Dp = D + 1;
    for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < npieces;
         p += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t b = piece_node[p];
        const uint32_t r0 = node_start[b] + (p - piece_start[b]) * kPieceRows;
        const uint32_t r1 = min(r0 + kPieceRows, node_start[b + 1]);
        const float* wb = w + (size_t)b * D;
        double wv[NQ], acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const uint32_t k = lane + 32 * q;
            wv[q] = k < D ? (double)wb[k] : 0.0;
            acc[q] = 0.0;
        }
        double ds = 0.0;
        for (uint32_t r = r0; r < r1; r += 32) {
            const uint32_t mrow = min(32u, r1 - r);
            uint32_t mypos = 0;
            uint64_t myrow = 0;
            if (lane < (int)mrow) {
                mypos = sorted[r + lane];
                myrow = sel ? (uint64_t)sel[mypos] : (uint64_t)mypos;
            }
            for (uint32_t j0 = 0; j0 < mrow; j0 += B) {
                float xv[B][NQ];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const uint64_t row = __shfl_sync(0xffffffffu, myrow, (j0 + j) & 31);
                    const float* xr = x + row * D;
                    const bool ok = j0 + j < mrow;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const uint32_t k = lane + 32 * q;
                        xv[j][q] = (ok && k < D) ? __ldg(xr + k) : 0.0f;
                    }
                }
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    if (j0 + j < mrow) {
                        double d2 = 0.0;
#pragma unroll
                        for (int q = 0; q < NQ; ++q) {
                            acc[q] += (double)xv[j][q];
                            if (want_dist && lane + 32 * q < D) {
                                const double dd = (double)xv[j][q] - wv[q];
                                d2 = fma(dd, dd, d2);
                            }
                        }
                        if (want_dist) {
#pragma unroll
                            for (int o = 16; o; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
                            const double dist = sqrt(d2 > 0.0 ? d2 : 0.0);
                            const uint32_t pos = __shfl_sync(0xffffffffu, mypos, (j0 + j) & 31);
                            if (dist_out && lane == 0) dist_out[pos] = dist;
                            ds += dist;
                        }
                    }
                }
            }
        }
        double* out = partial + (size_t)p * Dp;
        if (accumulate) {
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (lane + 32 * q < D) out[lane + 32 * q] = acc[q];
        }
        if (lane == 0) out[D] = ds;
    }
}

// Async-copy gather: a warp copies 32 rows per batch into a double-buffered
// shared-memory ring with cp.async (LDGSTS, 8 bytes per lane: one instruction
// moves a whole 200-B row), so ~2 x 32 rows per warp are in flight without
// holding registers; then it accumulates S_b = sum x in FP64 registers.
// Requires d even (8-byte aligned rows).  partial[p][D] = sum of exact
// distances when requested (needs w_b: d = x - w).
constexpr int kAsyncWarps = 8;

__global__ void __launch_bounds__(kAsyncWarps * 32, 2) k_gather_async(
    const float* __restrict__ x, const uint32_t* __restrict__ sel, const float* __restrict__ w,
    uint32_t P, uint32_t D, const uint32_t* __restrict__ sorted,
    const uint32_t* __restrict__ node_start, const uint32_t* __restrict__ piece_start,
    const uint32_t* __restrict__ piece_node, double* __restrict__ partial,
    double* __restrict__ dist_out, int want_dist, int accumulate) {
    extern __shared__ __align__(16) float gbuf[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t rowf = D;                                   // floats per smem row
    float* buf = gbuf + (size_t)warp * 2 * 32 * rowf;          // [2][32][D]
    const uint32_t npieces = piece_start[P];
    const uint32_t Dp = D + 1;
    const uint32_t ka = 2 * lane, kb = 2 * lane + 1;
    const bool oka = ka < D, okb = kb < D;

    auto issue = [&](const uint64_t* rowaddr_reg, uint32_t nrows, int slot) {
        float* dst = buf + (size_t)slot * 32 * rowf;
        for (uint32_t j = 0; j < nrows; ++j) {
            const uint64_t a = __shfl_sync(0xffffffffu, *rowaddr_reg, j);
            if (okb) {
                const uint32_t sdst = (uint32_t)__cvta_generic_to_shared(dst + j * rowf + ka);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sdst),
                             "l"(a + 4ull * ka)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    for (uint32_t p = blockIdx.x * kAsyncWarps + warp; p < npieces; p += gridDim.x * kAsyncWarps) {
        const uint32_t b = piece_node[p];
        const uint32_t r0 = node_start[b] + (p - piece_start[b]) * kPieceRows;
        const uint32_t r1 = min(r0 + kPieceRows, node_start[b + 1]);
        const uint32_t nb = (r1 - r0 + 31) / 32;  // batches of 32 rows (<= 8)
        uint64_t addr[8];
        uint32_t pos[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const uint32_t r = r0 + 32 * m + lane;
            pos[m] = r < r1 ? sorted[r] : 0u;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const uint64_t row = sel ? (uint64_t)sel[pos[m]] : (uint64_t)pos[m];
            addr[m] = reinterpret_cast<uint64_t>(x + row * D);
        }
        double w0 = 0.0, w1 = 0.0;
        if (want_dist) {
            const float* wb = w + (size_t)b * D;
            w0 = oka ? (double)wb[ka] : 0.0;
            w1 = okb ? (double)wb[kb] : 0.0;
        }
        double a0 = 0.0, a1 = 0.0, ds = 0.0;
        issue(&addr[0], min(32u, r1 - r0), 0);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m < (int)nb) {
                const uint32_t rows_m = min(32u, r1 - (r0 + 32 * m));
                if (m + 1 < (int)nb) {
                    issue(&addr[m + 1], min(32u, r1 - (r0 + 32 * (m + 1))), (m + 1) & 1);
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                __syncwarp();
                const float* bm = buf + (size_t)(m & 1) * 32 * rowf;
#pragma unroll 4
                for (uint32_t j = 0; j < rows_m; ++j) {
                    float2 v = make_float2(0.0f, 0.0f);
                    if (okb) v = *reinterpret_cast<const float2*>(bm + j * rowf + ka);
                    a0 += (double)v.x;
                    a1 += (double)v.y;
                    if (want_dist) {
                        const double d0 = oka ? (double)v.x - w0 : 0.0;
                        const double d1 = okb ? (double)v.y - w1 : 0.0;
                        double d2 = fma(d0, d0, d1 * d1);
#pragma unroll
                        for (int o = 16; o; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
                        const double dist = sqrt(d2 > 0.0 ? d2 : 0.0);
                        const uint32_t pp = __shfl_sync(0xffffffffu, pos[m], j);
                        if (dist_out && lane == 0) dist_out[pp] = dist;
                        ds += dist;
                    }
                }
                __syncwarp();  // buffer m&1 may be refilled by the next issue
            }
        }
        double* out = partial + (size_t)p * Dp;
        if (accumulate) {
            if (oka) out[ka] = a0;
            if (okb) out[kb] = a1;
        }
        if (lane == 0) out[D] = ds;
    }
}

// TMA gather: lane l of a warp moves row l of a 32-row batch with one 1-D bulk
// copy (`cp.async.bulk`, the 16-byte-aligned window around the 8-byte-aligned
// row, into a 16-byte-aligned slot) completing on the batch's mbarrier; two
// batches in flight per warp.  One instruction moves 32 rows (the cp.async
// variant needs one per row plus the address shuffles), so the accumulation —
// four independent FP64 chains per lane — is what the warp spends its issue
// slots on.  Needs d even and readable slack after the last row (the window
// may extend up to 8 bytes past it).
constexpr int kTmaWarps = 8;

// kExact: every feature value and distance is put on a fixed-point grid fixed
// by the data's global bounds (exact_scales) and summed in int64 — exact and so
// order-independent: the sums do not depend on pieces, chunks or ranks.
template <bool kExact>
__global__ void __launch_bounds__(kTmaWarps * 32, 2) k_gather_tma(
    const float* __restrict__ x, uint32_t ldx, const uint32_t* __restrict__ sel,
    const float* __restrict__ w, uint32_t P, uint32_t D, uint32_t slot,
    const uint32_t* __restrict__ sorted,
    const uint32_t* __restrict__ node_start, const uint32_t* __restrict__ piece_start,
    const uint32_t* __restrict__ piece_node, double* __restrict__ partial,
    double* __restrict__ dist_out, int want_dist, int accumulate,
    const float* __restrict__ xmax2, const float* __restrict__ w2max) {
    extern __shared__ __align__(128) uint8_t tsm[];
    __shared__ __align__(8) uint64_t bars[kTmaWarps][2];
    __shared__ double wsm[kTmaWarps][64];  // w_b in FP64 for the distance pass (d <= 64)
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* buf = tsm + (size_t)warp * 2 * 32 * slot;
    if (lane == 0) {
        ptx::mbar_init(&bars[warp][0], 1);
        ptx::mbar_init(&bars[warp][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase = 0;  // bit s = parity to wait for on buffer s
    const uint32_t npieces = piece_start[P];
    const uint32_t Dp = D + 1;
    const uint32_t ka = 2 * lane, kb = 2 * lane + 1;
    const bool oka = ka < D, okb = kb < D;
    const uint32_t rowb = D * 4;                 // bytes of a row
    const uint64_t strideb = (uint64_t)ldx * 4;  // bytes between rows (D, or 64 padded)
    double sx = 0.0, sd = 0.0;
    if (kExact) exact_scales(xmax2, w2max, &sx, &sd);

    // Batch copy: every run of consecutive packed rows (the BMU-ordered
    // residency, keeps most of a node's rows in runs) is one bulk copy of
    // its 16-byte-aligned window, issued by the run's first lane into that
    // lane's slot; a run of k rows fits the k slots it starts (window <= 4dk
    // + 16 <= k slot for k >= 2).  Padded or scattered rows are runs of one.
    // roff = this lane's row's byte offset in buffer s; returns true when the
    // batch is a single run (rows at the row stride from lane 0's offset).
    auto issue = [&](uint64_t row, uint32_t nrows, int s, uint32_t& roff) -> bool {
        const bool mine = lane < nrows;
        const uint64_t a = reinterpret_cast<uint64_t>(x) + row * strideb;
        const uint64_t prev = __shfl_up_sync(0xffffffffu, row, 1);
        const bool lead = mine && !(lane > 0 && strideb == rowb && row == prev + 1);
        const uint32_t leads = __ballot_sync(0xffffffffu, lead);
        const uint32_t below = leads & (0xffffffffu >> (31 - lane));  // leaders <= lane
        const uint32_t l = 31 - __clz(below);                          // this row's run leader
        const uint32_t above = leads & ~(0xffffffffu >> (31 - lane));
        const uint32_t k = (above ? (uint32_t)__ffs(above) - 1 : nrows) - lane;  // run rows (leaders)
        const uint64_t c0 = a & ~15ull;
        const uint32_t len = lead ? (uint32_t)(((a + (uint64_t)k * rowb + 15) & ~15ull) - c0) : 0u;
        roff = l * slot + __shfl_sync(0xffffffffu, (uint32_t)(a & 15), l) + (lane - l) * rowb;
        const uint32_t total = __reduce_add_sync(0xffffffffu, len);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) ptx::mbar_expect_tx(&bars[warp][s], total);
        __syncwarp();
        if (lead)
            ptx::bulk_g2s(buf + ((size_t)s * 32 + lane) * slot, reinterpret_cast<const void*>(c0),
                          len, &bars[warp][s]);
        return leads == 1u;
    };

    for (uint32_t p = blockIdx.x * kTmaWarps + warp; p < npieces; p += gridDim.x * kTmaWarps) {
        const uint32_t b = piece_node[p];
        const uint32_t r0 = node_start[b] + (p - piece_start[b]) * kPieceRows;
        const uint32_t r1 = min(r0 + kPieceRows, node_start[b + 1]);
        const uint32_t nb = (r1 - r0 + 31) / 32;  // batches of 32 rows (<= 8)
        uint32_t pos[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const uint32_t r = r0 + 32 * m + lane;
            pos[m] = r < r1 ? sorted[r] : 0u;
        }
        uint64_t rowid[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) rowid[m] = sel ? (uint64_t)sel[pos[m]] : (uint64_t)pos[m];
        if (want_dist) {
            const float* wb = w + (size_t)b * D;
            __syncwarp();  // previous piece's distance pass done with wsm
            for (uint32_t k = lane; k < D; k += 32) wsm[warp][k] = (double)wb[k];
            __syncwarp();
        }
        double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0, ds = 0.0;
        long long qa0 = 0, qa1 = 0, qc0 = 0, qc1 = 0, qds = 0;
        uint32_t roff[2];
        bool one[2];
        one[0] = issue(rowid[0], min(32u, r1 - r0), 0, roff[0]);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m < (int)nb) {
                const uint32_t rows_m = min(32u, r1 - (r0 + 32 * m));
                const int s = m & 1;
                if (m + 1 < (int)nb)
                    one[s ^ 1] =
                        issue(rowid[m + 1], min(32u, r1 - (r0 + 32 * (m + 1))), s ^ 1, roff[s ^ 1]);
                ptx::mbar_wait(&bars[warp][s], (phase >> s) & 1u);
                phase ^= 1u << s;
                const uint8_t* bs = buf + (size_t)s * 32 * slot;
                // lanes past the row's features re-read feature pair 0 (their
                // sums are never stored): no per-row branch
                const uint8_t* bl = bs + (okb ? 8 * lane : 0u);
                auto add2 = [&](float2 u, float2 v) {
                    if (kExact) {
                        qa0 += __double2ll_rn((double)u.x * sx);
                        qa1 += __double2ll_rn((double)u.y * sx);
                        qc0 += __double2ll_rn((double)v.x * sx);
                        qc1 += __double2ll_rn((double)v.y * sx);
                    } else {
                        a0 += (double)u.x;
                        a1 += (double)u.y;
                        c0 += (double)v.x;
                        c1 += (double)v.y;
                    }
                };
                uint32_t j = 0;
                if (one[s]) {  // one run: row j at lane 0's offset + j rowb
                    const uint8_t* bm = bl + __shfl_sync(0xffffffffu, roff[s], 0);
                    for (; j + 2 <= rows_m; j += 2) {
                        add2(*reinterpret_cast<const float2*>(bm),
                             *reinterpret_cast<const float2*>(bm + rowb));
                        bm += 2 * rowb;
                    }
                } else {
                    for (; j + 2 <= rows_m; j += 2)
                        add2(*reinterpret_cast<const float2*>(bl + __shfl_sync(0xffffffffu, roff[s], j)),
                             *reinterpret_cast<const float2*>(
                                 bl + __shfl_sync(0xffffffffu, roff[s], j + 1)));
                }
                if (j < rows_m) {
                    const float2 u =
                        *reinterpret_cast<const float2*>(bl + __shfl_sync(0xffffffffu, roff[s], j));
                    if (kExact) {
                        qa0 += __double2ll_rn((double)u.x * sx);
                        qa1 += __double2ll_rn((double)u.y * sx);
                    } else {
                        a0 += (double)u.x;
                        a1 += (double)u.y;
                    }
                }
                if (want_dist && lane < rows_m) {
                    // lane = row: exact FP64 distance to w_b, features in order
                    // 8-byte reads (d is even): the 208-B slot stride then costs a
                    // 2-way bank conflict instead of the 4-way of 4-byte reads
                    const float2* xr = reinterpret_cast<const float2*>(bs + roff[s]);
                    double d2 = 0.0;
                    for (uint32_t k2 = 0; k2 < D / 2; ++k2) {
                        const float2 v = xr[k2];
                        const double d0 = (double)v.x - wsm[warp][2 * k2];
                        d2 = fma(d0, d0, d2);
                        const double d1 = (double)v.y - wsm[warp][2 * k2 + 1];
                        d2 = fma(d1, d1, d2);
                    }
                    const double dist = sqrt(d2);
                    if (dist_out) dist_out[pos[m]] = dist;
                    if (kExact) qds += __double2ll_rn(dist * sd);
                    else ds += dist;
                }
                __syncwarp();  // buffer s is refilled by the issue of batch m + 2
            }
        }
        double* out = partial + (size_t)p * Dp;
        if (kExact) {  // int64 partials (<= 256 rows x 2^54) in the double slots
            if (accumulate) {
                if (oka) out[ka] = __longlong_as_double(qa0 + qc0);
                if (okb) out[kb] = __longlong_as_double(qa1 + qc1);
            }
            if (want_dist) {
#pragma unroll
                for (int o = 16; o; o >>= 1) qds += __shfl_xor_sync(0xffffffffu, qds, o);
            }
            if (lane == 0) out[D] = __longlong_as_double(qds);
        } else {
            if (accumulate) {
                if (oka) out[ka] = a0 + c0;
                if (okb) out[kb] = a1 + c1;
            }
            if (want_dist) {
#pragma unroll
                for (int o = 16; o; o >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, o);
            }
            if (lane == 0) out[D] = ds;
        }
    }
}

// sums[b][k] (+)= sum over the pieces of node b: one warp per (b, k), lanes
// stride the node's pieces, fixed xor tree (deterministic, skew-proof)
__global__ void k_piece_reduce(const double* __restrict__ partial,
                               const uint32_t* __restrict__ piece_start, uint32_t P, uint32_t D,
                               double* __restrict__ sums, int add, double rows) {
    const size_t e = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the pass's row count (k_add_rowcount)
        double* t = sums + (size_t)P * D + P + 1;
        *t = add ? *t + rows : rows;
    }
    if (e >= (size_t)P * D) return;
    const uint32_t Dp = D + 1;
    const uint32_t b = (uint32_t)(e / D), k = (uint32_t)(e % D);
    const uint32_t p0 = piece_start[b], p1 = piece_start[b + 1];
    double q0 = 0.0, q1 = 0.0;
    uint32_t p = p0 + lane;
    for (; p + 32 < p1; p += 64) {
        q0 += partial[(size_t)p * Dp + k];
        q1 += partial[(size_t)(p + 32) * Dp + k];
    }
    if (p < p1) q0 += partial[(size_t)p * Dp + k];
    double v = q0 + q1;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sums[e] = add ? sums[e] + v : v;
}

// distance sum over all pieces: fixed strided partition + fixed tree (deterministic)
__global__ void __launch_bounds__(1024) k_dist_reduce(const double* __restrict__ partial,
                                                      const uint32_t* __restrict__ piece_start,
                                                      uint32_t P, uint32_t D,
                                                      double* __restrict__ sums, int add) {
    __shared__ double red[1024];
    const uint32_t np = piece_start[P], Dp = D + 1;
    double s = 0.0;
    for (uint32_t p = threadIdx.x; p < np; p += 1024) s += partial[(size_t)p * Dp + D];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int off = 512; off; off >>= 1) {
        if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* t = sums + (size_t)P * D + P;
        t[0] = add ? t[0] + red[0] : red[0];
    }
}

__global__ void k_add_rowcount(double* __restrict__ sums, uint32_t P, uint32_t D, double rows,
                               int add) {
    double* t = sums + (size_t)P * D + P + 1;
    *t = add ? *t + rows : rows;
}

// ---- exact mode: int128 sums as three int64 limbs of 42 / 42 / 44 bits ------
// (limbs of up to 2^20 ranks or chunks add in int64 without overflow; the
// reduce step is a plain int64 sum, then exact_unpack recombines)

__device__ __forceinline__ void to_limbs(__int128 v, long long* l) {
    const long long m = (1ll << 42) - 1;
    l[0] = (long long)(v & m);
    l[1] = (long long)((v >> 42) & m);
    l[2] = (long long)(v >> 84);
}
__device__ __forceinline__ __int128 from_limbs(const long long* l) {
    return ((__int128)l[2] << 84) + ((__int128)l[1] << 42) + (__int128)l[0];
}
__device__ __forceinline__ __int128 warp_sum_i128(__int128 v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, o);
        const long long hi = __shfl_xor_sync(0xffffffffu, (long long)(v >> 64), o);
        v += ((__int128)hi << 64) | (__int128)lo;
    }
    return v;
}

// xs[e] limbs (+)= sum over node b's pieces of the int64 partials, e = b*D + k
__global__ void k_piece_reduce_exact(const double* __restrict__ partial,
                                     const uint32_t* __restrict__ piece_start, uint32_t P,
                                     uint32_t D, long long* __restrict__ xs, int add) {
    const size_t e = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= (size_t)P * D) return;
    const uint32_t Dp = D + 1;
    const uint32_t b = (uint32_t)(e / D), k = (uint32_t)(e % D);
    const uint32_t p0 = piece_start[b], p1 = piece_start[b + 1];
    __int128 v = 0;
    for (uint32_t p = p0 + lane; p < p1; p += 32)
        v += (__int128)__double_as_longlong(partial[(size_t)p * Dp + k]);
    v = warp_sum_i128(v);
    if (lane == 0) {
        long long l[3];
        to_limbs(v, l);
        long long* o = xs + 3 * e;
        for (int i = 0; i < 3; ++i) o[i] = add ? o[i] + l[i] : l[i];
    }
}

__global__ void __launch_bounds__(1024) k_dist_reduce_exact(const double* __restrict__ partial,
                                                            const uint32_t* __restrict__ piece_start,
                                                            uint32_t P, uint32_t D,
                                                            long long* __restrict__ xs, int add) {
    __shared__ long long red[32][2];
    const uint32_t np = piece_start[P], Dp = D + 1;
    __int128 v = 0;
    for (uint32_t p = threadIdx.x; p < np; p += 1024)
        v += (__int128)__double_as_longlong(partial[(size_t)p * Dp + D]);
    v = warp_sum_i128(v);
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5][0] = (long long)(unsigned long long)v;
        red[threadIdx.x >> 5][1] = (long long)(v >> 64);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 t = 0;
        for (int w = 0; w < 32; ++w)
            t += ((__int128)red[w][1] << 64) | (__int128)(unsigned long long)red[w][0];
        long long l[3];
        to_limbs(t, l);
        long long* o = xs + 3 * (size_t)P * D;
        for (int i = 0; i < 3; ++i) o[i] = add ? o[i] + l[i] : l[i];
    }
}

// the counts and the row total (exact f64 integers) join the int64 buffer, so
// the epoch's one reduce is a single int64 sum
__global__ void k_exact_pack(const double* __restrict__ sums, uint32_t P, uint32_t D,
                             long long* __restrict__ xs) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    long long* t = xs + 3 * ((size_t)P * D + 1);
    if (b < P) t[b] = (long long)sums[(size_t)P * D + b];
    if (b == 0) t[P] = (long long)sums[(size_t)P * D + P + 1];
}

// back to the f64 sums layout [S | c | sum dist | rows] for K3: each exact sum
// converted once (round to nearest) and scaled back by a power of two
__global__ void k_exact_unpack(const long long* __restrict__ xs, uint32_t P, uint32_t D,
                               const float* __restrict__ xmax2, const float* __restrict__ w2max,
                               double* __restrict__ sums) {
    double sx, sd;
    exact_scales(xmax2, w2max, &sx, &sd);
    const size_t n = (size_t)P * D;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n + P + 2;
         e += (size_t)gridDim.x * blockDim.x) {
        if (e < n) {
            sums[e] = (double)from_limbs(xs + 3 * e) / sx;
        } else if (e < n + P) {
            sums[e] = (double)xs[3 * (n + 1) + (e - n)];
        } else if (e == n + P) {
            sums[e] = (double)from_limbs(xs + 3 * n) / sd;
        } else {
            sums[e] = (double)xs[3 * (n + 1) + P];
        }
    }
}

// ---------------------------------------------------------------------------

int g_gather_kind = 0;  // diagnostics (TSOM option 97): 1 = cp.async gather

__global__ void k_pad_rows(const float* __restrict__ x, uint64_t n, uint32_t D,
                           float* __restrict__ xpad) {
    const uint64_t total = n * kPadFloats;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / kPadFloats;
        const uint32_t k = (uint32_t)(e % kPadFloats);
        xpad[e] = k < D ? x[r * D + k] : 0.0f;
    }
}

void launch_pad_rows(const float* x, uint64_t n, uint32_t D, float* xpad, cudaStream_t st) {
    if (n == 0) return;
    TSOM_LAUNCH(k_pad_rows<<<148 * 16, 256, 0, st>>>(x, n, D, xpad));
}

int launch_accumulate(const float* x, const uint32_t* sel, uint64_t n, uint32_t D,
                       const float* w, uint32_t P, const uint32_t* bmu, double* dist_out,
                       bool want_dist_sum, bool accumulate, bool first, const AccumScratch& s,
                       double* sums, int sm_count, cudaStream_t st, bool x_slack,
                       uint32_t ldx, const ExactSums* exact) {
    if (ldx == 0) ldx = D;
    const int add = first ? 0 : 1;
    if (n == 0) {
        if (first) cudaMemsetAsync(sums, 0, ((size_t)P * D + P + 2) * sizeof(double), st);
        if (exact && first) {
            cudaMemsetAsync(exact->xs, 0, exact_sums_words(P, D) * sizeof(long long), st);
        }
        return 0;
    }
    const bool want_dist = dist_out != nullptr || want_dist_sum;
    if (!accumulate && !want_dist) {  // BMU only: nothing to gather
        if (first) cudaMemsetAsync(sums, 0, ((size_t)P * D + P + 2) * sizeof(double), st);
        TSOM_LAUNCH(k_add_rowcount<<<1, 1, 0, st>>>(sums, P, D, (double)n, add));
        if (exact) {
            if (!add) cudaMemsetAsync(exact->xs, 0, 3 * ((size_t)P * D + 1) * sizeof(long long), st);
            TSOM_LAUNCH(k_exact_pack<<<(P + 255) / 256, 256, 0, st>>>(sums, P, D, exact->xs));
        }
        return 0;
    }
    const uint32_t nblk = (uint32_t)accum_blocks(n);
    // dynamic smem beyond 48 KB (P up to ~7000 nodes)
    ensure_smem_attr((const void*)k_hist, (size_t)P * 4);
    ensure_smem_attr((const void*)k_scatter, (size_t)kScatterWarps * P * 4);
    TSOM_LAUNCH(k_hist<<<nblk, 512, P * sizeof(uint32_t), st>>>(bmu, n, P, s.counts));
    TSOM_LAUNCH(k_colscan<<<(P + 31) / 32, 256, 0, st>>>(s.counts, nblk, P, s.totals));
    TSOM_LAUNCH(k_nodescan<<<1, 1024, 0, st>>>(s.totals, P, D, s.node_start, s.piece_start,
                                               s.piece_node, sums, add,
                                               (!want_dist && first) ? 1 : 0));
    {
        const uint64_t pmax = accum_pieces_max(n, P);
        const unsigned pb = (unsigned)std::min<uint64_t>((pmax + 255) / 256, (uint64_t)sm_count * 4);
        TSOM_LAUNCH(k_piece_nodes<<<pb, 256, 0, st>>>(s.piece_start, P, (uint32_t)pmax,
                                                      s.piece_node));
    }
    TSOM_LAUNCH(k_scatter<<<nblk, kScatterWarps * 32, (size_t)kScatterWarps * P * sizeof(uint32_t),
                            st>>>(bmu, n, P, s.counts, s.node_start, s.sorted));
    const uint64_t pieces = accum_pieces_max(n, P);
    const uint64_t warps = pieces < (uint64_t)sm_count * 32 ? pieces : (uint64_t)sm_count * 32;
    const unsigned gblocks = (unsigned)((warps * 32 + 255) / 256);
    const bool v2 = (D % 2 == 0) && D <= 64 && ((reinterpret_cast<uintptr_t>(x) & 7u) == 0);
    const size_t asmem = (size_t)kAsyncWarps * 2 * 32 * D * sizeof(float);
    const uint32_t slot = (D * 4 + 8 + 15) / 16 * 16;  // longest 16-B window of a row
    const size_t tsmem = (size_t)kTmaWarps * 2 * 32 * slot;
    // padded rows (a 256-B stride, line aligned): a row is exactly two 128-B
    // lines instead of two or three; only the TMA gather reads strided rows
    const bool use_pad = ldx != D;
    const bool tma = use_pad ||
        (v2 && x_slack && g_gather_kind == 0 && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) &&
         tsmem <= 110 * 1024);
    if (exact && !tma) return 1;  // exact sums need the TMA row gather (d even, <= 62)
    if (tma) {
        const uint64_t tblocks = (pieces + kTmaWarps - 1) / kTmaWarps;
        const unsigned tb = (unsigned)(tblocks < (uint64_t)sm_count * 2 ? tblocks : sm_count * 2);
        if (exact) {
            ensure_smem_attr((const void*)k_gather_tma<true>, tsmem);
            TSOM_LAUNCH(k_gather_tma<true><<<tb, kTmaWarps * 32, tsmem, st>>>(
                x, ldx, sel, w, P, D, slot, s.sorted, s.node_start, s.piece_start, s.piece_node,
                s.partial, dist_out, want_dist ? 1 : 0, accumulate ? 1 : 0, exact->xmax2,
                exact->w2max));
        } else {
            ensure_smem_attr((const void*)k_gather_tma<false>, tsmem);
            TSOM_LAUNCH(k_gather_tma<false><<<tb, kTmaWarps * 32, tsmem, st>>>(
                x, ldx, sel, w, P, D, slot, s.sorted, s.node_start, s.piece_start, s.piece_node,
                s.partial, dist_out, want_dist ? 1 : 0, accumulate ? 1 : 0, nullptr, nullptr));
        }
    } else if (v2 && D <= 64 && asmem <= 110 * 1024) {
        ensure_smem_attr((const void*)k_gather_async, asmem);
        const uint64_t ablocks = (pieces + kAsyncWarps - 1) / kAsyncWarps;
        const unsigned ab = (unsigned)(ablocks < (uint64_t)sm_count * 2 ? ablocks : sm_count * 2);
        TSOM_LAUNCH(k_gather_async<<<ab, kAsyncWarps * 32, asmem, st>>>(
            x, sel, w, P, D, s.sorted, s.node_start, s.piece_start, s.piece_node, s.partial,
            dist_out, want_dist ? 1 : 0, accumulate ? 1 : 0));
    } else {
        const int nq = (int)((D + 31) / 32);
#define TSOM_GATHER_ANY(NQ)                                                                     \
    TSOM_LAUNCH(k_gather_any<NQ><<<gblocks, 256, 0, st>>>(                                     \
        x, sel, w, P, D, s.sorted, s.node_start, s.piece_start, s.piece_node, s.partial,       \
        dist_out, want_dist ? 1 : 0, accumulate ? 1 : 0))
        switch (nq) {
            case 1: TSOM_GATHER_ANY(1); break;
            case 2: TSOM_GATHER_ANY(2); break;
            case 3: TSOM_GATHER_ANY(3); break;
            case 4: TSOM_GATHER_ANY(4); break;
            case 5: TSOM_GATHER_ANY(5); break;
            case 6: TSOM_GATHER_ANY(6); break;
            case 7: TSOM_GATHER_ANY(7); break;
            default: TSOM_GATHER_ANY(8); break;
        }
#undef TSOM_GATHER_ANY
    }
    const size_t m = (size_t)P * D;
    if (exact) {
        // S and the distance sum exact in the int64 limb buffer (zero when not
        // produced), then counts and rows joined: the one reduce is on exact->xs
        if (accumulate)
            TSOM_LAUNCH(k_piece_reduce_exact<<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(
                s.partial, s.piece_start, P, D, exact->xs, add));
        else if (!add)
            cudaMemsetAsync(exact->xs, 0, 3 * m * sizeof(long long), st);
        if (want_dist)
            TSOM_LAUNCH(k_dist_reduce_exact<<<1, 1024, 0, st>>>(s.partial, s.piece_start, P, D,
                                                                 exact->xs, add));
        else if (!add)
            cudaMemsetAsync(exact->xs + 3 * m, 0, 3 * sizeof(long long), st);
        TSOM_LAUNCH(k_add_rowcount<<<1, 1, 0, st>>>(sums, P, D, (double)n, add));
        TSOM_LAUNCH(k_exact_pack<<<(P + 255) / 256, 256, 0, st>>>(sums, P, D, exact->xs));
        return 0;
    }
    if (accumulate)
        TSOM_LAUNCH(k_piece_reduce<<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(
            s.partial, s.piece_start, P, D, sums, add, (double)n));
    if (want_dist)
        TSOM_LAUNCH(k_dist_reduce<<<1, 1024, 0, st>>>(s.partial, s.piece_start, P, D, sums, add));
    if (!accumulate) TSOM_LAUNCH(k_add_rowcount<<<1, 1, 0, st>>>(sums, P, D, (double)n, add));
    return 0;
}

void launch_exact_unpack(const ExactSums& ex, uint32_t P, uint32_t D, double* sums,
                         cudaStream_t st) {
    TSOM_LAUNCH(k_exact_unpack<<<148, 256, 0, st>>>(ex.xs, P, D, ex.xmax2, ex.w2max, sums));
}

size_t exact_sums_words(uint32_t P, uint32_t D) { return 3 * ((size_t)P * D + 1) + P + 1; }

void accum_scratch_bytes(uint64_t n, uint32_t P, uint32_t D, size_t out[7]) {
    const uint64_t nblk = accum_blocks(n), pieces = accum_pieces_max(n, P);
    out[0] = (size_t)nblk * P * 4;           // counts / offsets
    out[1] = (size_t)P * 4;                  // totals
    out[2] = (size_t)(P + 1) * 4;            // node_start
    out[3] = (size_t)(P + 1) * 4;            // piece_start
    out[4] = (size_t)pieces * 4;             // piece_node
    out[5] = (size_t)(n ? n : 1) * 4;        // sorted positions
    out[6] = (size_t)pieces * (D + 1) * 8;   // piece partials
}

}  // namespace tsom

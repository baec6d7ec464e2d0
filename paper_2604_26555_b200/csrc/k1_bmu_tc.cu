// k1_bmu_tc.cu — K1: BMU search as a tcgen05 3xTF32 tile GEMM with a fused
// top-2 epilogue (the samples x codebook distance matrix never reaches HBM).
//
// For every row x and node j the kernel evaluates  v_j = ||w_j||^2 - 2 x.w_j
// (trainer.hpp:282-308 without the row-constant ||x||^2) as one augmented dot
// product  x'.w'  with  x' = [x, 1, 1, 0..]  and  w' = [-2w, p1+p2, p3, 0..]
// (k_bmu.cu: k_prep_codebook, k_split_rows), K padded to 56 = 7 tf32 k-steps.
// 3xTF32: x' = xh + xl, w' = wh + wl (xh, wh exact tf32), and
//   x'.w' ~= xh.wh + xl.wh + xh.wl          (xl.wl ~ 2^-22 relative, dropped)
// accumulated in FP32 in TMEM.  Rows whose best/second-best gap falls inside
// the error window are re-checked in exact FP64 (k_rescan), so BMU indices are
// bit-identical to the reference.
//
// Work split: the codebook is cut into groups of gn <= 256 nodes.  A CTA keeps
// one group resident in shared memory (hi|lo, 2 * 14 * gn * 16 B) for its
// whole life and streams 128-row sample tiles (hi|lo, 57,344 B) through a
// 2-stage cp.async.bulk pipeline.  Warp roles (256 threads):
//   warp 0      : producer — bulk copies (mbarrier complete_tx)
//   warp 1      : MMA issuer — one elected thread, 21 tcgen05.mma per tile
//                 (M=128 rows x N=gn nodes x K=8, three products x 7 k-steps)
//   warp 2      : TMEM allocator (2 accumulator buffers x gn columns)
//   warps 4..7  : epilogue — warp q+4 owns TMEM lanes 32q.. (tile rows) and all
//                 columns; pipelined tcgen05.ld x32, eight independent top-2
//                 streams per thread, candidate enumeration for near-ties
// Samples sit on the TMEM lane axis, so no cross-lane reduction is needed.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "engine.h"

namespace tsom {

namespace {

constexpr int kThreads = 384;          // 4 role warps + 2 sets x 4 epilogue warps
constexpr uint32_t kEpiThreads = 128;   // arrivals per accumulator buffer (one set)
constexpr int kStages = 2;
constexpr uint32_t kTileBytes = 2u * kTcTileM * kTcKPad * 4u;  // 57,344 (hi + lo)
constexpr uint32_t kHalfTile = kTcTileM * kTcKPad * 4u;         // 28,672
constexpr int kKSteps = kTcKPad / 8;                             // 7

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (cute::UMMA::SmemDescriptor):
// [0,14) start>>4, [16,30) LBO>>4 (k-core stride), [32,46) SBO>>4 (8-row stride),
// [46,48) version = 1, [61,64) layout = SWIZZLE_NONE.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    return d;
}

// Instruction descriptor for kind::tf32: D = F32, A = B = TF32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
        "}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define TMEM_LD32(taddr, r)                                                                      \
    asm volatile(                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),            \
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),         \
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),         \
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),         \
          "=r"(r[31])                                                                            \
        : "r"(taddr))

#define TMEM_LD16(taddr, r)                                                                      \
    asm volatile(                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15}, [%16];"                                                                       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),            \
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                                                  \
        : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

}  // namespace

// branch-free top-2 step: strict < keeps the earliest j on ties, an exact tie
// lands in b2 (gap 0 => candidate enumeration)
__device__ __forceinline__ void top2_step(float v, uint32_t j, float& b1, uint32_t& i1,
                                          float& b2) {
    const float nb1 = fminf(b1, v);
    b2 = fminf(b2, fmaxf(b1, v));
    i1 = v < b1 ? j : i1;
    b1 = nb1;
}

__device__ __forceinline__ void top2_merge_dev(float& b1, uint32_t& i1, float& b2, float ob1,
                                               uint32_t oi1, float ob2) {
    if (ob1 < b1 || (ob1 == b1 && oi1 < i1)) {
        b2 = fminf(b1, ob2);
        b1 = ob1;
        i1 = oi1;
    } else {
        b2 = fminf(b2, ob1);
    }
}

// Candidate list of one (row, group): up to 4 local node indices (8 bits each)
// whose computed value lies within thr of the group's best; count 15 = overflow.
constexpr uint32_t kCandOverflow = 15u;

// kEnum = false (main pass): per (row, group) the top-2 (b1, i1, b2) only.
// kEnum = true (near-tie rows only, see k_merge_fast): per (row, group) the best
// value plus up to 8 local candidate ids within thr of it (count 15 = overflow),
// enumerated only in the groups flagged relevant for the row (rmask).
// dev_n (optional): row count read on the device (the near-tie list length).
template <bool kEnum>
__global__ void __launch_bounds__(kThreads, 1)
    k1_bmu_tc(const float* __restrict__ tiles, uint64_t n_host, const uint32_t* __restrict__ dev_n,
              uint32_t groups, uint32_t gn, const float* __restrict__ wsplit,
              const float* __restrict__ xn2, const float* __restrict__ w2max, float tau,
              const uint32_t* __restrict__ rmask, float* __restrict__ part) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint64_t n = dev_n ? min((uint64_t)*dev_n, n_host) : n_host;  // n_host caps dev_n
    const uint32_t ntiles = (uint32_t)((n + kTcTileM - 1) / kTcTileM);
    const uint32_t w_bytes = 2u * kTcKPad * gn * 4u;  // hi + lo of this CTA's group
    uint8_t* sW = smem;
    uint8_t* sX = smem + ((w_bytes + 1023u) & ~1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + kStages * kTileBytes);
    uint64_t* full_bar = bars;        // [kStages] X tile landed
    uint64_t* empty_bar = bars + 2;   // [kStages] MMAs done with X tile
    uint64_t* tfull_bar = bars + 4;   // [2] accumulator ready
    uint64_t* tempty_bar = bars + 6;  // [2] accumulator drained
    uint64_t* w_bar = bars + 8;       // codebook group landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g = blockIdx.x % groups;
    const uint32_t cta_in_group = blockIdx.x / groups;
    const uint32_t ctas_per_group = gridDim.x / groups;
    const uint32_t acc_cols = gn <= 32 ? 32 : (gn <= 64 ? 64 : (gn <= 128 ? 128 : 256));

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull_bar[a], 1);
            mbar_init(&tempty_bar[a], kEpiThreads);
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
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0 && ntiles > cta_in_group) {
            // resident codebook group (hi and lo halves, each < 2^20 B of tx count)
            mbar_expect_tx(w_bar, w_bytes);
            const float* wg = wsplit + (size_t)g * 2 * kTcKPad * gn;
            bulk_g2s(sW, wg, w_bytes / 2, w_bar);
            bulk_g2s(sW + w_bytes / 2, wg + (size_t)kTcKPad * gn, w_bytes / 2, w_bar);
            uint32_t stage = 0, phase = 0;
            for (uint32_t t = cta_in_group; t < ntiles; t += ctas_per_group) {
                mbar_wait(&empty_bar[stage], phase ^ 1);
                mbar_expect_tx(&full_bar[stage], kTileBytes);
                bulk_g2s(sX + stage * kTileBytes, tiles + (size_t)t * (kTileBytes / 4), kTileBytes,
                         &full_bar[stage]);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && ntiles > cta_in_group) {
            const uint32_t idesc = idesc_tf32(kTcTileM, gn);
            const uint32_t w_lbo = gn * 16u;
            const uint32_t sw = smem_u32(sW);
            const uint32_t sw_lo = sw + w_bytes / 2;
            mbar_wait(w_bar, 0);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            for (uint32_t t = cta_in_group; t < ntiles; t += ctas_per_group) {
                mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * acc_cols;
                const uint32_t sx = smem_u32(sX + stage * kTileBytes);
                const uint32_t sx_lo = sx + kHalfTile;
#pragma unroll
                for (int k = 0; k < kKSteps; ++k) {
                    const uint64_t ah = umma_desc(sx + k * 4096u, 2048u, 128u);
                    const uint64_t al = umma_desc(sx_lo + k * 4096u, 2048u, 128u);
                    const uint64_t bh = umma_desc(sw + k * 2u * w_lbo, w_lbo, 128u);
                    const uint64_t bl = umma_desc(sw_lo + k * 2u * w_lbo, w_lbo, 128u);
                    mma_tf32(d, ah, bh, idesc, k > 0 ? 1u : 0u);
                    mma_tf32(d, al, bh, idesc, 1u);
                    mma_tf32(d, ah, bl, idesc, 1u);
                }
                mma_commit(&empty_bar[stage]);  // X stage free once these MMAs retire
                mma_commit(&tfull_bar[acc]);    // accumulator ready for the epilogue
                if (++stage == kStages) {
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
        // 2 sets x 4 epilogue warps: set s drains accumulator buffer s (every
        // other tile), so two warps per SM sub-partition hide each other's
        // latency without exchanging anything.  Warp (set, q) owns TMEM lanes
        // 32q..32q+31 (= tile rows) and all gn columns; thread = row.
        const uint32_t q = warp & 3, set = (warp - 4) >> 2;
        const uint32_t row = q * 32 + lane;
        const uint32_t nfull = gn / 32, tail16 = (gn % 32) != 0;
        const uint32_t acc = set;
        uint32_t acc_phase = 0;
        for (uint32_t t = cta_in_group + set * ctas_per_group; t < ntiles;
             t += 2 * ctas_per_group) {
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * acc_cols;
            // pass 1: eight independent top-2 streams (ILP), TMEM loads pipelined
            float b1[8], b2[8];
            uint32_t i1[8];
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2) {
                b1[s2] = CUDART_INF_F;
                b2[s2] = CUDART_INF_F;
                i1[s2] = 0;
            }
            uint32_t ra[32], rb[32];
            if (nfull) TMEM_LD32(taddr, ra);
            for (uint32_t c = 0; c < nfull; c += 2) {
                tmem_wait_ld();
                if (c + 1 < nfull) TMEM_LD32(taddr + (c + 1) * 32, rb);
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    top2_step(__uint_as_float(ra[k]), c * 32 + k, b1[k & 7], i1[k & 7], b2[k & 7]);
                if (c + 1 < nfull) {
                    tmem_wait_ld();
                    if (c + 2 < nfull) TMEM_LD32(taddr + (c + 2) * 32, ra);
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        top2_step(__uint_as_float(rb[k]), (c + 1) * 32 + k, b1[k & 7], i1[k & 7],
                                  b2[k & 7]);
                }
            }
            if (tail16) {
                uint32_t r[16];
                TMEM_LD16(taddr + nfull * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    top2_step(__uint_as_float(r[k]), nfull * 32 + k, b1[k & 7], i1[k & 7], b2[k & 7]);
            }
#pragma unroll
            for (int s2 = 1; s2 < 8; ++s2)
                top2_merge_dev(b1[0], i1[0], b2[0], b1[s2], i1[s2], b2[s2]);
            const float B1 = b1[0], B2 = b2[0];
            const uint32_t I1 = i1[0];
            uint32_t w1 = I1, w2 = __float_as_uint(B2), w3 = 1;
            if (kEnum) {
                // enumerate the row's candidates v <= B1 + thr in ascending j
                const uint64_t prow = (uint64_t)t * kTcTileM + row;
                const bool relevant = prow < n && ((__ldg(rmask + prow) >> (g & 31)) & 1u);
                const float thr = relevant ? tau * (__ldg(xn2 + prow) + __ldg(w2max)) : 0.0f;
                const bool need = relevant && !(B2 - B1 > thr);
                w2 = 0;
                if (__any_sync(0xffffffffu, need)) {
                    const float lim = B1 + thr;
                    uint32_t pk0 = 0, pk1 = 0, nc = 0;
                    for (uint32_t cc = 0; cc < gn; cc += 16) {
                        uint32_t r[16];
                        TMEM_LD16(taddr + cc, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            if (need && __uint_as_float(r[k]) <= lim) {
                                const uint32_t id = (cc + k) << (8 * (nc & 3));
                                if (nc < 4) pk0 |= id;
                                else if (nc < 8) pk1 |= id;
                                ++nc;
                            }
                        }
                    }
                    if (need) {
                        w1 = pk0;
                        w2 = pk1;
                        w3 = (nc >= 1 && nc <= 8) ? nc : kCandOverflow;
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty_bar[acc]);  // this thread is done with the accumulator
            const uint64_t pos = (uint64_t)t * kTcTileM + row;
            if (pos < n) {
                float* pg = part + (size_t)g * (kEnum ? 4 : 3) * n;
                pg[pos] = B1;
                pg[n + pos] = __uint_as_float(w1);
                pg[2 * n + pos] = __uint_as_float(w2);
                if (kEnum) pg[3 * n + pos] = __uint_as_float(w3);
            }
            acc_phase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(2 * acc_cols));
    }
}

bool tc_supported(uint32_t P, uint32_t D) { return P >= 1 && D + 2 <= (uint32_t)kTcKPad; }

cudaError_t launch_bmu_tc(const float* tiles, uint64_t n, const uint32_t* dev_n, bool enumerate,
                          uint32_t P, const float* wsplit, const float* xn2,
                          const float* w2max, float tau, const uint32_t* rmask, float* part,
                          int sm_count, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint32_t gn = tc_group_width(P);
    const uint32_t groups = (P + gn - 1) / gn;
    const uint32_t ntiles = (uint32_t)((n + kTcTileM - 1) / kTcTileM);  // upper bound
    uint32_t per_group = (uint32_t)sm_count / groups;
    if (per_group < 1) per_group = 1;
    if (per_group > ntiles) per_group = ntiles;
    const uint32_t grid = per_group * groups;
    const uint32_t w_bytes = 2u * kTcKPad * gn * 4u;
    const size_t smem = ((w_bytes + 1023u) & ~1023u) + kStages * kTileBytes + 80;
    auto kern = enumerate ? k1_bmu_tc<true> : k1_bmu_tc<false>;
    static size_t attr[2] = {0, 0};
    if (attr[enumerate] < smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr[enumerate] = smem;
    }
    TSOM_LAUNCH(kern<<<grid, kThreads, smem, st>>>(tiles, n, dev_n, groups, gn, wsplit, xn2,
                                                   w2max, tau, rmask, part));
    return cudaGetLastError();
}

}  // namespace tsom

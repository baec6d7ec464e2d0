// k_order.cu — BMU-ordered residency of the bound rows (TSOM_OPT_ROW_ORDER,
// DESIGN.md §3-§4).  After a full pass, the resident rows are re-laid out in
// that pass's BMU order (K2's counting-sort output): rows that share a BMU sit
// next to each other, so K1's epilogue skips the column chunks no row of a warp
// needs and K2 gathers each node's rows with one bulk copy per 32 rows.  The
// engine keeps perm (position -> caller row id) and pinv (its inverse); every
// call still speaks caller row ids: selections are mapped through pinv,
// per-row outputs of full passes scattered back through perm.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace tsom {
namespace {

// dst row q (packed, D floats) = src row sorted[q] (stride ldx); perm_out[q] =
// perm_in[sorted[q]] (perm_in == nullptr: the identity; perm_out optional).  One warp per row
// group: lanes copy 8-byte pieces (d even) or floats.
__global__ void k_permute_rows(const float* __restrict__ src, uint32_t ldx,
                               const uint32_t* __restrict__ sorted, uint64_t n, uint32_t D,
                               float* __restrict__ dst, const uint32_t* __restrict__ perm_in,
                               uint32_t* __restrict__ perm_out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t q = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; q < n; q += warps) {
        const uint32_t r = __ldg(sorted + q);
        if (lane == 0 && perm_out) perm_out[q] = perm_in ? __ldg(perm_in + r) : r;
        const float* s = src + (uint64_t)r * ldx;
        float* d = dst + q * D;
        if ((D & 1u) == 0 && (ldx & 1u) == 0) {
            const float2* s2 = reinterpret_cast<const float2*>(s);
            float2* d2 = reinterpret_cast<float2*>(d);
            for (uint32_t k = lane; k < D / 2; k += 32) d2[k] = __ldg(s2 + k);
        } else {
            for (uint32_t k = lane; k < D; k += 32) d[k] = __ldg(s + k);
        }
    }
}

__global__ void k_invert(const uint32_t* __restrict__ perm, uint64_t n, uint32_t* __restrict__ pinv) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x)
        pinv[perm[q]] = (uint32_t)q;
}

// out[i] = pinv[sel[i]]: caller row ids -> positions
__global__ void k_map_ids(const uint32_t* __restrict__ sel, uint64_t n,
                          const uint32_t* __restrict__ pinv, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = __ldg(pinv + __ldg(sel + i));
}

// out[perm[q]] = v[q]: per-position values -> caller row order
template <typename T>
__global__ void k_unpermute(const T* __restrict__ v, const uint32_t* __restrict__ perm, uint64_t n,
                            T* __restrict__ out) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x)
        out[__ldg(perm + q)] = v[q];
}

unsigned grid_for(uint64_t n, int per_block) {
    const uint64_t b = (n + per_block - 1) / per_block;
    return (unsigned)(b < 148u * 16u ? (b ? b : 1) : 148u * 16u);
}

}  // namespace

void launch_permute_rows(const float* src, uint32_t ldx, const uint32_t* sorted, uint64_t n,
                         uint32_t D, float* dst, const uint32_t* perm_in, uint32_t* perm_out,
                         cudaStream_t st) {
    if (n == 0) return;
    TSOM_LAUNCH(k_permute_rows<<<grid_for(n, 8), 256, 0, st>>>(src, ldx, sorted, n, D, dst,
                                                               perm_in, perm_out));
}

void launch_invert_perm(const uint32_t* perm, uint64_t n, uint32_t* pinv, cudaStream_t st) {
    if (n == 0) return;
    TSOM_LAUNCH(k_invert<<<grid_for(n, 256), 256, 0, st>>>(perm, n, pinv));
}

void launch_map_ids(const uint32_t* sel, uint64_t n, const uint32_t* pinv, uint32_t* out,
                    cudaStream_t st) {
    if (n == 0) return;
    TSOM_LAUNCH(k_map_ids<<<grid_for(n, 256), 256, 0, st>>>(sel, n, pinv, out));
}

void launch_unpermute_u32(const uint32_t* v, const uint32_t* perm, uint64_t n, uint32_t* out,
                          cudaStream_t st) {
    if (n == 0) return;
    TSOM_LAUNCH(k_unpermute<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(v, perm, n, out));
}

void launch_unpermute_f64(const double* v, const uint32_t* perm, uint64_t n, double* out,
                          cudaStream_t st) {
    if (n == 0) return;
    TSOM_LAUNCH(k_unpermute<double><<<grid_for(n, 256), 256, 0, st>>>(v, perm, n, out));
}

}  // namespace tsom

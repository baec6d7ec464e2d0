// k_topology.cu — topology refresh on the device.
//
// The reference rebuilds the neighbourhood graph from the current codebook
// (refresh_topology, topology.hpp:439-451):
//   pairwise_sq_dists  topology.hpp:81-108   FP64 Gram, sequential k, clamp at 0
//   build_mst          topology.hpp:192-220  Kruskal, ties in (w, i, j) order
//   build_rng_graph    topology.hpp:229-258  strict blocker test max(d_ar, d_br) < d_ab
//   hop_distances      topology.hpp:292-325  all-pairs shortest hop counts (u16)
// Every value here is bit-identical to the reference:
//   * the Gram is evaluated with the reference's operation order and no
//     contraction (__dmul_rn / __dadd_rn), so d2[i][j] == d2[j][i] exactly;
//   * the MST under the strict total order (w, i, j) is unique, so Boruvka
//     (what runs here) returns Kruskal's tree;
//   * the RNG predicate is an OR over witnesses, independent of tiling;
//   * BFS from every source gives the same shortest hop counts as the
//     blocked Floyd-Warshall.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "engine.h"

namespace tsom {

// norms[i] = sum_k w_ik^2 (sequential, no FMA), topology.hpp:85-91
__global__ void k_gram_norms(const float* __restrict__ w, uint32_t P, uint32_t D,
                             double* __restrict__ norms) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const float* wi = w + (size_t)i * D;
    double s = 0.0;
    for (uint32_t k = 0; k < D; ++k) s = __dadd_rn(s, __dmul_rn((double)wi[k], (double)wi[k]));
    norms[i] = s;
}

// d2[i][j] = max(0, n_i + n_j - 2 dot(w_i, w_j)), diagonal exactly 0 (:93-106).
// Block: 32 x 8 threads over a 32 x 32 (i, j) tile, codebook rows staged in smem.
__global__ void __launch_bounds__(256) k_gram(const float* __restrict__ w, uint32_t P, uint32_t D,
                                              const double* __restrict__ norms,
                                              double* __restrict__ d2) {
    extern __shared__ float gs[];
    float* wi_s = gs;             // [32][D]
    float* wj_s = gs + 32 * D;    // [32][D]
    const uint32_t i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    for (uint32_t e = threadIdx.x; e < 32 * D; e += 256) {
        const uint32_t r = e / D, k = e % D;
        wi_s[e] = i0 + r < P ? w[(size_t)(i0 + r) * D + k] : 0.0f;
        wj_s[e] = j0 + r < P ? w[(size_t)(j0 + r) * D + k] : 0.0f;
    }
    __syncthreads();
    const uint32_t tj = threadIdx.x & 31, ti = threadIdx.x >> 5;
    const uint32_t j = j0 + tj;
    for (uint32_t ii = ti; ii < 32; ii += 8) {
        const uint32_t i = i0 + ii;
        if (i >= P || j >= P) continue;
        if (i == j) {
            d2[(size_t)i * P + j] = 0.0;
            continue;
        }
        double dot = 0.0;
        for (uint32_t k = 0; k < D; ++k)
            dot = __dadd_rn(dot, __dmul_rn((double)wi_s[ii * D + k], (double)wj_s[tj * D + k]));
        const double v = __dsub_rn(__dadd_rn(norms[i], norms[j]), __dmul_rn(2.0, dot));
        d2[(size_t)i * P + j] = v > 0.0 ? v : 0.0;
    }
}

// ---------------------------------------------------------------------------
// MST: Boruvka in one CTA (P <= 4096), edge order (w, i, j) with i < j.
// ---------------------------------------------------------------------------

__device__ __forceinline__ bool edge_less(double w1, uint32_t a1, uint32_t b1, double w2,
                                          uint32_t a2, uint32_t b2) {
    if (w1 != w2) return w1 < w2;
    if (a1 != a2) return a1 < a2;
    return b1 < b2;
}

__device__ uint32_t find_root(uint32_t* comp, uint32_t x) {
    while (comp[x] != x) x = comp[x];
    return x;
}

// edges out: (i, j) pairs, i < j, sorted lexicographically; returns count in *ne
// MST edges are marked in the P x P keep mask (a < b); k_rng_rowcount/k_rng_emit
// then list them in lexicographic order, as build_mst's final sort (:218).
__global__ void __launch_bounds__(1024) k_mst_boruvka(const double* __restrict__ d2, uint32_t P,
                                                      uint32_t* __restrict__ comp_g,
                                                      double* __restrict__ bw_g,
                                                      uint32_t* __restrict__ ba_g,
                                                      uint32_t* __restrict__ bb_g,
                                                      uint8_t* __restrict__ keep) {
    __shared__ int changed;
    __shared__ uint32_t ncomp;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) comp_g[i] = i;
    if (threadIdx.x == 0) ncomp = P;
    __syncthreads();
    while (ncomp > 1) {
        // 1. every node: its lightest edge leaving its component
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
            const uint32_t ci = comp_g[i];
            double bw = CUDART_INF;
            uint32_t ba = 0xFFFFFFFFu, bb = 0xFFFFFFFFu;
            for (uint32_t j = 0; j < P; ++j) {
                if (comp_g[j] == ci) continue;
                const double wv = d2[(size_t)i * P + j];
                const uint32_t a = i < j ? i : j, b = i < j ? j : i;
                if (edge_less(wv, a, b, bw, ba, bb)) {
                    bw = wv;
                    ba = a;
                    bb = b;
                }
            }
            bw_g[i] = bw;
            ba_g[i] = ba;
            bb_g[i] = bb;
        }
        __syncthreads();
        // 2. component minimum: the root (comp == index) scans its members
        for (uint32_t c = threadIdx.x; c < P; c += blockDim.x) {
            if (comp_g[c] != c) continue;
            double bw = CUDART_INF;
            uint32_t ba = 0xFFFFFFFFu, bb = 0xFFFFFFFFu;
            for (uint32_t i = 0; i < P; ++i) {
                if (comp_g[i] != c) continue;
                if (edge_less(bw_g[i], ba_g[i], bb_g[i], bw, ba, bb)) {
                    bw = bw_g[i];
                    ba = ba_g[i];
                    bb = bb_g[i];
                }
            }
            // stash the component's edge in slot c (read back below)
            bw_g[P + c] = bw;
            ba_g[P + c] = ba;
            bb_g[P + c] = bb;
        }
        __syncthreads();
        // 3. add the chosen edges (one thread, deterministic order) with union
        //    by index; duplicates (both sides chose the same edge) merge once
        if (threadIdx.x == 0) {
            for (uint32_t c = 0; c < P; ++c) {
                if (comp_g[c] != c) continue;
                const uint32_t a = ba_g[P + c], b = bb_g[P + c];
                if (a == 0xFFFFFFFFu) continue;
                const uint32_t ra = find_root(comp_g, a), rb = find_root(comp_g, b);
                if (ra == rb) continue;
                keep[(size_t)a * P + b] = 1;
                if (ra < rb) comp_g[rb] = ra; else comp_g[ra] = rb;
                --ncomp;
            }
        }
        __syncthreads();
        // 4. flatten component labels
        do {
            __syncthreads();
            if (threadIdx.x == 0) changed = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t p = comp_g[i], pp = comp_g[p];
                if (p != pp) {
                    comp_g[i] = pp;
                    changed = 1;
                }
            }
            __syncthreads();
        } while (changed);
        // roots must be their own label (c == comp[c]); after flattening the
        // root of each component is its smallest index, which the union kept
    }
}

// ---------------------------------------------------------------------------
// RNG: thread per candidate pair (a < b), witnesses r scanned with early exit.
// Emits a P x P byte mask; compaction in (a, b) order keeps the reference's
// lexicographic edge order.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_rng_mask(const double* __restrict__ d2, uint32_t P,
                                                  uint8_t* __restrict__ keep) {
    const uint32_t a = blockIdx.y;
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= P) return;
    const double* da = d2 + (size_t)a * P;
    for (uint32_t bb = b; bb < P; bb += gridDim.x * blockDim.x) {
        if (bb <= a) {
            keep[(size_t)a * P + bb] = 0;
            continue;
        }
        const double dab = da[bb];
        bool blocked = false;
        for (uint32_t r = 0; r < P && !blocked; ++r) {
            if (r == a || r == bb) continue;
            const double dar = da[r];
            const double dbr = d2[(size_t)r * P + bb];  // == d2[bb][r] (exactly symmetric)
            blocked = fmax(dar, dbr) < dab;
        }
        keep[(size_t)a * P + bb] = blocked ? 0 : 1;
    }
}

// compaction of the keep mask into sorted (a, b) pairs: one thread per row a
// counts, one CTA scans, rows write their edges in order.
__global__ void k_rng_rowcount(const uint8_t* __restrict__ keep, uint32_t P,
                               uint32_t* __restrict__ rowcnt) {
    const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= P) return;
    uint32_t c = 0;
    for (uint32_t b = a + 1; b < P; ++b) c += keep[(size_t)a * P + b];
    rowcnt[a] = c;
}

__global__ void k_rng_emit(const uint8_t* __restrict__ keep, uint32_t P,
                           const uint32_t* __restrict__ rowcnt, uint32_t* __restrict__ edges,
                           uint32_t* __restrict__ ne) {
    // single CTA: exclusive scan of row counts, then each row writes its edges
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t a = 0; a < P; ++a) run += rowcnt[a];
        *ne = run;
    }
    for (uint32_t a = threadIdx.x; a < P; a += blockDim.x) {
        uint32_t off = 0;
        for (uint32_t q = 0; q < a; ++q) off += rowcnt[q];
        for (uint32_t b = a + 1; b < P; ++b)
            if (keep[(size_t)a * P + b]) {
                edges[2 * off] = a;
                edges[2 * off + 1] = b;
                ++off;
            }
    }
}

// ---------------------------------------------------------------------------
// all-pairs hop counts: one CTA per BFS source, CSR adjacency, frontier in smem
// ---------------------------------------------------------------------------

__global__ void k_build_csr(const uint32_t* __restrict__ edges, const uint32_t* __restrict__ ne,
                            uint32_t P, uint32_t* __restrict__ deg, uint32_t* __restrict__ adj,
                            uint32_t* __restrict__ status) {
    // single CTA; P and edge counts are O(1e4)
    const uint32_t n = *ne;
    for (uint32_t i = threadIdx.x; i <= P; i += blockDim.x) deg[i] = 0;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
        const uint32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a >= P || b >= P) {
            atomicOr(status, 2u);  // edge index out of range
            continue;
        }
        atomicAdd(&deg[a + 1], 1u);
        atomicAdd(&deg[b + 1], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (uint32_t i = 0; i < P; ++i) deg[i + 1] += deg[i];
    __syncthreads();
    // fill: sequential per node for a deterministic adjacency order
    for (uint32_t v = threadIdx.x; v < P; v += blockDim.x) {
        uint32_t f = deg[v];
        for (uint32_t e = 0; e < n; ++e) {
            const uint32_t a = edges[2 * e], b = edges[2 * e + 1];
            if (a == v) adj[f++] = b;
            else if (b == v) adj[f++] = a;
        }
    }
}

__global__ void __launch_bounds__(256) k_bfs_all(const uint32_t* __restrict__ deg,
                                                 const uint32_t* __restrict__ adj, uint32_t P,
                                                 uint16_t* __restrict__ hops,
                                                 double* __restrict__ hopd,
                                                 uint32_t* __restrict__ status) {
    // dist_s[P] (u16), then the next-frontier bitmap mark_s[ceil(P/32)] (u32).
    // Level-synchronous: phase A only reads distances and sets bits of the
    // unvisited neighbours (atomicOr), phase B lets the owner thread of each
    // bitmap word assign level + 1 and clear the word — no shared location is
    // written by two threads without an atomic (racecheck-clean).
    extern __shared__ uint16_t dist_s[];
    uint32_t* mark_s = reinterpret_cast<uint32_t*>(dist_s + ((P + 1) & ~1u));
    const uint32_t words = (P + 31) / 32;
    const uint32_t src = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) dist_s[i] = i == src ? 0 : 0xFFFFu;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) mark_s[i] = 0u;
    __syncthreads();
    for (uint32_t level = 0;; ++level) {
        for (uint32_t v = threadIdx.x; v < P; v += blockDim.x) {
            if (dist_s[v] != level) continue;
            for (uint32_t e = deg[v]; e < deg[v + 1]; ++e) {
                const uint32_t u = adj[e];
                if (dist_s[u] == 0xFFFFu) atomicOr(&mark_s[u >> 5], 1u << (u & 31));
            }
        }
        __syncthreads();
        int grew = 0;
        for (uint32_t wd = threadIdx.x; wd < words; wd += blockDim.x) {
            uint32_t m = mark_s[wd];
            if (!m) continue;
            mark_s[wd] = 0u;
            grew = 1;
            while (m) {
                const uint32_t bit = __ffs(m) - 1;
                m &= m - 1;
                dist_s[wd * 32 + bit] = (uint16_t)(level + 1);
            }
        }
        if (!__syncthreads_or(grew)) break;
    }
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint16_t h = dist_s[i];
        if (h == 0xFFFFu) atomicOr(status, 1u);  // disconnected
        hops[(size_t)src * P + i] = h;
        hopd[(size_t)src * P + i] = (double)h;
    }
}

// ---------------------------------------------------------------------------

void launch_gram_only(const float* w, uint32_t P, uint32_t D, TopoScratch& s, cudaStream_t st) {
    TSOM_LAUNCH(k_gram_norms<<<(P + 255) / 256, 256, 0, st>>>(w, P, D, s.norms));
    const dim3 gg((P + 31) / 32, (P + 31) / 32);
    const size_t gsm = (size_t)64 * D * sizeof(float);
    if (gsm > 48 * 1024) cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm);
    TSOM_LAUNCH(k_gram<<<gg, 256, gsm, st>>>(w, P, D, s.norms, s.d2));
}

int launch_refresh_topology(const float* w, uint32_t P, uint32_t D, int kind, TopoScratch& s,
                            cudaStream_t st) {
    // kind: 2 = MST, 3 = RNG (TopologyKind values, topology.hpp:22)
    launch_gram_only(w, P, D, s, st);
    cudaMemsetAsync(s.ne, 0, sizeof(uint32_t), st);
    cudaMemsetAsync(s.status, 0, sizeof(uint32_t), st);
    if (kind == 2) {
        cudaMemsetAsync(s.keep, 0, (size_t)P * P, st);
        if (P > 1)
            TSOM_LAUNCH(k_mst_boruvka<<<1, 1024, 0, st>>>(s.d2, P, s.comp, s.bw, s.ba, s.bb,
                                                          s.keep));
    } else {
        const dim3 rg((P + 255) / 256, P);
        TSOM_LAUNCH(k_rng_mask<<<rg, 256, 0, st>>>(s.d2, P, s.keep));
    }
    TSOM_LAUNCH(k_rng_rowcount<<<(P + 255) / 256, 256, 0, st>>>(s.keep, P, s.rowcnt));
    TSOM_LAUNCH(k_rng_emit<<<1, 1024, 0, st>>>(s.keep, P, s.rowcnt, s.edges, s.ne));
    TSOM_LAUNCH(k_build_csr<<<1, 1024, 0, st>>>(s.edges, s.ne, P, s.deg, s.adj, s.status));
    const size_t bsm = (size_t)((P + 1) & ~1u) * sizeof(uint16_t) + (size_t)(P + 31) / 32 * 4;
    if (bsm > 48 * 1024) cudaFuncSetAttribute(k_bfs_all, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    TSOM_LAUNCH(k_bfs_all<<<P, 256, bsm, st>>>(s.deg, s.adj, P, s.hops, s.hopd, s.status));
    return 0;
}

}  // namespace tsom

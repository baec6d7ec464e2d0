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

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>

#include "engine.h"

namespace tsom {

namespace cg = cooperative_groups;

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

// The same Boruvka over the whole GPU: one cooperative launch, the phases of
// a round separated by grid-wide barriers — (1) a warp per vertex finds its
// lightest edge leaving its component, (2) a warp per component root the
// lightest over its members, (3) a thread per root records that edge (it is
// in the MST: the unique minimum across the cut under the total order) and
// hooks the component onto the other end's (a mutual pair keeps the smaller
// root), (4) every vertex follows the hooks to its new root.  Each round at
// least halves the components; a round with no edge found ends the loop.
// scratch: bw/ba/bb [2P] (vertex minima, then component minima), parent [P],
// cnt [2] (edges found per round, alternating), comp [P].
__device__ __forceinline__ void warp_edge_min(double& w, uint32_t& a, uint32_t& b) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ow = __shfl_xor_sync(0xffffffffu, w, o);
        const uint32_t oa = __shfl_xor_sync(0xffffffffu, a, o);
        const uint32_t ob = __shfl_xor_sync(0xffffffffu, b, o);
        if (edge_less(ow, oa, ob, w, a, b)) {
            w = ow;
            a = oa;
            b = ob;
        }
    }
}

__global__ void __launch_bounds__(256) k_mst_grid(const double* __restrict__ d2, uint32_t P,
                                                  uint32_t* __restrict__ comp,
                                                  double* __restrict__ bw, uint32_t* __restrict__ ba,
                                                  uint32_t* __restrict__ bb,
                                                  uint32_t* __restrict__ parent,
                                                  uint32_t* __restrict__ cnt,
                                                  uint8_t* __restrict__ keep) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const uint32_t lane = threadIdx.x & 31, gw = tid >> 5, nw = nth >> 5;
    for (uint32_t i = tid; i < P; i += nth) comp[i] = i;
    if (tid == 0) {
        cnt[0] = 0;
        cnt[1] = 0;
    }
    grid.sync();
    for (uint32_t round = 0;; ++round) {
        for (uint32_t i = gw; i < P; i += nw) {  // (1)
            const uint32_t ci = comp[i];
            double w = CUDART_INF;
            uint32_t a = 0xFFFFFFFFu, b = 0xFFFFFFFFu;
            for (uint32_t j = lane; j < P; j += 32) {
                if (comp[j] == ci) continue;
                const double wv = d2[(size_t)i * P + j];
                const uint32_t aa = i < j ? i : j, bb2 = i < j ? j : i;
                if (edge_less(wv, aa, bb2, w, a, b)) {
                    w = wv;
                    a = aa;
                    b = bb2;
                }
            }
            warp_edge_min(w, a, b);
            if (lane == 0) {
                bw[i] = w;
                ba[i] = a;
                bb[i] = b;
            }
        }
        grid.sync();
        for (uint32_t c = gw; c < P; c += nw) {  // (2)
            if (comp[c] != c) continue;  // (warp-uniform)
            double w = CUDART_INF;
            uint32_t a = 0xFFFFFFFFu, b = 0xFFFFFFFFu;
            for (uint32_t i = lane; i < P; i += 32)
                if (comp[i] == c && edge_less(bw[i], ba[i], bb[i], w, a, b)) {
                    w = bw[i];
                    a = ba[i];
                    b = bb[i];
                }
            warp_edge_min(w, a, b);
            if (lane == 0) {
                bw[P + c] = w;
                ba[P + c] = a;
                bb[P + c] = b;
            }
        }
        grid.sync();
        const uint32_t cur = round & 1u;
        for (uint32_t c = tid; c < P; c += nth) {  // (3)
            if (comp[c] != c) continue;
            const uint32_t a = ba[P + c], b = bb[P + c];
            if (a == 0xFFFFFFFFu) {
                parent[c] = c;
                continue;
            }
            keep[(size_t)a * P + b] = 1;
            const uint32_t t = comp[a] == c ? comp[b] : comp[a];
            const bool mutual = ba[P + t] == a && bb[P + t] == b;
            parent[c] = (mutual && c < t) ? c : t;
            atomicAdd(&cnt[cur], 1u);
        }
        grid.sync();
        if (*reinterpret_cast<volatile uint32_t*>(&cnt[cur]) == 0) break;  // one component
        for (uint32_t i = tid; i < P; i += nth) {  // (4)
            uint32_t r = comp[i];
            while (parent[r] != r) r = parent[r];
            comp[i] = r;
        }
        if (tid == 0) cnt[cur ^ 1u] = 0;
        grid.sync();
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

// RNG with nearest-first witnesses: every row a's other nodes sorted by d2
// (one CTA per row, bitonic sort in shared memory), then a thread per pair
// (a, b > a) scans a's list only while d_ar < d_ab — a node at least as far
// from a as b cannot block the pair (max(d_ar, d_br) < d_ab needs d_ar <
// d_ab) — and stops at the first witness.  Same predicate, same mask as
// k_rng_mask (an OR over the same witnesses); far pairs meet a witness among
// a's first few neighbours instead of after a scan in index order.
__global__ void __launch_bounds__(1024) k_rng_sort_rows(const double* __restrict__ d2, uint32_t P,
                                                        uint32_t P2, double* __restrict__ skey,
                                                        uint16_t* __restrict__ sidx) {
    extern __shared__ uint8_t rsm[];
    double* key = reinterpret_cast<double*>(rsm);
    uint16_t* idx = reinterpret_cast<uint16_t*>(key + P2);
    const uint32_t a = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < P2; i += blockDim.x) {
        key[i] = (i < P && i != a) ? d2[(size_t)a * P + i] : CUDART_INF;
        idx[i] = (uint16_t)(i < P ? i : 0);
    }
    __syncthreads();
    for (uint32_t k = 2; k <= P2; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < P2; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = key[i] > key[l] || (key[i] == key[l] && idx[i] > idx[l]);
                    if (gt == up) {
                        const double tk = key[i];
                        key[i] = key[l];
                        key[l] = tk;
                        const uint16_t ti = idx[i];
                        idx[i] = idx[l];
                        idx[l] = ti;
                    }
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i + 1 < P; i += blockDim.x) {  // (the INF self entry is last)
        skey[(size_t)a * P + i] = key[i];
        sidx[(size_t)a * P + i] = idx[i];
    }
}

__global__ void __launch_bounds__(256) k_rng_mask_sorted(const double* __restrict__ d2, uint32_t P,
                                                         const double* __restrict__ skey,
                                                         const uint16_t* __restrict__ sidx,
                                                         uint8_t* __restrict__ keep) {
    const uint32_t a = blockIdx.y;
    if (a >= P) return;
    const double* ka = skey + (size_t)a * P;
    const uint16_t* ia = sidx + (size_t)a * P;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < P; b += gridDim.x * blockDim.x) {
        if (b <= a) {
            keep[(size_t)a * P + b] = 0;
            continue;
        }
        const double dab = d2[(size_t)a * P + b];
        bool blocked = false;
        for (uint32_t q = 0; q + 1 < P; ++q) {
            const double dar = ka[q];
            if (!(dar < dab)) break;  // every later r is at least as far from a
            const uint32_t r = ia[q];
            if (r == b) continue;
            if (d2[(size_t)r * P + b] < dab) {  // == max(d_ar, d_br) < d_ab here
                blocked = true;
                break;
            }
        }
        keep[(size_t)a * P + b] = blocked ? 0 : 1;
    }
}

// compaction of the keep mask into sorted (a, b) pairs: a warp per row counts
// its edges (ballots over 32 columns at a time), one CTA scans the counts into
// row offsets, and a warp per row writes its edges in column order
__global__ void k_rng_rowcount(const uint8_t* __restrict__ keep, uint32_t P,
                               uint32_t* __restrict__ rowcnt) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < P; a += nw) {
        uint32_t c = 0;
        for (uint32_t b0 = 0; b0 < P; b0 += 32) {
            const uint32_t b = b0 + lane;
            c += __popc(__ballot_sync(0xffffffffu, b < P && b > a && keep[(size_t)a * P + b]));
        }
        if (lane == 0) rowcnt[a] = c;
    }
}

__global__ void __launch_bounds__(1024) k_rng_scan(uint32_t P, const uint32_t* __restrict__ rowcnt,
                                                   uint32_t* __restrict__ rowoff,
                                                   uint32_t* __restrict__ ne) {
    __shared__ uint32_t sc[1024];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < P; base += 1024) {
        const uint32_t a = base + threadIdx.x;
        const uint32_t v = a < P ? rowcnt[a] : 0u;
        sc[threadIdx.x] = v;
        __syncthreads();
        for (uint32_t off = 1; off < 1024; off <<= 1) {
            const uint32_t add = threadIdx.x >= off ? sc[threadIdx.x - off] : 0u;
            __syncthreads();
            sc[threadIdx.x] += add;
            __syncthreads();
        }
        if (a < P) rowoff[a] = carry + sc[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += sc[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *ne = carry;
}

__global__ void k_rng_emit(const uint8_t* __restrict__ keep, uint32_t P,
                           const uint32_t* __restrict__ rowoff, uint32_t* __restrict__ edges) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < P; a += nw) {
        uint32_t o = rowoff[a];
        for (uint32_t b0 = 0; b0 < P; b0 += 32) {
            const uint32_t b = b0 + lane;
            const bool k = b < P && b > a && keep[(size_t)a * P + b];
            const uint32_t m = __ballot_sync(0xffffffffu, k);
            if (k) {
                const uint32_t q = o + __popc(m & ((1u << lane) - 1u));
                edges[2 * q] = a;
                edges[2 * q + 1] = b;
            }
            o += __popc(m);
        }
    }
}

// degrees (atomic counts), then offsets by one CTA's scan, then the fill with
// an atomic cursor per node: the adjacency order within a node is arbitrary,
// which BFS hop counts do not depend on
__global__ void k_csr_degrees(const uint32_t* __restrict__ edges, const uint32_t* __restrict__ ne,
                              uint32_t P, uint32_t* __restrict__ deg, uint32_t* __restrict__ status) {
    const uint32_t n = *ne;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const uint32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a >= P || b >= P) {
            atomicOr(status, 2u);  // edge index out of range
            continue;
        }
        atomicAdd(&deg[a + 1], 1u);
        atomicAdd(&deg[b + 1], 1u);
    }
}

__global__ void __launch_bounds__(1024) k_csr_scan(uint32_t P, uint32_t* __restrict__ deg,
                                                   uint32_t* __restrict__ cursor) {
    __shared__ uint32_t sc[1024];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < P; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < P ? deg[i + 1] : 0u;
        sc[threadIdx.x] = v;
        __syncthreads();
        for (uint32_t off = 1; off < 1024; off <<= 1) {
            const uint32_t add = threadIdx.x >= off ? sc[threadIdx.x - off] : 0u;
            __syncthreads();
            sc[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < P) {
            deg[i + 1] = carry + sc[threadIdx.x];
            cursor[i] = carry + sc[threadIdx.x] - v;
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry += sc[1023];
        __syncthreads();
    }
}

__global__ void k_csr_fill(const uint32_t* __restrict__ edges, const uint32_t* __restrict__ ne,
                           uint32_t P, uint32_t* __restrict__ cursor, uint32_t* __restrict__ adj) {
    const uint32_t n = *ne;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const uint32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a >= P || b >= P) continue;
        adj[atomicAdd(&cursor[a], 1u)] = b;
        adj[atomicAdd(&cursor[b], 1u)] = a;
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
        if (P > 1) {
            // the grid-wide Boruvka (one cooperative launch); the one-CTA
            // version if the cooperative launch is refused
            // (scratch: parent = rowcnt, the round counters = deg[0..1], both
            // rewritten by the compaction below)
            static int blocks_per_sm = -1;
            if (blocks_per_sm < 0 &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_mst_grid, 256, 0) !=
                    cudaSuccess) {
                cudaGetLastError();
                blocks_per_sm = 0;
            }
            int dev = 0, sms = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const unsigned nb = (unsigned)std::min(std::max(blocks_per_sm, 0), 4) * (unsigned)sms;
            cudaError_t e = cudaErrorInvalidConfiguration;
            if (nb > 0) {
                const double* d2 = s.d2;
                uint32_t* comp = s.comp;
                double* bw = s.bw;
                uint32_t* ba = s.ba;
                uint32_t* bb = s.bb;
                uint32_t* parent = s.rowcnt;
                uint32_t* cnt = s.deg;
                uint8_t* keep = s.keep;
                void* args[] = {(void*)&d2, (void*)&P, (void*)&comp, (void*)&bw, (void*)&ba,
                                (void*)&bb, (void*)&parent, (void*)&cnt, (void*)&keep};
                ++g_launches;
                e = cudaLaunchCooperativeKernel((const void*)k_mst_grid, dim3(nb), dim3(256), args,
                                                0, st);
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                TSOM_LAUNCH(k_mst_boruvka<<<1, 1024, 0, st>>>(s.d2, P, s.comp, s.bw, s.ba, s.bb,
                                                              s.keep));
            }
        }
    } else {
        const dim3 rg((P + 255) / 256, P);
        uint32_t P2 = 1;
        while (P2 < P) P2 <<= 1;
        const size_t ssm = (size_t)P2 * (sizeof(double) + sizeof(uint16_t));
        if (P >= 64 && P2 <= 16384 && ssm <= 200 * 1024) {
            // (scratch: the sorted keys in hopd, the indices in hops — both
            // rewritten by the BFS below)
            if (ssm > 48 * 1024)
                cudaFuncSetAttribute(k_rng_sort_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ssm);
            TSOM_LAUNCH(k_rng_sort_rows<<<P, 1024, ssm, st>>>(s.d2, P, P2, s.hopd, s.hops));
            TSOM_LAUNCH(k_rng_mask_sorted<<<rg, 256, 0, st>>>(s.d2, P, s.hopd, s.hops, s.keep));
        } else {
            TSOM_LAUNCH(k_rng_mask<<<rg, 256, 0, st>>>(s.d2, P, s.keep));
        }
    }
    const unsigned wb = (P + 7) / 8;  // a warp per row, 8 warps per block
    TSOM_LAUNCH(k_rng_rowcount<<<wb, 256, 0, st>>>(s.keep, P, s.rowcnt));
    TSOM_LAUNCH(k_rng_scan<<<1, 1024, 0, st>>>(P, s.rowcnt, s.comp, s.ne));  // (comp: row offsets)
    TSOM_LAUNCH(k_rng_emit<<<wb, 256, 0, st>>>(s.keep, P, s.comp, s.edges));
    cudaMemsetAsync(s.deg, 0, (size_t)(P + 1) * sizeof(uint32_t), st);
    TSOM_LAUNCH(k_csr_degrees<<<(P + 255) / 256 * 4, 256, 0, st>>>(s.edges, s.ne, P, s.deg,
                                                                   s.status));
    TSOM_LAUNCH(k_csr_scan<<<1, 1024, 0, st>>>(P, s.deg, s.rowcnt));  // (rowcnt: fill cursors)
    TSOM_LAUNCH(k_csr_fill<<<(P + 255) / 256 * 4, 256, 0, st>>>(s.edges, s.ne, P, s.rowcnt, s.adj));
    const size_t bsm = (size_t)((P + 1) & ~1u) * sizeof(uint16_t) + (size_t)(P + 31) / 32 * 4;
    if (bsm > 48 * 1024) cudaFuncSetAttribute(k_bfs_all, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    TSOM_LAUNCH(k_bfs_all<<<P, 256, bsm, st>>>(s.deg, s.adj, P, s.hops, s.hopd, s.status));
    return 0;
}

}  // namespace tsom

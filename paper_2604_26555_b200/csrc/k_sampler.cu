// k_sampler.cu — the reference's per-epoch samplers on the device
// (sampling.hpp:46-157, rng.hpp:33-91), producing the same selections as
// toposom::Sampler for the same seed.
//
// Random stream: the sampler's Rng is std::mt19937_64 seeded with
// mix_seed(seed, SeedStream::sampler).  An epoch's draws are produced by G
// generators at once: generator g starts at draw g*L of the epoch, its state
// obtained from the epoch's start state with the jump polynomial t^(gL) mod
// phi (mt_jump.cpp): the start window is extended by 19937 + 311 words
// (k_mt_extend, one CTA), then every generator CTA computes its window as an
// XOR of shifted copies of that sequence held in shared memory, and twists /
// tempers its L outputs (k_mt_generate).  The state after the epoch's draws is
// read from the recorded untempered "tail" words, at the device-side draw count.
//
// select_random (sampling.hpp:56-73, Floyd): draw t_k = index(j + 1) for
// j = n - m + k (rejection sampling, rng.hpp:42-51 — rejections are detected
// and replayed sequentially); pick_j = t_k unless t_k was picked before, then
// j.  "Picked before" is decided without the hash set: t_k collides iff an
// earlier draw equals t_k (first-occurrence table) or t_k is an earlier j that
// itself collided — a chain through strictly smaller j.
//
// select_adaptive (sampling.hpp:101-139): key_i = -log(1 - real01) / w_i with
// w_i = (e_i/max e)^alpha + (a_i/max a)^beta, unseen rows first; the m
// smallest (seen, key) pairs win (radix select on 64-bit sortable keys), then
// the sorted index list.  update_adaptive (:143-157) on the device.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "engine.h"
#include "mt_jump.h"

namespace tsom {

namespace {

constexpr uint64_t kA = 0xB5026F5AA96619E9ULL, kUM = 0xFFFFFFFF80000000ULL,
                   kLM = 0x7FFFFFFFULL;

__device__ __forceinline__ uint64_t mt_step(uint64_t x0, uint64_t x1, uint64_t xm) {
    const uint64_t y = (x0 & kUM) | (x1 & kLM);
    return xm ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

constexpr int kT = 320;  // threads per MT CTA (>= 312)
constexpr uint32_t kCompactBlocks = 1184;  // segments of the first-digit compaction

// one twist of the 312-word window `cur` into `nxt` (both shared), by kT threads
__device__ __forceinline__ void twist(const uint64_t* cur, uint64_t* nxt) {
    const int k = threadIdx.x;
    if (k < 156) nxt[k] = mt_step(cur[k], cur[k + 1], cur[k + 156]);
    __syncthreads();
    if (k >= 156 && k < 311) nxt[k] = mt_step(cur[k], cur[k + 1], nxt[k - 156]);
    if (k == 311) nxt[311] = mt_step(cur[311], nxt[0], nxt[155]);
    __syncthreads();
}

// window[k] = XOR over the set bits i of the jump polynomial (s_j, 312
// words) of s_seq[i + k], k < 312.  The set-bit indices are first listed in
// s_idx (a block-wide scan of the words' popcounts), so the XOR loop is one
// broadcast index load and one sequence load per term.  All kT threads call.
__device__ __forceinline__ uint64_t jump_apply(const uint64_t* s_seq, const uint64_t* s_j,
                                               uint16_t* s_idx, uint32_t* s_wsum) {
    const int k = threadIdx.x, lane = k & 31, wid = k >> 5;
    const uint64_t bits0 = k < 312 ? s_j[k] : 0ull;
    const uint32_t c = __popcll(bits0);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    uint32_t base = 0, nt = 0;
    for (int w = 0; w < kT / 32; ++w) {
        const uint32_t v = s_wsum[w];
        if (w < wid) base += v;
        nt += v;
    }
    uint32_t pos = base + incl - c;
    for (uint64_t bits = bits0; bits; bits &= bits - 1)
        s_idx[pos++] = (uint16_t)(64 * k + __ffsll((long long)bits) - 1);
    __syncthreads();
    uint64_t a0 = 0, a1 = 0;
    if (k < 312) {
        uint32_t t = 0;
        for (; t + 4 <= nt; t += 4) {
            a0 ^= s_seq[s_idx[t] + k] ^ s_seq[s_idx[t + 1] + k];
            a1 ^= s_seq[s_idx[t + 2] + k] ^ s_seq[s_idx[t + 3] + k];
        }
        for (; t < nt; ++t) a0 ^= s_seq[s_idx[t] + k];
    }
    return a0 ^ a1;
}

constexpr size_t kJumpIdxBytes = (19937 + 64) * sizeof(uint16_t);

}  // namespace

// seq[0..312) = window, seq[312 .. 312 + 312 * twists) = the next untempered words
__global__ void __launch_bounds__(kT) k_mt_extend(const uint64_t* __restrict__ window,
                                                  uint32_t twists, uint64_t* __restrict__ seq) {
    __shared__ uint64_t buf[2][312];
    const int k = threadIdx.x;
    if (k < 312) {
        buf[0][k] = window[k];
        seq[k] = window[k];
    }
    __syncthreads();
    for (uint32_t t = 0; t < twists; ++t) {
        twist(buf[t & 1], buf[(t + 1) & 1]);
        if (k < 312) seq[312 + (size_t)t * 312 + k] = buf[(t + 1) & 1][k];
    }
}

// Generator g's start window (draw g*L): X[gL .. gL + 312) from the epoch's
// extended sequence and the jump polynomial jp[g] (g = 0 without jump0: the
// sequence itself).  One CTA per generator; ~210 KB of shared memory.
__global__ void __launch_bounds__(kT) k_mt_jump_all(const uint64_t* __restrict__ seq,
                                                    const uint64_t* __restrict__ jp, uint64_t L,
                                                    uint64_t total, uint64_t* __restrict__ wins,
                                                    int jump0) {
    extern __shared__ uint64_t sm[];
    uint64_t* s_seq = sm;                 // [mt::kSeq]
    uint64_t* s_j = sm + mt::kSeq;        // [312]
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_j + 312);
    __shared__ uint32_t s_wsum[kT / 32];
    const int k = threadIdx.x;
    const uint64_t g = blockIdx.x;
    if (g * L >= total) return;
    if (g == 0 && !jump0) {
        if (k < 312) wins[k] = seq[k];
        return;
    }
    for (int i = k; i < mt::kSeq; i += kT) s_seq[i] = seq[i];
    if (k < 312) s_j[k] = jp[g * 312 + k];
    __syncthreads();
    const uint64_t acc = jump_apply(s_seq, s_j, s_idx, s_wsum);
    if (k < 312) wins[g * 312 + k] = acc;
}

// Generator g: from its start window, `L` tempered outputs into draws[g*L ..)
// (bounded by total).  Untempered words at positions [tail0, tail0 + tail_len)
// (window coordinates of the epoch start: output q = temper(X[q + 312])) are
// copied to tail[].  5 KB of shared memory: several generator CTAs share an
// SM with the epoch's other kernels (the draws are made on a side stream).
__global__ void __launch_bounds__(kT) k_mt_generate(const uint64_t* __restrict__ wins, uint64_t L,
                                                    uint64_t total, uint64_t* __restrict__ draws,
                                                    uint64_t tail0, uint32_t tail_len,
                                                    uint64_t* __restrict__ tail) {
    __shared__ uint64_t s_w[2 * 312];
    const int k = threadIdx.x;
    const uint64_t g = blockIdx.x;
    const uint64_t q0 = g * L;
    if (q0 >= total) return;
    if (k < 312) s_w[k] = wins[g * 312 + k];
    __syncthreads();
    const uint64_t q1 = min(q0 + L, total);
    int cur = 0;
    for (uint64_t q = q0; q < q1; q += 312) {
        twist(s_w + cur * 312, s_w + (cur ^ 1) * 312);
        cur ^= 1;
        if (k < 312) {
            const uint64_t x = s_w[cur * 312 + k];
            const uint64_t qq = q + k;  // output index; x = X[qq + 312]
            if (qq < q1) draws[qq] = mt_temper(x);
            const uint64_t pos = qq + 312;
            if (pos >= tail0 && pos < tail0 + tail_len) tail[pos - tail0] = x;
        }
    }
}

// new window = X[delta .. delta + 312): from seq (delta + 312 <= kSeq) or tail
__global__ void k_mt_advance(const uint64_t* __restrict__ seq, const uint64_t* __restrict__ tail,
                             uint64_t tail0, uint32_t tail_len, const uint64_t* __restrict__ delta,
                             uint64_t* __restrict__ window, uint32_t* __restrict__ status) {
    const uint64_t d = *delta;
    const int k = threadIdx.x;
    if (k >= 312) return;
    const uint64_t pos = d + k;
    if (pos < (uint64_t)mt::kSeq) {
        window[k] = seq[pos];
    } else if (pos >= tail0 && pos < tail0 + tail_len) {
        window[k] = tail[pos - tail0];
    } else if (k == 0) {
        atomicOr(status, 4u);  // draws beyond the generated slack
    }
}

// window <- X[J .. J + 312) from the epoch-start sequence and jp = t^J mod phi
// (sharded adaptive: every rank skips the whole epoch's N draws at once)
__global__ void __launch_bounds__(kT) k_mt_jump_window(const uint64_t* __restrict__ seq,
                                                       const uint64_t* __restrict__ jp,
                                                       uint64_t* __restrict__ window) {
    extern __shared__ uint64_t sm2[];
    uint64_t* s_seq = sm2;
    uint64_t* s_j = sm2 + mt::kSeq;
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_j + 312);
    __shared__ uint32_t s_wsum[kT / 32];
    const int k = threadIdx.x;
    for (int i = k; i < mt::kSeq; i += kT) s_seq[i] = seq[i];
    if (k < 312) s_j[k] = jp[k];
    __syncthreads();
    const uint64_t acc = jump_apply(s_seq, s_j, s_idx, s_wsum);
    if (k < 312) window[k] = acc;
}

// ---------------------------------------------------------------------------
// select_random
// ---------------------------------------------------------------------------

// t_k = index(j + 1), j = n - m + k; flags rejections (x >= limit)
__global__ void k_rand_index(const uint64_t* __restrict__ draws, uint64_t n, uint64_t m,
                             uint32_t* __restrict__ t, uint32_t* __restrict__ first,
                             uint32_t* __restrict__ status) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bound = n - m + k + 1;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        const uint64_t x = draws[k];
        if (x >= limit) atomicOr(status, 1u);
        const uint32_t tk = (uint32_t)(x % bound);
        t[k] = tk;
        atomicMin(&first[tk], (uint32_t)k);
    }
}

// exact sequential replay when a rejection occurred (rng.hpp:42-51): every
// index() call consumes draws until one is below its limit
__global__ void k_rand_replay(const uint64_t* __restrict__ draws, uint64_t avail, uint64_t n,
                              uint64_t m, uint32_t* __restrict__ t, uint32_t* __restrict__ first,
                              uint64_t* __restrict__ delta, uint32_t* __restrict__ status) {
    if (!(*status & 1u)) return;
    uint64_t r = 0;
    for (uint64_t k = 0; k < m; ++k) {
        const uint64_t bound = n - m + k + 1;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t x;
        do {
            if (r >= avail) {
                atomicOr(status, 4u);
                return;
            }
            x = draws[r++];
        } while (x >= limit);
        t[k] = (uint32_t)(x % bound);
    }
    for (uint64_t k = 0; k < m; ++k) first[t[k]] = 0xFFFFFFFFu;
    for (uint64_t k = 0; k < m; ++k)
        if (first[t[k]] == 0xFFFFFFFFu) first[t[k]] = (uint32_t)k;
    *delta = r;
}

// Floyd's pick for every k (sampling.hpp:64-70), into the row bitmap
__global__ void k_rand_pick(const uint32_t* __restrict__ t, const uint32_t* __restrict__ first,
                            uint64_t n, uint64_t m, uint32_t* __restrict__ bitmap) {
    const uint64_t j0 = n - m;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        // collided(k) = dup(k) || (t_k in [j0, j0 + k) && collided(t_k - j0))
        uint64_t c = k;
        bool coll;
        while (true) {
            const uint32_t tc = t[c];
            if (first[tc] < (uint32_t)c) {
                coll = true;
                break;
            }
            if (tc >= j0 && tc < j0 + c) {
                c = tc - j0;
                continue;
            }
            coll = false;
            break;
        }
        const uint64_t pick = coll ? j0 + k : (uint64_t)t[k];
        atomicOr(&bitmap[pick >> 5], 1u << (pick & 31));
    }
}

// ---------------------------------------------------------------------------
// select_adaptive
// ---------------------------------------------------------------------------

// update_adaptive's "every age + 1, the observed rows 0" (sampling.hpp:143-157)
// is applied lazily: observe only marks its rows (kAgeMark), and the next
// select reads every age through age_now() and writes the result back while
// computing the keys, so no separate pass over the N ages is made.
constexpr uint32_t kAgeMark = 0xFFFFFFFFu;
__device__ __forceinline__ uint32_t age_now(uint32_t a, int pending) {
    return pending ? (a == kAgeMark ? 0u : a + 1u) : a;
}

__global__ void k_adapt_max(const double* __restrict__ err, const uint32_t* __restrict__ age,
                            uint64_t n, int pending, unsigned long long* __restrict__ mx) {
    double me = 0.0;
    uint32_t ma = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        me = fmax(me, err[i]);
        ma = max(ma, age_now(age[i], pending));
    }
    for (int o = 16; o; o >>= 1) {
        me = fmax(me, __shfl_xor_sync(0xffffffffu, me, o));
        ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&mx[0], (unsigned long long)__double_as_longlong(me));  // errors >= 0
        atomicMax(&mx[1], (unsigned long long)ma);
    }
}

__device__ __forceinline__ double pow_ref(double x, double e) {
    // pow(x, 1) and pow(x, 2) are exact in the reference's libm as well
    if (e == 1.0) return x;
    if (e == 2.0) return x * x;
    return pow(x, e);
}

// warp-aggregated shared-memory histogram increment: lanes with the same bin
// add once (the radix digits of the keys concentrate on few bins)
__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t bin, bool active) {
    const uint32_t key = active ? bin : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const uint32_t lane = threadIdx.x & 31;
    if (active && (__ffs(peers) - 1) == (int)lane) atomicAdd(&h[bin], (uint32_t)__popc(peers));
}

// sortable 64-bit key: (seen << 63) | bits(key), key >= 0 (sampling.hpp:116-133),
// and the histogram of the keys' first radix digit (bits 52-63, over every key,
// so no second pass over the N keys is made for it).  The age term
// a / max_age takes few values (ages count epochs): it comes from a per-block
// table of the same IEEE quotients for a < kAgeTab.
constexpr uint32_t kAgeTab = 1024;
__global__ void __launch_bounds__(256) k_adapt_keys(
    const double* __restrict__ err, uint32_t* __restrict__ age, const uint64_t* __restrict__ draws,
    uint64_t n, double alpha, double beta, int pending, const unsigned long long* __restrict__ mx,
    unsigned long long* __restrict__ keys, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[4096];
    __shared__ double agetab[kAgeTab];
    const double max_err = fmax(__longlong_as_double((long long)mx[0]), 1e-12);
    const double max_age = fmax((double)mx[1], 1e-12);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
    for (uint32_t a = threadIdx.x; a < kAgeTab; a += blockDim.x) agetab[a] = (double)a / max_age;
    __syncthreads();
    // kU elements per thread and step, all loads issued before the arithmetic
    constexpr int kU = 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * kU;
    for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x * kU; i0 < n; i0 += stride) {
        double e[kU];
        uint32_t a[kU];
        uint64_t dr[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint64_t i = i0 + (uint64_t)q * blockDim.x + threadIdx.x;
            const bool in = i < n;
            e[q] = in ? err[i] : 0.0;
            a[q] = in ? age[i] : 0u;
            dr[q] = in ? draws[i] : 0ull;
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint64_t i = i0 + (uint64_t)q * blockDim.x + threadIdx.x;
            const bool in = i < n;
            unsigned long long kb = 0;
            if (in) {
                const uint32_t an = age_now(a[q], pending);
                if (pending) age[i] = an;
                const double ta = an < kAgeTab ? agetab[an] : (double)an / max_age;
                const double w = pow_ref(e[q] / max_err, alpha) + pow_ref(ta, beta);
                const double u = 1.0 - (double)(dr[q] >> 11) * 0x1.0p-53;
                double key = w > 0.0 ? -log(u) / w : CUDART_INF;
                key = fmax(key, 0.0);  // -log(1) = -0
                const unsigned long long seen = e[q] != 1e30 ? 1ULL : 0ULL;
                kb = (seen << 63) | (unsigned long long)__double_as_longlong(key);
                keys[i] = kb;
            }
            hist_add(h, (uint32_t)(kb >> 52), in);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Keys in the first digit's chosen bucket -> cand[] with the histogram of
// the second digit (bits 40-51); the later digits then scan only these.
// Block b compacts keys [b*chunk, (b+1)*chunk) into its own segment of cand
// starting at b*chunk (no global counter); cnt[b] = its candidates.
__global__ void k_adapt_compact(const unsigned long long* __restrict__ keys, uint64_t n,
                                uint64_t chunk, const unsigned long long* __restrict__ sel_state,
                                unsigned long long* __restrict__ cand, uint32_t* __restrict__ cidx,
                                uint32_t* __restrict__ cnt, uint32_t* __restrict__ hist,
                                uint32_t* __restrict__ bitmap) {
    __shared__ uint32_t h[4096];
    __shared__ uint32_t fill;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
    if (threadIdx.x == 0) fill = 0;
    __syncthreads();
    const unsigned long long top = sel_state[0] >> 52;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t c0 = blockIdx.x * chunk, c1 = min(n, c0 + chunk);
    unsigned long long* out = cand + c0;
    uint32_t* oidx = cidx + c0;
    for (uint64_t i0 = c0; i0 < c1; i0 += blockDim.x) {
        const uint64_t i = i0 + threadIdx.x;
        const unsigned long long k = i < c1 ? keys[i] : ~0ULL;
        const bool in = i < c1 && (k >> 52) == top;
        // every key below the first digit's bucket is below the threshold: its
        // row is selected here, one bitmap word per warp (chunk and the warp's
        // rows are 32-aligned); the bucket's own rows are decided by
        // k_adapt_mark_cand once the threshold is complete
        const uint32_t take = __ballot_sync(0xffffffffu, i < c1 && (k >> 52) < top);
        if (lane == 0 && i < c1) bitmap[i >> 5] = take;
        const uint32_t ballot = __ballot_sync(0xffffffffu, in);
        if (ballot) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&fill, (uint32_t)__popc(ballot));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (in) {
                const uint32_t slot = base + __popc(ballot & ((1u << lane) - 1u));
                out[slot] = k;
                oidx[slot] = (uint32_t)i;
            }
            hist_add(h, (uint32_t)((k >> 40) & 4095ULL), in);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cnt[blockIdx.x] = fill;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// radix digit histogram over the compacted segments of k_adapt_compact
__global__ void k_adapt_hist_cand(const unsigned long long* __restrict__ cand, uint64_t chunk,
                                  const uint32_t* __restrict__ cnt,
                                  const unsigned long long* __restrict__ sel_state, int shift,
                                  int width, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sel_state[0];
    const unsigned long long hi_mask = ~0ULL << (shift + width);
    const unsigned long long dmask = (1ULL << width) - 1ULL;
    const unsigned long long* seg = cand + blockIdx.x * chunk;
    const uint32_t m = cnt[blockIdx.x];
    for (uint32_t i0 = 0; i0 < m; i0 += blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        const unsigned long long k = i < m ? seg[i] : 0ULL;
        hist_add(h, (uint32_t)((k >> shift) & dmask), i < m && (k & hi_mask) == prefix);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// sel_state = [prefix, need]: pick the digit where the running count reaches
// need (one block of 1024 threads, 4 bins each, block-wide inclusive scan)
__global__ void __launch_bounds__(1024) k_adapt_digit(uint32_t* __restrict__ hist, int shift,
                                                      unsigned long long* __restrict__ sel_state) {
    __shared__ unsigned long long wsum[32];
    __shared__ int found;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const unsigned long long need = sel_state[1];
    uint32_t h[4];
    unsigned long long loc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        h[i] = hist[4 * t + i];
        loc += h[i];
    }
    unsigned long long inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[wid] = inc;
    if (t == 0) found = 4095;
    __syncthreads();
    if (wid == 0) {
        unsigned long long v = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    // exclusive prefix before this thread's 4 bins
    unsigned long long cum = inc - loc + (wid ? wsum[wid - 1] : 0ULL);
    int d = -1;
    unsigned long long before = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (d < 0 && cum + h[i] >= need) {
            d = 4 * t + i;
            before = cum;
        }
        cum += h[i];
    }
    if (d >= 0) atomicMin(&found, d);
    __syncthreads();
    if (d >= 0 && d == found) {
        sel_state[0] |= (unsigned long long)d << shift;
        sel_state[1] = need - before;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) hist[4 * t + i] = 0;
}

// the first digit's bucket (k_adapt_compact's segments): rows with key < T,
// plus the first `need` rows with key == T (ties at the boundary are
// implementation-defined in the reference; counted in status).  The rows below
// the bucket were selected by the compaction.
__global__ void k_adapt_mark_cand(const unsigned long long* __restrict__ cand,
                                  const uint32_t* __restrict__ cidx, uint64_t chunk,
                                  const uint32_t* __restrict__ cnt,
                                  const unsigned long long* __restrict__ sel_state,
                                  uint32_t* __restrict__ bitmap, unsigned long long* __restrict__ eq) {
    const unsigned long long T = sel_state[0], need = sel_state[1];
    const unsigned long long* seg = cand + blockIdx.x * chunk;
    const uint32_t* sidx = cidx + blockIdx.x * chunk;
    const uint32_t m = cnt[blockIdx.x];
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const unsigned long long k = seg[i];
        bool take = k < T;
        if (k == T) take = atomicAdd(eq, 1ULL) < need;
        if (take) {
            const uint32_t r = sidx[i];
            atomicOr(&bitmap[r >> 5], 1u << (r & 31));
        }
    }
}

// update_adaptive: every age + 1, then selected rows get their distance, age 0
__global__ void k_adapt_age(uint32_t* __restrict__ age, uint64_t n) {  // materialise
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        age[i] = age_now(age[i], 1);
}
__global__ void k_adapt_observe(const uint32_t* __restrict__ sel, uint64_t m,
                                const double* __restrict__ dist, double* __restrict__ err,
                                uint32_t* __restrict__ age) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = sel[k];
        err[i] = dist[k];
        age[i] = kAgeMark;  // -> 0 at the next select (age_now)
    }
}

// sharded random: the rows of a sorted global selection that fall in this
// rank's range [off, off + n), as local ids; count -> *m_local
__global__ void k_local_slice(const uint32_t* __restrict__ glist, const unsigned long long* total,
                              uint64_t off, uint64_t n, uint32_t* __restrict__ out,
                              unsigned long long* __restrict__ m_local) {
    const uint64_t m = *total;
    // lower bounds by binary search (one thread), then a strided copy
    __shared__ uint64_t lo_hi[2];
    if (threadIdx.x < 2) {
        const uint64_t key = off + (threadIdx.x ? n : 0);
        uint64_t lo = 0, hi = m;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if ((uint64_t)glist[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        lo_hi[threadIdx.x] = lo;
    }
    __syncthreads();
    const uint64_t a = lo_hi[0], b = lo_hi[1];
    for (uint64_t i = a + threadIdx.x; i < b; i += blockDim.x) out[i - a] = (uint32_t)(glist[i] - off);
    if (threadIdx.x == 0) *m_local = b - a;
}

// equal-to-threshold keys of this rank -> eq slot; then this rank's share of
// the boundary ties in rank order (sel_state[1] = local need)
__global__ void k_adapt_eq(const unsigned long long* __restrict__ cand, uint64_t chunk,
                           const uint32_t* __restrict__ cnt,
                           const unsigned long long* __restrict__ sel_state,
                           unsigned long long* __restrict__ slot) {
    // keys equal to T are in the first digit's bucket: its segments only
    const unsigned long long T = sel_state[0];
    const unsigned long long* seg = cand + blockIdx.x * chunk;
    const uint32_t m = cnt[blockIdx.x];
    unsigned long long c = 0;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) c += seg[i] == T;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(slot, c);
}
__global__ void k_tie_quota(const unsigned long long* __restrict__ eq, int world, int rank,
                            unsigned long long* __restrict__ sel_state) {
    unsigned long long need = sel_state[1], before = 0;
    for (int r = 0; r < rank; ++r) before += eq[r];
    const unsigned long long mine = eq[rank];
    sel_state[1] = need > before ? (need - before < mine ? need - before : mine) : 0ULL;
}

// ---------------------------------------------------------------------------
// bitmap -> sorted index list
// ---------------------------------------------------------------------------

__global__ void k_bitmap_count(const uint32_t* __restrict__ bitmap, uint64_t words,
                               uint32_t* __restrict__ bcount) {
    // one block = 1024 words
    __shared__ uint32_t s[32];
    const uint64_t w = blockIdx.x * 1024ull + threadIdx.x;
    uint32_t c = w < words ? __popc(bitmap[w]) : 0u;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t v = s[threadIdx.x];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) bcount[blockIdx.x] = v;
    }
}

// exclusive scan of the per-block counts in place, 1024 at a time (warp
// scans, then a scan of the warp sums); *total = the sum
__global__ void __launch_bounds__(1024) k_block_scan(uint32_t* __restrict__ bcount, uint64_t nb,
                                                     unsigned long long* __restrict__ total) {
    __shared__ uint32_t wsum[32];
    __shared__ unsigned long long carry;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < nb; base += 1024) {
        const uint64_t b = base + threadIdx.x;
        const uint32_t c = b < nb ? bcount[b] : 0u;
        uint32_t inc = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if ((int)lane >= o) inc += v;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            uint32_t v = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
                if ((int)lane >= o) v += u;
            }
            wsum[lane] = v;  // inclusive over the warps
        }
        __syncthreads();
        const uint32_t before = (wid ? wsum[wid - 1] : 0u) + inc - c;
        if (b < nb) bcount[b] = (uint32_t)(carry + before);
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void k_bitmap_write(const uint32_t* __restrict__ bitmap, uint64_t words,
                               const uint32_t* __restrict__ boff, uint32_t* __restrict__ out) {
    __shared__ uint32_t wsum[32];
    const uint64_t w = blockIdx.x * 1024ull + threadIdx.x;
    const uint32_t bits = w < words ? bitmap[w] : 0u;
    const uint32_t c = __popc(bits);
    // exclusive scan of c over the block
    uint32_t inc = c;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    uint32_t pos = boff[blockIdx.x] + inc - c + (wid ? wsum[wid - 1] : 0u);
    uint32_t b = bits;
    while (b) {
        const int i = __ffs(b) - 1;
        b &= b - 1;
        out[pos++] = (uint32_t)(w * 32 + i);
    }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

namespace {
constexpr uint32_t kSlack = 4096;  // extra draws for rejection replays
}

int sampler_setup(SamplerState& s, int kind, uint64_t n, uint64_t m, uint64_t seed, double alpha,
                  double beta, int sm_count) {
    if (s.side) cudaStreamSynchronize(s.side);  // no generation of a previous setup in flight
    s.pre = false;
    s.age_pending = false;
    s.want_gen = false;
    s.kind = kind;
    s.n = n;
    s.m = m;
    s.alpha = alpha;
    s.beta = beta;
    if (!s.sharded) {
        s.gN = n;
        s.off = 0;
    }
    const uint64_t gN = s.gN;
    s.draws_per_epoch = 0;
    // random: every rank draws the whole epoch's m indices (Floyd is global);
    // adaptive: each rank draws for its own rows, at its offset of the stream
    if (kind == 1 && m < gN) s.draws_per_epoch = m;
    if (kind == 2) s.draws_per_epoch = n;
    const uint64_t stream_off = kind == 2 ? s.off : 0;
    s.jump0 = stream_off > 0;
    // Rng(seed, SeedStream::sampler): mt19937_64(mix_seed(seed, 3)) (rng.hpp:12-37)
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (3 + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    uint64_t w[312];
    mt::seed_window(z ^ (z >> 31), w);
    if (s.window.ensure(312 * 8) != cudaSuccess) return 4;
    if (h2d_blocking(s.window.p, w, 312 * 8) != cudaSuccess) return 4;
    if (s.misc.ensure(128) != cudaSuccess) return 4;
    if (s.sharded && s.slots.ensure((size_t)std::max(1, s.world) * 8) != cudaSuccess) return 4;
    if (kind == 2 && s.sharded) {
        // the stream advances by gN draws per epoch, whatever this rank's share
        const std::vector<uint64_t> JN = mt::jump_poly(gN);
        if (s.jN.ensure(312 * 8) != cudaSuccess) return 4;
        if (h2d_blocking(s.jN.p, JN.data(), 312 * 8) != cudaSuccess) return 4;
    }
    if (!s.draws_per_epoch) return 0;
    const uint64_t total = s.draws_per_epoch + kSlack;
    uint64_t G = (total + 65535) / 65536;
    // two generators per SM: the jumps (one ~210-KB CTA each) run in two
    // waves, the generation itself in small CTAs that halve the sequential
    // twist rounds per generator
    G = std::max<uint64_t>(1, std::min<uint64_t>(G, 2ull * (uint64_t)sm_count));
    const uint64_t L = (total + G - 1) / G;
    s.G = (uint32_t)G;
    s.L = L;
    // jump polynomials t^(stream_off + gL) mod phi (host, once per configuration)
    std::vector<uint64_t> jp(G * 312, 0);
    if (G > 1 || stream_off > 0) {
        const std::vector<uint64_t> J = mt::jump_poly(L);
        std::vector<uint64_t> cur = stream_off > 0 ? mt::jump_poly(stream_off) : J;
        for (uint64_t g = stream_off > 0 ? 0 : 1; g < G; ++g) {
            std::copy(cur.begin(), cur.end(), jp.begin() + g * 312);
            if (g + 1 < G) cur = mt::mul_poly(cur, J);
        }
    }
    if (s.jp.ensure(jp.size() * 8) != cudaSuccess) return 4;
    if (s.gwin.ensure(G * 312 * 8) != cudaSuccess) return 4;
    if (h2d_blocking(s.jp.p, jp.data(), jp.size() * 8) != cudaSuccess) return 4;
    const uint32_t twists = (mt::kSeq - 312 + 311) / 312;
    s.tail0 = s.draws_per_epoch;
    s.tail_len = 312 + kSlack;
    for (int b = 0; b < 2; ++b) {
        if (s.seqb[b].ensure((312 + (size_t)twists * 312) * 8) != cudaSuccess) return 4;
        if (s.drawsb[b].ensure(total * 8) != cudaSuccess) return 4;
        if (s.tailb[b].ensure((size_t)s.tail_len * 8) != cudaSuccess) return 4;
    }
    s.cur = 0;
    s.pre = false;
    if (!s.side && cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking) != cudaSuccess) return 4;
    if (!s.ev_adv && cudaEventCreateWithFlags(&s.ev_adv, cudaEventDisableTiming) != cudaSuccess)
        return 4;
    if (!s.ev_gen && cudaEventCreateWithFlags(&s.ev_gen, cudaEventDisableTiming) != cudaSuccess)
        return 4;
    if (kind == 2) {
        if (s.err.ensure(n * 8) != cudaSuccess || s.age.ensure(n * 4) != cudaSuccess ||
            s.keys.ensure(n * 8) != cudaSuccess || s.hist.ensure(4096 * 4) != cudaSuccess ||
            s.cand.ensure(n * 8) != cudaSuccess || s.cidx.ensure(n * 4) != cudaSuccess ||
            s.ccnt.ensure(kCompactBlocks * 4) != cudaSuccess)
            return 4;
        // last_error = kUnseenError (sampling.hpp:81, 91), age = 0
        const size_t chunk = 1 << 20;
        std::vector<double> init(std::min<uint64_t>(n, chunk), 1e30);
        for (uint64_t i = 0; i < n; i += chunk)
            if (h2d_blocking(s.err.as<double>() + i, init.data(),
                             std::min<uint64_t>(chunk, n - i) * 8) != cudaSuccess)
                return 4;
        if (cudaMemset(s.age.p, 0, n * 4) != cudaSuccess) return 4;
        if (cudaMemset(s.hist.p, 0, 4096 * 4) != cudaSuccess) return 4;
        // legacy-stream memsets: complete before the sampler's own streams use them
        if (cudaStreamSynchronize(0) != cudaSuccess) return 4;
    }
    if (kind == 1) {
        if (s.first.ensure(gN * 4) != cudaSuccess || s.tidx.ensure(m * 4) != cudaSuccess) return 4;
        if (s.sharded && s.glist.ensure(m * 4) != cudaSuccess) return 4;
    }
    return 0;
}

// the epoch's draws (k_mt_extend + k_mt_generate) into buffer b
static void generate_draws(SamplerState& s, int b, cudaStream_t st) {
    const uint32_t twists = (mt::kSeq - 312 + 311) / 312;
    TSOM_LAUNCH(k_mt_extend<<<1, kT, 0, st>>>(s.window.as<uint64_t>(), twists,
                                              s.seqb[b].as<uint64_t>()));
    const size_t smem = (mt::kSeq + 312) * 8 + kJumpIdxBytes;
    ensure_smem_attr((const void*)k_mt_jump_all, smem);
    ensure_smem_attr((const void*)k_mt_jump_window, smem);
    const uint64_t total = s.draws_per_epoch + kSlack;
    TSOM_LAUNCH(k_mt_jump_all<<<s.G, kT, smem, st>>>(s.seqb[b].as<uint64_t>(), s.jp.as<uint64_t>(),
                                                     s.L, total, s.gwin.as<uint64_t>(), s.jump0));
    TSOM_LAUNCH(k_mt_generate<<<s.G, kT, 0, st>>>(s.gwin.as<uint64_t>(), s.L, total,
                                                  s.drawsb[b].as<uint64_t>(), s.tail0, s.tail_len,
                                                  s.tailb[b].as<uint64_t>()));
}

// bitmap of `n` rows -> sorted ids in `out`; total count -> misc[3]
static void bitmap_to_list(SamplerState& s, uint64_t n, uint32_t* out, cudaStream_t st) {
    const uint64_t words = (n + 31) / 32;
    const uint64_t nb = (words + 1023) / 1024;
    TSOM_LAUNCH(k_bitmap_count<<<(unsigned)nb, 1024, 0, st>>>(s.bitmap.as<uint32_t>(), words,
                                                               s.bcount.as<uint32_t>()));
    TSOM_LAUNCH(k_block_scan<<<1, 1024, 0, st>>>(s.bcount.as<uint32_t>(), nb,
                                               reinterpret_cast<unsigned long long*>(
                                                   s.misc.as<uint64_t>() + 3)));
    TSOM_LAUNCH(k_bitmap_write<<<(unsigned)nb, 1024, 0, st>>>(s.bitmap.as<uint32_t>(), words,
                                                               s.bcount.as<uint32_t>(), out));
}

// misc: [0] delta (draws used), [1] status (u32: 1 rejection, 2 boundary tie,
// 4 slack exceeded), [2] tie count, [3] selected count, [4..5] adaptive max,
// [6..7] radix state
int sampler_select(SamplerState& s, uint32_t* out, uint64_t* m_out, int sm_count, cudaStream_t st) {
    const uint64_t n = s.n, gN = s.gN;
    uint64_t* misc = s.misc.as<uint64_t>();
    cudaMemsetAsync(misc, 0, 64, st);
    if (s.kind == 0 || (s.kind == 1 && s.m >= gN)) {
        *m_out = n;
        return -1;  // identity selection: the caller uses "all rows"
    }
    // random sharded: the whole gN-row bitmap (Floyd is global)
    const uint64_t bits = s.kind == 1 ? gN : n;
    const uint64_t words = (bits + 31) / 32;
    const uint64_t nb = (words + 1023) / 1024;
    if (s.bitmap.ensure(words * 4) != cudaSuccess || s.bcount.ensure(nb * 4 + 4) != cudaSuccess)
        return 4;
    cudaMemsetAsync(s.bitmap.p, 0, words * 4, st);
    const int b = s.cur;
    if (s.pre)
        cudaStreamWaitEvent(st, s.ev_gen, 0);  // generated during the previous epoch
    else
        generate_draws(s, b, st);
    s.pre = false;
    s.want_gen = false;
    const uint64_t* draws = s.drawsb[b].as<uint64_t>();
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((std::max(s.m, bits) + 255) / 256, (uint64_t)sm_count * 16));
    uint32_t* status = reinterpret_cast<uint32_t*>(misc + 1);
    auto* total = reinterpret_cast<unsigned long long*>(misc + 3);
    bool ok = true;
    if (s.kind == 1) {
        const uint64_t m = s.m;
        cudaMemsetAsync(s.first.p, 0xFF, gN * 4, st);
        cudaMemcpyAsync(misc, &m, 8, cudaMemcpyHostToDevice, st);  // delta = m (no rejection)
        TSOM_LAUNCH(k_rand_index<<<grid, 256, 0, st>>>(draws, gN, m, s.tidx.as<uint32_t>(),
                                                       s.first.as<uint32_t>(), status));
        TSOM_LAUNCH(k_rand_replay<<<1, 1, 0, st>>>(draws, s.draws_per_epoch + kSlack, gN, m,
                                                   s.tidx.as<uint32_t>(), s.first.as<uint32_t>(),
                                                   misc, status));
        TSOM_LAUNCH(k_rand_pick<<<grid, 256, 0, st>>>(s.tidx.as<uint32_t>(), s.first.as<uint32_t>(),
                                                      gN, m, s.bitmap.as<uint32_t>()));
        if (s.sharded) {
            bitmap_to_list(s, gN, s.glist.as<uint32_t>(), st);
            TSOM_LAUNCH(k_local_slice<<<1, 1024, 0, st>>>(s.glist.as<uint32_t>(), total, s.off, n, out,
                                                          total));
        } else {
            bitmap_to_list(s, n, out, st);
        }
    } else {
        const uint64_t m = std::min(s.m, gN);
        cudaMemcpyAsync(misc, &gN, 8, cudaMemcpyHostToDevice, st);  // delta = gN draws
        auto* mx = reinterpret_cast<unsigned long long*>(misc + 4);
        const int pending = s.age_pending ? 1 : 0;
        TSOM_LAUNCH(k_adapt_max<<<grid, 256, 0, st>>>(s.err.as<double>(), s.age.as<uint32_t>(), n,
                                                      pending, mx));
        if (s.sharded) ok &= s.allreduce(mx, 2, 1);  // the maxima over all rows
        auto* rs = reinterpret_cast<unsigned long long*>(misc + 6);
        const unsigned long long st0[2] = {0ULL, (unsigned long long)m};
        cudaMemcpyAsync(rs, st0, 16, cudaMemcpyHostToDevice, st);
        auto* keys = reinterpret_cast<unsigned long long*>(s.keys.p);
        auto* cand = reinterpret_cast<unsigned long long*>(s.cand.p);
        uint32_t* ccnt = s.ccnt.as<uint32_t>();
        // (a multiple of 32: a compaction warp's rows fill whole bitmap words)
        const uint64_t chunk = ((n + kCompactBlocks - 1) / kCompactBlocks + 31) / 32 * 32;
        TSOM_LAUNCH(k_adapt_keys<<<grid, 256, 0, st>>>(s.err.as<double>(), s.age.as<uint32_t>(),
                                                       draws, n, s.alpha, s.beta, pending, mx, keys,
                                                       s.hist.as<uint32_t>()));
        s.age_pending = false;  // the keys pass wrote the ages back
        // digits of the 64-bit key: bits 52-63, 40-51, 28-39, 16-27, 4-15, 0-3.
        // Digit 0 scans every key, digit 1 comes with the compaction of digit
        // 0's bucket, digits 2-5 scan only that bucket.  Sharded: each digit
        // histogram summed over the ranks (the same digit is then picked
        // everywhere: one global threshold).
        const int shifts[6] = {52, 40, 28, 16, 4, 0}, widths[6] = {12, 12, 12, 12, 12, 4};
        for (int d = 0; d < 6; ++d) {
            // (digit 0's histogram came with the keys, k_adapt_keys)
            if (d == 1)
                TSOM_LAUNCH(k_adapt_compact<<<kCompactBlocks, 256, 0, st>>>(
                    keys, n, chunk, rs, cand, s.cidx.as<uint32_t>(), ccnt, s.hist.as<uint32_t>(),
                    s.bitmap.as<uint32_t>()));
            else if (d >= 2)
                TSOM_LAUNCH(k_adapt_hist_cand<<<kCompactBlocks, 256, 0, st>>>(
                    cand, chunk, ccnt, rs, shifts[d], widths[d], s.hist.as<uint32_t>()));
            if (s.sharded) ok &= s.allreduce(s.hist.p, 4096, 0);
            TSOM_LAUNCH(k_adapt_digit<<<1, 1024, 0, st>>>(s.hist.as<uint32_t>(), shifts[d], rs));
        }
        if (s.sharded) {  // boundary ties: taken in rank order
            auto* eq = reinterpret_cast<unsigned long long*>(s.slots.p);
            cudaMemsetAsync(eq, 0, (size_t)s.world * 8, st);
            TSOM_LAUNCH(k_adapt_eq<<<kCompactBlocks, 256, 0, st>>>(cand, chunk, ccnt, rs,
                                                                    eq + s.rank));
            ok &= s.allreduce(eq, (size_t)s.world, 2);
            TSOM_LAUNCH(k_tie_quota<<<1, 1, 0, st>>>(eq, s.world, s.rank, rs));
        }
        TSOM_LAUNCH(k_adapt_mark_cand<<<kCompactBlocks, 256, 0, st>>>(
            cand, s.cidx.as<uint32_t>(), chunk, ccnt, rs, s.bitmap.as<uint32_t>(),
            reinterpret_cast<unsigned long long*>(misc + 2)));
        bitmap_to_list(s, n, out, st);
    }
    if (!ok) return 5;
    // the stream continues after the draws actually used
    if (s.kind == 2 && s.sharded)
        TSOM_LAUNCH(k_mt_jump_window<<<1, kT, (mt::kSeq + 312) * 8 + kJumpIdxBytes, st>>>(
            s.seqb[b].as<uint64_t>(), s.jN.as<uint64_t>(), s.window.as<uint64_t>()));
    else
        TSOM_LAUNCH(k_mt_advance<<<1, 320, 0, st>>>(s.seqb[b].as<uint64_t>(),
                                                    s.tailb[b].as<uint64_t>(), s.tail0, s.tail_len,
                                                    misc, s.window.as<uint64_t>(), status));
    // the next epoch's draws depend only on the advanced stream state; they are
    // generated on the side stream while this epoch trains (sampler_pregenerate,
    // started once the BMU kernel has finished so it does not compete with it)
    s.cur = b ^ 1;
    s.want_gen = true;
    if (s.sharded) {  // this rank's share is only known on the device
        unsigned long long mloc = 0;
        cudaMemcpyAsync(&mloc, total, 8, cudaMemcpyDeviceToHost, st);
        if (s.sync) {
            if (!s.sync(st)) return 5;
        } else {
            cudaStreamSynchronize(st);
        }
        *m_out = mloc;
    } else {
        *m_out = s.kind == 1 ? s.m : std::min(s.m, n);
    }
    return 0;
}

void sampler_pregenerate(SamplerState& s, cudaEvent_t after) {
    if (!s.want_gen) return;
    s.want_gen = false;
    cudaStreamWaitEvent(s.side, after, 0);
    generate_draws(s, s.cur, s.side);
    cudaEventRecord(s.ev_gen, s.side);
    s.pre = true;
}

void sampler_release(SamplerState& s) {
    if (s.side) cudaStreamSynchronize(s.side);
    for (DevBuf* d : {&s.window, &s.jp, &s.gwin, &s.misc, &s.seqb[0], &s.seqb[1], &s.drawsb[0],
                      &s.drawsb[1], &s.tailb[0], &s.tailb[1], &s.err, &s.age, &s.keys, &s.hist, &s.cand, &s.cidx, &s.ccnt,
                      &s.first, &s.tidx, &s.bitmap, &s.bcount, &s.sel})
        d->release();
    if (s.ev_adv) cudaEventDestroy(s.ev_adv);
    if (s.ev_gen) cudaEventDestroy(s.ev_gen);
    if (s.side) cudaStreamDestroy(s.side);
    s = SamplerState();
}

void sampler_observe(SamplerState& s, const uint32_t* sel, uint64_t m, const double* dist,
                     int sm_count, cudaStream_t st) {
    if (s.kind != 2) return;
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((s.n + 255) / 256, (uint64_t)sm_count * 16));
    if (s.age_pending)  // two observes without a select in between
        TSOM_LAUNCH(k_adapt_age<<<grid, 256, 0, st>>>(s.age.as<uint32_t>(), s.n));
    if (m)
        TSOM_LAUNCH(k_adapt_observe<<<grid, 256, 0, st>>>(sel, m, dist, s.err.as<double>(),
                                                          s.age.as<uint32_t>()));
    s.age_pending = true;
}

void sampler_materialize_ages(SamplerState& s, int sm_count, cudaStream_t st) {
    if (s.kind != 2 || !s.age_pending) return;
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((s.n + 255) / 256, (uint64_t)sm_count * 16));
    TSOM_LAUNCH(k_adapt_age<<<grid, 256, 0, st>>>(s.age.as<uint32_t>(), s.n));
    s.age_pending = false;
}

}  // namespace tsom

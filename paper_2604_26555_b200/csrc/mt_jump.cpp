// mt_jump.cpp — jump-ahead for the reference's random stream (host side).
//
// The samplers draw from toposom::Rng = std::mt19937_64 (rng.hpp:33-91).  To
// produce an epoch's draws on the GPU with many independent generators, each
// generator starts at its own offset of the SAME stream: the state at output
// q + L is obtained from the outputs around q with the jump polynomial
//     J_L(t) = t^L mod phi(t),
// phi the characteristic polynomial of the MT19937-64 transition (degree
// 19937): every bit sequence of the untempered words X[k] satisfies phi, so
//     X[q + L + j] = XOR_{i : J_L[i] = 1} X[q + i + j]   (j = 0..311).
// phi is recovered once by Berlekamp-Massey from 2 * 19937 output bits; the
// polynomial arithmetic (carry-less multiply, reduction by a byte table) runs
// on the host once per sampler configuration.  Pure CPU code: exercised by the
// CPU test suite through tsom_mt_selftest.
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include <immintrin.h>

#include "mt_jump.h"

namespace tsom {
namespace mt {

namespace {

constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 63) / 64;  // 312: polynomials of degree < 19937
constexpr uint64_t kA = 0xB5026F5AA96619E9ULL, kUM = 0xFFFFFFFF80000000ULL,
                   kLM = 0x7FFFFFFFULL;

inline uint64_t step(uint64_t x0, uint64_t x1, uint64_t xm) {
    const uint64_t y = (x0 & kUM) | (x1 & kLM);
    return xm ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
}

using Poly = std::vector<uint64_t>;  // bit i = coefficient of t^i

inline bool getbit(const Poly& p, size_t i) { return (p[i >> 6] >> (i & 63)) & 1ULL; }
inline void flip(Poly& p, size_t i) { p[i >> 6] ^= 1ULL << (i & 63); }

// carry-less 64 x 64 -> 128: PCLMULQDQ when the host has it, else portable
__attribute__((target("pclmul,sse2"))) inline void clmul_hw(uint64_t a, uint64_t b, uint64_t& lo,
                                                           uint64_t& hi) {
    const __m128i r = _mm_clmulepi64_si128(_mm_set_epi64x(0, (long long)a),
                                           _mm_set_epi64x(0, (long long)b), 0x00);
    lo = (uint64_t)_mm_cvtsi128_si64(r);
    hi = (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(r, r));
}

inline void clmul_sw(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
    uint64_t l = 0, h = 0;
    for (int i = 0; i < 64; ++i)
        if ((b >> i) & 1ULL) {
            l ^= a << i;
            if (i) h ^= a >> (64 - i);
        }
    lo = l;
    hi = h;
}

struct Field {
    Poly phi;  // kWords + 1 words, bit kDeg set
    // red[k][v]: (byte v at bit kDeg + 8k) reduced mod phi, k = 0..7 — reduces
    // 64 excess bits at a time
    std::vector<Poly> red;
};

Field* g_field = nullptr;
std::once_flag g_once;

// the first 2 * kDeg + 64 untempered words X[312 + k] of a seeded generator
std::vector<uint64_t> raw_words(uint64_t seed, size_t count) {
    std::vector<uint64_t> x(312 + count);
    x[0] = seed;
    for (int i = 1; i < 312; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (size_t k = 0; k < count; ++k) x[312 + k] = step(x[k], x[k + 1], x[k + 156]);
    return x;
}

// Berlekamp-Massey over GF(2) on bit 0 of X[312 + k]: the minimal polynomial
// of the transition (degree 19937).  Returns phi with phi_j = C_{L-j}.
Poly berlekamp_massey() {
    const size_t N = 2 * kDeg + 64;
    const std::vector<uint64_t> x = raw_words(0x1234567ULL, N);
    // r = reversed sequence: r[k] = s[N - 1 - k], s[k] = bit0 of X[312 + k]
    const size_t rw = (N + 63) / 64 + 2;
    std::vector<uint64_t> r(rw, 0);
    for (size_t k = 0; k < N; ++k)
        if (x[312 + k] & 1ULL) {
            const size_t p = N - 1 - k;
            r[p >> 6] |= 1ULL << (p & 63);
        }
    auto rbits = [&](size_t off) -> uint64_t {  // 64 bits of r from bit `off`
        const size_t w = off >> 6, b = off & 63;
        uint64_t v = r[w] >> b;
        if (b && w + 1 < rw) v |= r[w + 1] << (64 - b);
        return v;
    };
    const size_t cw = (N + 63) / 64 + 2;
    std::vector<uint64_t> C(cw, 0), B(cw, 0), T;
    C[0] = B[0] = 1;
    size_t L = 0, m = 1;
    for (size_t n = 0; n < N; ++n) {
        // d = sum_{i=0..L} C_i s[n - i] = sum_i C_i r[N - 1 - n + i]
        uint64_t acc = 0;
        const size_t base = N - 1 - n;
        for (size_t w = 0; w * 64 <= L; ++w) {
            uint64_t c = C[w];
            if ((w + 1) * 64 > L + 1) c &= (L + 1 - w * 64 >= 64) ? ~0ULL : ((1ULL << ((L + 1) - w * 64)) - 1);
            acc ^= c & rbits(base + w * 64);
        }
        const int d = __builtin_parityll(acc);
        if (!d) {
            ++m;
            continue;
        }
        const bool grow = 2 * L <= n;
        if (grow) T = C;
        // C ^= B << m
        const size_t ws = m >> 6, bs = m & 63;
        for (size_t w = cw; w-- > ws;) {
            uint64_t v = B[w - ws] << bs;
            if (bs && w - ws >= 1) v |= B[w - ws - 1] >> (64 - bs);
            C[w] ^= v;
        }
        if (grow) {
            L = n + 1 - L;
            B = T;
            m = 1;
        } else {
            ++m;
        }
    }
    Poly phi(kWords + 1, 0);
    for (size_t j = 0; j <= L; ++j)
        if ((C[(L - j) >> 6] >> ((L - j) & 63)) & 1ULL) flip(phi, j);
    return phi;
}

// reduce a product (up to 2 * kDeg bits) mod phi in place; result < kDeg bits.
// Excess bits are folded 64 at a time from the top: bits [lo, top) = e stand
// for e * t^lo = e * t^(lo - kDeg) * t^kDeg, and the byte tables hold
// (byte << 8k) * t^kDeg mod phi; shifted by lo - kDeg they land below lo.
void reduce(const Field& f, Poly& p) {
    for (size_t top = p.size() * 64; top > (size_t)kDeg;) {
        const size_t lo = top >= (size_t)kDeg + 64 ? top - 64 : (size_t)kDeg;
        uint64_t e = 0;
        for (size_t i = lo; i < top; ++i)
            if (getbit(p, i)) {
                e |= 1ULL << (i - lo);
                flip(p, i);
            }
        const size_t sh = lo - kDeg, ws = sh >> 6, bs = sh & 63;
        for (int k = 0; k < 8; ++k) {
            const uint32_t v = (uint32_t)((e >> (8 * k)) & 0xFFu);
            if (!v) continue;
            const Poly& r = f.red[k * 256 + v];
            for (size_t w = 0; w < (size_t)kWords; ++w) {
                if (!r[w]) continue;
                p[w + ws] ^= r[w] << bs;
                if (bs) p[w + ws + 1] ^= r[w] >> (64 - bs);
            }
        }
        top = lo;
    }
    p.resize(kWords);
    const int tail = kDeg - 64 * (kWords - 1);
    p[kWords - 1] &= (tail == 64) ? ~0ULL : ((1ULL << tail) - 1);
}

void init_field() {
    auto* f = new Field();
    f->phi = berlekamp_massey();
    // t^(kDeg + b) mod phi for b = 0..63, by repeated multiplication with t
    std::vector<Poly> tb(64);
    Poly cur(kWords + 2, 0);
    // t^kDeg mod phi = phi - t^kDeg
    for (int w = 0; w < kWords + 1; ++w) cur[w] = f->phi[w];
    flip(cur, kDeg);
    for (int b = 0; b < 64; ++b) {
        tb[b] = Poly(cur.begin(), cur.begin() + kWords);
        // cur *= t, then reduce the one bit that may reach kDeg
        for (int w = kWords + 1; w > 0; --w) cur[w] = (cur[w] << 1) | (cur[w - 1] >> 63);
        cur[0] <<= 1;
        if (getbit(cur, kDeg)) {
            flip(cur, kDeg);
            for (int w = 0; w < kWords + 1; ++w) cur[w] ^= f->phi[w] & (w == kDeg / 64 ? ~(1ULL << (kDeg & 63)) : ~0ULL);
        }
    }
    f->red.assign(8 * 256, Poly(kWords, 0));
    for (int k = 0; k < 8; ++k)
        for (int v = 1; v < 256; ++v) {
            Poly& r = f->red[k * 256 + v];
            for (int b = 0; b < 8; ++b)
                if ((v >> b) & 1)
                    for (int w = 0; w < kWords; ++w) r[w] ^= tb[8 * k + b][w];
        }
    g_field = f;
}

const Field& field() {
    std::call_once(g_once, init_field);
    return *g_field;
}

Poly mulmod(const Poly& a, const Poly& b) {
    const Field& f = field();
    static const bool hw = __builtin_cpu_supports("pclmul");
    Poly p(2 * kWords + 2, 0);
    for (int i = 0; i < kWords; ++i) {
        if (!a[i]) continue;
        for (int j = 0; j < kWords; ++j) {
            if (!b[j]) continue;
            uint64_t lo, hi;
            if (hw)
                clmul_hw(a[i], b[j], lo, hi);
            else
                clmul_sw(a[i], b[j], lo, hi);
            p[i + j] ^= lo;
            p[i + j + 1] ^= hi;
        }
    }
    reduce(f, p);
    return p;
}

Poly sqrmod(const Poly& a) {
    const Field& f = field();
    Poly p(2 * kWords + 2, 0);
    for (int i = 0; i < kWords; ++i) {
        uint64_t lo = 0, hi = 0;
        for (int b = 0; b < 32; ++b) {
            lo |= ((a[i] >> b) & 1ULL) << (2 * b);
            hi |= ((a[i] >> (b + 32)) & 1ULL) << (2 * b);
        }
        p[2 * i] = lo;
        p[2 * i + 1] = hi;
    }
    reduce(f, p);
    return p;
}

Poly pow_t(uint64_t e) {
    Poly r(kWords, 0);
    r[0] = 1;  // t^0
    int top = 63;
    while (top >= 0 && !((e >> top) & 1ULL)) --top;
    for (int b = top; b >= 0; --b) {
        r = sqrmod(r);
        if ((e >> b) & 1ULL) {
            // r *= t
            Poly s(kWords + 1, 0);
            for (int w = kWords; w > 0; --w) s[w] = (r[w] << 1) | (r[w - 1] >> 63);
            s[0] = r[0] << 1;
            if (getbit(s, kDeg)) {
                flip(s, kDeg);
                for (int w = 0; w < kWords; ++w) s[w] ^= field().phi[w];
                flip(s, kDeg);  // phi's own top bit cancelled above
            }
            s.resize(kWords);
            r = s;
        }
    }
    return r;
}

}  // namespace

int degree() { return kDeg; }

std::vector<uint64_t> jump_poly(uint64_t L) { return pow_t(L); }

std::vector<uint64_t> mul_poly(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
    return mulmod(a, b);
}

// window (312 untempered words) at output offset L of a stream whose untempered
// words from the current window are seq[0 .. 312 + 19937 + 311) — host reference
// of the device kernel
void apply_jump(const std::vector<uint64_t>& J, const uint64_t* seq, uint64_t* out) {
    for (int j = 0; j < 312; ++j) out[j] = 0;
    for (int i = 0; i < kDeg; ++i)
        if ((J[i >> 6] >> (i & 63)) & 1ULL)
            for (int j = 0; j < 312; ++j) out[j] ^= seq[i + j];
}

void extend(const uint64_t* window, size_t count, uint64_t* seq) {
    std::memcpy(seq, window, 312 * sizeof(uint64_t));
    for (size_t k = 0; k < count; ++k) seq[312 + k] = step(seq[k], seq[k + 1], seq[k + 156]);
}

uint64_t temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

void seed_window(uint64_t seed, uint64_t* window) {
    window[0] = seed;
    for (int i = 1; i < 312; ++i)
        window[i] = 6364136223846793005ULL * (window[i - 1] ^ (window[i - 1] >> 62)) + i;
}

}  // namespace mt
}  // namespace tsom

namespace tsom {
namespace mt {

// Jump a seeded generator by L through the polynomial and compare the window
// and the next 1000 outputs with plain sequential generation.  0 = identical.
int selftest(uint64_t seed, uint64_t L) {
    std::vector<uint64_t> w(312);
    seed_window(seed, w.data());
    // sequential reference: X[0 .. L + 312 + 1000 + 312)
    const size_t total = (size_t)L + 312 + 1312;
    std::vector<uint64_t> ref(312 + total);
    extend(w.data(), total, ref.data());
    // jump
    std::vector<uint64_t> seq(kSeq + 1);
    extend(w.data(), kSeq + 1 - 312, seq.data());
    std::vector<uint64_t> jw(312);
    apply_jump(jump_poly(L), seq.data(), jw.data());
    int bad = 0;
    if ((jw[0] & 0xFFFFFFFF80000000ULL) != (ref[L] & 0xFFFFFFFF80000000ULL)) ++bad;
    for (int j = 1; j < 312; ++j) bad += jw[j] != ref[L + j];
    std::vector<uint64_t> cont(312 + 1000);
    extend(jw.data(), 1000, cont.data());
    for (int k = 0; k < 1000; ++k) bad += temper(cont[312 + k]) != temper(ref[L + 312 + k]);
    return bad;
}

}  // namespace mt
}  // namespace tsom

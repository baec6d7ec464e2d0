// host_synth.cpp — the SURVEY.md §8(d) Gaussian-mixture rows on the host,
// value-identical to the reference's generator, on all host cores.
//
// The stream is one toposom::Rng(seed, SeedStream::synth) (rng.hpp:21-37):
// the n_comp x d centres real(-4, 4) first, then per row m = index(n_comp) and
// d draws of gaussian() (Box-Muller, the second value of each pair cached,
// rng.hpp:64-76), x = f32(mu[m][k] + g).  Without an index() rejection (a
// draw >= 2^64 - (2^64 mod n_comp), probability ~n_comp / 2^64) row r starts
// at output
//     q(r) = n_comp d + r + 2 ceil(r d / 2)
// of the mt19937_64 stream, so each thread jumps its generator straight to
// its first row (t^q mod phi, mt_jump.cpp) and generates its rows with the
// reference's arithmetic (glibc log / sqrt / sin / cos, no FMA contraction:
// compiled with -ffp-contract=off like the reference's Release flags).  A row
// whose index draw is rejected shifts every later row: then the whole set is
// regenerated sequentially.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "mt_jump.h"

namespace tsom {
namespace {

constexpr uint64_t kA = 0xB5026F5AA96619E9ULL, kUM = 0xFFFFFFFF80000000ULL,
                   kLM = 0x7FFFFFFFULL;

// std::mt19937_64 continued from a window of 312 untempered words
struct Mt {
    uint64_t w[312];
    int i = 312;
    explicit Mt(const uint64_t* window) { std::memcpy(w, window, sizeof(w)); }
    void twist() {
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (w[k] & kUM) | (w[k + 1 < 312 ? k + 1 : 0] & kLM);
            w[k] = w[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
        }
        i = 0;
    }
    uint64_t operator()() {
        if (i == 312) twist();
        return mt::temper(w[i++]);
    }
};

// toposom::Rng's draws (rng.hpp:42-76) over an Mt
struct Draws {
    Mt g;
    double cached = 0.0;
    bool has_cached = false;
    explicit Draws(const uint64_t* window) : g(window) {}
    double real01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    double gaussian() {
        if (has_cached) {
            has_cached = false;
            return cached;
        }
        const double u1 = 1.0 - real01();
        const double u2 = real01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.14159265358979323846 * u2;
        cached = r * std::sin(theta);
        has_cached = true;
        return r * std::cos(theta);
    }
};

uint64_t synth_seed(uint64_t seed) {  // mix_seed(seed, SeedStream::synth = 4), rng.hpp:12-18
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (4 + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// rows [r0, r1) (into out + r * d) from a generator positioned at row r0;
// false on a rejection
bool gen_rows(Draws& rg, const std::vector<double>& mu, float* out, uint64_t r0, uint64_t r1,
              uint32_t d, uint32_t n_comp) {
    const uint64_t un = n_comp, limit = UINT64_MAX - UINT64_MAX % un;
    for (uint64_t r = r0; r < r1; ++r) {
        const uint64_t x = rg.g();
        if (x >= limit) return false;
        const size_t m = static_cast<size_t>(x % un);
        float* row = out + r * d;
        for (uint32_t k = 0; k < d; ++k)
            row[k] = static_cast<float>(mu[m * d + k] + rg.gaussian());
    }
    return true;
}

}  // namespace
}  // namespace tsom

extern "C" int tsom_synth_gmm_host(float* out, uint64_t row0, uint64_t n, uint32_t d,
                                   uint64_t seed, uint32_t n_comp, uint32_t threads) {
    using namespace tsom;
    if ((!out && n) || d < 1 || n_comp < 1) return 1;  // TSOM_ERR_INVALID
    uint64_t window[312];
    mt::seed_window(synth_seed(seed), window);
    Draws head(window);
    std::vector<double> mu((size_t)n_comp * d);
    for (auto& v : mu) v = -4.0 + (4.0 - -4.0) * head.real01();  // real(-4, 4), rng.hpp:47
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t min_rows = 65536;  // below this the jumps cost more than they save
    uint64_t T = std::min<uint64_t>(threads, std::max<uint64_t>(1, n / min_rows));
    if (row0 > 0) T = std::max<uint64_t>(T, 1);
    // the reference order, one generator from row 0 (rejections redrawn as
    // index() does); rows before row0 are drawn and dropped
    auto sequential = [&] {
        Draws rg(window);
        for (uint64_t i = 0; i < (uint64_t)n_comp * d; ++i) rg.real01();
        const uint64_t un = n_comp, limit = UINT64_MAX - UINT64_MAX % un;
        for (uint64_t r = 0; r < row0 + n; ++r) {
            uint64_t x;
            do {
                x = rg.g();
            } while (x >= limit);
            const size_t m = static_cast<size_t>(x % un);
            for (uint32_t k = 0; k < d; ++k) {
                const double g = rg.gaussian();
                if (r >= row0) out[(r - row0) * d + k] = static_cast<float>(mu[m * d + k] + g);
            }
        }
        return 0;
    };
    if (T <= 1 && row0 == 0) return sequential();
    // untempered words from the seed window, the input of every jump
    std::vector<uint64_t> seq(mt::kSeq + 1);
    mt::extend(window, seq.size() - 312, seq.data());
    const uint64_t C = (uint64_t)n_comp * d, per = (n + T - 1) / T;
    std::vector<char> ok(T, 1);
    std::vector<std::thread> pool;
    for (uint64_t t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            // rows [r0, r1) of the stream, written from out[(r0 - row0) * d]
            const uint64_t r0 = row0 + std::min(n, t * per), r1 = row0 + std::min(n, t * per + per);
            if (r0 >= r1) return;
            // a pending cached gaussian at row r0 (r0 d odd) is the second half
            // of the pair drawn just before its index draw: start 2 draws early
            const bool carry = ((r0 * d) & 1ULL) != 0;
            const uint64_t q = C + r0 + 2 * ((r0 * d + 1) / 2) - (carry ? 2 : 0);
            uint64_t jw[312];
            mt::apply_jump(mt::jump_poly(q), seq.data(), jw);
            Draws rg(jw);
            if (carry) {
                rg.has_cached = false;
                rg.gaussian();  // recompute the pair; its sin half is now cached
            }
            ok[t] = gen_rows(rg, mu, out - row0 * d, r0, r1, d, n_comp);
        });
    for (auto& th : pool) th.join();
    for (char o : ok)
        if (!o) return sequential();  // an index() rejection shifted the stream
    return 0;
}

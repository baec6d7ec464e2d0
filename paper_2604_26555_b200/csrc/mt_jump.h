// mt_jump.h — host-side jump-ahead of std::mt19937_64 (see mt_jump.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace tsom {
namespace mt {

constexpr int kN = 312;      // state words
constexpr int kSeq = 20248;  // untempered words a jump reads: 19937 + 311

int degree();
// t^L mod phi (312 words, bit i = coefficient of t^i)
std::vector<uint64_t> jump_poly(uint64_t L);
std::vector<uint64_t> mul_poly(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b);
// out[j] = XOR_{i: J_i} seq[i + j], j < 312 (host reference of the device jump)
void apply_jump(const std::vector<uint64_t>& J, const uint64_t* seq, uint64_t* out);
// seq[0..312) = window, then `count` more untempered words by the recurrence
void extend(const uint64_t* window, size_t count, uint64_t* seq);
uint64_t temper(uint64_t x);
// std::mt19937_64(seed) state words (the window before output 0)
void seed_window(uint64_t seed, uint64_t* window);
// jump-vs-sequential self check (0 = identical)
int selftest(uint64_t seed, uint64_t L);

}  // namespace mt
}  // namespace tsom

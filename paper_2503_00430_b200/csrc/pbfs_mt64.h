// mt19937_64 ([rand.predef]: w=64 n=312 m=156 r=31), bit-identical to
// std::mt19937_64 -- the draw stream of the reference generator
// (generator.cpp:16-29) -- with O(p^2) jump-ahead so the stream can be cut
// into chunks that host threads generate in parallel.
//
// Jump-ahead (the polynomial method of Haramoto, Matsumoto, Nishimura,
// Panneton and L'Ecuyer, "Efficient jump ahead for F2-linear random number
// generators", 2008): the state transition T is linear over GF(2); on the
// 19937-dimensional subspace every reachable state lives in, its minimal
// polynomial phi has degree p = 19937. phi is recovered once by
// Berlekamp-Massey from 2p output bits, and T^J s = g(T) s with
// g = t^J mod phi, evaluated by Horner's rule on the state: p steps of one
// generator word each plus a state XOR per set coefficient.
#pragma once

#include <cstdint>
#include <vector>

namespace pbfs {

class Mt64 {
 public:
  static constexpr int N = 312, M = 156;
  explicit Mt64(uint64_t seed) {
    s_[0] = seed;
    for (int i = 1; i < N; ++i) s_[i] = 6364136223846793005ULL * (s_[i - 1] ^ (s_[i - 1] >> 62)) + i;
  }
  // Twists the state and writes the next N outputs. The twist is split into
  // its two dependency-free halves so the compiler vectorises it.
  void block(uint64_t* out) {
    constexpr uint64_t U = 0xFFFFFFFF80000000ULL, L = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    uint64_t* mt = s_;
    for (int i = 0; i < N - M; ++i) {
      const uint64_t y = (mt[i] & U) | (mt[i + 1] & L);
      mt[i] = mt[i + M] ^ (y >> 1) ^ ((0 - (y & 1)) & A);
    }
    for (int i = N - M; i < N - 1; ++i) {
      const uint64_t y = (mt[i] & U) | (mt[i + 1] & L);
      mt[i] = mt[i + M - N] ^ (y >> 1) ^ ((0 - (y & 1)) & A);
    }
    {
      const uint64_t y = (mt[N - 1] & U) | (mt[0] & L);
      mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ ((0 - (y & 1)) & A);
    }
    for (int i = 0; i < N; ++i) out[i] = temper(mt[i]);
  }
  static uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
  }
  // The raw state: after b calls of block() it holds X_{312b .. 312b+311} of
  // the linear recurrence, the values the NEXT block() twists.
  uint64_t* state() { return s_; }
  const uint64_t* state() const { return s_; }

 private:
  uint64_t s_[N];
};

// g(t) = t^J mod phi(t), as packed coefficients (bit k = coefficient of t^k).
std::vector<uint64_t> mt64_jump_poly(uint64_t J);

// Replaces `state` (an Mt64 state after at least one block(), i.e. on the
// reachable subspace) by T^J state for the J that `poly` = mt64_jump_poly(J)
// was made for: afterwards block() continues the stream J draws further on.
// J must be a multiple of 312 for the block() alignment to carry over.
void mt64_jump(uint64_t* state, const std::vector<uint64_t>& poly);

}  // namespace pbfs

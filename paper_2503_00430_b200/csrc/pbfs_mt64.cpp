// Jump-ahead for mt19937_64 (see pbfs_mt64.h): Berlekamp-Massey for the
// minimal polynomial phi of the transition, t^J mod phi by square-and-
// multiply over GF(2), Horner evaluation of g(T) on a state.
#include "pbfs_mt64.h"

#include <algorithm>
#include <cstring>
#include <mutex>

namespace pbfs {
namespace {

constexpr int kDeg = 19937;                // degree of phi (MT19937-64's period exponent)
constexpr int kWords = (kDeg + 64) / 64;   // coefficient words of a polynomial of degree <= kDeg
constexpr uint64_t kU = 0xFFFFFFFF80000000ULL, kL = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;

using Bits = std::vector<uint64_t>;

inline bool get_bit(const Bits& b, int i) { return (b[i >> 6] >> (i & 63)) & 1u; }
inline void flip_bit(Bits& b, int i) { b[i >> 6] ^= uint64_t{1} << (i & 63); }

// dst ^= src << shift (bit shift, dst sized to hold the result).
void xor_shifted(Bits& dst, const Bits& src, int src_bits, int shift) {
  const int ws = shift >> 6, bs = shift & 63;
  const int nw = (src_bits + 63) >> 6;
  for (int i = 0; i < nw && i + ws < static_cast<int>(dst.size()); ++i) {
    const uint64_t w = src[i];
    if (!w) continue;
    dst[i + ws] ^= w << bs;
    if (bs && i + ws + 1 < static_cast<int>(dst.size())) dst[i + ws + 1] ^= w >> (64 - bs);
  }
}

// Minimal polynomial of the output bit sequence (bit 0 of each draw), which
// for MT19937-64 is phi itself (phi is primitive). Returned in the
// characteristic-polynomial orientation: bit k = coefficient of t^k, bit
// kDeg set.
Bits compute_phi() {
  const int nbits = 2 * kDeg + 64;
  std::vector<uint8_t> s(nbits);
  {
    Mt64 mt(5489u);
    uint64_t buf[Mt64::N];
    for (int i = 0; i < nbits; i += Mt64::N) {
      mt.block(buf);
      for (int j = 0; j < Mt64::N && i + j < nbits; ++j) s[i + j] = buf[j] & 1u;
    }
  }
  // Berlekamp-Massey over GF(2). C, B: connection polynomials (bit i =
  // coefficient of x^i); R holds the recent sequence reversed (bit i =
  // s_{n-i}), so the discrepancy is the parity of C & R.
  const int cap = kDeg + 128;
  const int cw = (cap + 63) / 64;
  Bits C(cw, 0), B(cw, 0), R(cw, 0), Tmp;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  for (int n = 0; n < nbits; ++n) {
    for (int i = cw - 1; i > 0; --i) R[i] = (R[i] << 1) | (R[i - 1] >> 63);
    R[0] = (R[0] << 1) | s[n];
    uint64_t par = 0;
    const int lw = (L >> 6) + 1;
    for (int i = 0; i < lw && i < cw; ++i) par ^= C[i] & R[i];
    if (!(__builtin_popcountll(par) & 1)) {
      ++m;
    } else if (2 * L <= n) {
      Tmp = C;
      xor_shifted(C, B, cap - m, m);
      L = n + 1 - L;
      B = Tmp;
      m = 1;
    } else {
      xor_shifted(C, B, cap - m, m);
      ++m;
    }
  }
  // C(x) = 1 + c1 x + ... + cL x^L  ->  phi(t) = t^L + c1 t^(L-1) + ... + cL.
  Bits phi(kWords, 0);
  for (int i = 0; i <= L; ++i) {
    if (get_bit(C, i)) flip_bit(phi, L - i);
  }
  if (L != kDeg) phi.clear();  // not MT19937-64's recurrence: refuse to jump
  return phi;
}

const Bits& phi() {
  static Bits p;
  static std::once_flag once;
  std::call_once(once, [] { p = compute_phi(); });
  return p;
}

// r <- r mod phi for r of degree < 2 * kDeg (bits from the top down).
void reduce(Bits& r, const Bits& ph) {
  for (int i = 2 * kDeg; i >= kDeg; --i) {
    if (get_bit(r, i)) xor_shifted(r, ph, kDeg + 1, i - kDeg);
  }
}

// Spreads the 32 bits of x to the even bit positions of a 64-bit word.
inline uint64_t spread(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFULL;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFULL;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0FULL;
  v = (v | (v << 2)) & 0x3333333333333333ULL;
  v = (v | (v << 1)) & 0x5555555555555555ULL;
  return v;
}

}  // namespace

std::vector<uint64_t> mt64_jump_poly(uint64_t J) {
  const Bits& ph = phi();
  if (ph.empty()) return {};
  const int big = 2 * kWords + 2;
  Bits r(big, 0);
  r[0] = 1;  // t^0
  int top = 63;
  while (top >= 0 && !((J >> top) & 1u)) --top;
  for (int b = top; b >= 0; --b) {
    // r <- r^2 (GF(2): coefficient k moves to 2k)
    Bits sq(big, 0);
    for (int i = 0; i < kWords; ++i) {
      sq[2 * i] = spread(static_cast<uint32_t>(r[i]));
      sq[2 * i + 1] = spread(static_cast<uint32_t>(r[i] >> 32));
    }
    reduce(sq, ph);
    r.swap(sq);
    if ((J >> b) & 1u) {
      // r <- r * t
      for (int i = big - 1; i > 0; --i) r[i] = (r[i] << 1) | (r[i - 1] >> 63);
      r[0] <<= 1;
      if (get_bit(r, kDeg)) xor_shifted(r, ph, kDeg + 1, 0);
    }
  }
  r.resize(kWords);
  return r;
}

void mt64_jump(uint64_t* state, const std::vector<uint64_t>& poly) {
  constexpr int N = Mt64::N, Mo = Mt64::M;
  // Accumulator as a ring buffer: logical word j lives at acc[(h + j) % N].
  uint64_t acc[N];
  std::memset(acc, 0, sizeof(acc));
  int h = 0;
  int d = kDeg;
  while (d >= 0 && !get_bit(poly, d)) --d;
  for (int i = d; i >= 0; --i) {
    // acc <- T acc (one new word of the recurrence; the oldest drops out)
    {
      const uint64_t a0 = acc[h], a1 = acc[h + 1 < N ? h + 1 : h + 1 - N];
      const uint64_t am = acc[h + Mo < N ? h + Mo : h + Mo - N];
      const uint64_t y = (a0 & kU) | (a1 & kL);
      acc[h] = am ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
      h = h + 1 < N ? h + 1 : 0;
    }
    if (get_bit(poly, i)) {
      // acc <- acc + state
      for (int j = 0; j < N - h; ++j) acc[h + j] ^= state[j];
      for (int j = N - h; j < N; ++j) acc[j - (N - h)] ^= state[j];
    }
  }
  // Horner: acc = (...(g_d T + g_{d-1}) T + ...) state = sum_i g_i T^i state
  // (the first T acts on the zero accumulator).
  for (int j = 0; j < N; ++j) state[j] = acc[(h + j) % N];
}

}  // namespace pbfs

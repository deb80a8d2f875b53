// Host-side widening microbenchmark (the pbfs_bfs_batch e2e bound): 1 B level
// codes -> uint32 distances (0xFF -> 0xFFFFFFFF) for 2^26 vertices, T threads,
// SSE2 / AVX2 non-temporal vs plain stores. Prints destination GB/s.
//   g++ -O3 -march=native -pthread tools/ubench_widen.cpp -o build_ab/ubench_widen
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static void widen_sse(const uint8_t* s, uint32_t* d, size_t b, size_t e, bool nt) {
  const __m128i ones = _mm_set1_epi32(-1);
  for (size_t i = b; i + 16 <= e; i += 16) {
    const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i m = _mm_cmpeq_epi8(x, ones);
    const __m128i lo = _mm_unpacklo_epi8(x, m), hi = _mm_unpackhi_epi8(x, m);
    const __m128i mlo = _mm_unpacklo_epi8(m, m), mhi = _mm_unpackhi_epi8(m, m);
    __m128i* o = reinterpret_cast<__m128i*>(d + i);
    __m128i r0 = _mm_unpacklo_epi16(lo, mlo), r1 = _mm_unpackhi_epi16(lo, mlo);
    __m128i r2 = _mm_unpacklo_epi16(hi, mhi), r3 = _mm_unpackhi_epi16(hi, mhi);
    if (nt) {
      _mm_stream_si128(o, r0); _mm_stream_si128(o + 1, r1);
      _mm_stream_si128(o + 2, r2); _mm_stream_si128(o + 3, r3);
    } else {
      _mm_store_si128(o, r0); _mm_store_si128(o + 1, r1);
      _mm_store_si128(o + 2, r2); _mm_store_si128(o + 3, r3);
    }
  }
  _mm_sfence();
}
#ifdef __AVX2__
static void widen_avx2(const uint8_t* s, uint32_t* d, size_t b, size_t e) {
  for (size_t i = b; i + 8 <= e; i += 8) {
    const __m128i x = _mm_loadl_epi64(reinterpret_cast<const __m128i*>(s + i));
    __m256i w = _mm256_cvtepu8_epi32(x);
    const __m256i m = _mm256_cmpeq_epi32(w, _mm256_set1_epi32(0xFF));
    w = _mm256_or_si256(w, m);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), w);
  }
  _mm_sfence();
}
#endif

int main() {
  const size_t n = size_t{1} << 26;
  uint8_t* src = static_cast<uint8_t*>(aligned_alloc(64, n));
  uint32_t* dst = static_cast<uint32_t*>(aligned_alloc(64, n * 4));
  for (size_t i = 0; i < n; ++i) src[i] = static_cast<uint8_t>(i % 9 == 0 ? 0xFF : i % 7);
  std::memset(dst, 0, n * 4);
  const unsigned hw = std::thread::hardware_concurrency();
  std::printf("hardware threads %u\n", hw);
  for (int variant = 0; variant < 3; ++variant) {
#ifndef __AVX2__
    if (variant == 2) continue;
#endif
    for (unsigned T : {1u, 4u, 8u, 12u, 16u, 24u, 32u}) {
      if (T > hw) continue;
      double best = 1e30;
      for (int rep = 0; rep < 5; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t) {
          th.emplace_back([&, t] {
            const size_t b = (n * t / T) & ~size_t{63}, e = t + 1 == T ? n : (n * (t + 1) / T) & ~size_t{63};
            if (variant == 0) widen_sse(src, dst, b, e, true);
            if (variant == 1) widen_sse(src, dst, b, e, false);
#ifdef __AVX2__
            if (variant == 2) widen_avx2(src, dst, b, e);
#endif
          });
        }
        for (auto& x : th) x.join();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (s < best) best = s;
      }
      std::printf("%-10s T=%2u  %.3f ms  %.1f GB/s dst\n",
                  variant == 0 ? "sse2-nt" : variant == 1 ? "sse2-plain" : "avx2-nt", T, best * 1e3,
                  n * 4 / best / 1e9);
    }
  }
  return 0;
}

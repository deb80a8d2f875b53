// Host-side graph library: seeded generators, the parallel CSR builder, the
// classifier, source selection and the CSR1 format. Same public semantics as
// the reference's proj/core graph layer (generator.cpp, csr_graph.cpp,
// graph_stats.cpp, graph_io.cpp, tools/bfsbench.cpp:pick_sources), rebuilt for
// multi-GB graphs: no O(m log m) global sort, no value-initialised buffers,
// the mt19937_64 stream cut into chunks by jump-ahead (pbfs_mt64.h) and
// generated on every host thread.
#include <immintrin.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "pbfs_internal.h"
#include "pbfs_mt64.h"

namespace pbfs {

namespace {
thread_local std::string g_last_error;
}

pbfs_status fail(pbfs_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}
void clear_error() { g_last_error.clear(); }

unsigned resolve_threads(uint32_t requested) {
  if (requested) return requested;
  unsigned hw = std::thread::hardware_concurrency();
  return hw ? hw : 1;
}

const char* last_error_cstr() { return g_last_error.c_str(); }

namespace {

// PBFS_GEN_TIMING=1: phase times of the generator / builder on stderr.
struct PhaseClock {
  bool on;
  std::chrono::steady_clock::time_point t0;
  PhaseClock() : on(std::getenv("PBFS_GEN_TIMING") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pbfs gen] %-18s %8.3f s\n", what,
                 std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  }
};

// Sequential draw stream with block refills (for the small generators).
class Stream {
 public:
  explicit Stream(uint64_t seed) : mt_(seed) {}
  uint64_t next() {
    if (pos_ == Mt64::N) {
      mt_.block(buf_);
      pos_ = 0;
    }
    return buf_[pos_++];
  }
  // Sampler::bounded (generator.cpp:22-26)
  uint64_t bounded(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
  }
  // Sampler::unit (generator.cpp:29)
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

 private:
  Mt64 mt_;
  uint64_t buf_[Mt64::N];
  int pos_ = Mt64::N;
};

// Quadrant thresholds of generator.cpp:35-37,75-84. unit() < T exactly when
// (draw >> 11) < T * 2^53, and T * 2^53 is an integer for T in [0.5, 1), so
// the comparison chain runs on integers with identical outcomes.
struct KronThresholds {
  uint64_t a, ab, abc;
  KronThresholds() {
    constexpr double kA = 0.57, kB = 0.19, kC = 0.19;
    a = static_cast<uint64_t>(kA * 0x1.0p53);
    ab = static_cast<uint64_t>((kA + kB) * 0x1.0p53);
    abc = static_cast<uint64_t>((kA + kB + kC) * 0x1.0p53);
  }
};

void kron_convert(const uint64_t* draws, uint64_t samples, uint32_t scale,
                  const KronThresholds& t, uint32_t* pairs) {
  for (uint64_t s = 0; s < samples; ++s) {
    const uint64_t* d = draws + s * scale;
    uint64_t row = 0, col = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      const uint64_t r = d[l] >> 11;
      const uint64_t rb = r >= t.ab;                       // c or d quadrant
      const uint64_t cb = (r >= t.a && r < t.ab) | (r >= t.abc);  // b or d quadrant
      row = (row << 1) | rb;
      col = (col << 1) | cb;
    }
    pairs[2 * s] = static_cast<uint32_t>(row);
    pairs[2 * s + 1] = static_cast<uint32_t>(col);
  }
}

void uniform_convert(const uint64_t* draws, uint64_t samples, uint64_t n, uint32_t* pairs) {
  for (uint64_t s = 0; s < samples; ++s) {
    pairs[2 * s] = static_cast<uint32_t>((static_cast<unsigned __int128>(draws[2 * s]) * n) >> 64);
    pairs[2 * s + 1] =
        static_cast<uint32_t>((static_cast<unsigned __int128>(draws[2 * s + 1]) * n) >> 64);
  }
}

// generator.cpp:51-89 — the sample loop. Sample s consumes draws
// [s * per, (s + 1) * per) of ONE mt19937_64 stream, so the stream is cut
// into chunks of whole samples whose start states are reached by jump-ahead
// (pbfs_mt64.h): every host thread generates and converts its own chunks,
// and the pairs are bit-identical to the sequential stream for any thread
// count.
void sample_pairs(uint32_t kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                  unsigned threads, uint32_t* pairs) {
  const uint64_t n = uint64_t{1} << scale;
  const uint64_t samples = n * edge_factor;
  const uint32_t per = kind == PBFS_GEN_KRONECKER ? scale : 2;
  KronThresholds thr;
  PhaseClock jclk;
  // Chunks: a multiple of 312 samples (so of 312 draws too), about four per
  // thread for balance; tiny streams stay one chunk.
  const uint64_t want = (samples + 4ull * threads - 1) / (4ull * threads);
  uint64_t chunk = std::max<uint64_t>(Mt64::N * 16, (want + Mt64::N - 1) / Mt64::N * Mt64::N);
  uint64_t nchunks = threads > 1 ? (samples + chunk - 1) / chunk : 1;
  if (nchunks <= 1) chunk = samples;
  std::vector<std::vector<uint64_t>> start(std::max<uint64_t>(nchunks, 1));
  {
    Mt64 mt(seed);
    start[0].assign(mt.state(), mt.state() + Mt64::N);
    if (nchunks > 1) {
      // W_312 (after one twist) is on the reachable subspace; chunk k starts
      // at draw k * chunk * per.
      uint64_t tmp[Mt64::N];
      mt.block(tmp);
      std::vector<uint64_t> cur(mt.state(), mt.state() + Mt64::N);
      const uint64_t stride = chunk * per;
      const std::vector<uint64_t> first = mt64_jump_poly(stride - Mt64::N);
      const std::vector<uint64_t> step = nchunks > 2 ? mt64_jump_poly(stride) : first;
      if (first.empty() || step.empty()) {
        nchunks = 1;  // cannot jump: one chunk, front to back
        chunk = samples;
      }
      for (uint64_t k = 1; k < nchunks; ++k) {
        mt64_jump(cur.data(), k == 1 ? first : step);
        start[k] = cur;
      }
    }
  }
  jclk.mark("sample: jump setup");
  auto run_chunk = [&](uint64_t k, std::vector<uint64_t>& buf) {
    Mt64 mt(0);
    std::memcpy(mt.state(), start[k].data(), Mt64::N * sizeof(uint64_t));
    const uint64_t first = k * chunk;
    const uint64_t count = std::min(chunk, samples - first);
    // Batches of whole samples and whole twists (multiples of 312 samples).
    const uint64_t batch = Mt64::N * 16;
    buf.resize(batch * per);
    uint64_t tmp[Mt64::N];
    for (uint64_t done = 0; done < count;) {
      const uint64_t cnt = std::min(batch, count - done);
      const uint64_t draws = cnt * per;
      uint64_t produced = 0;
      while (produced + Mt64::N <= draws) {
        mt.block(buf.data() + produced);
        produced += Mt64::N;
      }
      if (produced < draws) {
        mt.block(tmp);
        std::memcpy(buf.data() + produced, tmp, (draws - produced) * sizeof(uint64_t));
      }
      if (kind == PBFS_GEN_KRONECKER) {
        kron_convert(buf.data(), cnt, scale, thr, pairs + 2 * (first + done));
      } else {
        uniform_convert(buf.data(), cnt, n, pairs + 2 * (first + done));
      }
      done += cnt;
    }
  };
  std::atomic<uint64_t> next{0};
  parallel_for_threads(nchunks > 1 ? threads : 1, [&](unsigned) {
    std::vector<uint64_t> buf;
    for (;;) {
      const uint64_t k = next.fetch_add(1);
      if (k >= nchunks) break;
      run_chunk(k, buf);
    }
  });
}

// Config-3 mesh (restated in oracle/pbfs_oracle.c
// orc_mesh_pairs): row-major right-then-down keep draws, then shortcuts.
std::vector<uint32_t> mesh_pairs(const pbfs_gen_spec& s) {
  const uint64_t side = s.mesh_side;
  const uint64_t n = side * side;
  std::vector<uint32_t> pairs;
  pairs.reserve(2 * (2 * side * (side - 1) + s.mesh_shortcuts));
  Stream rng(s.seed);
  for (uint64_t r = 0; r < side; ++r) {
    for (uint64_t c = 0; c < side; ++c) {
      const uint32_t u = static_cast<uint32_t>(r * side + c);
      if (c + 1 < side && rng.unit() < s.mesh_keep) {
        pairs.push_back(u);
        pairs.push_back(u + 1);
      }
      if (r + 1 < side && rng.unit() < s.mesh_keep) {
        pairs.push_back(u);
        pairs.push_back(static_cast<uint32_t>(u + side));
      }
    }
  }
  const int64_t R = s.mesh_radius;
  for (uint64_t i = 0; i < s.mesh_shortcuts; ++i) {
    const uint64_t u = rng.bounded(n);
    const int64_t ur = static_cast<int64_t>(u / side), uc = static_cast<int64_t>(u % side);
    for (;;) {
      const int64_t dr = static_cast<int64_t>(rng.bounded(2 * R + 1)) - R;
      const int64_t dc = static_cast<int64_t>(rng.bounded(2 * R + 1)) - R;
      const int64_t man = (dr < 0 ? -dr : dr) + (dc < 0 ? -dc : dc);
      const int64_t tr = ur + dr, tc = uc + dc;
      if (man < 1 || man > R || tr < 0 || tc < 0 || tr >= static_cast<int64_t>(side) ||
          tc >= static_cast<int64_t>(side)) {
        continue;
      }
      pairs.push_back(static_cast<uint32_t>(u));
      pairs.push_back(static_cast<uint32_t>(tr * static_cast<int64_t>(side) + tc));
      break;
    }
  }
  return pairs;
}

bool is_symmetric(const HostCsr& g, unsigned threads) {
  std::atomic<bool> ok{true};
  parallel_for_threads(threads, [&](unsigned t) {
    const uint64_t b = g.n * t / threads, e = g.n * (t + 1) / threads;
    for (uint64_t u = b; u < e && ok.load(std::memory_order_relaxed); ++u) {
      for (uint64_t k = g.offsets[u]; k < g.offsets[u + 1]; ++k) {
        const uint32_t v = g.col[k];
        const uint32_t* lo = g.col.get() + g.offsets[v];
        const uint32_t* hi = g.col.get() + g.offsets[v + 1];
        if (!std::binary_search(lo, hi, static_cast<uint32_t>(u))) {
          ok = false;
          break;
        }
      }
    }
  });
  return ok;
}

}  // namespace

// csr_graph.cpp:11-55, restructured as a parallel bucketed counting sort:
//   1. per-thread histograms of arcs per fine source bucket (2^k vertices),
//      grouped into coarse buckets of balanced arc counts,
//   2. scatter (src<<32|dst) keys bucket-major,
//   3. per bucket: counting sort by row, per-row sort + unique, degrees,
//      dst compacted in place,
//   4. offsets by prefix sum, columns copied out bucket by bucket.
pbfs_status build_csr_impl(const uint32_t* pairs, uint64_t npairs, uint64_t n, bool symmetrize,
                           bool drop_self_loops, unsigned threads, HostCsr* out,
                           std::unique_ptr<uint32_t[]>* owned_pairs = nullptr) {
  if (n > 0x7fffffffULL) {
    return fail(PBFS_E_INPUT, "vertex count " + std::to_string(n) +
                                  " exceeds the supported maximum 2147483647");
  }
  threads = std::max(1u, std::min<unsigned>(threads, npairs / 4096 + 1));
  PhaseClock clk;
  // Range check (csr_graph.cpp:18-24): report the first offending pair.
  std::atomic<uint64_t> bad{UINT64_MAX};
  parallel_for_threads(threads, [&](unsigned t) {
    const uint64_t b = npairs * t / threads, e = npairs * (t + 1) / threads;
    for (uint64_t i = b; i < e; ++i) {
      if (pairs[2 * i] >= n || pairs[2 * i + 1] >= n) {
        uint64_t cur = bad.load();
        while (i < cur && !bad.compare_exchange_weak(cur, i)) {
        }
        break;
      }
    }
  });
  if (bad.load() != UINT64_MAX) {
    const uint64_t i = bad.load();
    return fail(PBFS_E_INPUT, "edge (" + std::to_string(pairs[2 * i]) + ", " +
                                  std::to_string(pairs[2 * i + 1]) +
                                  ") references a vertex >= " + std::to_string(n));
  }

  // Fine buckets of 2^shift vertices (<= 65536 of them) for the histogram;
  // runs of fine buckets are grouped into coarse buckets of about
  // total / (16 threads) arcs each, so RMAT's low-id hub region (several % of
  // all arcs in a few thousand vertices) is not one thread's straggler.
  int shift = 0;
  while ((n >> shift) > 65536) ++shift;
  const uint64_t nfine = n ? ((n - 1) >> shift) + 1 : 1;
  std::vector<uint64_t> fine(static_cast<size_t>(threads) * nfine, 0);
  parallel_for_threads(threads, [&](unsigned t) {
    uint64_t* h = fine.data() + t * nfine;
    const uint64_t b = npairs * t / threads, e = npairs * (t + 1) / threads;
    for (uint64_t i = b; i < e; ++i) {
      const uint32_t s = pairs[2 * i], d = pairs[2 * i + 1];
      if (s == d) {
        if (!drop_self_loops) ++h[s >> shift];
        continue;
      }
      ++h[s >> shift];
      if (symmetrize) ++h[d >> shift];
    }
  });
  uint64_t total = 0;
  std::vector<uint64_t> fine_sum(nfine, 0);
  for (unsigned t = 0; t < threads; ++t) {
    for (uint64_t f = 0; f < nfine; ++f) fine_sum[f] += fine[t * nfine + f];
  }
  for (uint64_t f = 0; f < nfine; ++f) total += fine_sum[f];
  const uint64_t target = std::max<uint64_t>(total / (16ull * threads) + 1, 1ull << 16);
  std::vector<uint32_t> f2c(nfine);
  std::vector<uint64_t> cv0;  // first vertex of each coarse bucket (+ n at the end)
  {
    uint64_t acc = 0;
    for (uint64_t f = 0; f < nfine; ++f) {
      if (f == 0 || acc >= target) {
        cv0.push_back(f << shift);
        acc = 0;
      }
      f2c[f] = static_cast<uint32_t>(cv0.size() - 1);
      acc += fine_sum[f];
    }
    cv0.push_back(n);
  }
  const uint64_t nbuckets = cv0.size() - 1;
  // bucket-major, thread-minor positions
  std::vector<uint64_t> hist(static_cast<size_t>(threads) * nbuckets, 0);
  for (unsigned t = 0; t < threads; ++t) {
    for (uint64_t f = 0; f < nfine; ++f) hist[t * nbuckets + f2c[f]] += fine[t * nfine + f];
  }
  fine.clear();
  fine.shrink_to_fit();
  std::vector<uint64_t> bucket_start(nbuckets + 1, 0);
  {
    uint64_t run = 0;
    for (uint64_t bk = 0; bk < nbuckets; ++bk) {
      bucket_start[bk] = run;
      for (unsigned t = 0; t < threads; ++t) {
        uint64_t c = hist[t * nbuckets + bk];
        hist[t * nbuckets + bk] = run;
        run += c;
      }
    }
    bucket_start[nbuckets] = run;
  }
  std::unique_ptr<uint64_t[], FreeDeleter> keys(
      static_cast<uint64_t*>(std::malloc((total ? total : 1) * sizeof(uint64_t))));
  if (!keys) return fail(PBFS_E_CAPACITY, "host allocation failed for " + std::to_string(total) + " arcs");
  parallel_for_threads(threads, [&](unsigned t) {
    uint64_t* pos = hist.data() + t * nbuckets;
    const uint64_t b = npairs * t / threads, e = npairs * (t + 1) / threads;
    for (uint64_t i = b; i < e; ++i) {
      const uint64_t s = pairs[2 * i], d = pairs[2 * i + 1];
      if (s == d) {
        if (!drop_self_loops) keys[pos[f2c[s >> shift]]++] = (s << 32) | d;
        continue;
      }
      keys[pos[f2c[s >> shift]]++] = (s << 32) | d;
      if (symmetrize) keys[pos[f2c[d >> shift]]++] = (d << 32) | s;
    }
  });
  hist.clear();
  hist.shrink_to_fit();
  clk.mark("build: scatter");
  // Peak host memory at RMAT-28 is pairs + keys; the pairs are dead from here.
  if (owned_pairs) owned_pairs->reset();

  out->n = n;
  out->offsets.reset(new (std::nothrow) uint64_t[n + 1]);
  if (!out->offsets) return fail(PBFS_E_CAPACITY, "host allocation failed (offsets)");
  std::vector<uint64_t> bucket_unique(nbuckets, 0);
  // Largest buckets first (dynamic assignment balances the tail).
  std::vector<uint64_t> order(nbuckets);
  for (uint64_t bk = 0; bk < nbuckets; ++bk) order[bk] = bk;
  std::sort(order.begin(), order.end(), [&](uint64_t x, uint64_t y) {
    return bucket_start[x + 1] - bucket_start[x] > bucket_start[y + 1] - bucket_start[y];
  });
  std::atomic<uint64_t> next_bucket{0};
  uint32_t* colbuf = reinterpret_cast<uint32_t*>(keys.get());
  // Per bucket: counting sort of its keys by source row (the degrees go
  // straight into offsets[v+1]), then each row's destinations sorted and
  // deduplicated (sort + unique per row = the reference's global pair sort
  // + unique, csr_graph.cpp:35-36) and compacted as u32 at the start of the
  // bucket's own key range, which has been fully read by then.
  parallel_for_threads(threads, [&](unsigned) {
    std::vector<uint32_t> tmp;
    std::vector<uint64_t> pos;
    for (;;) {
      const uint64_t oi = next_bucket.fetch_add(1);
      if (oi >= nbuckets) break;
      const uint64_t bk = order[oi];
      const uint64_t* kb = keys.get() + bucket_start[bk];
      const uint64_t K = bucket_start[bk + 1] - bucket_start[bk];
      const uint64_t v0 = cv0[bk], v1 = cv0[bk + 1];
      uint64_t* deg = out->offsets.get() + v0 + 1;
      const uint64_t rows = v1 - v0;
      std::fill(deg, deg + rows, 0);
      for (uint64_t i = 0; i < K; ++i) ++deg[(kb[i] >> 32) - v0];
      pos.resize(rows);
      uint64_t run = 0;
      for (uint64_t j = 0; j < rows; ++j) {
        pos[j] = run;
        run += deg[j];
      }
      tmp.resize(K);
      for (uint64_t i = 0; i < K; ++i) tmp[pos[(kb[i] >> 32) - v0]++] = static_cast<uint32_t>(kb[i]);
      uint32_t* cdst = colbuf + 2 * bucket_start[bk];
      uint64_t out_i = 0;
      for (uint64_t j = 0; j < rows; ++j) {
        uint32_t* rb = tmp.data() + pos[j] - deg[j];
        uint32_t* re = tmp.data() + pos[j];
        if (re - rb > 1) {
          std::sort(rb, re);
          re = std::unique(rb, re);
        }
        const uint64_t u = static_cast<uint64_t>(re - rb);
        std::memcpy(cdst + out_i, rb, u * sizeof(uint32_t));
        out_i += u;
        deg[j] = u;
      }
      bucket_unique[bk] = out_i;
    }
  });
  clk.mark("build: sort+unique");
  // Offsets: bucket bases, then rows (parallel per bucket).
  std::vector<uint64_t> bucket_base(nbuckets + 1, 0);
  for (uint64_t bk = 0; bk < nbuckets; ++bk) bucket_base[bk + 1] = bucket_base[bk] + bucket_unique[bk];
  const uint64_t m = bucket_base[nbuckets];
  out->m = m;
  out->offsets[0] = 0;
  next_bucket = 0;
  parallel_for_threads(threads, [&](unsigned) {
    for (;;) {
      const uint64_t bk = next_bucket.fetch_add(1);
      if (bk >= nbuckets) break;
      const uint64_t v0 = cv0[bk], v1 = cv0[bk + 1];
      uint64_t run = bucket_base[bk];
      for (uint64_t v = v0; v < v1; ++v) {
        run += out->offsets[v + 1];
        out->offsets[v + 1] = run;
      }
    }
  });
  // Columns: slide every bucket's compacted u32 run to its final position in
  // the same buffer (destinations never pass the sources: bucket_base[bk] <=
  // 2 * bucket_start[bk], and buckets move in ascending order), then shrink.
  for (uint64_t bk = 0; bk < nbuckets; ++bk) {
    std::memmove(colbuf + bucket_base[bk], colbuf + 2 * bucket_start[bk],
                 bucket_unique[bk] * sizeof(uint32_t));
  }
  void* shrunk = std::realloc(keys.get(), (m ? m : 1) * sizeof(uint32_t));
  if (!shrunk) return fail(PBFS_E_CAPACITY, "host reallocation failed (columns)");
  keys.release();
  out->col.reset(static_cast<uint32_t*>(shrunk));
  clk.mark("build: offsets+cols");
  out->symmetric = symmetrize ? true : is_symmetric(*out, threads);
  return PBFS_OK;
}

#if defined(__x86_64__) && defined(__GNUC__)
// One 64 B line of output per 16 codes: vpmovzxbd, the unreached code patched
// to all-ones under a mask, one vmovntdq. A line written by a single store
// never leaves a write-combining buffer half filled, which matters when the
// inbound DMA of the next transfer shares the memory system.
__attribute__((target("avx512f,avx512bw,avx512vl")))
static void widen_codes_avx512_impl(const uint8_t* src, uint32_t* dst, uint64_t b, uint64_t e,
                                    uint32_t bits) {
  uint64_t i = b;
  const __m512i ones = _mm512_set1_epi32(-1);
  if (bits == 4) {
    const __m128i nib = _mm_set1_epi8(0x0F);
    for (; i + 16 <= e; i += 16) {
      const __m128i x = _mm_loadl_epi64(reinterpret_cast<const __m128i*>(src + (i >> 1)));
      const __m128i lo = _mm_and_si128(x, nib), hi = _mm_and_si128(_mm_srli_epi16(x, 4), nib);
      const __m128i y = _mm_unpacklo_epi8(lo, hi);  // vertex order: even = low nibble
      const __mmask16 un = _mm_cmpeq_epi8_mask(y, nib);
      _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i),
                          _mm512_mask_mov_epi32(_mm512_cvtepu8_epi32(y), un, ones));
    }
    for (; i < e; ++i) {
      const uint32_t c = (src[i >> 1] >> ((i & 1) * 4)) & 0xFu;
      dst[i] = c == 0xF ? 0xFFFFFFFFu : c;
    }
  } else {
    const __m128i ff = _mm_set1_epi8(static_cast<char>(0xFF));
    for (; i + 16 <= e; i += 16) {
      const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
      const __mmask16 un = _mm_cmpeq_epi8_mask(x, ff);
      _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i),
                          _mm512_mask_mov_epi32(_mm512_cvtepu8_epi32(x), un, ones));
    }
    for (; i < e; ++i) dst[i] = src[i] == 0xFF ? 0xFFFFFFFFu : src[i];
  }
  _mm_sfence();
}
bool widen_codes_avx512(const uint8_t* src, uint32_t* dst, uint64_t b, uint64_t e, uint32_t bits) {
  static const bool have = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                           __builtin_cpu_supports("avx512vl") && !std::getenv("PBFS_NO_AVX512");
  if (!have || (bits != 4 && bits != 8) || (reinterpret_cast<uintptr_t>(dst + b) & 63) || (b & 1)) {
    return false;
  }
  widen_codes_avx512_impl(src, dst, b, e, bits);
  return true;
}
#else
bool widen_codes_avx512(const uint8_t*, uint32_t*, uint64_t, uint64_t, uint32_t) { return false; }
#endif

pbfs_status validate_csr_view(const pbfs_csr* c, unsigned threads) {
  if (c->vertex_count > 0x7fffffffULL) {
    return fail(PBFS_E_FORMAT, "vertex count " + std::to_string(c->vertex_count) +
                                   " exceeds the supported maximum");
  }
  if (c->offset_bytes != 4 && c->offset_bytes != 8) {
    return fail(PBFS_E_FORMAT, "offset width must be 4 or 8 bytes");
  }
  if (!c->row_offsets || (c->edge_count && !c->column_indices)) {
    return fail(PBFS_E_FORMAT, "null CSR array");
  }
  if (csr_offset(c, 0) != 0) return fail(PBFS_E_FORMAT, "offset array must start at 0");
  if (csr_offset(c, c->vertex_count) != c->edge_count) {
    return fail(PBFS_E_FORMAT, "offset array ends at " + std::to_string(csr_offset(c, c->vertex_count)) +
                                   " but edge count is " + std::to_string(c->edge_count));
  }
  const uint64_t n = c->vertex_count, m = c->edge_count;
  threads = std::max(1u, std::min<unsigned>(threads, n / 65536 + 1));
  std::vector<std::string> errs(threads);
  auto first_error = [&]() -> pbfs_status {
    for (auto& e : errs) {
      if (!e.empty()) return fail(PBFS_E_FORMAT, e);
    }
    return PBFS_OK;
  };
  // Pass 1: every offset is non-decreasing and <= m before any column is
  // read (a crafted offset must not send pass 2 outside column_indices).
  parallel_for_threads(threads, [&](unsigned t) {
    const uint64_t b = n * t / threads, e = n * (t + 1) / threads;
    for (uint64_t v = b; v < e; ++v) {
      const uint64_t lo = csr_offset(c, v), hi = csr_offset(c, v + 1);
      if (lo > hi) {
        errs[t] = "offset array decreases at vertex " + std::to_string(v);
        return;
      }
      if (hi > m) {
        errs[t] = "offset of vertex " + std::to_string(v + 1) + " exceeds the edge count";
        return;
      }
    }
  });
  pbfs_status st = first_error();
  if (st != PBFS_OK) return st;
  // Pass 2: neighbour ids in range and strictly increasing per row.
  parallel_for_threads(threads, [&](unsigned t) {
    const uint64_t b = n * t / threads, e = n * (t + 1) / threads;
    for (uint64_t v = b; v < e; ++v) {
      const uint64_t lo = csr_offset(c, v), hi = csr_offset(c, v + 1);
      for (uint64_t k = lo; k < hi; ++k) {
        const uint32_t x = c->column_indices[k];
        if (x >= n) {
          errs[t] = "vertex " + std::to_string(v) + " has a neighbor " + std::to_string(x) +
                    " outside the graph";
          return;
        }
        if (k > lo && c->column_indices[k - 1] >= x) {
          errs[t] = "adjacency list of vertex " + std::to_string(v) + " is not strictly increasing";
          return;
        }
      }
    }
  });
  return first_error();
}

}  // namespace pbfs

using namespace pbfs;

extern "C" {

pbfs_status pbfs_build_csr(const uint32_t* pairs, uint64_t npairs, uint64_t vertex_count,
                           uint32_t symmetrize, uint32_t drop_self_loops, uint32_t threads,
                           pbfs_host_csr** out) {
  if (!out || (npairs && !pairs)) return fail(PBFS_E_INPUT, "null argument");
  auto* h = new (std::nothrow) pbfs_host_csr;
  if (!h) return fail(PBFS_E_CAPACITY, "host allocation failed");
  pbfs_status st = build_csr_impl(pairs, npairs, vertex_count, symmetrize != 0,
                                  drop_self_loops != 0, resolve_threads(threads), &h->g);
  if (st != PBFS_OK) {
    delete h;
    return st;
  }
  *out = h;
  return PBFS_OK;
}

// pbfs_build_csr over generator-owned pairs, which the builder frees as soon
// as it has scattered them.
static pbfs_status build_to_handle(const uint32_t* pairs, uint64_t npairs, uint64_t n,
                                   uint32_t drop_self_loops, unsigned threads, pbfs_host_csr** out,
                                   std::unique_ptr<uint32_t[]>* owned) {
  auto* h = new (std::nothrow) pbfs_host_csr;
  if (!h) return fail(PBFS_E_CAPACITY, "host allocation failed");
  pbfs_status st = build_csr_impl(pairs, npairs, n, true, drop_self_loops != 0, threads, &h->g, owned);
  if (st != PBFS_OK) {
    delete h;
    return st;
  }
  *out = h;
  return PBFS_OK;
}

pbfs_status pbfs_generate(const pbfs_gen_spec* spec, pbfs_host_csr** out) {
  if (!spec || !out) return fail(PBFS_E_INPUT, "null argument");
  const unsigned threads = resolve_threads(spec->threads);
  std::vector<uint32_t> pairs;
  uint64_t n = 0;
  if (spec->kind == PBFS_GEN_MESH) {
    if (spec->mesh_side < 2 || static_cast<uint64_t>(spec->mesh_side) * spec->mesh_side > 0x7fffffffULL) {
      return fail(PBFS_E_CONFIG, "mesh side must be in [2, 46340]");
    }
    if (!(spec->mesh_keep >= 0.0 && spec->mesh_keep <= 1.0) || spec->mesh_radius < 1) {
      return fail(PBFS_E_CONFIG, "mesh keep probability must be in [0, 1] and radius >= 1");
    }
    n = static_cast<uint64_t>(spec->mesh_side) * spec->mesh_side;
    pairs = mesh_pairs(*spec);
  } else if (spec->kind == PBFS_GEN_UNIFORM || spec->kind == PBFS_GEN_KRONECKER) {
    // generator.cpp:42-50
    if (spec->scale < 1) return fail(PBFS_E_CONFIG, "generator scale must be at least 1");
    if (spec->edge_factor < 1) return fail(PBFS_E_CONFIG, "generator edge factor must be at least 1");
    if (spec->scale > 30) {
      return fail(PBFS_E_CAPACITY, "generator scale " + std::to_string(spec->scale) +
                                       " exceeds the 32-bit vertex id space");
    }
    n = uint64_t{1} << spec->scale;
    const uint64_t samples = n * spec->edge_factor;
    // Raw buffer: a value-initialised vector would zero-fill 8.6 GB at scale 26.
    std::unique_ptr<uint32_t[]> raw(new (std::nothrow) uint32_t[2 * samples]);
    if (!raw) {
      return fail(PBFS_E_CAPACITY, "host allocation failed for " + std::to_string(samples) + " samples");
    }
    PhaseClock clk;
    sample_pairs(spec->kind, spec->scale, spec->edge_factor, spec->seed, threads, raw.get());
    clk.mark("sample pairs");
    return build_to_handle(raw.get(), samples, n, spec->drop_self_loops, threads, out, &raw);
  } else {
    return fail(PBFS_E_CONFIG, "unknown generator kind");
  }
  return pbfs_build_csr(pairs.data(), pairs.size() / 2, n, 1, spec->drop_self_loops, threads, out);
}

pbfs_status pbfs_host_csr_view(const pbfs_host_csr* h, pbfs_csr* view) {
  if (!h || !view) return fail(PBFS_E_INPUT, "null argument");
  view->vertex_count = h->g.n;
  view->edge_count = h->g.m;
  view->row_offsets = h->g.offsets.get();
  view->column_indices = h->g.col.get();
  view->offset_bytes = 8;
  view->symmetric = h->g.symmetric ? 1 : 0;
  return PBFS_OK;
}

pbfs_status pbfs_host_csr_free(pbfs_host_csr* h) {
  delete h;
  return PBFS_OK;
}

pbfs_status pbfs_compute_stats(const pbfs_csr* c, double threshold, pbfs_stats* out) {
  if (!c || !out) return fail(PBFS_E_INPUT, "null argument");
  if (c->vertex_count == 0) return fail(PBFS_E_INPUT, "cannot compute stats for an empty graph");
  out->vertex_count = c->vertex_count;
  out->edge_count = c->edge_count;
  out->average_degree = static_cast<double>(c->edge_count) / static_cast<double>(c->vertex_count);
  uint64_t mx = 0;
  for (uint64_t v = 0; v < c->vertex_count; ++v) {
    mx = std::max(mx, csr_offset(c, v + 1) - csr_offset(c, v));
  }
  out->max_degree = mx;
  out->large_diameter = out->average_degree < threshold ? 1 : 0;
  out->reserved = 0;
  return PBFS_OK;
}

pbfs_status pbfs_pick_sources(const pbfs_csr* c, uint32_t count, uint64_t seed, uint32_t* out) {
  if (!c || (count && !out)) return fail(PBFS_E_INPUT, "null argument");
  if (count == 0) return fail(PBFS_E_CONFIG, "source count must be positive");
  bool any = false;
  for (uint64_t v = 0; v < c->vertex_count && !any; ++v) any = csr_offset(c, v + 1) > csr_offset(c, v);
  if (!any) return fail(PBFS_E_CONFIG, "graph has no vertex with positive degree; pass --source-list");
  Stream rng(seed);
  uint32_t got = 0;
  while (got < count) {
    const uint32_t v = static_cast<uint32_t>(rng.next() % c->vertex_count);
    if (csr_offset(c, v + 1) > csr_offset(c, v)) out[got++] = v;
  }
  return PBFS_OK;
}

// graph_io.cpp:70-85 — little-endian CSR1 (this library only targets
// little-endian hosts, so arrays are written directly).
pbfs_status pbfs_save_csr1(const pbfs_csr* c, const char* path) {
  if (!c || !path) return fail(PBFS_E_INPUT, "null argument");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(PBFS_E_INPUT, std::string("cannot open file for writing: ") + path);
  bool ok = std::fwrite("CSR1", 1, 4, f) == 4;
  ok = ok && std::fwrite(&c->vertex_count, 8, 1, f) == 1;
  ok = ok && std::fwrite(&c->edge_count, 8, 1, f) == 1;
  if (c->offset_bytes == 8) {
    ok = ok && std::fwrite(c->row_offsets, 8, c->vertex_count + 1, f) == c->vertex_count + 1;
  } else {
    for (uint64_t i = 0; ok && i <= c->vertex_count; ++i) {
      const uint64_t o = csr_offset(c, i);
      ok = std::fwrite(&o, 8, 1, f) == 1;
    }
  }
  ok = ok && std::fwrite(c->column_indices, 4, c->edge_count, f) == c->edge_count;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(PBFS_E_INPUT, std::string("write failure on file: ") + path);
  return PBFS_OK;
}

// graph_io.cpp:87-119
pbfs_status pbfs_load_csr1(const char* path, pbfs_host_csr** out) {
  if (!path || !out) return fail(PBFS_E_INPUT, "null argument");
  FILE* f = std::fopen(path, "rb");
  const std::string name = path;
  if (!f) return fail(PBFS_E_INPUT, "cannot open file for reading: " + name);
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CSR1", 4) != 0) {
    std::fclose(f);
    return fail(PBFS_E_FORMAT, name + ": missing CSR1 header");
  }
  uint64_t n = 0, m = 0;
  if (std::fread(&n, 8, 1, f) != 1 || std::fread(&m, 8, 1, f) != 1) {
    std::fclose(f);
    return fail(PBFS_E_FORMAT, name + ": truncated header");
  }
  if (n > 0x7fffffffULL) {
    std::fclose(f);
    return fail(PBFS_E_FORMAT, name + ": vertex count exceeds the supported maximum");
  }
  // The header's counts must describe exactly the bytes that follow it
  // (graph_io.cpp:100-116 rejects short and trailing data): checked before
  // any allocation, so a crafted m cannot wrap m * 4 or over-allocate.
  const long long here = ftello(f);
  long long end = -1;
  if (here >= 0 && fseeko(f, 0, SEEK_END) == 0) end = ftello(f);
  if (end < 0 || fseeko(f, here, SEEK_SET) != 0) {
    std::fclose(f);
    return fail(PBFS_E_FORMAT, name + ": cannot determine the file size");
  }
  const uint64_t body = static_cast<uint64_t>(end - here);
  const uint64_t off_bytes = (n + 1) * 8;
  if (body < off_bytes) {
    std::fclose(f);
    return fail(PBFS_E_FORMAT, name + ": truncated graph data");
  }
  if (m > (body - off_bytes) / 4) {
    std::fclose(f);
    return fail(PBFS_E_FORMAT, name + ": truncated graph data");
  }
  auto* h = new (std::nothrow) pbfs_host_csr;
  if (!h) {
    std::fclose(f);
    return fail(PBFS_E_CAPACITY, name + ": host allocation failed");
  }
  h->g.n = n;
  h->g.m = m;
  h->g.offsets.reset(new (std::nothrow) uint64_t[n + 1]);
  h->g.col.reset(static_cast<uint32_t*>(std::malloc((m ? m : 1) * sizeof(uint32_t))));
  if (!h->g.offsets || !h->g.col) {
    std::fclose(f);
    delete h;
    return fail(PBFS_E_CAPACITY, name + ": host allocation failed");
  }
  bool ok = std::fread(h->g.offsets.get(), 8, n + 1, f) == n + 1;
  ok = ok && std::fread(h->g.col.get(), 4, m, f) == m;
  if (!ok) {
    std::fclose(f);
    delete h;
    return fail(PBFS_E_FORMAT, name + ": truncated graph data");
  }
  const bool trailing = std::fgetc(f) != EOF;
  std::fclose(f);
  if (trailing) {
    delete h;
    return fail(PBFS_E_FORMAT, name + ": trailing bytes after graph data");
  }
  pbfs_csr view;
  pbfs_host_csr_view(h, &view);
  pbfs_status st = validate_csr_view(&view, resolve_threads(0));
  if (st != PBFS_OK) {
    delete h;
    return st;
  }
  h->g.symmetric = is_symmetric(h->g, resolve_threads(0));
  *out = h;
  return PBFS_OK;
}

}  // extern "C"

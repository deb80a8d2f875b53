// Host-side graph library: seeded generators, the parallel CSR builder, the
// classifier, source selection and the CSR1 format. Same public semantics as
// the reference's proj/core graph layer (generator.cpp, csr_graph.cpp,
// graph_stats.cpp, graph_io.cpp, tools/bfsbench.cpp:pick_sources), rebuilt for
// multi-GB graphs: no O(m log m) global sort, no value-initialised buffers,
// the mt19937_64 stream generated in twist-sized blocks on one thread while
// other threads turn draws into edge pairs.
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "pbfs_internal.h"

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

// ---------------------------------------------------------------------------
// mt19937_64 ([rand.predef]) producing whole 312-word twists at a time. The
// twist is split into its two dependency-free halves so the compiler
// vectorises it; outputs are bit-identical to std::mt19937_64.
class Mt64 {
 public:
  static constexpr int N = 312, M = 156;
  explicit Mt64(uint64_t seed) {
    s_[0] = seed;
    for (int i = 1; i < N; ++i) s_[i] = 6364136223846793005ULL * (s_[i - 1] ^ (s_[i - 1] >> 62)) + i;
  }
  // Writes the next N outputs.
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
    for (int i = 0; i < N; ++i) {
      uint64_t y = mt[i];
      y ^= (y >> 29) & 0x5555555555555555ULL;
      y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
      y ^= (y << 37) & 0xFFF7EEE000000000ULL;
      y ^= y >> 43;
      out[i] = y;
    }
  }

 private:
  uint64_t s_[N];
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

// generator.cpp:51-89 — the sample loop, pipelined: the calling thread fills
// draw buffer k while `threads-1` workers convert buffer k-1 into pairs.
void sample_pairs(uint32_t kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                  unsigned threads, uint32_t* pairs) {
  const uint64_t n = uint64_t{1} << scale;
  const uint64_t samples = n * edge_factor;
  const uint32_t per = kind == PBFS_GEN_KRONECKER ? scale : 2;
  // Batch = a whole number of samples and of twists (lcm via 312 * per).
  const uint64_t batch_samples =
      std::max<uint64_t>(Mt64::N, (uint64_t{1} << 20) / per / Mt64::N * Mt64::N);
  const uint64_t batch_draws = batch_samples * per;  // multiple of 312
  std::vector<uint64_t> buf[2] = {std::vector<uint64_t>(batch_draws),
                                  std::vector<uint64_t>(batch_draws)};
  Mt64 mt(seed);
  KronThresholds thr;
  const unsigned workers = threads > 1 ? threads - 1 : 1;
  auto convert = [&](const uint64_t* draws, uint64_t first, uint64_t count) {
    // The workers outlive this call: capture the batch by value.
    auto work = [=, &thr](unsigned t) {
      const uint64_t b = first + count * t / workers;
      const uint64_t e = first + count * (t + 1) / workers;
      const uint64_t* d = draws + (b - first) * per;
      if (kind == PBFS_GEN_KRONECKER) {
        kron_convert(d, e - b, scale, thr, pairs + 2 * b);
      } else {
        uniform_convert(d, e - b, n, pairs + 2 * b);
      }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < workers; ++t) pool.emplace_back(work, t);
    return pool;
  };
  std::vector<std::thread> pending;
  uint64_t done = 0;
  int cur = 0;
  while (done < samples) {
    const uint64_t count = std::min(batch_samples, samples - done);
    const uint64_t draws = count * per;
    uint64_t* out = buf[cur].data();
    // Whole twists; the stream is consumed exactly `draws` deep because the
    // last batch is the only partial one and nothing is drawn after it.
    uint64_t produced = 0;
    uint64_t tmp[Mt64::N];
    while (produced + Mt64::N <= draws) {
      mt.block(out + produced);
      produced += Mt64::N;
    }
    if (produced < draws) {
      mt.block(tmp);
      std::memcpy(out + produced, tmp, (draws - produced) * sizeof(uint64_t));
    }
    for (auto& th : pending) th.join();
    pending = convert(out, done, count);
    done += count;
    cur ^= 1;
  }
  for (auto& th : pending) th.join();
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
//   1. per-thread histograms of arcs per source bucket (2^k vertices each),
//   2. scatter (src<<32|dst) keys bucket-major,
//   3. per bucket: sort + unique + per-row degree, dst compacted in place,
//   4. offsets by prefix sum, columns copied out bucket by bucket.
pbfs_status build_csr_impl(const uint32_t* pairs, uint64_t npairs, uint64_t n, bool symmetrize,
                           bool drop_self_loops, unsigned threads, HostCsr* out,
                           std::unique_ptr<uint32_t[]>* owned_pairs = nullptr) {
  if (n > 0x7fffffffULL) {
    return fail(PBFS_E_INPUT, "vertex count " + std::to_string(n) +
                                  " exceeds the supported maximum 2147483647");
  }
  threads = std::max(1u, std::min<unsigned>(threads, npairs / 4096 + 1));
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

  int shift = 0;
  while ((n >> shift) > 4096) ++shift;  // <= 4096 buckets
  const uint64_t nbuckets = n ? ((n - 1) >> shift) + 1 : 1;
  std::vector<uint64_t> hist(static_cast<size_t>(threads) * nbuckets, 0);
  parallel_for_threads(threads, [&](unsigned t) {
    uint64_t* h = hist.data() + t * nbuckets;
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
  // bucket-major, thread-minor positions
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
  const uint64_t total = bucket_start[nbuckets];
  std::unique_ptr<uint64_t[], FreeDeleter> keys(
      static_cast<uint64_t*>(std::malloc((total ? total : 1) * sizeof(uint64_t))));
  if (!keys) return fail(PBFS_E_CAPACITY, "host allocation failed for " + std::to_string(total) + " arcs");
  parallel_for_threads(threads, [&](unsigned t) {
    uint64_t* pos = hist.data() + t * nbuckets;
    const uint64_t b = npairs * t / threads, e = npairs * (t + 1) / threads;
    for (uint64_t i = b; i < e; ++i) {
      const uint64_t s = pairs[2 * i], d = pairs[2 * i + 1];
      if (s == d) {
        if (!drop_self_loops) keys[pos[s >> shift]++] = (s << 32) | d;
        continue;
      }
      keys[pos[s >> shift]++] = (s << 32) | d;
      if (symmetrize) keys[pos[d >> shift]++] = (d << 32) | s;
    }
  });
  hist.clear();
  hist.shrink_to_fit();
  // Peak host memory at RMAT-28 is pairs + keys; the pairs are dead from here.
  if (owned_pairs) owned_pairs->reset();

  out->n = n;
  out->offsets.reset(new (std::nothrow) uint64_t[n + 1]);
  if (!out->offsets) return fail(PBFS_E_CAPACITY, "host allocation failed (offsets)");
  std::vector<uint64_t> bucket_unique(nbuckets, 0);
  std::atomic<uint64_t> next_bucket{0};
  uint32_t* colbuf = reinterpret_cast<uint32_t*>(keys.get());
  parallel_for_threads(threads, [&](unsigned) {
    for (;;) {
      const uint64_t bk = next_bucket.fetch_add(1);
      if (bk >= nbuckets) break;
      uint64_t* kb = keys.get() + bucket_start[bk];
      uint64_t* ke = keys.get() + bucket_start[bk + 1];
      std::sort(kb, ke);
      ke = std::unique(kb, ke);
      const uint64_t cnt = static_cast<uint64_t>(ke - kb);
      bucket_unique[bk] = cnt;
      const uint64_t v0 = bk << shift, v1 = std::min<uint64_t>(n, (bk + 1) << shift);
      for (uint64_t v = v0; v < v1; ++v) out->offsets[v + 1] = 0;
      // Degrees into offsets[v+1]; destinations compacted in place as u32
      // (write index 4i never passes read index 8i).
      uint32_t* cdst = colbuf + 2 * bucket_start[bk];
      for (uint64_t i = 0; i < cnt; ++i) {
        const uint64_t k = kb[i];
        ++out->offsets[(k >> 32) + 1];
        cdst[i] = static_cast<uint32_t>(k);
      }
    }
  });
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
      const uint64_t v0 = bk << shift, v1 = std::min<uint64_t>(n, (bk + 1) << shift);
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
  out->symmetric = symmetrize ? true : is_symmetric(*out, threads);
  return PBFS_OK;
}

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
    sample_pairs(spec->kind, spec->scale, spec->edge_factor, spec->seed, threads, raw.get());
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

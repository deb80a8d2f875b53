/* TEST INFRASTRUCTURE ONLY — see pbfs_oracle.h. Plain C, single-threaded,
 * deliberately naive; shares no code with the product library. */
#include "pbfs_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 ([rand.predef]: w=64 n=312 m=156 r=31) ------------------ */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (uint32_t i = 1; i < MT_N; ++i) {
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + i;
  }
  s->idx = MT_N;
}

/* The twist of all 312 words, written as its three index ranges so no
 * modulo sits in the loop (same recurrence as the textbook form
 * x[i] = x[(i+m) % n] ^ A(upper(x[i]) | lower(x[(i+1) % n]))). */
static void mt64_twist(orc_mt64* s) {
  uint64_t* x = s->mt;
  uint32_t i = 0;
  for (; i < MT_N - MT_M; ++i) {
    const uint64_t y = (x[i] & MT_UPPER) | (x[i + 1] & MT_LOWER);
    x[i] = x[i + MT_M] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
  }
  for (; i < MT_N - 1; ++i) {
    const uint64_t y = (x[i] & MT_UPPER) | (x[i + 1] & MT_LOWER);
    x[i] = x[i + MT_M - MT_N] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
  }
  {
    const uint64_t y = (x[MT_N - 1] & MT_UPPER) | (x[0] & MT_LOWER);
    x[MT_N - 1] = x[MT_M - 1] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
  }
  s->idx = 0;
}

static inline uint64_t mt64_next(orc_mt64* s) {
  if (s->idx >= MT_N) mt64_twist(s);
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint64_t orc_mt64_next(orc_mt64* s) { return mt64_next(s); }

/* Sampler::bounded / Sampler::unit — generator.cpp:22-29 */
static inline uint64_t bounded(orc_mt64* s, uint64_t n) {
  return (uint64_t)(((unsigned __int128)mt64_next(s) * n) >> 64);
}
static inline double unit(orc_mt64* s) {
  return (double)(mt64_next(s) >> 11) * 0x1.0p-53;
}

/* generator.cpp:41-89 */
int orc_generate_pairs(int kind, uint32_t scale, uint32_t edge_factor,
                       uint64_t seed, uint32_t* pairs) {
  if (scale < 1 || edge_factor < 1 || scale > 30) return -1;
  const uint64_t n = (uint64_t)1 << scale;
  const uint64_t samples = n * edge_factor;
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  for (uint64_t i = 0; i < samples; ++i) {
    uint64_t row = 0, col = 0;
    if (kind == 0) {
      row = bounded(&s, n);
      col = bounded(&s, n);
    } else {
      /* generator.cpp:75-84's quadrant chain r < a | < a+b | < a+b+c | else,
       * as comparisons (same double thresholds, no branches):
       * row bit set for quadrants c and d, column bit for b and d. */
      const double ta = 0.57, tab = 0.57 + 0.19, tabc = 0.57 + 0.19 + 0.19;
      for (uint32_t l = 0; l < scale; ++l) {
        const double r = unit(&s);
        const uint64_t rb = r >= tab;
        const uint64_t cb = ((uint64_t)(r >= ta) & (uint64_t)(r < tab)) | (uint64_t)(r >= tabc);
        row = (row << 1) | rb;
        col = (col << 1) | cb;
      }
    }
    pairs[2 * i] = (uint32_t)row;
    pairs[2 * i + 1] = (uint32_t)col;
  }
  return 0;
}

/* Ascending sort of a row: insertion sort for short rows, else an LSD radix
 * sort (four 8-bit digits) through `tmp` (len entries). */
static void sort_u32(uint32_t* a, uint64_t len, uint32_t* tmp) {
  if (len <= 32) {
    for (uint64_t i = 1; i < len; ++i) {
      const uint32_t x = a[i];
      uint64_t j = i;
      while (j > 0 && a[j - 1] > x) {
        a[j] = a[j - 1];
        --j;
      }
      a[j] = x;
    }
    return;
  }
  uint64_t count[256];
  uint32_t* src = a;
  uint32_t* dst = tmp;
  for (int shift = 0; shift < 32; shift += 8) {
    memset(count, 0, sizeof(count));
    for (uint64_t i = 0; i < len; ++i) count[(src[i] >> shift) & 0xFF]++;
    uint64_t sum = 0;
    for (int d = 0; d < 256; ++d) {
      const uint64_t c = count[d];
      count[d] = sum;
      sum += c;
    }
    for (uint64_t i = 0; i < len; ++i) dst[count[(src[i] >> shift) & 0xFF]++] = src[i];
    uint32_t* t = src;
    src = dst;
    dst = t;
  }
  /* four passes: the result is back in a */
}

/* csr_graph.cpp:11-55: the reference sorts all (src, dst) pairs and drops
 * duplicates; the same set, per source row: count arcs per row, place each
 * arc's dst in its row, then sort + unique every row. */
uint64_t orc_build_csr(const uint32_t* pairs, uint64_t npairs, uint64_t n,
                       int symmetrize, int drop_self_loops, uint64_t* offsets,
                       uint32_t* col) {
  for (uint64_t i = 0; i < 2 * npairs; ++i) {
    if (pairs[i] >= n) return UINT64_MAX;
  }
  memset(offsets, 0, sizeof(uint64_t) * (n + 1));
  for (uint64_t i = 0; i < npairs; ++i) {
    const uint32_t a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b && drop_self_loops) continue;
    offsets[a + 1]++;
    if (symmetrize && a != b) offsets[b + 1]++;
  }
  for (uint64_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
  uint64_t* pos = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  memcpy(pos, offsets, sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < npairs; ++i) {
    const uint32_t a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b && drop_self_loops) continue;
    col[pos[a]++] = b;
    if (symmetrize && a != b) col[pos[b]++] = a;
  }
  free(pos);
  /* Rows are compacted forward in place: row v's unique run is written at
   * m <= offsets[v], its own start. */
  uint64_t maxdeg = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (offsets[v + 1] - offsets[v] > maxdeg) maxdeg = offsets[v + 1] - offsets[v];
  }
  uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (maxdeg ? maxdeg : 1));
  uint64_t m = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t b = offsets[v], e = offsets[v + 1];
    sort_u32(col + b, e - b, tmp);
    offsets[v] = m;
    for (uint64_t k = b; k < e; ++k) {
      if (k == b || col[k] != col[k - 1]) col[m++] = col[k];
    }
  }
  offsets[n] = m;
  free(tmp);
  return m;
}

/* kernels.cpp:19-41 */
int orc_bfs_serial(uint64_t n, const uint64_t* offsets, const uint32_t* col,
                   uint32_t source, uint32_t* dist) {
  if (source >= n) return -1;
  uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint64_t v = 0; v < n; ++v) dist[v] = 0xFFFFFFFFu;
  uint64_t head = 0, tail = 0;
  dist[source] = 0;
  queue[tail++] = source;
  while (head < tail) {
    const uint32_t u = queue[head++];
    const uint32_t nd = dist[u] + 1;
    for (uint64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
      const uint32_t v = col[e];
      if (dist[v] == 0xFFFFFFFFu) {
        dist[v] = nd;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  return 0;
}

/* tests/support/graphs.hpp:138-156 */
int orc_relaxation(uint64_t n, const uint64_t* offsets, const uint32_t* col,
                   uint32_t source, uint32_t* dist) {
  if (source >= n) return -1;
  for (uint64_t v = 0; v < n; ++v) dist[v] = 0xFFFFFFFFu;
  dist[source] = 0;
  int changed = 1;
  while (changed) {
    changed = 0;
    for (uint64_t u = 0; u < n; ++u) {
      if (dist[u] == 0xFFFFFFFFu) continue;
      for (uint64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
        const uint32_t v = col[e];
        if (dist[u] + 1 < dist[v]) {
          dist[v] = dist[u] + 1;
          changed = 1;
        }
      }
    }
  }
  return 0;
}

/* tools/bfsbench.cpp:221-234 */
int orc_pick_sources(uint64_t n, const uint64_t* offsets, uint32_t count,
                     uint64_t seed, uint32_t* out) {
  int any = 0;
  for (uint64_t v = 0; v < n && !any; ++v) any = offsets[v + 1] > offsets[v];
  if (!any) return -1;
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  uint32_t got = 0;
  while (got < count) {
    const uint32_t v = (uint32_t)(mt64_next(&s) % n);
    if (offsets[v + 1] > offsets[v]) out[got++] = v;
  }
  return 0;
}

/* tests/support/graphs.hpp:177-215, layered from exact distances. */
uint32_t orc_simulate_phases(uint64_t n, uint64_t m, const uint64_t* offsets,
                             const uint32_t* dist, double threshold,
                             int beamer, double alpha, double beta,
                             uint8_t* phases, uint32_t cap) {
  uint32_t deepest = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (dist[v] != 0xFFFFFFFFu && dist[v] > deepest) deepest = dist[v];
  }
  const uint32_t layers = deepest + 1;
  uint64_t* size = (uint64_t*)calloc(layers, sizeof(uint64_t));
  uint64_t* degree = (uint64_t*)calloc(layers, sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) {
    if (dist[v] == 0xFFFFFFFFu) continue;
    size[dist[v]]++;
    degree[dist[v]] += offsets[v + 1] - offsets[v];
  }
  const double dn = (double)n;
  int top_down = 1;
  uint64_t unvisited = m;
  uint64_t prev = 0;
  uint32_t out = 0;
  for (uint32_t d = 0; d < layers; ++d) {
    unvisited -= degree[d];
    if (beamer) {
      if (top_down) {
        if ((double)degree[d] > (double)unvisited / alpha) top_down = 0;
      } else if ((double)size[d] < dn / beta && size[d] < prev) {
        top_down = 1;
      }
    } else {
      top_down = (double)size[d] < threshold * dn;
    }
    if (out < cap) phases[out] = top_down ? 0 : 1;
    ++out;
    prev = size[d];
  }
  free(size);
  free(degree);
  return out;
}

/* graph_stats.cpp:9-25 */
void orc_stats(uint64_t n, uint64_t m, const uint64_t* offsets,
               double threshold, double* avg_degree, uint64_t* max_degree,
               int* large_diameter) {
  *avg_degree = (double)m / (double)n;
  uint64_t mx = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t d = offsets[v + 1] - offsets[v];
    if (d > mx) mx = d;
  }
  *max_degree = mx;
  *large_diameter = *avg_degree < threshold;
}

uint64_t orc_mesh_pairs(uint32_t side, double keep, uint64_t shortcuts,
                        uint32_t radius, uint64_t seed, uint32_t* pairs) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  const uint64_t n = (uint64_t)side * side;
  uint64_t k = 0;
  for (uint32_t r = 0; r < side; ++r) {
    for (uint32_t c = 0; c < side; ++c) {
      const uint32_t u = r * side + c;
      if (c + 1 < side && unit(&s) < keep) {
        pairs[2 * k] = u;
        pairs[2 * k + 1] = u + 1;
        ++k;
      }
      if (r + 1 < side && unit(&s) < keep) {
        pairs[2 * k] = u;
        pairs[2 * k + 1] = u + side;
        ++k;
      }
    }
  }
  const int64_t R = radius;
  for (uint64_t i = 0; i < shortcuts; ++i) {
    const uint64_t u = bounded(&s, n);
    const int64_t ur = (int64_t)(u / side), uc = (int64_t)(u % side);
    for (;;) {
      const int64_t dr = (int64_t)bounded(&s, 2 * R + 1) - R;
      const int64_t dc = (int64_t)bounded(&s, 2 * R + 1) - R;
      const int64_t man = (dr < 0 ? -dr : dr) + (dc < 0 ? -dc : dc);
      const int64_t tr = ur + dr, tc = uc + dc;
      if (man < 1 || man > R || tr < 0 || tc < 0 || tr >= side || tc >= side) continue;
      pairs[2 * k] = (uint32_t)u;
      pairs[2 * k + 1] = (uint32_t)(tr * side + tc);
      ++k;
      break;
    }
  }
  return k;
}

void orc_component(uint64_t n, const uint64_t* offsets, const uint32_t* dist,
                   uint64_t* n_reached, uint64_t* arcs_reached) {
  uint64_t nr = 0, ar = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (dist[v] == 0xFFFFFFFFu) continue;
    ++nr;
    ar += offsets[v + 1] - offsets[v];
  }
  *n_reached = nr;
  *arcs_reached = ar;
}

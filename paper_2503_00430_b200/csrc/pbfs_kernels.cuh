// Device side of the B200-native level-synchronous BFS (arXiv 2503.00430).
//
// ONE persistent cooperative kernel runs a whole traversal: every CTA walks
// the same level loop and takes every control decision redundantly from
// counters it reads right after a grid barrier, so the host is not involved
// between levels (the reference needs a std::barrier round and a serial
// single-worker section per level, kernels.cpp:165-173,384-464). Per level:
//
//   top-down  (kernels.cpp:262-338): warps grab 32-entry slices of the frontier
//     queue; vertices of degree <= kHeavyDeg are expanded warp-cooperatively
//     (shuffle scan of degrees + per-lane owner search, so a warp reads one
//     coalesced 128 B span of `col` per step); hubs are split into
//     kChunk-edge items expanded by the whole grid after a barrier. Claims:
//       kClaimCas    atomicCAS on dist            (BFS-Conventional)
//       kClaimPlain  plain same-value dist stores (BFS-NonAtomic, duplicates)
//       kClaimBitmap test-then-atomicOr on the bit-packed visited set, then a
//                    plain dist store            (BFS-Hybrid / VisitedBitmap)
//     Discoveries go to a per-warp shared-memory buffer flushed with one
//     atomicAdd per 256 entries (the GPU form of LocalFrontier +
//     reserve_and_flush, frontier.hpp:58-98).
//   bottom-up (kernels.cpp:340-382): warps own 16-word (512-vertex) groups of
//     the visited bitmap, compact the unvisited ids into shared memory and
//     scan each one's adjacency until the first frontier-bitmap hit (early
//     exit). Owner-exclusive: next/visited words are written with plain
//     stores, no atomics.
//   control (kernels.cpp:384-464,487-513): distinct size read from the level
//     counter; `top_down = (double)distinct < thr * (double)n` evaluated in
//     IEEE double exactly like the reference; representation conversions
//     (queue <-> bitmap) only when the direction flips.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

#include "pbfs.h"

namespace pbfs {
namespace dev {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kHeavyDeg = 256;  // degree above which a vertex is split
constexpr uint32_t kChunk = 1024;    // edges per heavy work item
constexpr int kPushBuf = 256;        // per-warp discovery buffer (entries)
constexpr int kGroupWords = 16;      // bottom-up: bitmap words per warp group
constexpr int kGroupVerts = kGroupWords * 32;
constexpr uint32_t kUnreached = 0xFFFFFFFFu;

enum Claim : int { kClaimCas = 0, kClaimPlain = 1, kClaimBitmap = 2 };
enum Policy : int { kPolicyTopDown = 0, kPolicyFraction = 1, kPolicyBeamer = 2 };

// Per-level counters, ring of 4 indexed by depth & 3 (a slot is re-zeroed two
// levels after its readers are provably past it).
struct alignas(128) LevelCnt {
  unsigned long long produced;  // distinct discoveries (next frontier size)
  unsigned long long raw;       // queue pushes (next queue length)
  unsigned long long edges;     // adjacency entries examined
  unsigned long long degree;    // degree sum of discoveries (Beamer m_f)
  unsigned long long violations;
  unsigned int td_cursor;       // frontier slice grab
  unsigned int heavy_count;     // heavy items appended
  unsigned int heavy_cursor;    // heavy items grabbed
  unsigned int conv_count;      // bitmap -> queue compaction length
  unsigned int mark_cursor;
  unsigned int pad[5];
};

struct alignas(128) Ctl {
  unsigned long long bar_count;  // monotone arrivals (grid barrier)
  unsigned long long pad0[15];
  unsigned int exit_count;
  unsigned int pad1[31];
  LevelCnt cnt[4];
  unsigned int overflow;  // PBFS_E_CAPACITY raised on device
  unsigned int levels;
  unsigned int bu_levels;
  unsigned int pad2;
  unsigned long long reached;
  unsigned long long violations;
  unsigned long long edges;
};

struct HeavyItem {
  unsigned long long beg;
  unsigned long long end;
};

template <typename OffT>
struct Params {
  const OffT* __restrict__ rowptr;
  const uint32_t* __restrict__ col;
  uint32_t* dist;
  uint32_t* visited;
  uint32_t* bm[2];
  const uint32_t* init_mask;
  uint32_t* queue[2];
  HeavyItem* heavy;
  Ctl* ctl;
  pbfs_level* records;
  unsigned long long qcap;
  unsigned long long heavy_cap;
  unsigned long long n;
  unsigned long long m;
  unsigned long long max_degree;
  uint32_t words;  // bitmap words, multiple of kGroupWords
  uint32_t rec_cap;
  uint32_t source;
  int policy;
  int validate;
  double threshold;
  double alpha;
  double beta;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free grid barrier on a monotone 64-bit arrival counter: barrier k
// completes when the counter reaches k * gridDim.x. Thread 0 of each CTA
// publishes the CTA's writes (fence), arrives, spins with acquire loads, and
// fences again so the whole CTA observes every other CTA's writes.
struct GridBarrier {
  Ctl* ctl;
  unsigned long long target;
  __device__ __forceinline__ void sync() {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&ctl->bar_count, 1ull);
      while (ld_acquire(&ctl->bar_count) < target) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
  }
};

// Per-warp discovery buffer in shared memory (LocalFrontier analogue).
struct WarpPush {
  uint32_t* buf;  // kPushBuf entries in smem
  int count;      // warp-uniform
  __device__ __forceinline__ void flush(uint32_t* out, unsigned long long* counter,
                                        unsigned long long cap, unsigned int* overflow) {
    __syncwarp();
    if (count) {
      unsigned long long base = 0;
      if (lane_id() == 0) base = atomicAdd(counter, (unsigned long long)count);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + count <= cap) {
        for (int i = lane_id(); i < count; i += 32) out[base + i] = buf[i];
      } else if (lane_id() == 0) {
        atomicExch(overflow, 1u);
      }
    }
    count = 0;
    __syncwarp();
  }
  __device__ __forceinline__ void push(bool want, uint32_t v, uint32_t* out,
                                       unsigned long long* counter, unsigned long long cap,
                                       unsigned int* overflow) {
    const unsigned mask = __ballot_sync(0xffffffffu, want);
    if (!mask) return;
    const int k = __popc(mask);
    if (count + k > kPushBuf) flush(out, counter, cap, overflow);
    if (want) buf[count + __popc(mask & lanemask_lt())] = v;
    count += k;
  }
};

// Edge (u -> v) at depth d: the claim discipline of the variant. Returns
// whether v is appended to the next queue; *distinct says whether this
// append is the vertex's first discovery.
template <int C, typename OffT>
__device__ __forceinline__ bool visit(const Params<OffT>& p, uint32_t v, uint32_t nd,
                                      bool& distinct, unsigned long long& viol) {
  const uint32_t w = v >> 5, bit = 1u << (v & 31);
  if constexpr (C == kClaimCas) {
    // kernels.cpp:282-290: claim by compare-exchange from kUnreached.
    if (ld_relaxed(&p.dist[v]) == kUnreached &&
        atomicCAS(&p.dist[v], kUnreached, nd) == kUnreached) {
      distinct = true;
      return true;
    }
    return false;
  } else if constexpr (C == kClaimPlain) {
    // kernels.cpp:291-301: load, compare, plain store; racing writers all
    // store the same nd, so duplicates are possible but values are not.
    const uint32_t cur = ld_relaxed(&p.dist[v]);
    if (nd < cur) {
      if (p.validate && cur != kUnreached) ++viol;  // kernels.cpp:294
      p.dist[v] = nd;
      // The visited bitmap is only a distinct-count ledger here.
      const uint32_t old = atomicOr(&p.visited[w], bit);
      distinct = !(old & bit);
      return true;
    }
    return false;
  } else {
    // kernels.cpp:302-320: test the visited bit, claim it, store dist inline.
    if (!(ld_relaxed(&p.visited[w]) & bit)) {
      const uint32_t old = atomicOr(&p.visited[w], bit);
      if (!(old & bit)) {
        p.dist[v] = nd;
        distinct = true;
        return true;
      }
    }
    return false;
  }
}

template <typename OffT>
__device__ __forceinline__ unsigned long long degree_of(const Params<OffT>& p, uint32_t v) {
  return (unsigned long long)(p.rowptr[v + 1] - p.rowptr[v]);
}

struct WarpTally {
  unsigned long long produced = 0, raw = 0, edges = 0, degree = 0, viol = 0;
};

// One warp-cooperative step over up to 32 edges: lane processes edge e of the
// batch (owner found by a shuffle binary search over inclusive degree sums).
template <int C, typename OffT>
__device__ __forceinline__ void td_light_batch(const Params<OffT>& p, uint32_t nd, OffT beg,
                                               uint32_t deg, uint32_t* qout, WarpPush& wp,
                                               LevelCnt* cnt, WarpTally& t) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  uint32_t incl = deg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(FULL, incl, o);
    if (lane >= (unsigned)o) incl += x;
  }
  const uint32_t total = __shfl_sync(FULL, incl, 31);
  const uint32_t excl = incl - deg;
  for (uint32_t e0 = 0; e0 < total; e0 += 32) {
    const uint32_t e = e0 + lane;
    int j = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const uint32_t x = __shfl_sync(FULL, incl, j + step - 1);
      if (x <= e) j += step;
    }
    const OffT ob = __shfl_sync(FULL, beg, j);
    const uint32_t oex = __shfl_sync(FULL, excl, j);
    bool want = false, distinct = false;
    uint32_t v = 0;
    if (e < total) {
      v = __ldg(&p.col[ob + (e - oex)]);
      want = visit<C>(p, v, nd, distinct, t.viol);
    }
    if (distinct) {
      ++t.produced;
      if (p.policy == kPolicyBeamer) t.degree += degree_of(p, v);
    }
    t.raw += want;
    wp.push(want, v, qout, &cnt->raw, p.qcap, &p.ctl->overflow);
  }
}

template <int C, typename OffT>
__device__ void td_phase_light(const Params<OffT>& p, uint32_t depth, const uint32_t* qin,
                               unsigned long long qlen, uint32_t* qout, WarpPush& wp,
                               LevelCnt* cnt, WarpTally& t) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  for (;;) {
    unsigned int base = 0;
    if (lane == 0) base = atomicAdd(&cnt->td_cursor, 32u);
    base = __shfl_sync(FULL, base, 0);
    if (base >= qlen) break;
    const unsigned long long i = (unsigned long long)base + lane;
    OffT beg = 0, end = 0;
    if (i < qlen) {
      const uint32_t u = qin[i];
      beg = __ldg(&p.rowptr[u]);
      end = __ldg(&p.rowptr[u + 1]);
    }
    unsigned long long deg = (unsigned long long)(end - beg);
    t.edges += deg;
    if (deg > kHeavyDeg) {
      // Hub: split into kChunk-edge items for the grid-wide heavy pass.
      const unsigned int items = (unsigned int)((deg + kChunk - 1) / kChunk);
      const unsigned int slot = atomicAdd(&cnt->heavy_count, items);
      if ((unsigned long long)slot + items <= p.heavy_cap) {
        for (unsigned int k = 0; k < items; ++k) {
          const unsigned long long b = (unsigned long long)beg + (unsigned long long)k * kChunk;
          const unsigned long long e = b + kChunk < (unsigned long long)end ? b + kChunk
                                                                            : (unsigned long long)end;
          p.heavy[slot + k] = HeavyItem{b, e};
        }
      } else {
        atomicExch(&p.ctl->overflow, 1u);
      }
      deg = 0;
    }
    td_light_batch<C>(p, nd, beg, (uint32_t)deg, qout, wp, cnt, t);
  }
}

template <int C, typename OffT>
__device__ void td_phase_heavy(const Params<OffT>& p, uint32_t depth, unsigned int items,
                               uint32_t* qout, WarpPush& wp, LevelCnt* cnt, WarpTally& t) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  for (;;) {
    unsigned int it = 0;
    if (lane == 0) it = atomicAdd(&cnt->heavy_cursor, 1u);
    it = __shfl_sync(FULL, it, 0);
    if (it >= items) break;
    const HeavyItem h = p.heavy[it];
    for (unsigned long long e0 = h.beg; e0 < h.end; e0 += 128) {
      // Four independent coalesced loads in flight per lane.
      uint32_t v[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned long long e = e0 + k * 32 + lane;
        ok[k] = e < h.end;
        v[k] = ok[k] ? __ldg(&p.col[e]) : 0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bool distinct = false;
        const bool want = ok[k] && visit<C>(p, v[k], nd, distinct, t.viol);
        if (distinct) {
          ++t.produced;
          if (p.policy == kPolicyBeamer) t.degree += degree_of(p, v[k]);
        }
        t.raw += want;
        wp.push(want, v[k], qout, &cnt->raw, p.qcap, &p.ctl->overflow);
      }
    }
  }
}

// Bottom-up over all vertices (kernels.cpp:340-382).
template <typename OffT>
__device__ void bu_phase(const Params<OffT>& p, uint32_t depth, const uint32_t* front,
                         uint32_t* next, uint32_t* list, uint32_t* found, WarpTally& t) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  const unsigned warps_total = gridDim.x * kWarps;
  const unsigned gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t groups = p.words / kGroupWords;
  for (uint32_t g = gw; g < groups; g += warps_total) {
    const uint32_t w = g * kGroupWords + (lane & (kGroupWords - 1));
    const bool owner = lane < (unsigned)kGroupWords;
    const uint32_t vis = owner ? p.visited[w] : 0xffffffffu;
    const uint32_t unv = ~vis;
    const uint32_t c = __popc(unv);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    const uint32_t total = __shfl_sync(FULL, incl, 31);
    if (total == 0) {
      if (owner) next[w] = 0;
      continue;
    }
    {
      uint32_t pos = incl - c;
      uint32_t bits = unv;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        list[pos++] = w * 32 + b;
      }
    }
    if (owner) found[lane] = 0;
    __syncwarp();
    for (uint32_t k = 0; k < total; k += 32) {
      const uint32_t idx = k + lane;
      if (idx < total) {
        const uint32_t v = list[idx];
        const OffT beg = __ldg(&p.rowptr[v]);
        const OffT end = __ldg(&p.rowptr[v + 1]);
        for (OffT e = beg; e < end; ++e) {
          const uint32_t u = __ldg(&p.col[e]);
          ++t.edges;
          if ((front[u >> 5] >> (u & 31)) & 1u) {
            p.dist[v] = nd;
            atomicOr(&found[(v >> 5) - g * kGroupWords], 1u << (v & 31));
            ++t.produced;
            if (p.policy == kPolicyBeamer) t.degree += (unsigned long long)(end - beg);
            break;
          }
        }
      }
    }
    __syncwarp();
    if (owner) {
      const uint32_t f = found[lane];
      next[w] = f;
      if (f) p.visited[w] = vis | f;
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void warp_flush_tally(LevelCnt* cnt, WarpTally& t, bool add_raw) {
  const unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t.produced += __shfl_xor_sync(FULL, t.produced, o);
    t.raw += __shfl_xor_sync(FULL, t.raw, o);
    t.edges += __shfl_xor_sync(FULL, t.edges, o);
    t.degree += __shfl_xor_sync(FULL, t.degree, o);
    t.viol += __shfl_xor_sync(FULL, t.viol, o);
  }
  if (lane_id() == 0) {
    if (t.produced) atomicAdd(&cnt->produced, t.produced);
    if (t.edges) atomicAdd(&cnt->edges, t.edges);
    if (t.degree) atomicAdd(&cnt->degree, t.degree);
    if (t.viol) atomicAdd(&cnt->violations, t.viol);
    (void)add_raw;
  }
  t = WarpTally{};
}

template <int C, typename OffT>
__global__ void __launch_bounds__(kThreads) bfs_persistent(Params<OffT> p) {
  __shared__ uint32_t s_list[kWarps][kGroupVerts];  // BU id list / TD push buffer
  __shared__ uint32_t s_found[kWarps][kGroupWords];
  const unsigned warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  const unsigned long long tid = (unsigned long long)blockIdx.x * kThreads + threadIdx.x;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * kThreads;
  Ctl* ctl = p.ctl;
  GridBarrier bar{ctl, 0};
  WarpPush wp{s_list[warp], 0};
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

  // ---- init (Engine ctor + seed, kernels.cpp:72-102,144-163) ------------
  const uint32_t src = p.source;
  {
    uint4* d4 = reinterpret_cast<uint4*>(p.dist);
    const unsigned long long n4 = p.n / 4;
    for (unsigned long long i = tid; i < n4; i += nthreads) {
      uint4 val = make_uint4(kUnreached, kUnreached, kUnreached, kUnreached);
      if ((src >> 2) == i) (&val.x)[src & 3] = 0;
      d4[i] = val;
    }
    for (unsigned long long i = n4 * 4 + tid; i < p.n; i += nthreads) p.dist[i] = i == src ? 0 : kUnreached;
    for (unsigned long long w = tid; w < p.words; w += nthreads) {
      const uint32_t sb = (w == (src >> 5)) ? (1u << (src & 31)) : 0u;
      p.visited[w] = p.init_mask[w] | sb;
      p.bm[0][w] = sb;
    }
    if (leader) {
      p.queue[0][0] = src;
      for (int s = 0; s < 4; ++s) {
        LevelCnt z{};
        ctl->cnt[s] = z;
      }
      ctl->overflow = 0;
    }
  }
  const unsigned long long src_deg = degree_of(p, src);
  // decide_direction for the seed frontier (kernels.cpp:154-156)
  auto decide = [&](bool cur_td, unsigned long long produced, unsigned long long produced_deg,
                    unsigned long long consumed, unsigned long long unvisited_edges) -> bool {
    if (p.policy == kPolicyTopDown) return true;
    if (p.policy == kPolicyFraction) return (double)produced < p.threshold * (double)p.n;
    if (cur_td) {
      if ((double)produced_deg > (double)unvisited_edges / p.alpha) return false;
      return true;
    }
    if ((double)produced < (double)p.n / p.beta && produced < consumed) return true;
    return false;
  };
  unsigned long long unvisited_edges = p.m - src_deg;
  bool td = decide(true, 1, src_deg, 0, unvisited_edges);
  int qcur = 0;              // queue index holding the current frontier (TD)
  int fcur = 0;              // bitmap index holding the current frontier (BU)
  unsigned long long qlen = 1;       // current frontier queue length (raw)
  unsigned long long cur_raw = 1, cur_distinct = 1;
  unsigned long long reached = 0, edges_total = 0, viol_total = 0;
  unsigned int bu_levels = 0;
  unsigned long long t_start = leader ? globaltimer() : 0;
  bar.sync();

  uint32_t depth = 0;
  for (;; ++depth) {
    LevelCnt* cnt = &ctl->cnt[depth & 3];
    if (leader) {
      LevelCnt z{};
      ctl->cnt[(depth + 2) & 3] = z;
    }
    WarpTally t;
    if (td) {
      uint32_t* qout = p.queue[qcur ^ 1];
      td_phase_light<C>(p, depth, p.queue[qcur], qlen, qout, wp, cnt, t);
      if (p.max_degree > kHeavyDeg) {
        bar.sync();
        const unsigned int items = *(volatile unsigned int*)&cnt->heavy_count;
        if (items) td_phase_heavy<C>(p, depth, items, qout, wp, cnt, t);
      }
      wp.flush(qout, &cnt->raw, p.qcap, &ctl->overflow);
    } else {
      bu_phase(p, depth, p.bm[fcur], p.bm[fcur ^ 1], s_list[warp], s_found[warp], t);
    }
    warp_flush_tally(cnt, t, false);
    bar.sync();

    // ---- single section (kernels.cpp:384-464), evaluated by every CTA ----
    const unsigned long long produced = *(volatile unsigned long long*)&cnt->produced;
    const unsigned long long raw = td ? *(volatile unsigned long long*)&cnt->raw : produced;
    const unsigned long long edges = *(volatile unsigned long long*)&cnt->edges;
    const unsigned long long pdeg = *(volatile unsigned long long*)&cnt->degree;
    const unsigned int overflow = *(volatile unsigned int*)&ctl->overflow;
    if (leader) {
      const unsigned long long now = globaltimer();
      if (depth < p.rec_cap) {
        pbfs_level r;
        r.depth = depth;
        r.phase = td ? PBFS_TOP_DOWN : PBFS_BOTTOM_UP;
        r.frontier_size = cur_raw;
        r.distinct_size = cur_distinct;
        r.duplicate_count = cur_raw - cur_distinct;
        r.edges_examined = edges;
        r.flush_events = 0;
        r.elapsed_ns = (long long)(now - t_start);
        p.records[depth] = r;
      }
      t_start = now;
      viol_total += *(volatile unsigned long long*)&cnt->violations;
    }
    reached += cur_distinct;
    edges_total += edges;
    bu_levels += td ? 0 : 1;
    if (overflow || raw == 0) break;
    unvisited_edges -= pdeg;
    const unsigned long long consumed = cur_distinct;
    const bool next_td = decide(td, produced, pdeg, consumed, unvisited_edges);
    if (td && next_td) {
      qcur ^= 1;
      qlen = raw;
    } else if (!td && !next_td) {
      fcur ^= 1;
    } else if (td && !next_td) {
      // Entering bottom-up: frontier bitmap from the produced queue
      // (mark_bitmap_from_dense, kernels.cpp:243-260).
      uint32_t* fb = p.bm[fcur];
      for (unsigned long long w = tid; w < p.words; w += nthreads) fb[w] = 0;
      bar.sync();
      const uint32_t* q = p.queue[qcur ^ 1];
      for (unsigned long long i = tid; i < raw; i += nthreads) {
        const uint32_t v = q[i];
        atomicOr(&fb[v >> 5], 1u << (v & 31));
      }
      bar.sync();
    } else {
      // Entering top-down: ascending queue from the produced bitmap
      // (count_bitmap_slice / write_dense_slice, kernels.cpp:225-241).
      const uint32_t* nb = p.bm[fcur ^ 1];
      uint32_t* q = p.queue[qcur];
      const unsigned warps_total = gridDim.x * kWarps;
      const unsigned gw = blockIdx.x * kWarps + warp;
      for (uint32_t base = gw * 32; base < p.words; base += warps_total * 32) {
        const uint32_t w = base + lane;
        const uint32_t word = w < p.words ? nb[w] : 0u;
        const uint32_t c = __popc(word);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= (unsigned)o) incl += x;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        if (!total) continue;
        unsigned int off = 0;
        if (lane == 0) off = atomicAdd(&cnt->conv_count, total);
        off = __shfl_sync(0xffffffffu, off, 0);
        uint32_t pos = off + incl - c;
        uint32_t bits = word;
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          q[pos++] = w * 32 + b;
        }
      }
      bar.sync();
      qlen = *(volatile unsigned int*)&cnt->conv_count;
    }
    td = next_td;
    cur_raw = raw;
    cur_distinct = produced;
  }

  if (leader) {
    ctl->levels = depth + 1;
    ctl->bu_levels = bu_levels;
    ctl->reached = reached;
    ctl->edges = edges_total;
    ctl->violations = viol_total;
  }
  // Self-reset of the barrier for the next launch: the last CTA out clears it
  // (every CTA has left its final spin before incrementing exit_count).
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int out = atomicAdd(&ctl->exit_count, 1u);
    if (out == gridDim.x - 1) {
      ctl->bar_count = 0;
      ctl->exit_count = 0;
      __threadfence();
    }
  }
}

// Reached-component reduction over the last distance array (metric inputs).
template <typename OffT>
__global__ void component_kernel(const OffT* __restrict__ rowptr, const uint32_t* __restrict__ dist,
                                 unsigned long long n, unsigned long long* out) {
  unsigned long long nr = 0, ar = 0;
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (unsigned long long)gridDim.x * blockDim.x) {
    if (dist[v] != kUnreached) {
      ++nr;
      ar += (unsigned long long)(rowptr[v + 1] - rowptr[v]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nr += __shfl_xor_sync(0xffffffffu, nr, o);
    ar += __shfl_xor_sync(0xffffffffu, ar, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], nr);
    atomicAdd(&out[1], ar);
  }
}

}  // namespace dev
}  // namespace pbfs

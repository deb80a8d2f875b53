// 1D vertex-partitioned BFS: one partition per GPU, one
// frontier-bitmap allgather per level.
//
//   * Ownership by a bijective hash pi on [0, 2^k) (multiply by an odd
//     constant, xor-shift, multiply again; identity + padding when n is not a
//     power of two): rank r owns the vertices with pi(v) in [r*nloc,
//     (r+1)*nloc), so every rank holds an equal share of the RMAT arcs
//     (unpermuted RMAT puts ~42 % of arcs on one of 8 contiguous ranks).
//   * Numbering by gid(v) = owner * nloc + the vertex's rank among its
//     owner's vertices in original order: order-preserving inside each
//     partition, so sorted adjacency lists stay sorted (and RMAT's dense
//     low-id hub region stays dense) -- the probe locality the single-GPU
//     kernel lives on (pi's own order costs ~40 % of top-down speed).
//   * Rank r owns gids [r*nloc, (r+1)*nloc) and stores
//       - the ROW slice: full adjacency of its owned vertices (neighbours as
//         gids) -- bottom-up scans it against the replicated frontier;
//       - the COLUMN slice: for every gid u, u's owned neighbours as local ids,
//         ascending (u's own list filtered by owner; the graph is symmetric)
//         -- top-down expands the whole replicated frontier over it.
//     Either way discoveries are owner-local: dist / visited stores stay
//     local and the claim atomics never cross a GPU.
//   * After each level every rank holds only its own slice of the next
//     frontier bitmap; the host exchanges slices with one allgather (NCCL
//     over NVLink, in place) and every rank then derives the identical
//     distinct count, direction and termination from the full bitmap.
//
// The per-rank level code is the single-GPU engine's device code
// (pbfs_kernels.cuh: td_phase_light / td_phase_heavy / bu_phase /
// compact_bitmap) run over partition-shaped Params, one launch per phase.
// Partitions on the SAME device may share the full bitmaps ("loopback"),
// which turns the allgather into a no-op; tests use it to check G-way
// partitioned traversals bit-exactly on one B200.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "pbfs_internal.h"
#include "pbfs_kernels.cuh"
#include "pbfs_part_impl.h"

using namespace pbfs;
using namespace pbfs::dev;
using namespace pbfs::part;


namespace {

// ---- partition-build kernels ---------------------------------------------------
// Ownership: rank of v = pi(v) / nloc (the hash balances RMAT's arcs).
// Numbering: gid(v) = owner * nloc + (number of vertices u < v with the same
// owner) -- the ORDER-PRESERVING local index. A hub's sorted neighbour list
// stays sorted (and, on RMAT, dense in low ids) inside every partition, so
// the probes of a warp hit few bitmap lines, as on one GPU; pi's own order
// would scatter them.
__global__ void k_owner_flags(uint64_t n, Relabel rl, uint64_t nloc, uint32_t r,
                              uint32_t* flags) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    flags[v] = pi_fwd(rl, v) / nloc == r ? 1u : 0u;
  }
}

__global__ void k_owner_gid(uint64_t n, Relabel rl, uint64_t nloc, uint32_t r,
                            const uint32_t* __restrict__ rank_in, uint32_t* gid, uint32_t* inv) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (pi_fwd(rl, v) / nloc == r) {
      const uint64_t g = r * nloc + rank_in[v];
      gid[v] = (uint32_t)g;
      inv[g] = (uint32_t)v;
    }
  }
}

template <typename OffT>
__global__ void k_local_degrees(const OffT* __restrict__ rowptr, uint64_t n,
                                const uint32_t* __restrict__ inv, uint64_t lo, uint64_t nloc,
                                unsigned long long* deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nloc;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = inv[lo + i];
    deg[i] = v < n ? (unsigned long long)(rowptr[v + 1] - rowptr[v]) : 0ull;
  }
}

// Warp per owned vertex: its neighbour list, renumbered to gids, is its row
// of the row slice (bottom-up).
template <typename OffT>
__global__ void k_fill_rows(const OffT* __restrict__ rowptr, const uint32_t* __restrict__ col,
                            uint64_t n, const uint32_t* __restrict__ gid,
                            const uint32_t* __restrict__ inv, uint64_t lo, uint64_t nloc,
                            const unsigned long long* __restrict__ rowloc, uint32_t* colrow) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; i < nloc;
       i += warps) {
    const uint64_t v = inv[lo + i];
    if (v >= n) continue;
    const uint64_t b = rowptr[v], e = rowptr[v + 1], out = rowloc[i];
    for (uint64_t k = b + lane; k < e; k += 32) colrow[out + (k - b)] = gid[col[k]];
  }
}

// Column slice (top-down): for every vertex u, its neighbours owned by this
// rank as local ids. The graph is symmetric, so that is u's own neighbour
// list filtered by owner -- written in list order, hence ascending. Pass 1
// counts (indexed by gid(u)), pass 2 fills with a warp ballot compaction.
template <typename OffT>
__global__ void k_col_count(const OffT* __restrict__ rowptr, const uint32_t* __restrict__ col,
                            uint64_t n, const uint32_t* __restrict__ gid, uint64_t lo,
                            uint64_t nloc, unsigned long long* colcnt) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t u = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; u < n;
       u += warps) {
    unsigned long long c = 0;
    for (uint64_t k = rowptr[u] + lane; k < rowptr[u + 1]; k += 32) {
      const uint64_t w = gid[col[k]];
      c += (w >= lo && w < lo + nloc) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) colcnt[gid[u]] = c;
  }
}

template <typename OffT>
__global__ void k_col_fill(const OffT* __restrict__ rowptr, const uint32_t* __restrict__ col,
                           uint64_t n, const uint32_t* __restrict__ gid, uint64_t lo,
                           uint64_t nloc, const unsigned long long* __restrict__ colptr,
                           uint32_t* colcol) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t u = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; u < n;
       u += warps) {
    unsigned long long out = colptr[gid[u]];
    const uint64_t e = rowptr[u + 1];
    for (uint64_t k0 = rowptr[u]; k0 < e; k0 += 32) {
      const uint64_t k = k0 + lane;
      uint64_t w = 0;
      bool mine = false;
      if (k < e) {
        w = gid[col[k]];
        mine = w >= lo && w < lo + nloc;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, mine);
      if (mine) colcol[out + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)(w - lo);
      out += __popc(bal);
    }
  }
}

__global__ void k_col_stats(const unsigned long long* __restrict__ colptr, uint64_t npad,
                            unsigned long long* maxdeg, unsigned long long* heavy_items) {
  unsigned long long mx = 0, hv = 0;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < npad;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = colptr[u + 1] - colptr[u];
    mx = d > mx ? d : mx;
    if (d > kHeavyDeg) hv += (d + kChunk - 1) / kChunk;
  }
  atomicMax(maxdeg, mx);
  if (hv) atomicAdd(heavy_items, hv);
}

__global__ void k_first_nbr(const unsigned long long* __restrict__ rowloc,
                            const uint32_t* __restrict__ colrow, uint64_t nloc, uint32_t* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nloc;
       i += (uint64_t)gridDim.x * blockDim.x) {
    first[i] = rowloc[i] < rowloc[i + 1] ? colrow[rowloc[i]] : 0u;
  }
}

__global__ void k_local_mask(const unsigned long long* __restrict__ rowloc, uint64_t nloc,
                             uint64_t words, uint32_t* mask) {
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m = 0;
    for (int b = 0; b < 32; ++b) {
      const uint64_t i = w * 32 + b;
      if (i >= nloc || rowloc[i + 1] == rowloc[i]) m |= 1u << b;  // isolated / padding
    }
    mask[w] = m;
  }
}

// ---- per-level kernels -------------------------------------------------------------
// The level state lives on the device so a host can enqueue several levels
// ahead without a sync: every level kernel reads it first and returns when
// the traversal is done or the level goes the other direction, and
// k_decide (one thread) applies the 5 % rule. The host's only per-level
// knowledge is the bitmap parity (fcur flips every level), which names the
// `next` buffer it allgathers.
__global__ void k_begin(uint32_t* dist, uint32_t* visited, const uint32_t* mask, uint64_t nloc,
                        uint64_t lwords, uint32_t* front, uint32_t* next, uint64_t clear_lo,
                        uint64_t clear_words, const uint32_t* __restrict__ gid, uint32_t source,
                        uint64_t lo, bool shared, uint32_t* queue, PartState* st, bool seed_td) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t src_pi = gid[source];
  const bool owner = src_pi >= lo && src_pi < lo + nloc;
  const bool set_src_bit = !shared || owner;
  for (uint64_t i = tid; i < nloc; i += nth) dist[i] = (owner && i == src_pi - lo) ? 0u : kUnreached;
  for (uint64_t w = tid; w < lwords; w += nth) {
    uint32_t m = mask[w];
    if (owner && w == (src_pi - lo) / 32) m |= 1u << ((src_pi - lo) & 31);
    visited[w] = m;
  }
  for (uint64_t w = tid; w < clear_words; w += nth) {
    const uint64_t gw = clear_lo + w;
    front[gw] = (set_src_bit && gw == src_pi / 32) ? (1u << (src_pi & 31)) : 0u;
    next[gw] = 0u;
  }
  if (tid == 0) {
    queue[0] = (uint32_t)src_pi;
    PartState z{};
    z.qlen = 1;
    z.cur_distinct = 1;
    z.td = seed_td ? 1u : 0u;
    *st = z;
  }
}

// Zero this rank's slice of the next bitmap (top-down marks into it).
__global__ void k_clear(uint32_t* bm0, uint32_t* bm1, uint64_t lo_word, uint64_t words,
                        const PartState* st) {
  if (st->done || !st->td) return;
  uint32_t* p = (st->fcur ? bm0 : bm1) + lo_word;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
       w += (uint64_t)gridDim.x * blockDim.x) {
    p[w] = 0u;
  }
}

template <typename OffT>
__global__ void __launch_bounds__(kThreads) k_td_light(Params<OffT> p, uint32_t* q0,
                                                       uint32_t* q1, uint32_t* bm0, uint32_t* bm1,
                                                       uint64_t lo_word, const PartState* st) {
  if (st->done || !st->td) return;
  __shared__ uint32_t s_buf[kWarps][kPushBuf];
  WarpPush wp{s_buf[threadIdx.x >> 5], 0};
  WarpTally t;
  LevelCnt* cnt = &p.ctl->cnt[0];
  uint32_t* mark = (st->fcur ? bm0 : bm1) + lo_word;
  td_phase_light<kClaimBitmap>(p, st->depth, q0, st->qlen, q1, wp, cnt, t, mark, nullptr);
  wp.flush(q1, &cnt->raw, p.qcap, &p.ctl->overflow);
  warp_flush_tally(cnt, t, false);
}

template <typename OffT>
__global__ void __launch_bounds__(kThreads) k_td_heavy(Params<OffT> p, uint32_t* q1,
                                                       uint32_t* bm0, uint32_t* bm1,
                                                       uint64_t lo_word, const PartState* st) {
  if (st->done || !st->td) return;
  __shared__ uint32_t s_buf[kWarps][kPushBuf];
  WarpPush wp{s_buf[threadIdx.x >> 5], 0};
  WarpTally t;
  LevelCnt* cnt = &p.ctl->cnt[0];
  uint32_t* mark = (st->fcur ? bm0 : bm1) + lo_word;
  const unsigned int items = *(volatile unsigned int*)&cnt->heavy_count;
  if (items) td_phase_heavy<kClaimBitmap>(p, st->depth, items, q1, wp, cnt, t, mark);
  wp.flush(q1, &cnt->raw, p.qcap, &p.ctl->overflow);
  warp_flush_tally(cnt, t, false);
}

template <typename OffT>
__global__ void __launch_bounds__(kThreads) k_bu(Params<OffT> p, uint32_t* bm0, uint32_t* bm1,
                                                 uint64_t lo_word, const PartState* st) {
  if (st->done || st->td) return;
  __shared__ uint32_t s_list[kWarps][kListCap];
  __shared__ uint32_t s_found[kWarps][kGroupWords];
  const unsigned warp = threadIdx.x >> 5;
  const uint32_t* front = st->fcur ? bm1 : bm0;
  uint32_t* next_local = (st->fcur ? bm0 : bm1) + lo_word;
  WarpTally t;
  bu_phase(p, st->depth, front, next_local, s_list[warp], s_found[warp], t,
           &p.ctl->cnt[0].bu_cursor, false);
  warp_flush_tally(&p.ctl->cnt[0], t, false);
}

// Distinct size of the gathered next frontier (same value on every rank).
__global__ void k_popcount(const uint32_t* __restrict__ bm0, const uint32_t* __restrict__ bm1,
                           uint64_t words, PartState* st) {
  if (st->done) return;
  const uint32_t* bm = st->fcur ? bm0 : bm1;
  unsigned long long c = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
       w += (uint64_t)gridDim.x * blockDim.x) {
    c += __popc(bm[w]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&st->distinct, c);
}

// single_section + decide_direction (kernels.cpp:384-464, :487-513) for one
// partition: record the level, stop on an empty frontier, else flip the
// bitmaps, apply the 5 % rule and request the queue compaction for a
// top-down level.
__global__ void k_decide(PartState* st, Ctl* ctl, pbfs_level* recs, int policy, double threshold,
                         unsigned long long n) {
  if (st->done) return;
  const unsigned long long produced = st->distinct;
  LevelCnt* cnt = &ctl->cnt[0];
  if (st->depth < kPartRecCap) {
    pbfs_level r{};
    r.depth = st->depth;
    r.phase = st->td ? PBFS_TOP_DOWN : PBFS_BOTTOM_UP;
    r.frontier_size = st->cur_distinct;
    r.distinct_size = st->cur_distinct;
    r.edges_examined = cnt->edges;  // this rank's share
    recs[st->depth] = r;
  }
  if (produced == 0) {
    st->done = 1;
    return;
  }
  const bool next_td = policy == kPolicyTopDown || (double)produced < threshold * (double)n;
  st->fcur ^= 1u;
  st->cur_distinct = produced;
  st->distinct = 0;
  st->depth += 1;
  st->td = next_td ? 1u : 0u;
  st->compact = next_td ? 1u : 0u;
  ctl->cnt[1].conv_count = 0;
  // The next level's counters start from zero.
  LevelCnt z{};
  ctl->cnt[0] = z;
}

// Every rank compacts the FULL gathered frontier (gids) into its queue.
__global__ void k_compact(const uint32_t* bm0, const uint32_t* bm1, uint64_t words,
                          uint32_t* queue, LevelCnt* cnt, const PartState* st) {
  if (!st->compact) return;
  compact_bitmap(const_cast<uint32_t*>(st->fcur ? bm1 : bm0), queue, (uint32_t)words,
                 &cnt->conv_count, false);
}

__global__ void k_set_qlen(const LevelCnt* cnt, PartState* st) {
  if (!st->compact) return;
  st->qlen = cnt->conv_count;
  st->compact = 0;
}

__global__ void k_unrelabel(const uint32_t* __restrict__ dist_pi, uint64_t n,
                            const uint32_t* __restrict__ gid, uint32_t* dist) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    dist[v] = dist_pi[gid[v]];
  }
}

}  // namespace

namespace {

pbfs_status cuda_fail_p(cudaError_t e, const char* what) {
  cudaGetLastError();
  return fail(PBFS_E_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}
#define PCUDA(call, what)                                   \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess) return cuda_fail_p(_e, what);    \
  } while (0)

template <typename T>
pbfs_status palloc(pbfs_part* g, T** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PBFS_E_CAPACITY, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  g->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return PBFS_OK;
}

void part_release(pbfs_part* g) { pbfs::part::release(g); }

// Launch on `s` with a persisting-L2 window over [base, base + bytes): the
// top-down kernels keep the local visited slice resident against the col
// stream, bottom-up the frontier bitmap it probes.
template <typename... KArgs, typename... Args>
cudaError_t launch_window(void (*kern)(KArgs...), int grid, cudaStream_t s, const void* base,
                          size_t bytes, size_t persist, Args... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(kThreads);
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  int nattr = 0;
  if (persist && bytes) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr[0].val.accessPolicyWindow.num_bytes = bytes;
    attr[0].val.accessPolicyWindow.hitRatio =
        std::min(1.0f, static_cast<float>(persist) / static_cast<float>(bytes));
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    nattr = 1;
  }
  lc.attrs = attr;
  lc.numAttrs = nattr;
  return cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...);
}

}  // namespace

namespace pbfs {
namespace part {

void release(pbfs_part* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  for (void* p : g->allocs) cudaFree(p);
  if (g->st_host) cudaFreeHost(g->st_host);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

Params<unsigned long long> td_params(const pbfs_part* g) {
  Params<unsigned long long> p{};
  p.rowptr = g->colptr;
  p.col = g->colcol;
  p.dist = g->dist;
  p.visited = g->visited;
  p.heavy = g->heavy;
  p.ctl = g->ctl;
  p.qcap = g->nloc + 1;
  p.heavy_cap = g->heavy_cap;
  p.heavy_deg = kHeavyDeg;
  p.chunk_log2 = __builtin_ctz(kChunk);
  p.n = g->nloc;
  p.words = (uint32_t)g->lwords;
  p.policy = g->policy;
  p.threshold = g->threshold;
  return p;
}

Params<unsigned long long> bu_params(const pbfs_part* g) {
  Params<unsigned long long> p{};
  p.rowptr = g->rowloc;
  p.col = g->colrow;
  p.first_nbr = g->first;
  p.dist = g->dist;
  p.visited = g->visited;
  p.ctl = g->ctl;
  p.n = g->nloc;
  p.words = (uint32_t)g->lwords;
  p.policy = g->policy;
  p.threshold = g->threshold;
  return p;
}

}  // namespace part
}  // namespace pbfs

namespace {

template <typename OffT>
pbfs_status build_partition(pbfs_part* g, const OffT* rowptr, const uint32_t* col) {
  cudaStream_t s = g->stream;
  const int blocks = g->grid;
  pbfs_status st;
  // Scan scratch sized for every scan below.
  size_t tmp_bytes = 0, t1 = 0, t2 = 0, t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, static_cast<uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), (int64_t)g->n, s);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, static_cast<unsigned long long*>(nullptr),
                                static_cast<unsigned long long*>(nullptr), (int64_t)(g->nloc + 1), s);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, static_cast<unsigned long long*>(nullptr),
                                static_cast<unsigned long long*>(nullptr), (int64_t)(g->npad + 1), s);
  tmp_bytes = std::max({t1, t2, t3, size_t{16}});
  void* tmp = nullptr;
  PCUDA(cudaMalloc(&tmp, tmp_bytes), "scan scratch");
  auto bail = [&](pbfs_status x) {
    cudaFree(tmp);
    return x;
  };
  // 1. gid / inv maps: one flag scan per owner rank.
  if ((st = palloc(g, &g->gid, g->n * 4 + 16)) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->inv, g->npad * 4 + 16)) != PBFS_OK) return bail(st);
  PCUDA(cudaMemsetAsync(g->inv, 0xFF, g->npad * 4, s), "memset");
  {
    uint32_t *flags = nullptr, *rank_in = nullptr;
    PCUDA(cudaMalloc(&flags, g->n * 4 + 16), "flags");
    if (cudaMalloc(&rank_in, g->n * 4 + 16) != cudaSuccess) {
      cudaFree(flags);
      cudaGetLastError();
      return bail(fail(PBFS_E_CAPACITY, "partition build scratch"));
    }
    for (uint32_t r = 0; r < g->world; ++r) {
      k_owner_flags<<<blocks, 256, 0, s>>>(g->n, g->rl, g->nloc, r, flags);
      cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, rank_in, (int64_t)g->n, s);
      k_owner_gid<<<blocks, 256, 0, s>>>(g->n, g->rl, g->nloc, r, rank_in, g->gid, g->inv);
    }
    cudaError_t e = cudaStreamSynchronize(s);
    cudaFree(flags);
    cudaFree(rank_in);
    if (e != cudaSuccess) return bail(cuda_fail_p(e, "gid maps"));
  }
  // 2. Row slice: owned vertices' lists, neighbours as gids.
  unsigned long long* deg = nullptr;
  if ((st = palloc(g, &g->rowloc, (g->nloc + 1) * 8)) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &deg, (g->nloc + 1) * 8)) != PBFS_OK) return bail(st);
  PCUDA(cudaMemsetAsync(deg, 0, (g->nloc + 1) * 8, s), "memset");
  k_local_degrees<OffT><<<blocks, 256, 0, s>>>(rowptr, g->n, g->inv, g->lo, g->nloc, deg);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, g->rowloc, (int64_t)(g->nloc + 1), s);
  unsigned long long mloc = 0;
  PCUDA(cudaMemcpyAsync(&mloc, g->rowloc + g->nloc, 8, cudaMemcpyDeviceToHost, s), "read m_loc");
  PCUDA(cudaStreamSynchronize(s), "partition scan");
  g->m_loc = mloc;
  if ((st = palloc(g, &g->colrow, (g->m_loc + 16) * 4)) != PBFS_OK) return bail(st);
  k_fill_rows<OffT><<<blocks, 256, 0, s>>>(rowptr, col, g->n, g->gid, g->inv, g->lo, g->nloc,
                                           g->rowloc, g->colrow);
  // 3. Column slice: every vertex's owned neighbours, ascending local ids.
  unsigned long long* colcnt = nullptr;
  if ((st = palloc(g, &colcnt, (g->npad + 1) * 8)) != PBFS_OK) return bail(st);
  PCUDA(cudaMemsetAsync(colcnt, 0, (g->npad + 1) * 8, s), "memset");
  k_col_count<OffT><<<blocks, 256, 0, s>>>(rowptr, col, g->n, g->gid, g->lo, g->nloc, colcnt);
  if ((st = palloc(g, &g->colptr, (g->npad + 1) * 8)) != PBFS_OK) return bail(st);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, colcnt, g->colptr, (int64_t)(g->npad + 1), s);
  if ((st = palloc(g, &g->colcol, (g->m_loc + 8) * 4)) != PBFS_OK) return bail(st);
  k_col_fill<OffT><<<blocks, 256, 0, s>>>(rowptr, col, g->n, g->gid, g->lo, g->nloc, g->colptr,
                                          g->colcol);
  unsigned long long* stats = deg;  // reuse: [0] maxdeg, [1] heavy items
  PCUDA(cudaMemsetAsync(stats, 0, 16, s), "memset");
  k_col_stats<<<blocks, 256, 0, s>>>(g->colptr, g->npad, stats, stats + 1);
  unsigned long long hs[2];
  PCUDA(cudaMemcpyAsync(hs, stats, 16, cudaMemcpyDeviceToHost, s), "read stats");
  if ((st = palloc(g, &g->mask, g->lwords * 4)) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->first, (g->nloc + 1) * 4)) != PBFS_OK) return bail(st);
  k_first_nbr<<<blocks, 256, 0, s>>>(g->rowloc, g->colrow, g->nloc, g->first);
  k_local_mask<<<blocks, 256, 0, s>>>(g->rowloc, g->nloc, g->lwords, g->mask);
  PCUDA(cudaGetLastError(), "partition kernels");
  PCUDA(cudaStreamSynchronize(s), "partition build");
  cudaFree(tmp);
  g->col_maxdeg = hs[0];
  g->heavy_cap = hs[1];
  return PBFS_OK;
}

pbfs_status part_create_impl(uint64_t n, bool symmetric, int device, const void* rowptr,
                             const uint32_t* col, uint32_t offb, const pbfs_part_options* opt,
                             pbfs_part** out);
}  // namespace

namespace pbfs {
namespace part {
pbfs_status create(uint64_t n, bool symmetric, int device, const void* rowptr, const uint32_t* col,
                   uint32_t offb, const pbfs_part_options* opt, pbfs_part** out) {
  return part_create_impl(n, symmetric, device, rowptr, col, offb, opt, out);
}
}  // namespace part
}  // namespace pbfs

extern "C" {

pbfs_status pbfs_part_create(const pbfs_graph* full, const pbfs_part_options* opt,
                             pbfs_part** out) {
  if (!full || !opt || !out) return fail(PBFS_E_INPUT, "null argument");
  pbfs_graph_info gi;
  pbfs_status st = pbfs_graph_get_info(full, &gi);
  if (st != PBFS_OK) return st;
  const void* rowptr = nullptr;
  const uint32_t* col = nullptr;
  uint32_t offb = 0;
  if ((st = pbfs_graph_device_arrays(full, &rowptr, &col, &offb)) != PBFS_OK) return st;
  return part_create_impl(gi.vertex_count, gi.symmetric != 0, gi.device, rowptr, col, offb, opt,
                          out);
}

pbfs_status pbfs_part_create_device(const pbfs_csr* dcsr, int32_t device,
                                    const pbfs_part_options* opt, pbfs_part** out) {
  if (!dcsr || !opt || !out) return fail(PBFS_E_INPUT, "null argument");
  if (dcsr->offset_bytes != 4 && dcsr->offset_bytes != 8) {
    return fail(PBFS_E_FORMAT, "offset width must be 4 or 8 bytes");
  }
  return part_create_impl(dcsr->vertex_count, dcsr->symmetric != 0, device, dcsr->row_offsets,
                          dcsr->column_indices, dcsr->offset_bytes, opt, out);
}

}  // extern "C"

namespace {
pbfs_status part_create_impl(uint64_t n, bool symmetric, int device, const void* rowptr,
                             const uint32_t* col, uint32_t offb, const pbfs_part_options* opt,
                             pbfs_part** out) {
  if (opt->world < 1 || opt->rank >= opt->world) return fail(PBFS_E_CONFIG, "bad rank/world");
  if (!symmetric) {
    return fail(PBFS_E_INPUT, "the vertex partition needs a symmetric graph (its column "
                              "slice is the transpose of the row slice)");
  }
  pbfs_status st;
  struct {
    uint64_t vertex_count;
    int32_t device;
  } gi{n, device};
  auto* g = new (std::nothrow) pbfs_part;
  if (!g) return fail(PBFS_E_CAPACITY, "host allocation failed");
  g->device = gi.device;
  g->rank = opt->rank;
  g->world = opt->world;
  g->n = gi.vertex_count;
  g->offb = offb;
  // Padded id space: a power of two (hashed relabel) or the next multiple of
  // 512 * world (identity), so every rank's slice is whole 16-word groups.
  uint32_t k = 0;
  while ((1ull << k) < g->n) ++k;
  const bool pow2 = (1ull << k) == g->n;
  const uint64_t quantum = 512ull * g->world;
  // The hashed bijection lives on [0, 2^k): its equal ownership ranges
  // [r * n / world, ...) tile it exactly only when world divides 2^k into
  // whole 512-vertex groups, i.e. world is a power of two and n >= quantum.
  // Any other world size (3, 5, 6, 7) takes identity + padding.
  const bool world_pow2 = (g->world & (g->world - 1)) == 0;
  if (pow2 && world_pow2 && opt->relabel && g->n >= quantum) {
    g->npad = g->n;
    g->rl = make_relabel(k, true);
  } else {
    g->npad = (g->n + quantum - 1) / quantum * quantum;
    g->rl = make_relabel(k, false);
  }
  g->nloc = g->npad / g->world;
  g->lo = g->nloc * g->rank;
  g->words_total = g->npad / 32;
  g->lwords = g->nloc / 32;
  g->shared = opt->shared_frontier && opt->shared_next;
  cudaSetDevice(g->device);
  auto bail = [&](pbfs_status s2) {
    part_release(g);
    return s2;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bail(cuda_fail_p(e, "stream"));
  int occ = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, g->device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_td_light<unsigned long long>, kThreads, 0);
  g->grid = prop.multiProcessorCount * std::max(occ, 1);
  st = offb == 8 ? build_partition<unsigned long long>(g, static_cast<const unsigned long long*>(rowptr), col)
                 : build_partition<uint32_t>(g, static_cast<const uint32_t*>(rowptr), col);
  if (st != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->dist, g->nloc * 4 + 16)) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->visited, g->lwords * 4)) != PBFS_OK) return bail(st);
  if (g->shared) {
    g->bm[0] = static_cast<uint32_t*>(opt->shared_frontier);
    g->bm[1] = static_cast<uint32_t*>(opt->shared_next);
  } else {
    if ((st = palloc(g, &g->bm[0], g->words_total * 4)) != PBFS_OK) return bail(st);
    if ((st = palloc(g, &g->bm[1], g->words_total * 4)) != PBFS_OK) return bail(st);
  }
  if ((st = palloc(g, &g->queue[0], (g->npad + 1) * 4)) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->queue[1], (g->npad + 1) * 4)) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->heavy, std::max<uint64_t>(g->heavy_cap, 1) * sizeof(HeavyItem))) != PBFS_OK)
    return bail(st);
  if ((st = palloc(g, &g->ctl, sizeof(Ctl))) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->st, sizeof(PartState))) != PBFS_OK) return bail(st);
  if ((st = palloc(g, &g->recs, kPartRecCap * sizeof(pbfs_level))) != PBFS_OK) return bail(st);
  if ((e = cudaMallocHost(&g->st_host, sizeof(PartState))) != cudaSuccess)
    return bail(cuda_fail_p(e, "pinned state"));
  PCUDA(cudaMemset(g->ctl, 0, sizeof(Ctl)), "memset");
  // Persisting-L2 set-aside (process-wide limit, only ever raised) for the
  // level kernels' windows: the larger of the local visited slice and the
  // full frontier bitmap.
  if (prop.persistingL2CacheMaxSize > 0) {
    const size_t want = std::min<size_t>(std::max<size_t>(g->lwords, g->words_total) * 4,
                                         prop.persistingL2CacheMaxSize);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur >= want || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
      g->persist = std::max(cur, want);
    }
    cudaGetLastError();
  }
  *out = g;
  return PBFS_OK;
}
}  // namespace

extern "C" {

pbfs_status pbfs_part_destroy(pbfs_part* g) {
  part_release(g);
  return PBFS_OK;
}

pbfs_status pbfs_part_get_info(const pbfs_part* g, pbfs_part_info* info) {
  if (!g || !info) return fail(PBFS_E_INPUT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->vertex_count = g->n;
  info->padded_count = g->npad;
  info->local_first = g->lo;
  info->local_count = g->nloc;
  info->local_arcs = g->m_loc;
  info->words_total = g->words_total;
  info->words_local = g->lwords;
  info->rank = g->rank;
  info->world = g->world;
  info->relabel_hashed = g->rl.hashed;
  info->frontier = g->bm[g->fcur];
  info->next = g->bm[g->fcur ^ 1];
  info->dist_local = g->dist;
  info->depth = g->depth;
  info->top_down = g->td ? 1u : 0u;
  return PBFS_OK;
}

pbfs_status pbfs_part_relabel(const pbfs_part* g, uint64_t v, uint64_t* pi_v) {
  if (!g || !pi_v) return fail(PBFS_E_INPUT, "null argument");
  if (v >= g->n) return fail(PBFS_E_INPUT, "vertex out of range");
  uint32_t x = 0;
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  PCUDA(cudaMemcpy(&x, g->gid + v, 4, cudaMemcpyDeviceToHost), "gid");
  *pi_v = x;
  return PBFS_OK;
}

pbfs_status pbfs_part_begin(pbfs_part* g, uint32_t source, const pbfs_config* cfg, void* stream) {
  if (!g || !cfg) return fail(PBFS_E_INPUT, "null argument");
  pbfs_status st = pbfs_config_validate(cfg);
  if (st != PBFS_OK) return st;
  if (cfg->variant != PBFS_HYBRID && cfg->variant != PBFS_VISITED_INLINE) {
    return fail(PBFS_E_CONFIG, "the partitioned engine runs the hybrid (5 % rule) traversal");
  }
  if (source >= g->n) {
    return fail(PBFS_E_INPUT, "source vertex " + std::to_string(source) +
                                  " is out of range for a graph with " + std::to_string(g->n) +
                                  " vertices");
  }
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  g->policy = cfg->force_top_down_only ? kPolicyTopDown : kPolicyFraction;
  g->threshold = cfg->hybrid_threshold_fraction;
  g->fcur = 0;
  g->depth = 0;
  g->issued = 0;
  g->td = true;
  const uint64_t clear_lo = g->shared ? g->lo / 32 : 0;
  const uint64_t clear_words = g->shared ? g->lwords : g->words_total;
  // decide_direction for the seed (kernels.cpp:154-156); the size-fraction
  // rule does not need the source degree.
  const bool seed_td = g->policy == kPolicyTopDown || 1.0 < g->threshold * (double)g->n;
  PCUDA(cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), s), "memset ctl");
  k_begin<<<g->grid, 256, 0, s>>>(g->dist, g->visited, g->mask, g->nloc, g->lwords, g->bm[0],
                                  g->bm[1], clear_lo, clear_words, g->gid, source, g->lo,
                                  g->shared, g->queue[0], g->st, seed_td);
  PCUDA(cudaGetLastError(), "begin");
  return PBFS_OK;
}

// Enqueues one level's local work; needs no host knowledge of the level's
// direction (the kernels read it on the device).
pbfs_status pbfs_part_step(pbfs_part* g, void* stream) {
  if (!g) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  const uint64_t lo_word = g->lo / 32;
  k_clear<<<g->grid, 256, 0, s>>>(g->bm[0], g->bm[1], lo_word, g->lwords, g->st);
  Params<unsigned long long> tp = td_params(g);
  const size_t vbytes = g->lwords * 4;
  PCUDA(launch_window(k_td_light<unsigned long long>, g->grid, s, g->visited, vbytes, g->persist,
                      tp, g->queue[0], g->queue[1], g->bm[0], g->bm[1], lo_word,
                      (const PartState*)g->st),
        "top-down launch");
  if (g->col_maxdeg > kHeavyDeg) {
    PCUDA(launch_window(k_td_heavy<unsigned long long>, g->grid, s, g->visited, vbytes,
                        g->persist, tp, g->queue[1], g->bm[0], g->bm[1], lo_word,
                        (const PartState*)g->st),
          "top-down launch");
  }
  Params<unsigned long long> bp = bu_params(g);
  // The frontier bitmap the bottom-up probes: its parity is known here.
  PCUDA(launch_window(k_bu<unsigned long long>, g->grid, s, g->bm[g->fcur], g->words_total * 4,
                      g->persist, bp, g->bm[0], g->bm[1], lo_word, (const PartState*)g->st),
        "bottom-up launch");
  return PBFS_OK;
}

pbfs_status pbfs_part_end_level_async(pbfs_part* g, void* stream) {
  if (!g) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  k_popcount<<<g->grid, 256, 0, s>>>(g->bm[0], g->bm[1], g->words_total, g->st);
  k_decide<<<1, 1, 0, s>>>(g->st, g->ctl, g->recs, g->policy, g->threshold, g->n);
  k_compact<<<g->grid, kThreads, 0, s>>>(g->bm[0], g->bm[1], g->words_total, g->queue[0],
                                         &g->ctl->cnt[1], g->st);
  k_set_qlen<<<1, 1, 0, s>>>(&g->ctl->cnt[1], g->st);
  PCUDA(cudaGetLastError(), "level end");
  g->fcur ^= 1;  // host parity: names the next level's allgather target
  ++g->issued;
  return PBFS_OK;
}

pbfs_status pbfs_part_poll(pbfs_part* g, void* stream, uint32_t* done, uint32_t* levels) {
  if (!g || !done) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  unsigned int overflow = 0;
  PCUDA(cudaMemcpyAsync(g->st_host, g->st, sizeof(PartState), cudaMemcpyDeviceToHost, s), "read");
  PCUDA(cudaMemcpyAsync(&overflow, &g->ctl->overflow, 4, cudaMemcpyDeviceToHost, s), "read");
  PCUDA(cudaStreamSynchronize(s), "level");
  if (overflow) return fail(PBFS_E_CAPACITY, "partition frontier overflow");
  *done = g->st_host->done;
  g->depth = g->st_host->depth;
  g->td = g->st_host->td != 0;
  if (levels) *levels = g->st_host->depth + (g->st_host->done ? 1u : 0u);
  return PBFS_OK;
}

pbfs_status pbfs_part_level_record(pbfs_part* g, uint32_t depth, pbfs_level* rec) {
  if (!g || !rec) return fail(PBFS_E_INPUT, "null argument");
  if (depth >= kPartRecCap) return fail(PBFS_E_CAPACITY, "level beyond the record capacity");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  PCUDA(cudaMemcpy(rec, g->recs + depth, sizeof(pbfs_level), cudaMemcpyDeviceToHost), "record");
  return PBFS_OK;
}

pbfs_status pbfs_part_end_level(pbfs_part* g, void* stream, uint32_t* done, pbfs_level* rec) {
  if (!g || !done) return fail(PBFS_E_INPUT, "null argument");
  const uint32_t depth = g->issued;
  pbfs_status st = pbfs_part_end_level_async(g, stream);
  if (st != PBFS_OK) return st;
  if ((st = pbfs_part_poll(g, stream, done, nullptr)) != PBFS_OK) return st;
  if (rec) return pbfs_part_level_record(g, depth, rec);
  return PBFS_OK;
}

pbfs_status pbfs_part_unrelabel(pbfs_part* g, const uint32_t* dist_pi, uint32_t* dist,
                                void* stream) {
  if (!g || !dist_pi || !dist) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  k_unrelabel<<<g->grid, 256, 0, s>>>(dist_pi, g->n, g->gid, dist);
  PCUDA(cudaGetLastError(), "unrelabel");
  return PBFS_OK;
}

pbfs_status pbfs_part_component(pbfs_part* g, uint64_t* n_reached, uint64_t* arcs_reached) {
  if (!g || !n_reached || !arcs_reached) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  unsigned long long* out = reinterpret_cast<unsigned long long*>(&g->ctl->cnt[2]);
  PCUDA(cudaMemsetAsync(out, 0, 16, g->stream), "memset");
  // component_kernel (pbfs_kernels.cuh) over the row slice: local degrees.
  component_kernel<unsigned long long><<<g->grid, 256, 0, g->stream>>>(g->rowloc, g->dist,
                                                                         g->nloc, out);
  unsigned long long h[2];
  PCUDA(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, g->stream), "read");
  PCUDA(cudaStreamSynchronize(g->stream), "component");
  *n_reached = h[0];
  *arcs_reached = h[1];
  return PBFS_OK;
}

pbfs_status pbfs_part_copy_dist(pbfs_part* g, uint32_t* host_out) {
  if (!g || !host_out) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  PCUDA(cudaStreamSynchronize(g->stream), "sync");
  PCUDA(cudaMemcpy(host_out, g->dist, g->nloc * 4, cudaMemcpyDeviceToHost), "copy dist");
  return PBFS_OK;
}

pbfs_status pbfs_part_unrelabel_host(const pbfs_part* g, const uint32_t* dist_pi, uint32_t* dist) {
  if (!g || !dist_pi || !dist) return fail(PBFS_E_INPUT, "null argument");
  auto* gm = const_cast<pbfs_part*>(g);
  if (gm->gid_host.size() != g->n) {
    gm->gid_host.resize(g->n);
    PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
    PCUDA(cudaMemcpy(gm->gid_host.data(), g->gid, g->n * 4, cudaMemcpyDeviceToHost), "gid map");
  }
  for (uint64_t v = 0; v < g->n; ++v) dist[v] = dist_pi[gm->gid_host[v]];
  return PBFS_OK;
}

pbfs_status pbfs_part_sync(pbfs_part* g, void* stream) {
  if (!g) return fail(PBFS_E_INPUT, "null argument");
  PCUDA(cudaSetDevice(g->device), "cudaSetDevice");
  PCUDA(cudaStreamSynchronize(stream ? static_cast<cudaStream_t>(stream) : g->stream), "sync");
  return PBFS_OK;
}

}  // extern "C"

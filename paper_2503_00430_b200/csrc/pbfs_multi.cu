// Multi-partition BFS with the frontier exchange fused into the level
// kernels (the next step DESIGN.md §6 named in round 1).
//
// The 1D vertex partition of pbfs_part.cu (hashed ownership, order-preserving
// gids, row slice for bottom-up, column slice for top-down), run as ONE
// persistent cooperative launch per device for a whole traversal. A launch
// carries every partition placed on its device (its CTAs split evenly), so
// the same code runs
//   * one partition per GPU of an NVLink/NVSwitch box (one process drives all
//     devices; peers' buffers are reached through peer access), and
//   * several partitions on one GPU ("loopback"), which is how the protocol
//     is tested bit-exactly on a single B200: partitions never share buffers,
//     every exchange goes through the same peer stores and flags.
//
// Per level, partition p (its CTAs):
//   top-down  expands the replicated frontier -- a queue of P segments, one
//             per partition -- over its column slice (td_phase_light /
//             td_phase_heavy, pbfs_kernels.cuh). Discoveries are owner-local
//             (dist / visited / claim atomics never leave p), and every
//             per-warp flush writes p's discoveries (as gids) into p's
//             segment of EVERY partition's next queue: the allgather of the
//             frontier is the level's own stores, tile by tile.
//   bottom-up scans p's unvisited vertices against the replicated frontier
//             bitmap; every 32-word group of p's next-bitmap slice is stored
//             locally and into every peer's bitmap at the same offset.
//   then      each CTA releases its stores at system scope, the partition
//             barrier gives p's level counters, and p's first CTA writes
//             {sequence, discoveries, edges} into slot p of every
//             partition's exchange block. Every CTA of every partition polls
//             the P slots of its OWN exchange block (local memory) until all
//             carry this exchange's sequence number: that single flag round
//             replaces the host round trip + NCCL allgather + decision
//             launches of pbfs_part.cu. All partitions then take the same
//             decision (the reference's IEEE-double 5 % rule on the summed
//             distinct count, kernels.cpp:494-497) and termination
//             (raw == 0, kernels.cpp:440-443).
// Conversions: bottom-up -> top-down compacts the (replicated, complete)
// bitmap locally into segment 0; top-down -> bottom-up rebuilds p's slice of
// the frontier bitmap from its distances and pushes it (one more exchange).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
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

namespace pbfs {
namespace multi {

constexpr int kMaxParts = 8;

// One exchange record: written by partition q into slot q of every
// partition's block (sequence last, with release semantics).
struct alignas(64) XSlot {
  unsigned long long seq;       // (run << 32) | (exchange index + 1)
  unsigned long long produced;  // q's distinct discoveries (= queue pushes)
  unsigned long long edges;     // q's adjacency entries examined
  unsigned long long pad[5];
};
// Double-buffered by exchange parity: a slot is rewritten two exchanges
// later, by which time every reader has copied it (see the kernel).
struct Xchg {
  XSlot slot[2][kMaxParts];
};

// Everything one partition's CTAs need, in device memory (read through a
// const __restrict__ pointer, so the level loops keep what they use in
// registers). Pointers to other partitions' buffers are peer pointers
// (unified addressing) or same-device pointers in loopback.
struct PartDev {
  Params<unsigned long long> td;  // column slice: rowptr = colptr (gid-indexed), col = local ids
  Params<unsigned long long> bu;  // row slice: rowptr = rowloc (local), col = gids
  uint32_t* bm[2];                // own full frontier bitmaps (words_total)
  uint32_t* q[2];                 // own frontier queues: P segments of seg_cap
  uint32_t* peer_bm[kMaxParts][2];
  uint32_t* peer_q[kMaxParts][2];
  Xchg* peer_x[kMaxParts];  // [rank] is this partition's own block
  Ctl* ctl;                 // partition barrier word + level counters
  pbfs_level* recs;
  const uint32_t* mask;     // lwords: isolated / padding bits of the local slice
  uint32_t* dist;           // nloc, gid order
  uint32_t* visited;        // lwords
  unsigned long long lo, nloc, lwords, words_total, seg_cap, col_maxdeg;
  uint32_t rank, rec_cap;
};

struct MultiParams {
  const PartDev* parts;  // all P partitions (this device's copy of the array)
  unsigned long long n;  // vertices of the graph (the 5 % rule's denominator)
  uint32_t P;            // partitions of the traversal
  uint32_t first;        // first partition of this launch
  uint32_t count;        // partitions in this launch
  uint32_t ctas_per_part;
  uint32_t source_gid;
  uint32_t run;          // traversal number: exchange sequence numbers never repeat
  int policy;
  double threshold;
};

// The replicated top-down frontier: P segments, segment r holding
// partition r's discoveries of the previous level (pre = prefix lengths).
struct SegQueue {
  const uint32_t* base;
  unsigned long long stride;
  const unsigned long long* pre;  // shared memory, nseg + 1 entries
  int nseg;
  __device__ __forceinline__ uint32_t operator[](unsigned long long i) const {
    int r = 0;
    while (r + 1 < nseg && i >= pre[r + 1]) ++r;
    return base[(unsigned long long)r * stride + (i - pre[r])];
  }
};

// Memory-model scope of the exchange: system scope when partitions sit on
// different GPUs (peer stores over NVLink), GPU scope when every partition
// shares one device (loopback), where the partition barrier's own
// release/acquire already covers the peer stores.
template <bool kSys>
__device__ __forceinline__ void st_relaxed_x(unsigned long long* p, unsigned long long v) {
  if constexpr (kSys) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  } else {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  }
}
template <bool kSys>
__device__ __forceinline__ unsigned long long ld_relaxed_x(const unsigned long long* p) {
  unsigned long long v;
  if constexpr (kSys) {
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  } else {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  }
  return v;
}
template <bool kSys>
__device__ __forceinline__ void fence_x() {
  if constexpr (kSys) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  } else {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
}

template <bool kSys>
__global__ void __launch_bounds__(kThreads, kMinBlocks) bfs_multi(MultiParams mp) {
  __shared__ __align__(16) uint32_t s_list[kWarps][kListCap];
  __shared__ uint32_t s_found[kWarps][kGroupWords];
  __shared__ unsigned long long s_snap[8];
  __shared__ unsigned long long s_pre[kMaxParts + 1];
  __shared__ unsigned long long s_x[kMaxParts][2];  // this exchange: discoveries, edges
  __shared__ uint32_t* s_dst[kMaxParts];             // push targets of the current phase
  const unsigned cpp = mp.ctas_per_part;
  const uint32_t me = mp.first + blockIdx.x / cpp;
  const VGrid vg{blockIdx.x % cpp, cpp};
  const PartDev* __restrict__ D = mp.parts + me;
  const uint32_t P = mp.P;
  const unsigned warp = threadIdx.x >> 5;
  const unsigned long long tid = (unsigned long long)vg.cta * kThreads + threadIdx.x;
  const unsigned long long nthreads = (unsigned long long)cpp * kThreads;
  Ctl* ctl = D->ctl;
  GridBarrier bar{ctl, s_snap, vg};
  const CntSnap snap{s_snap};
  const bool leader = vg.cta == cpp - 1 && threadIdx.x == 0;
  const bool recorder = leader && me == 0;
  const unsigned long long lo = D->lo, nloc = D->nloc, lwords = D->lwords;
  const unsigned long long lo_word = lo / 32;
  const uint32_t src = mp.source_gid;
  const bool owner = src >= lo && src < lo + nloc;

  // ---- init (Engine ctor + seed, kernels.cpp:72-102,144-163), per partition
  for (unsigned long long i = tid; i < nloc; i += nthreads) {
    D->dist[i] = (owner && i == src - lo) ? 0u : kUnreached;
  }
  for (unsigned long long w = tid; w < lwords; w += nthreads) {
    uint32_t m = D->mask[w];
    if (owner && w == (src - lo) / 32) m |= 1u << ((src - lo) & 31);
    D->visited[w] = m;
  }
  // Only bm[0] (the seed frontier) and q[0] (the seed queue) are written
  // here: a faster partition may already be storing level 0's output into
  // this partition's bm[1] / q[1] (every bottom-up level rewrites whole
  // words of its slice, so bm[1] needs no clearing).
  for (unsigned long long w = tid; w < D->words_total; w += nthreads) {
    D->bm[0][w] = w == src / 32 ? (1u << (src & 31)) : 0u;
  }
  if (leader) {
    D->q[0][0] = src;  // segment 0 holds the seed frontier
    for (int s = 0; s < 4; ++s) {
      LevelCnt z{};
      ctl->cnt[s] = z;
    }
    ctl->overflow = 0;
  }
  if (threadIdx.x == 0) {
    s_pre[0] = 0;
    for (uint32_t r = 1; r <= P; ++r) s_pre[r] = 1;  // [1, 0, 0, ...]
  }
  auto decide = [&](unsigned long long produced) -> bool {
    if (mp.policy == kPolicyTopDown) return true;
    return (double)produced < mp.threshold * (double)mp.n;
  };
  bool td = decide(1);
  int qcur = 0, fcur = 0;
  unsigned long long cur_distinct = 1, reached = 0, edges_total = 0;
  unsigned int bu_levels = 0;
  uint32_t xstep = 0;  // exchanges so far in this traversal
  unsigned long long t_start = recorder ? globaltimer() : 0;
  bar.sync();

  // One exchange: publish (a, b), wait for every partition's, leave the P
  // pairs in s_x. Callers have released their peer stores (release_cta) and
  // passed the partition barrier first. One fence per side: the writer
  // stores every value, fences, then every sequence number; a reader polls
  // the sequence numbers, fences, then reads the values.
  auto exchange = [&](unsigned long long a, unsigned long long b) {
    const unsigned long long seq = ((unsigned long long)mp.run << 32) | (xstep + 1);
    const int par = xstep & 1;
    if (vg.cta == 0 && threadIdx.x == 0) {
      for (uint32_t r = 0; r < P; ++r) {
        XSlot* sl = &D->peer_x[r]->slot[par][me];
        st_relaxed_x<kSys>(&sl->produced, a);
        st_relaxed_x<kSys>(&sl->edges, b);
      }
      fence_x<kSys>();
      for (uint32_t r = 0; r < P; ++r) st_relaxed_x<kSys>(&D->peer_x[r]->slot[par][me].seq, seq);
    }
    if (threadIdx.x == 0) {
      Xchg* x = D->peer_x[me];
      const unsigned long long t0 = globaltimer();
      for (uint32_t r = 0; r < P; ++r) {
        while (ld_relaxed_x<kSys>(&x->slot[par][r].seq) != seq) {
          // A partition that never arrives (a peer launch that failed to
          // start) must not wedge the device: abort the launch after 30 s.
          if (globaltimer() - t0 > 30000000000ull) __trap();
        }
      }
      fence_x<kSys>();
      for (uint32_t r = 0; r < P; ++r) {
        s_x[r][0] = ld_relaxed_x<kSys>(&x->slot[par][r].produced);
        s_x[r][1] = ld_relaxed_x<kSys>(&x->slot[par][r].edges);
      }
    }
    ++xstep;
    __syncthreads();
  };
  // Every CTA's stores to other GPUs' memory, made visible system-wide
  // before the partition barrier that precedes an exchange (on one GPU the
  // barrier's release/acquire at GPU scope covers them).
  auto release_cta = [&]() {
    if constexpr (kSys) {
      __syncthreads();
      if (threadIdx.x == 0) fence_x<true>();
    }
  };

  uint32_t depth = 0;
  for (;; ++depth) {
    LevelCnt* cnt = &ctl->cnt[depth & 3];
    if (leader) {
      LevelCnt z{};
      ctl->cnt[(depth + 2) & 3] = z;
    }
    WarpTally t;
    const int qn = qcur ^ 1;
    if (td) {
      // Push targets: this partition's segment of every partition's next queue.
      if (threadIdx.x < P) s_dst[threadIdx.x] = D->peer_q[threadIdx.x][qn] + (unsigned long long)me * D->seg_cap;
      __syncthreads();
      WarpPushT<true> wp{s_list[warp], 0, s_dst, (int)P, (uint32_t)lo};
      const SegQueue qv{D->q[qcur], D->seg_cap, s_pre, (int)P};
      const unsigned long long qlen = s_pre[P];
      td_phase_light<kClaimBitmap>(D->td, depth, qv, qlen, nullptr, wp, cnt, t, nullptr, nullptr, vg);
      if (D->col_maxdeg > D->td.heavy_deg) {
        bar.sync(cnt);
        const unsigned int items = (unsigned long long)snap.heavy_count() < D->td.heavy_cap
                                       ? snap.heavy_count()
                                       : (unsigned int)D->td.heavy_cap;
        if (items) td_phase_heavy<kClaimBitmap>(D->td, depth, items, nullptr, wp, cnt, t, nullptr, vg);
      }
      wp.flush(nullptr, &cnt->raw, D->seg_cap, &ctl->overflow);
    } else {
      // Targets: this partition's slice of every OTHER partition's next bitmap.
      if (threadIdx.x + 1 < P) {
        s_dst[threadIdx.x] = D->peer_bm[threadIdx.x < me ? threadIdx.x : threadIdx.x + 1][fcur ^ 1] + lo_word;
      }
      __syncthreads();
      bu_phase(D->bu, depth, D->bm[fcur], D->bm[fcur ^ 1] + lo_word, s_list[warp], s_found[warp], t,
               &cnt->bu_cursor, false, vg, NextPeers{s_dst, (int)P - 1});
    }
    warp_flush_tally(cnt, t, false);
    release_cta();
    bar.sync(cnt);
    exchange(snap.produced(), snap.edges());
    fcur ^= 1;

    // ---- single section (kernels.cpp:384-464), identical in every CTA ----
    unsigned long long produced = 0, edges = 0;
    for (uint32_t r = 0; r < P; ++r) {
      produced += s_x[r][0];
      edges += s_x[r][1];
    }
    if (recorder) {
      const unsigned long long now = globaltimer();
      if (depth < D->rec_cap) {
        pbfs_level rec;
        rec.depth = depth;
        rec.phase = td ? PBFS_TOP_DOWN : PBFS_BOTTOM_UP;
        rec.frontier_size = cur_distinct;
        rec.distinct_size = cur_distinct;
        rec.duplicate_count = 0;
        rec.edges_examined = edges;
        rec.flush_events = 0;
        rec.elapsed_ns = (long long)(now - t_start);
        D->recs[depth] = rec;
      }
      t_start = now;
    }
    reached += cur_distinct;
    edges_total += edges;
    bu_levels += td ? 0 : 1;
    if (produced == 0) break;
    const bool next_td = decide(produced);
    if (td && next_td) {
      // The pushed segments are the next frontier: lengths from the exchange.
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (uint32_t r = 0; r < P; ++r) {
          s_pre[r] = run;
          run += s_x[r][0];
        }
        s_pre[P] = run;
      }
      qcur ^= 1;
    } else if (!td && next_td) {
      // Entering top-down: every partition compacts the complete replicated
      // bitmap into segment 0 of its own queue (kernels.cpp:225-241).
      compact_bitmap(D->bm[fcur], D->q[qcur], (uint32_t)D->words_total, &cnt->conv_count, false,
                     nullptr, false, vg);
      bar.sync(cnt);
      if (threadIdx.x == 0) {
        s_pre[0] = 0;
        for (uint32_t r = 1; r <= P; ++r) s_pre[r] = snap.conv_count();
      }
    } else if (td && !next_td) {
      // Entering bottom-up: this partition's slice of the frontier bitmap
      // from its distances (front_from_dist), stored locally and into every
      // peer's bitmap, then one more exchange so every copy is complete.
      const uint32_t nd = depth + 1;
      for (unsigned long long w = tid; w < lwords; w += nthreads) {
        uint32_t bits = 0;
        const uint32_t reachw = __ldcg(&D->visited[w]) & ~__ldg(&D->mask[w]);
        if (reachw) {
          const uint4* d4 = reinterpret_cast<const uint4*>(D->dist + w * 32);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint4 a = __ldcs(d4 + k);
            bits |= (uint32_t)(a.x == nd) << (4 * k) | (uint32_t)(a.y == nd) << (4 * k + 1) |
                    (uint32_t)(a.z == nd) << (4 * k + 2) | (uint32_t)(a.w == nd) << (4 * k + 3);
          }
          bits &= reachw;
        }
        for (uint32_t r = 0; r < P; ++r) D->peer_bm[r][fcur][lo_word + w] = bits;
      }
      release_cta();
      bar.sync();
      exchange(0, 0);
    }
    // bottom-up -> bottom-up: the pushed slices already form the frontier.
    td = next_td;
    cur_distinct = produced;
  }
  if (recorder) {
    ctl->levels = depth + 1;
    ctl->bu_levels = bu_levels;
    ctl->reached = reached;
    ctl->edges = edges_total;
  }
}

// Hub items of the column slice when a small frontier splits hubs into
// 2^kSmallChunkLog2-edge items (td_phase_light), for hubs above heavy_deg.
__global__ void k_small_items(const unsigned long long* __restrict__ colptr, uint64_t npad,
                              uint32_t heavy_deg, unsigned long long* items) {
  unsigned long long c = 0;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < npad;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = colptr[u + 1] - colptr[u];
    if (d > heavy_deg) c += (d + (1ull << kSmallChunkLog2) - 1) >> kSmallChunkLog2;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(items, c);
}

__global__ void k_unrelabel_gather(const uint32_t* __restrict__ dist_pi, uint64_t n,
                                   const uint32_t* __restrict__ gid, uint32_t* dist) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    dist[v] = dist_pi[gid[v]];
  }
}

}  // namespace multi
}  // namespace pbfs

using namespace pbfs::multi;

struct pbfs_multi {
  std::mutex mu;
  uint64_t n = 0, m = 0;
  uint32_t P = 0;
  std::vector<int> part_dev;         // device of each partition
  std::vector<pbfs_part*> parts;
  std::vector<std::vector<void*>> allocs;  // per partition, freed on its device
  std::vector<uint32_t*> q[2];       // per partition
  std::vector<Xchg*> xchg;
  std::vector<uint32_t> gid_host;    // vertex -> gid
  uint64_t seg_cap = 0;
  // launch groups: one per distinct device
  struct Group {
    int device = 0;
    uint32_t first = 0, count = 0, ctas_per_part = 0;
    // visited | bm[0] | bm[1] of every partition of this device in ONE block,
    // under the launch's persisting-L2 window (the probe working set must not
    // be evicted by the multi-GB column stream, as in the single-GPU engine).
    uint32_t* bitmaps = nullptr;
    size_t bitmap_bytes = 0;
    size_t persist = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t start = nullptr, end = nullptr;
    PartDev* parts_dev = nullptr;  // this device's copy of the descriptor array
  };
  std::vector<Group> groups;
  cudaEvent_t all_done = nullptr;  // on group 0's device, after every group's end
  uint32_t* dist_pi = nullptr;     // group 0's device: npad
  uint32_t* dist_out = nullptr;    // group 0's device: n
  uint32_t* gid_dev0 = nullptr;    // group 0's device: n (partition 0's map)
  uint64_t npad = 0;
  uint32_t run = 0;
  bool launched = false;
  // System-scope exchange: partitions span several GPUs, or
  // PBFS_MULTI_SYS_SCOPE=1 (test hook: the multi-GPU memory-model path on
  // one GPU).
  bool sys = false;
  pbfs_config last_cfg{};
};

namespace {

pbfs_status cuda_fail_m(cudaError_t e, const char* what) {
  cudaGetLastError();
  return fail(PBFS_E_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}
#define MCUDA(call, what)                                  \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return cuda_fail_m(_e, what);   \
  } while (0)

void multi_release(pbfs_multi* m) {
  if (!m) return;
  for (auto& g : m->groups) {
    cudaSetDevice(g.device);
    if (g.parts_dev) cudaFree(g.parts_dev);
    if (g.bitmaps) cudaFree(g.bitmaps);
    if (g.start) cudaEventDestroy(g.start);
    if (g.end) cudaEventDestroy(g.end);
    if (g.stream) cudaStreamDestroy(g.stream);
  }
  if (!m->groups.empty()) {
    cudaSetDevice(m->groups[0].device);
    if (m->all_done) cudaEventDestroy(m->all_done);
    if (m->dist_pi) cudaFree(m->dist_pi);
    if (m->dist_out) cudaFree(m->dist_out);
    if (m->gid_dev0) cudaFree(m->gid_dev0);
  }
  for (uint32_t i = 0; i < m->parts.size(); ++i) {
    cudaSetDevice(m->part_dev[i]);
    for (void* p : m->allocs[i]) cudaFree(p);
    pbfs::part::release(m->parts[i]);
  }
  delete m;
}

template <typename T>
pbfs_status malloc_on(pbfs_multi* m, uint32_t part, T** p, size_t bytes) {
  void* q = nullptr;
  if (cudaMalloc(&q, bytes ? bytes : 16) != cudaSuccess) {
    cudaGetLastError();
    return fail(PBFS_E_CAPACITY, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  m->allocs[part].push_back(q);
  *p = static_cast<T*>(q);
  return PBFS_OK;
}

}  // namespace

extern "C" {

pbfs_status pbfs_multi_create(const pbfs_csr* csr, const int32_t* devices, uint32_t num_partitions,
                              pbfs_multi** out) {
  if (!csr || !devices || !out) return fail(PBFS_E_INPUT, "null argument");
  if (num_partitions < 1 || num_partitions > static_cast<uint32_t>(kMaxParts)) {
    return fail(PBFS_E_CONFIG, "partition count must be in [1, " + std::to_string(kMaxParts) + "]");
  }
  pbfs_status st = validate_csr_view(csr, resolve_threads(0));
  if (st != PBFS_OK) return st;
  if (!csr->symmetric) {
    return fail(PBFS_E_INPUT, "the vertex partition needs a symmetric graph (its column slice "
                              "is the transpose of the row slice)");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(PBFS_E_DEVICE, "no CUDA device available: the BFS kernels need a B200 "
                               "(there is no CPU fallback)");
  }
  for (uint32_t i = 0; i < num_partitions; ++i) {
    if (devices[i] < 0 || devices[i] >= ndev) return fail(PBFS_E_CONFIG, "device ordinal out of range");
  }
  int prev = 0;
  cudaGetDevice(&prev);
  auto* m = new (std::nothrow) pbfs_multi;
  if (!m) return fail(PBFS_E_CAPACITY, "host allocation failed");
  auto bail = [&](pbfs_status s2) {
    multi_release(m);
    cudaSetDevice(prev);
    return s2;
  };
  m->n = csr->vertex_count;
  m->m = csr->edge_count;
  m->P = num_partitions;
  m->part_dev.assign(devices, devices + num_partitions);
  m->allocs.resize(num_partitions);
  m->parts.assign(num_partitions, nullptr);
  m->q[0].assign(num_partitions, nullptr);
  m->q[1].assign(num_partitions, nullptr);
  m->xchg.assign(num_partitions, nullptr);
  // Peer access between every pair of distinct devices (NVLink / NVSwitch).
  for (uint32_t a = 0; a < num_partitions; ++a) {
    for (uint32_t b = 0; b < num_partitions; ++b) {
      const int da = devices[a], db = devices[b];
      if (da == db) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, da, db);
      if (!can) return bail(fail(PBFS_E_DEVICE, "device " + std::to_string(da) +
                                                    " cannot access device " + std::to_string(db) +
                                                    " (no peer path)"));
      cudaSetDevice(da);
      cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return bail(cuda_fail_m(e, "peer access"));
      cudaGetLastError();
    }
  }
  // Partitions: the full CSR visits each device once; that device's
  // partitions are built from it on the device (pbfs::part::create), then
  // the copy is freed.
  const uint64_t n = m->n, e = m->m;
  for (uint32_t i = 0; i < num_partitions;) {
    const int dev = devices[i];
    uint32_t j = i;
    while (j < num_partitions && devices[j] == dev) ++j;
    MCUDA(cudaSetDevice(dev), "cudaSetDevice");
    void* rowptr = nullptr;
    uint32_t* col = nullptr;
    if (cudaMalloc(&rowptr, (n + 1) * 8) != cudaSuccess || cudaMalloc(&col, e * 4 + 64) != cudaSuccess) {
      cudaGetLastError();
      if (rowptr) cudaFree(rowptr);
      return bail(fail(PBFS_E_CAPACITY, "device allocation for the partition build failed"));
    }
    cudaError_t ce = cudaSuccess;
    if (csr->offset_bytes == 8) {
      ce = cudaMemcpy(rowptr, csr->row_offsets, (n + 1) * 8, cudaMemcpyHostToDevice);
    } else {
      std::vector<uint64_t> w(n + 1);
      for (uint64_t v = 0; v <= n; ++v) w[v] = csr_offset(csr, v);
      ce = cudaMemcpy(rowptr, w.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    }
    if (ce == cudaSuccess && e) ce = cudaMemcpy(col, csr->column_indices, e * 4, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
      cudaFree(rowptr);
      cudaFree(col);
      return bail(cuda_fail_m(ce, "upload for the partition build"));
    }
    for (uint32_t k = i; k < j && st == PBFS_OK; ++k) {
      pbfs_part_options opt{};
      opt.rank = k;
      opt.world = num_partitions;
      opt.relabel = 1;
      st = pbfs::part::create(n, true, dev, rowptr, col, 8, &opt, &m->parts[k]);
    }
    cudaFree(rowptr);
    cudaFree(col);
    if (st != PBFS_OK) return bail(st);
    i = j;
  }
  pbfs_part* p0 = m->parts[0];
  m->npad = p0->npad;
  m->seg_cap = p0->nloc + 1;
  // Per partition: the P-segment queues and the exchange block.
  for (uint32_t i = 0; i < num_partitions; ++i) {
    MCUDA(cudaSetDevice(devices[i]), "cudaSetDevice");
    const uint64_t qbytes = (static_cast<uint64_t>(num_partitions) * m->seg_cap + 16) * 4;
    if ((st = malloc_on(m, i, &m->q[0][i], qbytes)) != PBFS_OK) return bail(st);
    if ((st = malloc_on(m, i, &m->q[1][i], qbytes)) != PBFS_OK) return bail(st);
    if ((st = malloc_on(m, i, &m->xchg[i], sizeof(Xchg))) != PBFS_OK) return bail(st);
    MCUDA(cudaMemset(m->xchg[i], 0, sizeof(Xchg)), "memset exchange block");
  }
  // Launch groups: one per distinct device, partitions of a device contiguous.
  for (uint32_t i = 0; i < num_partitions;) {
    uint32_t j = i;
    while (j < num_partitions && devices[j] == devices[i]) ++j;
    for (const auto& g : m->groups) {
      if (g.device == devices[i]) {
        return bail(fail(PBFS_E_CONFIG, "partitions placed on one device must be listed "
                                        "contiguously"));
      }
    }
    pbfs_multi::Group grp;
    grp.device = devices[i];
    grp.first = i;
    grp.count = j - i;
    m->groups.push_back(grp);
    i = j;
  }
  // Descriptors (identical bytes on every device: unified addressing).
  // Per device: one block holding every local partition's visited slice,
  // then their full bitmaps. The launch's persisting-L2 window covers the
  // whole block when the device holds one partition (its probe working set,
  // as in the single-GPU engine); with several partitions on one device
  // (loopback) only the visited slices -- the replicated full bitmaps would
  // crowd the set-aside (PBFS_MULTI_WINDOW=all|visited|none overrides).
  std::vector<uint32_t*> vis(num_partitions), bm0(num_partitions), bm1(num_partitions);
  const char* wenv = std::getenv("PBFS_MULTI_WINDOW");
  for (auto& grp : m->groups) {
    MCUDA(cudaSetDevice(grp.device), "cudaSetDevice");
    size_t vwords = 0, words = 0;
    for (uint32_t i = grp.first; i < grp.first + grp.count; ++i) {
      vwords += m->parts[i]->lwords;
      words += m->parts[i]->lwords + 2 * m->parts[i]->words_total;
    }
    MCUDA(cudaMalloc(&grp.bitmaps, words * 4), "bitmap block");
    uint32_t* at = grp.bitmaps;
    for (uint32_t i = grp.first; i < grp.first + grp.count; ++i) {
      vis[i] = at;
      at += m->parts[i]->lwords;
    }
    for (uint32_t i = grp.first; i < grp.first + grp.count; ++i) {
      bm0[i] = at;
      at += m->parts[i]->words_total;
      bm1[i] = at;
      at += m->parts[i]->words_total;
    }
    bool all = grp.count == 1;
    if (wenv && std::strcmp(wenv, "all") == 0) all = true;
    if (wenv && std::strcmp(wenv, "visited") == 0) all = false;
    grp.bitmap_bytes = (all ? words : vwords) * 4;
    cudaDeviceProp prop;
    MCUDA(cudaGetDeviceProperties(&prop, grp.device), "props");
    const bool none = wenv && std::strcmp(wenv, "none") == 0;
    if (!none && prop.persistingL2CacheMaxSize > 0 && prop.accessPolicyMaxWindowSize > 0) {
      grp.bitmap_bytes = std::min<size_t>(grp.bitmap_bytes, prop.accessPolicyMaxWindowSize);
      const size_t want = std::min<size_t>(grp.bitmap_bytes, prop.persistingL2CacheMaxSize);
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (cur >= want || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
        grp.persist = std::max(cur, want);
      }
      cudaGetLastError();
    }
  }
  // Top-down hub items: the partition's own capacity, or the small-frontier
  // split's (2^kSmallChunkLog2-edge items) if larger; graphs of >= 2^30
  // local arcs take the single-GPU engine's big split.
  std::vector<HeavyItem*> heavy(num_partitions);
  std::vector<unsigned long long> heavy_cap(num_partitions);
  for (uint32_t i = 0; i < num_partitions; ++i) {
    pbfs_part* g = m->parts[i];
    MCUDA(cudaSetDevice(g->device), "cudaSetDevice");
    unsigned long long* cnt = nullptr;
    if ((st = malloc_on(m, i, &cnt, 8)) != PBFS_OK) return bail(st);
    MCUDA(cudaMemset(cnt, 0, 8), "memset");
    k_small_items<<<1184, 256>>>(g->colptr, g->npad, kHeavyDeg, cnt);
    unsigned long long small = 0;
    MCUDA(cudaMemcpy(&small, cnt, 8, cudaMemcpyDeviceToHost), "small items");
    heavy_cap[i] = std::max<unsigned long long>(g->heavy_cap, small);
    if ((st = malloc_on(m, i, &heavy[i], std::max<unsigned long long>(heavy_cap[i], 1) *
                                              sizeof(HeavyItem))) != PBFS_OK) {
      return bail(st);
    }
  }
  std::vector<PartDev> desc(num_partitions);
  for (uint32_t i = 0; i < num_partitions; ++i) {
    pbfs_part* g = m->parts[i];
    PartDev& d = desc[i];
    std::memset(&d, 0, sizeof(d));
    d.td = pbfs::part::td_params(g);
    d.bu = pbfs::part::bu_params(g);
    d.td.qcap = m->seg_cap;
    d.td.visited = d.bu.visited = vis[i];
    d.td.heavy = heavy[i];
    d.td.heavy_cap = heavy_cap[i];
    {
      const char* sc = std::getenv("PBFS_MULTI_SMALL_CHUNKS");  // A/B knob
      d.td.small_chunks = sc && sc[0] == '0' ? 0 : 1;
    }
    if (g->m_loc >= kBigArcs) {
      d.td.heavy_deg = kHeavyDegBig;
      d.td.chunk_log2 = __builtin_ctz(kChunkBig);
    }
    d.bm[0] = bm0[i];
    d.bm[1] = bm1[i];
    d.q[0] = m->q[0][i];
    d.q[1] = m->q[1][i];
    for (uint32_t r = 0; r < num_partitions; ++r) {
      d.peer_bm[r][0] = bm0[r];
      d.peer_bm[r][1] = bm1[r];
      d.peer_q[r][0] = m->q[0][r];
      d.peer_q[r][1] = m->q[1][r];
      d.peer_x[r] = m->xchg[r];
    }
    d.ctl = g->ctl;
    d.recs = g->recs;
    d.rec_cap = pbfs::part::kPartRecCap;
    d.mask = g->mask;
    d.dist = g->dist;
    d.visited = vis[i];
    d.lo = g->lo;
    d.nloc = g->nloc;
    d.lwords = g->lwords;
    d.words_total = g->words_total;
    d.seg_cap = m->seg_cap;
    d.col_maxdeg = g->col_maxdeg;
    d.rank = i;
  }
  {
    const char* fs = std::getenv("PBFS_MULTI_SYS_SCOPE");
    m->sys = m->groups.size() > 1 || (fs && fs[0] == '1');
  }
  for (auto& grp : m->groups) {
    MCUDA(cudaSetDevice(grp.device), "cudaSetDevice");
    MCUDA(cudaStreamCreateWithFlags(&grp.stream, cudaStreamNonBlocking), "stream");
    MCUDA(cudaEventCreate(&grp.start), "event");
    MCUDA(cudaEventCreate(&grp.end), "event");
    MCUDA(cudaMalloc(&grp.parts_dev, sizeof(PartDev) * num_partitions), "descriptors");
    MCUDA(cudaMemcpy(grp.parts_dev, desc.data(), sizeof(PartDev) * num_partitions,
                     cudaMemcpyHostToDevice), "descriptors");
    cudaDeviceProp prop;
    MCUDA(cudaGetDeviceProperties(&prop, grp.device), "props");
    const bool sys = m->sys;
    const void* fn = sys ? reinterpret_cast<const void*>(&bfs_multi<true>)
                         : reinterpret_cast<const void*>(&bfs_multi<false>);
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 25);
    int occ = 0;
    MCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, 0), "occupancy");
    if (occ < 1) return bail(fail(PBFS_E_DEVICE, "multi-partition kernel cannot be resident"));
    const uint32_t grid = static_cast<uint32_t>(prop.multiProcessorCount * occ);
    grp.ctas_per_part = grid / grp.count;
    if (grp.ctas_per_part < 1) return bail(fail(PBFS_E_CONFIG, "too many partitions per device"));
  }
  MCUDA(cudaSetDevice(m->groups[0].device), "cudaSetDevice");
  MCUDA(cudaEventCreate(&m->all_done), "event");
  MCUDA(cudaMalloc(&m->dist_pi, m->npad * 4 + 16), "gather buffer");
  MCUDA(cudaMalloc(&m->dist_out, n * 4 + 16), "distance buffer");
  MCUDA(cudaMalloc(&m->gid_dev0, n * 4 + 16), "gid map");
  m->gid_host.resize(n);
  MCUDA(cudaSetDevice(devices[0]), "cudaSetDevice");
  MCUDA(cudaMemcpy(m->gid_host.data(), p0->gid, n * 4, cudaMemcpyDeviceToHost), "gid map");
  MCUDA(cudaSetDevice(m->groups[0].device), "cudaSetDevice");
  MCUDA(cudaMemcpy(m->gid_dev0, m->gid_host.data(), n * 4, cudaMemcpyHostToDevice), "gid map");
  cudaSetDevice(prev);
  *out = m;
  return PBFS_OK;
}

pbfs_status pbfs_multi_destroy(pbfs_multi* m) {
  multi_release(m);
  return PBFS_OK;
}

pbfs_status pbfs_multi_get_info(const pbfs_multi* m, pbfs_multi_info* info) {
  if (!m || !info) return fail(PBFS_E_INPUT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->vertex_count = m->n;
  info->edge_count = m->m;
  info->partitions = m->P;
  info->devices = static_cast<uint32_t>(m->groups.size());
  info->padded_count = m->npad;
  info->ctas_per_partition = m->groups.empty() ? 0 : m->groups[0].ctas_per_part;
  info->relabel_hashed = m->parts[0]->rl.hashed;
  for (uint32_t i = 0; i < m->P && i < 8; ++i) info->local_arcs[i] = m->parts[i]->m_loc;
  return PBFS_OK;
}

pbfs_status pbfs_multi_bfs_async(pbfs_multi* m, uint32_t source, const pbfs_config* cfg) {
  if (!m || !cfg) return fail(PBFS_E_INPUT, "null argument");
  std::lock_guard<std::mutex> lock(m->mu);
  pbfs_status st = pbfs_config_validate(cfg);
  if (st != PBFS_OK) return st;
  if (cfg->variant != PBFS_HYBRID && cfg->variant != PBFS_VISITED_INLINE) {
    return fail(PBFS_E_CONFIG, "the multi-partition engine runs the hybrid (5 % rule) traversal "
                               "(or its top-down-only dispatch)");
  }
  if (source >= m->n) {
    return fail(PBFS_E_INPUT, "source vertex " + std::to_string(source) +
                                  " is out of range for a graph with " + std::to_string(m->n) +
                                  " vertices");
  }
  int prev = 0;
  cudaGetDevice(&prev);
  ++m->run;
  MultiParams mp{};
  mp.n = m->n;
  mp.P = m->P;
  mp.source_gid = m->gid_host[source];
  mp.run = m->run;
  mp.policy = cfg->force_top_down_only ? kPolicyTopDown : kPolicyFraction;
  mp.threshold = cfg->hybrid_threshold_fraction;
  // Every group waits for the previous traversal's completion on group 0
  // (its buffers are reused) before it starts.
  for (size_t gi = 0; gi < m->groups.size(); ++gi) {
    auto& grp = m->groups[gi];
    MCUDA(cudaSetDevice(grp.device), "cudaSetDevice");
    if (m->launched) MCUDA(cudaStreamWaitEvent(grp.stream, m->all_done, 0), "order");
    MCUDA(cudaEventRecord(grp.start, grp.stream), "event");
  }
  for (auto& grp : m->groups) {
    MCUDA(cudaSetDevice(grp.device), "cudaSetDevice");
    mp.parts = grp.parts_dev;
    mp.first = grp.first;
    mp.count = grp.count;
    mp.ctas_per_part = grp.ctas_per_part;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grp.count * grp.ctas_per_part);
    lc.blockDim = dim3(kThreads);
    lc.stream = grp.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    int nattr = 1;
    if (grp.persist) {
      attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
      attr[1].val.accessPolicyWindow.base_ptr = grp.bitmaps;
      attr[1].val.accessPolicyWindow.num_bytes = grp.bitmap_bytes;
      attr[1].val.accessPolicyWindow.hitRatio =
          std::min(1.0f, static_cast<float>(grp.persist) / static_cast<float>(grp.bitmap_bytes));
      attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      nattr = 2;
    }
    lc.attrs = attr;
    lc.numAttrs = nattr;
    // System-scope exchange only when the partitions span several GPUs.
    cudaError_t e = m->sys ? cudaLaunchKernelEx(&lc, bfs_multi<true>, mp)
                           : cudaLaunchKernelEx(&lc, bfs_multi<false>, mp);
    if (e != cudaSuccess) {
      cudaSetDevice(prev);
      return cuda_fail_m(e, "multi-partition traversal launch");
    }
    MCUDA(cudaEventRecord(grp.end, grp.stream), "event");
  }
  auto& g0 = m->groups[0];
  MCUDA(cudaSetDevice(g0.device), "cudaSetDevice");
  for (size_t gi = 1; gi < m->groups.size(); ++gi) {
    MCUDA(cudaStreamWaitEvent(g0.stream, m->groups[gi].end, 0), "join");
  }
  MCUDA(cudaEventRecord(m->all_done, g0.stream), "event");
  m->launched = true;
  m->last_cfg = *cfg;
  cudaSetDevice(prev);
  return PBFS_OK;
}

pbfs_status pbfs_multi_sync(pbfs_multi* m, float* device_ms) {
  if (!m) return fail(PBFS_E_INPUT, "null argument");
  std::lock_guard<std::mutex> lock(m->mu);
  if (!m->launched) return PBFS_OK;
  auto& g0 = m->groups[0];
  MCUDA(cudaSetDevice(g0.device), "cudaSetDevice");
  MCUDA(cudaEventSynchronize(m->all_done), "multi-partition traversal");
  for (uint32_t i = 0; i < m->P; ++i) {
    MCUDA(cudaSetDevice(m->part_dev[i]), "cudaSetDevice");
    unsigned int overflow = 0;
    MCUDA(cudaMemcpy(&overflow, &m->parts[i]->ctl->overflow, 4, cudaMemcpyDeviceToHost), "read");
    if (overflow) return fail(PBFS_E_CAPACITY, "partition frontier overflow");
  }
  if (device_ms) {
    MCUDA(cudaSetDevice(g0.device), "cudaSetDevice");
    MCUDA(cudaEventElapsedTime(device_ms, g0.start, m->all_done), "elapsed");
  }
  return PBFS_OK;
}

pbfs_status pbfs_multi_stream(pbfs_multi* m, void** stream) {
  if (!m || !stream) return fail(PBFS_E_INPUT, "null argument");
  *stream = m->groups[0].stream;
  return PBFS_OK;
}

pbfs_status pbfs_multi_bfs(pbfs_multi* m, uint32_t source, const pbfs_config* cfg,
                           uint32_t* dist_host, pbfs_level* levels, uint32_t levels_cap,
                           pbfs_run_info* info) {
  pbfs_status st = pbfs_multi_bfs_async(m, source, cfg);
  if (st != PBFS_OK) return st;
  float ms = 0.f;
  if ((st = pbfs_multi_sync(m, &ms)) != PBFS_OK) return st;
  std::lock_guard<std::mutex> lock(m->mu);
  int prev = 0;
  cudaGetDevice(&prev);
  auto& g0 = m->groups[0];
  if (dist_host) {
    // Gather every partition's gid-order slice on group 0's device, map back
    // to vertex ids there, one D2H copy.
    MCUDA(cudaSetDevice(g0.device), "cudaSetDevice");
    for (uint32_t i = 0; i < m->P; ++i) {
      pbfs_part* p = m->parts[i];
      MCUDA(cudaMemcpyPeerAsync(m->dist_pi + p->lo, g0.device, p->dist, p->device, p->nloc * 4,
                                g0.stream), "gather distances");
    }
    MCUDA(cudaSetDevice(g0.device), "cudaSetDevice");
    k_unrelabel_gather<<<1184, 256, 0, g0.stream>>>(m->dist_pi, m->n, m->gid_dev0, m->dist_out);
    MCUDA(cudaGetLastError(), "unrelabel");
    MCUDA(cudaMemcpyAsync(dist_host, m->dist_out, m->n * 4, cudaMemcpyDeviceToHost, g0.stream),
          "read distances");
    MCUDA(cudaStreamSynchronize(g0.stream), "gather");
  }
  pbfs_part* p0 = m->parts[0];
  MCUDA(cudaSetDevice(p0->device), "cudaSetDevice");
  Ctl ctl;
  MCUDA(cudaMemcpy(&ctl, p0->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost), "read control");
  if (levels && levels_cap) {
    const uint32_t k = std::min<uint32_t>(std::min<uint32_t>(ctl.levels, pbfs::part::kPartRecCap),
                                          levels_cap);
    MCUDA(cudaMemcpy(levels, p0->recs, k * sizeof(pbfs_level), cudaMemcpyDeviceToHost), "read trace");
  }
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->levels = ctl.levels;
    info->bottom_up_levels = ctl.bu_levels;
    info->reached = ctl.reached;
    info->edges_examined = ctl.edges;
    info->device_ms = ms;
  }
  cudaSetDevice(prev);
  if (levels && ctl.levels > pbfs::part::kPartRecCap) {
    return fail(PBFS_E_CAPACITY, "traversal depth exceeds the partitioned trace capacity");
  }
  return PBFS_OK;
}

pbfs_status pbfs_multi_join(pbfs_multi* m, void* stream) {
  if (!m || !stream) return fail(PBFS_E_INPUT, "null argument");
  std::lock_guard<std::mutex> lock(m->mu);
  if (!m->launched) return PBFS_OK;
  MCUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), m->all_done, 0), "join");
  return PBFS_OK;
}

pbfs_status pbfs_multi_trace(pbfs_multi* m, pbfs_level* levels, uint32_t levels_cap,
                             uint32_t* count) {
  if (!m || !count || (levels_cap && !levels)) return fail(PBFS_E_INPUT, "null argument");
  pbfs_status st = pbfs_multi_sync(m, nullptr);
  if (st != PBFS_OK) return st;
  std::lock_guard<std::mutex> lock(m->mu);
  int prev = 0;
  cudaGetDevice(&prev);
  pbfs_part* p0 = m->parts[0];
  MCUDA(cudaSetDevice(p0->device), "cudaSetDevice");
  unsigned int nlev = 0;
  MCUDA(cudaMemcpy(&nlev, &p0->ctl->levels, sizeof(nlev), cudaMemcpyDeviceToHost), "read control");
  const uint32_t k = std::min<uint32_t>(std::min<uint32_t>(nlev, pbfs::part::kPartRecCap), levels_cap);
  if (k) MCUDA(cudaMemcpy(levels, p0->recs, k * sizeof(pbfs_level), cudaMemcpyDeviceToHost), "read trace");
  *count = k;
  cudaSetDevice(prev);
  if (nlev > pbfs::part::kPartRecCap) {
    return fail(PBFS_E_CAPACITY, "the last traversal was deeper than the partitioned trace buffer");
  }
  return PBFS_OK;
}

pbfs_status pbfs_multi_component(pbfs_multi* m, uint64_t* n_reached, uint64_t* arcs_reached) {
  if (!m || !n_reached || !arcs_reached) return fail(PBFS_E_INPUT, "null argument");
  pbfs_status st = pbfs_multi_sync(m, nullptr);
  if (st != PBFS_OK) return st;
  uint64_t nr = 0, ar = 0;
  for (uint32_t i = 0; i < m->P; ++i) {
    uint64_t a = 0, b = 0;
    if ((st = pbfs_part_component(m->parts[i], &a, &b)) != PBFS_OK) return st;
    nr += a;
    ar += b;
  }
  *n_reached = nr;
  *arcs_reached = ar;
  return PBFS_OK;
}

}  // extern "C"

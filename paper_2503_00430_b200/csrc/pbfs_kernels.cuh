// Device side of the B200-native level-synchronous BFS (arXiv 2503.00430).
//
// ONE persistent cooperative kernel runs a whole traversal: every CTA walks
// the same level loop and takes every control decision redundantly from
// counters it reads right after a grid barrier, so the host is not involved
// between levels (the reference needs a std::barrier round and a serial
// single-worker section per level, kernels.cpp:165-173,384-464). Per level:
//
//   top-down  (kernels.cpp:262-338): warps take frontier slices of 32
//     vertices (fewer on small frontiers; static first slice, atomic cursor
//     only for large frontiers); vertices of degree <= kHeavyDeg are expanded
//     warp-cooperatively (shuffle scan of degrees, PBFS_SLOTS edge slots per
//     lane, owner found by a shuffle binary search); hubs are split into
//     kChunk-edge items reserved with one atomicAdd per warp and expanded by
//     the whole grid after a barrier, 32 consecutive sorted neighbours per warp
//     load. Every batch issues all its col loads, then all probes, then all
//     claim atomics (predicated, no branches) before consuming any result.
//     Claims:
//       kClaimCas    atomicCAS on dist            (BFS-Conventional)
//       kClaimPlain  plain same-value dist stores + idempotent red.or into a
//                    next-frontier bitmap         (BFS-NonAtomic, duplicates)
//       kClaimBitmap visited-word probe through L1 (a set bit is final), a
//                    clear bit straight to atom.or, plain dist store
//                    (BFS-Hybrid / VisitedBitmap; the partitioned engine also
//                    red.ors winners into the next-frontier bitmap it ships)
//     Winners go to a per-warp shared-memory buffer flushed with one
//     atomicAdd per <= kPushBuf entries (the GPU form of LocalFrontier +
//     reserve_and_flush, frontier.hpp:58-98). Hub-free graphs run top-down
//     only take the latency-mode path (td_phase_latency).
//   bottom-up (kernels.cpp:340-382): warps own 32-word (1024-vertex) groups
//     of the visited bitmap and list the unvisited ids in shared memory;
//     each lane probes its vertex's first neighbour (dense first_nbr array,
//     coalesced) against the frontier bitmap, and the misses scan on in
//     aligned 8-entry windows with lane refill until the first hit (early
//     exit). Owner-exclusive: next/visited words are plain stores.
//   control (kernels.cpp:384-464,487-513): distinct size read from the level
//     counter; `top_down = (double)distinct < thr * (double)n` evaluated in
//     IEEE double exactly like the reference; bottom-up -> top-down compacts
//     the bitmap into a queue, top-down -> bottom-up rebuilds the frontier
//     bitmap from dist (front_from_dist).
#pragma once

#include <cooperative_groups.h>
#include <cstddef>
#include <cstdint>

#include "pbfs.h"

namespace pbfs {
namespace dev {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef PBFS_MIN_BLOCKS
#define PBFS_MIN_BLOCKS 3
#endif
#ifndef PBFS_SLOTS
#define PBFS_SLOTS 8  // edge slots per lane in the top-down batches
#endif
#ifndef PBFS_HEAVY_DEG
#define PBFS_HEAVY_DEG 128
#endif
#ifndef PBFS_PROBE
// Visited-bit probe of the bitmap claim: 0 = L1 probe, L2 re-probe of clear
// bits, then the claim atomic; 1 = L2 probe only; 2 = L1 probe straight to
// the atomic; 3 = the atomic alone (A/B knob). Measured on RMAT-26 (GTEPS,
// profiles/r01_ab.txt): 0: 367, 1: 398, 2: 411, 3: 167 -- a set bit seen in
// L1 is final, a clear one is settled by the atomic's returned word, and a
// separate L2 re-probe costs more round trips than the atomics it saves.
#define PBFS_PROBE 2
#endif
#ifndef PBFS_PRED_TD
#define PBFS_PRED_TD 1  // predicated-off probes for dead top-down slots (A/B knob)
#endif
// dist probe of the CAS / plain-store top-down variants: 0 = L2 (ld.cg) for
// every slot, 1 = through L1 (ld.ca; a set distance is final, a stale
// kUnreached is settled by the CAS / is a benign same-value store), dead
// slots predicated off; 2 = ld.cg, dead slots predicated off (A/B knobs).
// RMAT-26 / ER-24 GTEPS (profiles/r02/ab.txt): CAS 0: 85.5 / 84.3,
// 1: 90.7 / 83.1, 2: 91.5 / 86.4; plain 0: 91.3 / 88.4, 1: 105.1 / 89.4,
// 2: 96.5 / 91.1.
#ifndef PBFS_HOT_MODE
#define PBFS_HOT_MODE 0  // visited-probe L1 policy by word index (ld_hot_if; 0 = plain ld.ca)
#endif
#ifndef PBFS_HOT_WORDS
#define PBFS_HOT_WORDS 16384
#endif
#ifndef PBFS_CAS_PROBE
#define PBFS_CAS_PROBE 2
#endif
#ifndef PBFS_PLAIN_PROBE
#define PBFS_PLAIN_PROBE 1
#endif
#ifndef PBFS_TIMELINE
#define PBFS_TIMELINE 0  // diagnostic per-level timeline in LevelRecord::flush_events
#endif
#ifndef PBFS_CHUNK
#define PBFS_CHUNK 512
#endif
#ifndef PBFS_LAT_SPREAD
#define PBFS_LAT_SPREAD 1  // latency mode: adaptive slice width, slices dealt over CTAs (A/B knob)
#endif
constexpr int kMinBlocks = PBFS_MIN_BLOCKS;  // resident CTAs per SM the register budget targets
// Hub split for graphs below kBigArcs directed arcs; larger graphs take
// kHeavyDegBig / kChunkBig (their levels are long enough that fewer, larger
// items beat finer balance). Per graph in Params::heavy_deg / chunk_log2.
constexpr uint32_t kHeavyDeg = PBFS_HEAVY_DEG;  // degree above which a vertex is split
constexpr uint32_t kChunk = PBFS_CHUNK;  // edges per heavy work item (power of two)
constexpr uint32_t kHeavyDegBig = 2 * PBFS_HEAVY_DEG;
constexpr uint32_t kChunkBig = 2 * PBFS_CHUNK;
constexpr unsigned long long kBigArcs = 1ull << 30;
// Frontiers of at most kSmallFrontier vertices split hubs into 64-edge items:
// a level with a handful of hubs otherwise keeps only a few hundred warps busy.
#ifndef PBFS_SMALL_Q
#define PBFS_SMALL_Q 4096
#endif
#ifndef PBFS_SMALL_CHUNK_LOG2
#define PBFS_SMALL_CHUNK_LOG2 8
#endif
constexpr unsigned long long kSmallFrontier = PBFS_SMALL_Q;
// Reduction claim (bfs_persistent): top-down levels from this many frontier
// vertices claim with no-return reds (per-graph override PBFS_RED_MINQ, 0 = off).
#ifndef PBFS_RED_MINQ
#define PBFS_RED_MINQ 65536
#endif
constexpr uint32_t kRedMinQ = PBFS_RED_MINQ;
// Test hooks: run the size-gated paths on small graphs (parity coverage).
constexpr uint32_t kForceSparseBu = 1;     // sparse bottom-up tasks at every level
constexpr uint32_t kForceWideCompact = 2;  // 8-words-per-lane compaction
constexpr uint32_t kForceBigSplit = 4;     // the >= 2^30-arc hub split
constexpr uint32_t kForcePack = 8;         // pbfs_bfs_batch's narrow transfers at any size
constexpr uint32_t kSmallChunkLog2 = PBFS_SMALL_CHUNK_LOG2;
// Per-warp shared-memory buffers: discovery buffer (top-down) / unvisited-id
// list (bottom-up), same storage. Their size sets the CTA's shared memory and
// with it the L1 left for the probes (PBFS_LIST_CAP A/B knob).
#ifndef PBFS_LIST_CAP
#define PBFS_LIST_CAP 512
#endif
constexpr int kPushBuf = PBFS_LIST_CAP;  // per-warp discovery buffer (entries)
constexpr int kGroupWords = 32;      // bitmap words per warp group (one per lane)
constexpr int kListCap = PBFS_LIST_CAP;  // bottom-up: unvisited ids listed per round
static_assert(kPushBuf >= 32 * PBFS_SLOTS, "a top-down batch must fit the discovery buffer");
#ifndef PBFS_BU_SLOTS
#define PBFS_BU_SLOTS 4
#endif
#ifndef PBFS_BU_WIN
#define PBFS_BU_WIN 8
#endif
constexpr int kBuWin = PBFS_BU_WIN;        // bottom-up scan window (4, 8 or 16 entries)
static_assert(kBuWin == 4 || kBuWin == 8 || kBuWin == 16, "PBFS_BU_WIN must be 4, 8 or 16");
constexpr int kBuSlots = PBFS_BU_SLOTS;    // unvisited vertices per lane in flight
// 32-word groups per bottom-up task: 1 (finest balance), or kBuSparseGroups
// on a sparse level (few unvisited vertices left), where a task is mostly
// settled words and the round trips, not the scans, are the cost.
constexpr int kBuSparseGroups = 8;
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
  unsigned int bu_cursor;       // bottom-up task grab (after the static first)
  unsigned int pad[5];
};

static_assert(offsetof(LevelCnt, degree) == 24 && offsetof(LevelCnt, heavy_count) == 44 &&
                  offsetof(LevelCnt, conv_count) == 52,
              "CntSnap offsets");

// Views into a GridBarrier snapshot of a LevelCnt's first 64 bytes.
struct CntSnap {
  const unsigned long long* w;
  __device__ __forceinline__ unsigned long long produced() const { return w[0]; }
  __device__ __forceinline__ unsigned long long raw() const { return w[1]; }
  __device__ __forceinline__ unsigned long long edges() const { return w[2]; }
  __device__ __forceinline__ unsigned long long degree() const { return w[3]; }
  __device__ __forceinline__ unsigned int heavy_count() const { return (unsigned int)(w[5] >> 32); }
  __device__ __forceinline__ unsigned int conv_count() const { return (unsigned int)(w[6] >> 32); }
};

struct alignas(128) Ctl {
  unsigned int bar_word;  // grid barrier: bit 31 flips once per completed barrier
  unsigned int pad0[31];
  LevelCnt cnt[4];
  // Latency mode's multi-level rounds (latency_round): round r counts in
  // row r & 3 (indices kLk*); a row is re-zeroed two rounds ahead.
  alignas(128) unsigned long long latk[4][32];
  unsigned int overflow;  // PBFS_E_CAPACITY raised on device
  unsigned int levels;
  unsigned int bu_levels;
  unsigned int obs_count;  // observer log: entries appended by bottom-up levels' compaction
  unsigned long long reached;
  unsigned long long violations;
  unsigned long long edges;
};

// Bits per vertex of the packed host transfer for a traversal of `levels`
// levels (distances 0 .. levels-1, plus the all-ones unreached code): 4-bit
// codes when every level fits a nibble (RMAT: 7-9 levels), then 1 or 2 bytes;
// 32 = no pack. pack_width is the same in whole bytes, rounded up (what
// pbfs_run_info::transfer_width reports).
__host__ __device__ __forceinline__ uint32_t pack_bits(uint32_t levels, uint32_t min_bits = 4) {
  const uint32_t b = levels < 0xF ? 4u : levels < 0xFF ? 8u : levels < 0xFFFF ? 16u : 32u;
  return b < min_bits ? min_bits : b;  // min_bits = 8: no nibble codes (PBFS_PACK_MIN_BITS, A/B knob)
}
__host__ __device__ __forceinline__ uint32_t pack_width(uint32_t levels, uint32_t min_bits = 4) {
  const uint32_t b = pack_bits(levels, min_bits);
  return b < 8 ? 1u : b / 8;
}
// Bytes of a packed copy of n distances (whole 16 B vectors for the nibble codes).
__host__ __device__ __forceinline__ unsigned long long packed_bytes(unsigned long long n, uint32_t bits) {
  return bits == 4 ? ((n + 31) / 32) * 16 : n * (bits / 8);
}

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
  const uint32_t* __restrict__ first_nbr;  // col[rowptr[v]] (0 for isolated v), n entries
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
  unsigned long long isolated;  // zero-degree vertices pre-set in init_mask
  uint32_t heavy_deg;   // hub split threshold (kHeavyDeg or kHeavyDegBig)
  uint32_t chunk_log2;  // log2 of edges per heavy item
  uint32_t small_chunks;  // heavy_cap covers kSmallChunkLog2 items on small frontiers
  uint32_t force;         // kForce* test hooks (PBFS_FORCE_MODES at graph creation)
  void* pack;             // optional: narrow copy of dist for the host transfer (see pack_bits)
  uint32_t pack_min_bits = 4;
  // Latency mode (deep, hub-free graphs run top-down only, e.g. config 3's
  // mesh): 16 B queue entries {v, degree, row offset lo, hi}, see td_phase_latency.
  uint4* lq[2];
  int latency;
  // Observer log (test instrumentation, kernel_config.hpp:26-36): every
  // produced frontier appended as it was formed -- top-down the next queue
  // (as pushed), bottom-up the produced bitmap's ids; nullptr = off.
  uint32_t* obs;
  unsigned long long obs_cap;
  uint32_t source;
  int policy;
  int validate;
  double threshold;
  double alpha;
  double beta;
  uint32_t red_minq = 0;  // reduction claim from this frontier length (0 = off; bfs_persistent)
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// The CTAs one traversal runs on: the whole launch (single-GPU engine), or
// one partition's share of a launch that carries several partitions of the
// multi-partition engine (pbfs_multi.cu). Every work-distribution loop and
// the grid barrier take it instead of reading blockIdx / gridDim.
struct VGrid {
  unsigned cta;   // this CTA's index among the traversal's CTAs
  unsigned ctas;  // CTAs of the traversal
};
__device__ __forceinline__ VGrid hw_grid() { return VGrid{blockIdx.x, gridDim.x}; }
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
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Predicated claim atomics: one SASS instruction under a predicate instead of
// a divergent branch per edge slot. `old` keeps its input when not executed.
__device__ __forceinline__ uint32_t atom_or_if(bool pred, uint32_t* addr, uint32_t val,
                                               uint32_t old) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q atom.global.or.b32 %0, [%1], %3;\n\t}"
      : "+r"(old)
      : "l"(addr), "r"((uint32_t)pred), "r"(val));
  return old;
}
__device__ __forceinline__ uint32_t atom_cas_if(bool pred, uint32_t* addr, uint32_t cmp,
                                                uint32_t val, uint32_t old) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q atom.global.cas.b32 %0, [%1], %3, %4;\n\t}"
      : "+r"(old)
      : "l"(addr), "r"((uint32_t)pred), "r"(cmp), "r"(val));
  return old;
}
__device__ __forceinline__ uint32_t ld_cg_if(bool pred, const uint32_t* addr, uint32_t dflt) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q ld.global.cg.u32 %0, [%2];\n\t}"
      : "+r"(dflt)
      : "r"((uint32_t)pred), "l"(addr));
  return dflt;
}
// Predicated L1-allocating load (dead slots issue no request at all).
__device__ __forceinline__ uint32_t ld_ca_if(bool pred, const uint32_t* addr, uint32_t dflt) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q ld.global.ca.u32 %0, [%2];\n\t}"
      : "+r"(dflt)
      : "r"((uint32_t)pred), "l"(addr));
  return dflt;
}
// Predicated visited probe with an L1 eviction policy by word index (A/B
// knob PBFS_HOT_MODE / PBFS_HOT_WORDS): RMAT's hub core (the lowest ids) is
// the L1-reusable part of the bitmap, the rest is a flood of one-touch lines.
//   1: hot ld.ca,                 cold ld.L1::no_allocate
//   2: hot ld.L1::evict_last,     cold ld.L1::evict_first
//   3: hot ld.L1::evict_last,     cold ld.ca
template <int M>
__device__ __forceinline__ uint32_t ld_hot_if(bool pred, bool hot, const uint32_t* addr,
                                              uint32_t dflt) {
  const uint32_t h = (uint32_t)(pred && hot), c = (uint32_t)(pred && !hot);
  if constexpr (M == 1) {
    asm volatile(
        "{\n\t.reg .pred h, c;\n\tsetp.ne.b32 h, %1, 0;\n\tsetp.ne.b32 c, %2, 0;\n\t"
        "@h ld.global.ca.u32 %0, [%3];\n\t@c ld.global.L1::no_allocate.u32 %0, [%3];\n\t}"
        : "+r"(dflt) : "r"(h), "r"(c), "l"(addr));
  } else if constexpr (M == 2) {
    asm volatile(
        "{\n\t.reg .pred h, c;\n\tsetp.ne.b32 h, %1, 0;\n\tsetp.ne.b32 c, %2, 0;\n\t"
        "@h ld.global.L1::evict_last.u32 %0, [%3];\n\t@c ld.global.L1::evict_first.u32 %0, [%3];\n\t}"
        : "+r"(dflt) : "r"(h), "r"(c), "l"(addr));
  } else {
    asm volatile(
        "{\n\t.reg .pred h, c;\n\tsetp.ne.b32 h, %1, 0;\n\tsetp.ne.b32 c, %2, 0;\n\t"
        "@h ld.global.L1::evict_last.u32 %0, [%3];\n\t@c ld.global.ca.u32 %0, [%3];\n\t}"
        : "+r"(dflt) : "r"(h), "r"(c), "l"(addr));
  }
  return dflt;
}
__device__ __forceinline__ void red_or_if(bool pred, uint32_t* addr, uint32_t val) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
      "@q red.global.or.b32 [%1], %2;\n\t}" ::"r"((uint32_t)pred), "l"(addr), "r"(val));
}
// Read-only graph arrays (`col`, `rowptr`) streamed without allocating in L1:
// L1 is kept for the skewed visited / frontier bitmap probes, where RMAT hub
// words hit (measured: L1-cacheable skewed probes 380 G/s vs 125 G/s at L2,
// tools/ubench_probe.cu).
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_stream(const unsigned long long* p) {
  unsigned long long v;
  asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier on one 32-bit word (tools/ubench_barrier.cu: 2.0 us at 444
// CTAs vs 2.4 us for a two-level counter tree with sc fences). Every CTA adds
// 1 except CTA 0, which adds 2^31 - (grid - 1): each barrier adds exactly
// 2^31, so bit 31 flips when the last CTA arrives and the low bits return to
// their start value -- no reset between barriers or launches. Thread 0's
// release-add publishes the CTA's writes (ordered before it by
// __syncthreads); the spin is relaxed, since an acquire load per iteration
// would invalidate the SM's L1 under the CTAs still working, and one
// acquire fence follows it.
struct GridBarrier {
  Ctl* ctl;
  unsigned long long* snap;  // shared memory, 8 x u64
  VGrid vg = hw_grid();
  // `src` (optional, 64 B, 16 B aligned): thread 0 copies it into `snap`
  // after the barrier, so a CTA reads the level counters with one request
  // instead of every thread polling the same L2 line; `src2` likewise into
  // snap[8..15].
  __device__ __forceinline__ void sync(const void* src = nullptr, const void* src2 = nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned nb = vg.cta == 0 ? 0x80000000u - (vg.ctas - 1) : 1u;
      unsigned old;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;"
                   : "=r"(old) : "l"(&ctl->bar_word), "r"(nb) : "memory");
      while (((old ^ ld_relaxed(&ctl->bar_word)) & 0x80000000u) == 0) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (src) {
        const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
        const ulonglong2 a = __ldcg(s2), b = __ldcg(s2 + 1), c = __ldcg(s2 + 2), d = __ldcg(s2 + 3);
        snap[0] = a.x; snap[1] = a.y; snap[2] = b.x; snap[3] = b.y;
        snap[4] = c.x; snap[5] = c.y; snap[6] = d.x; snap[7] = d.y;
      }
      if (src2) {
        const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src2);
        const ulonglong2 a = __ldcg(s2), b = __ldcg(s2 + 1), c = __ldcg(s2 + 2), d = __ldcg(s2 + 3);
        snap[8] = a.x; snap[9] = a.y; snap[10] = b.x; snap[11] = b.y;
        snap[12] = c.x; snap[13] = c.y; snap[14] = d.x; snap[15] = d.y;
      }
    }
    __syncthreads();
  }
  // The barrier, then warp 0 copies the 32 u64 at src into snap[0..31].
  __device__ __forceinline__ void sync32(const unsigned long long* src) {
    __syncthreads();
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) {
        const unsigned nb = vg.cta == 0 ? 0x80000000u - (vg.ctas - 1) : 1u;
        unsigned old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;"
                     : "=r"(old) : "l"(&ctl->bar_word), "r"(nb) : "memory");
        while (((old ^ ld_relaxed(&ctl->bar_word)) & 0x80000000u) == 0) {
        }
      }
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      snap[threadIdx.x] = __ldcg(src + threadIdx.x);
    }
    __syncthreads();
  }
};

// Per-warp discovery buffer in shared memory (LocalFrontier analogue).
// kPeers (the multi-partition engine, pbfs_multi.cu): a flush writes the
// entries, offset by `lo` (local id -> global id), into `ndst` queue segments
// -- this partition's segment in every partition's queue, peers' included --
// so the frontier exchange rides on the level's own stores.
template <bool kPeers>
struct WarpPushT {
  uint32_t* buf;  // kPushBuf entries in smem
  int count;      // warp-uniform
  uint32_t* const* dst = nullptr;  // kPeers: smem array of ndst segment bases
  int ndst = 0;
  uint32_t lo = 0;
  __device__ __forceinline__ void flush(uint32_t* out, unsigned long long* counter,
                                        unsigned long long cap, unsigned int* overflow) {
    __syncwarp();
    if (count) {
      unsigned long long base = 0;
      if (lane_id() == 0) base = atomicAdd(counter, (unsigned long long)count);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + count <= cap) {
        if constexpr (kPeers) {
          for (int r = 0; r < ndst; ++r) {
            uint32_t* o = dst[r] + base;
            for (int i = lane_id(); i < count; i += 32) o[i] = buf[i] + lo;
          }
        } else {
          for (int i = lane_id(); i < count; i += 32) out[base + i] = buf[i];
        }
      } else if (lane_id() == 0) {
        atomicExch(overflow, 1u);
      }
    }
    count = 0;
    __syncwarp();
  }
  // Appends lane-local winners v[k] (bit k of winmask) of a K-slot batch with
  // one warp scan and at most one flush.
  template <int K>
  __device__ __forceinline__ void push_many(uint32_t winmask, const uint32_t (&v)[K],
                                            uint32_t* out, unsigned long long* counter,
                                            unsigned long long cap, unsigned int* overflow) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lane = lane_id();
    const uint32_t c = __popc(winmask);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    const int total = (int)__shfl_sync(FULL, incl, 31);
    if (total == 0) return;
    if (count + total > kPushBuf) flush(out, counter, cap, overflow);
    uint32_t pos = count + incl - c;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if ((winmask >> k) & 1u) buf[pos++] = v[k];
    }
    count += total;
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
using WarpPush = WarpPushT<false>;

template <typename OffT>
__device__ __forceinline__ unsigned long long degree_of(const Params<OffT>& p, uint32_t v) {
  return (unsigned long long)(ld_stream(&p.rowptr[v + 1]) - ld_stream(&p.rowptr[v]));
}

struct WarpTally {
  unsigned long long produced = 0, raw = 0, edges = 0, degree = 0, viol = 0;
};

// Probe word for the claim test. kClaimBitmap probes `visited` through L1
// first (see claim_batch); the dist probes of the CAS / plain variants go to
// L2 (random 4 B over n words, no reuse).
template <int C, typename OffT>
__device__ __forceinline__ uint32_t probe_word(const Params<OffT>& p, uint32_t v) {
  if constexpr (C == kClaimBitmap) {
    if constexpr (PBFS_PROBE == 1) return __ldcg(&p.visited[v >> 5]);
    return __ldca(&p.visited[v >> 5]);
  } else {
    return __ldcg(&p.dist[v]);
  }
}

// The claim discipline of each variant for K edges (u -> v[k]) of one lane,
// in three stages so nothing waits on a single round trip: all K probe
// loads, then all K claim atomics (results consumed only afterwards), then
// the dist stores and queue appends. okm bit k marks a live edge slot.
template <int C, int K, typename OffT, class WP>
__device__ __forceinline__ void claim_batch(const Params<OffT>& p, uint32_t nd,
                                            const uint32_t (&v)[K], uint32_t okm,
                                            uint32_t* qout, WP& wp, LevelCnt* cnt,
                                            WarpTally& t, uint32_t* obm, uint32_t* rbm = nullptr) {
  // Unconditional probes (dead slots hold a valid vertex id): predicated
  // loads end up in separate blocks that ptxas interleaves with their uses,
  // serialising the round trips this batching exists to overlap.
  uint32_t w[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if constexpr (C == kClaimBitmap && PBFS_PROBE == 3) {
      w[k] = 0;
    } else if constexpr (C == kClaimBitmap && PBFS_PROBE == 2 && PBFS_PRED_TD && PBFS_HOT_MODE) {
      w[k] = ld_hot_if<PBFS_HOT_MODE>((okm >> k) & 1u, (v[k] >> 5) < (uint32_t)PBFS_HOT_WORDS,
                                      &p.visited[v[k] >> 5], 0xffffffffu);
    } else if constexpr (C == kClaimBitmap && PBFS_PROBE == 2 && PBFS_PRED_TD) {
      // Dead slots issue no probe (read back as "visited").
      w[k] = ld_ca_if((okm >> k) & 1u, &p.visited[v[k] >> 5], 0xffffffffu);
    } else if constexpr (C != kClaimBitmap &&
                         (C == kClaimCas ? PBFS_CAS_PROBE : PBFS_PLAIN_PROBE) == 1) {
      w[k] = ld_ca_if((okm >> k) & 1u, &p.dist[v[k]], 0u);
    } else if constexpr (C != kClaimBitmap &&
                         (C == kClaimCas ? PBFS_CAS_PROBE : PBFS_PLAIN_PROBE) == 2) {
      w[k] = ld_cg_if((okm >> k) & 1u, &p.dist[v[k]], 0u);
    } else {
      w[k] = probe_word<C>(p, v[k]);
    }
  }
  if (C == kClaimBitmap && rbm != nullptr) {
    // Reduction claim (big top-down levels, see bfs_persistent): every slot
    // that saw a clear visited bit stores nd (racing writers store the same
    // value) and sets the bit in `visited` and in the next-frontier bitmap
    // `rbm` with no-return reds -- nothing waits on a claim round trip. The
    // distinct next frontier is the bitmap, counted and compacted after the
    // level; a stale clear bit only costs a redundant red.
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t bit = 1u << (v[k] & 31);
      const bool go = ((okm >> k) & 1u) && !(w[k] & bit);
      if (go) p.dist[v[k]] = nd;
      red_or_if(go, &p.visited[v[k] >> 5], bit);
      red_or_if(go, &rbm[v[k] >> 5], bit);
    }
    return;
  }
  if constexpr (C == kClaimPlain) {
    // kernels.cpp:291-301: compare, plain store; racing writers all store the
    // same nd, so duplicates are possible but values are not. Every racing
    // writer also ORs the same bit into the next-frontier bitmap (no-return
    // RED, idempotent like the reference's same-value byte stores):
    // duplicates are counted (raw) but collapse in the bitmap, which is
    // compacted into the next queue after the level.
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (((okm >> k) & 1u) && nd < w[k]) {
        if (p.validate && w[k] != kUnreached) ++t.viol;  // kernels.cpp:294
        p.dist[v[k]] = nd;
        ++t.raw;
        atomicOr(&p.bm[1][v[k] >> 5], 1u << (v[k] & 31));
      }
    }
    (void)qout;
    (void)wp;
    (void)cnt;
  } else {
    if constexpr (C == kClaimBitmap && PBFS_PROBE == 0) {
      // Stage 1b: an L1 hit is authoritative for bits set before this level
      // (the grid barrier's fence invalidated L1) -- RMAT hub words stay hot
      // there and never touch the hot L2 slices. A clear bit may be stale
      // with respect to this level's claims, so it is re-probed at L2 before
      // paying for an atomic.
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t bit = 1u << (v[k] & 31);
        w[k] = ld_cg_if(((okm >> k) & 1u) && !(w[k] & bit), &p.visited[v[k] >> 5], w[k]);
      }
    }
    // Stage 2: predicated claim atomics, all issued before any result is used.
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = (okm >> k) & 1u;
      if constexpr (C == kClaimCas) {
        // kernels.cpp:282-290: claim by compare-exchange from kUnreached.
        w[k] = atom_cas_if(live && w[k] == kUnreached, &p.dist[v[k]], kUnreached, nd, 0u);
      } else {
        // kernels.cpp:302-320: test the visited bit, then claim it.
        const uint32_t bit = 1u << (v[k] & 31);
        w[k] = atom_or_if(live && !(w[k] & bit), &p.visited[v[k] >> 5], bit, 0xffffffffu);
      }
    }
    // Stage 3: winners store dist inline (plain store) and are appended.
    uint32_t winmask = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool won = C == kClaimCas ? w[k] == kUnreached : !(w[k] & (1u << (v[k] & 31)));
      winmask |= (uint32_t)won << k;
      if constexpr (C == kClaimBitmap) {
        if (won) p.dist[v[k]] = nd;
        // Winners mark the next-frontier bitmap (no-return red) where the
        // caller needs it during the level (partitions exchange it); the
        // single-GPU engine passes obm = nullptr and rebuilds the bitmap from
        // dist only when bottom-up follows (front_from_dist): the reds cost
        // ~7 % of a huge top-down level.
        red_or_if(won && obm != nullptr, &obm[v[k] >> 5], 1u << (v[k] & 31));
      }
    }
    t.produced += __popc(winmask);
    if (p.policy == kPolicyBeamer) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if ((winmask >> k) & 1u) t.degree += degree_of(p, v[k]);
      }
    }
    wp.push_many<K>(winmask, v, qout, &cnt->raw, p.qcap, &p.ctl->overflow);
  }
}

// Warp-cooperative expansion of up to 32 light vertices (lane i holds vertex
// i's [beg, beg+deg)): inclusive shuffle scan of the degrees, then 4x32 edges
// per step, each lane locating its owner by a 5-step shuffle binary search.
template <int C, typename OffT, class WP>
__device__ __forceinline__ void td_light_batch(const Params<OffT>& p, uint32_t nd, OffT beg,
                                               uint32_t deg, uint32_t* qout, WP& wp,
                                               LevelCnt* cnt, WarpTally& t, uint32_t* obm,
                                               uint32_t* rbm = nullptr) {
  constexpr int K = PBFS_SLOTS;
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
  if (total == 0) return;
  // First edge of the batch: owner = first lane with a non-empty range.
  const unsigned nz = __ballot_sync(FULL, deg != 0);
  const OffT b0 = __shfl_sync(FULL, beg, __ffs(nz) - 1);
  for (uint32_t e0 = 0; e0 < total; e0 += 32 * K) {
    uint32_t v[K];
    uint32_t okm = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t e = e0 + 32 * k + lane;
      int j = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t x = __shfl_sync(FULL, incl, j + step - 1);
        if (x <= e) j += step;
      }
      const OffT ob = __shfl_sync(FULL, beg, j);
      const uint32_t oex = __shfl_sync(FULL, excl, j);
      const bool ok = e < total;
      okm |= (uint32_t)ok << k;
      // Dead slots re-read the batch's first edge (always valid): no branch.
      const unsigned long long ei = ok ? (unsigned long long)ob + (e - oex) : (unsigned long long)b0;
      v[k] = ld_stream(&p.col[ei]);
    }
    claim_batch<C, K>(p, nd, v, okm, qout, wp, cnt, t, obm, rbm);
  }
}

// Static-first work distribution: warp gw takes slice gw first and only
// then falls back to an atomic cursor, so a tiny frontier costs no atomics.
template <int C, typename OffT, class QV = const uint32_t*, class WP = WarpPush>
__device__ void td_phase_light(const Params<OffT>& p, uint32_t depth, QV qin,
                               unsigned long long qlen, uint32_t* qout, WP& wp,
                               LevelCnt* cnt, WarpTally& t, uint32_t* obm, uint32_t* stale,
                               VGrid vg = hw_grid(), uint32_t* rbm = nullptr) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  const unsigned warps_total = vg.ctas * kWarps;
  // Slice width: 32 frontier vertices per warp, fewer on a frontier smaller
  // than one full slice per warp, so its edges spread over more warps instead
  // of queueing up as batches (each a dependent round-trip chain) in a few.
  uint32_t W = 32;
  while (W > 1 && (unsigned long long)warps_total * (W / 2) >= qlen) W /= 2;
  unsigned long long base = (unsigned long long)(vg.cta * kWarps + (threadIdx.x >> 5)) * W;
  while (base < qlen) {
    const unsigned long long i = base + lane;
    OffT beg = 0, end = 0;
    if (lane < W && i < qlen) {
      const uint32_t u = qin[i];
      beg = __ldg(&p.rowptr[u]);
      end = __ldg(&p.rowptr[u + 1]);
      // The stale bitmap's set bits are exactly this input frontier: zero
      // their words so it can be the next level's mark target.
      if (stale) stale[u >> 5] = 0;
    }
    unsigned long long deg = (unsigned long long)(end - beg);
    t.edges += deg;
    // Hubs: split into 2^chunk_log2-edge items for the grid-wide heavy pass; the
    // warp reserves all its items with one atomicAdd (a per-vertex atomic on
    // one counter serialises at L2 when a level holds ~1e6 hubs).
    const bool hub = deg > p.heavy_deg;
    const uint32_t clog = qlen <= kSmallFrontier && p.small_chunks ? kSmallChunkLog2 : p.chunk_log2;
    const unsigned long long chunk = 1ull << clog;
    const unsigned int my_items = hub ? (unsigned int)((deg + chunk - 1) >> clog) : 0u;
    if (__any_sync(FULL, hub)) {
      unsigned int incl = my_items;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int x = __shfl_up_sync(FULL, incl, o);
        if (lane >= (unsigned)o) incl += x;
      }
      const unsigned int wtotal = __shfl_sync(FULL, incl, 31);
      unsigned int wbase = 0;
      if (lane == 0) wbase = atomicAdd(&cnt->heavy_count, wtotal);
      wbase = __shfl_sync(FULL, wbase, 0);
      if ((unsigned long long)wbase + wtotal <= p.heavy_cap) {
        const unsigned int slot = wbase + incl - my_items;
        for (unsigned int k = 0; k < my_items; ++k) {
          const unsigned long long b = (unsigned long long)beg + (unsigned long long)k * chunk;
          const unsigned long long e = b + chunk < (unsigned long long)end ? b + chunk
                                                                            : (unsigned long long)end;
          p.heavy[slot + k] = HeavyItem{b, e};
        }
      } else if (lane == 0) {
        atomicExch(&p.ctl->overflow, 1u);
      }
    }
    if (hub) deg = 0;
    td_light_batch<C>(p, nd, beg, (uint32_t)deg, qout, wp, cnt, t, obm, rbm);
    // The static first slices cover small frontiers entirely: no cursor
    // round trip at all (the common case on deep, narrow graphs).
    if (qlen <= (unsigned long long)warps_total * W) break;
    unsigned int nb = 0;
    if (lane == 0) nb = atomicAdd(&cnt->td_cursor, 32u);
    base = (unsigned long long)warps_total * 32 + __shfl_sync(FULL, nb, 0);
  }
}

// Hub chunks: 16 coalesced 128 B `col` loads per warp step, laid out so the
// 32 lanes of every load (and hence of every visited-bitmap probe and claim
// that follows) hold 32 CONSECUTIVE neighbours of the sorted adjacency list.
// A hub's neighbours are dense in id space, so one probe instruction touches
// ~2-3 distinct 128 B bitmap lines instead of ~32 -- the L1TEX line rate, not
// DRAM, is what bounds a random-probe loop on this part.
template <int C, typename OffT, class WP = WarpPush>
__device__ void td_phase_heavy(const Params<OffT>& p, uint32_t depth, unsigned int items,
                               uint32_t* qout, WP& wp, LevelCnt* cnt, WarpTally& t,
                               uint32_t* obm, VGrid vg = hw_grid(), uint32_t* rbm = nullptr) {
  constexpr int K = PBFS_SLOTS;
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  const unsigned warps_total = vg.ctas * kWarps;
  unsigned int it = vg.cta * kWarps + (threadIdx.x >> 5);
  while (it < items) {
    const HeavyItem h = p.heavy[it];
    const uint32_t* base = p.col + h.beg;
    const uint32_t len = (uint32_t)(h.end - h.beg);
    for (uint32_t e0 = 0; e0 < len; e0 += 32 * K) {
      uint32_t v[K];
      uint32_t okm = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t e = e0 + 32 * k + lane;
        const bool ok = e < len;
        okm |= (uint32_t)ok << k;
        v[k] = ld_stream(&base[ok ? e : 0u]);
      }
      claim_batch<C, K>(p, nd, v, okm, qout, wp, cnt, t, obm, rbm);
    }
    // Items are equal-sized (2^chunk_log2 edges but a hub's last one): a static
    // round-robin balances them without a contended cursor.
    it += warps_total;
  }
  (void)FULL;
  (void)cnt;
}

// ---- latency mode ---------------------------------------------------------------
// A deep graph (config 3: ~3900 levels of ~4 K vertices) is bound by one
// level's dependent chain, not by bytes: queue -> rowptr -> col -> probe ->
// claim -> flush, then the barrier. On a hub-free graph run top-down only the
// chain loses two round trips: queue entries carry the row range {v, degree,
// beg} (the winner loads rowptr in the shadow of its claim atomic, for every
// live slot at once), and the claim is the atom.or alone (its returned word
// settles the race; the L1 probe only saves atomics when most targets are
// visited, which costs an extra round trip here).

// Per-warp buffer of 16 B entries in the warp's s_list slice.
struct WarpPush4 {
  uint4* buf;  // kPushBuf / 4 entries
  int count;   // warp-uniform
  __device__ __forceinline__ void flush(uint4* out, unsigned long long* counter,
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
};

template <int K, typename OffT>
__device__ __forceinline__ void claim_latency(const Params<OffT>& p, uint32_t nd,
                                              const uint32_t (&v)[K], uint32_t okm, uint4* qout,
                                              WarpPush4& wp, LevelCnt* cnt, WarpTally& t) {
  constexpr int kCap = kPushBuf / 4;
  uint32_t w[K];
  OffT b0[K], b1[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t bit = 1u << (v[k] & 31);
    w[k] = atom_or_if((okm >> k) & 1u, &p.visited[v[k] >> 5], bit, 0xffffffffu);
    b0[k] = ld_stream(&p.rowptr[v[k]]);  // dead slots hold a valid id
    b1[k] = ld_stream(&p.rowptr[v[k] + 1]);
  }
  uint32_t winmask = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool won = !(w[k] & (1u << (v[k] & 31)));
    winmask |= (uint32_t)won << k;
    if (won) p.dist[v[k]] = nd;
  }
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  // Appended in halves of K / 2 slots, so a half's winners (<= 16 K) always
  // fit the kPushBuf / 4-entry buffer after a flush.
  static_assert(kCap >= 16 * K, "latency-mode discovery buffer");
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t hm = (winmask >> (h * K / 2)) & ((1u << (K / 2)) - 1u);
    const uint32_t c = __popc(hm);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    const int total = (int)__shfl_sync(FULL, incl, 31);
    if (total == 0) continue;
    t.produced += c;
    if (wp.count + total > kCap) wp.flush(qout, &cnt->raw, p.qcap, &p.ctl->overflow);
    uint32_t pos = wp.count + incl - c;
#pragma unroll
    for (int k = h * K / 2; k < (h + 1) * K / 2; ++k) {
      if ((winmask >> k) & 1u) {
        const unsigned long long b = (unsigned long long)b0[k];
        wp.buf[pos++] = make_uint4(v[k], (uint32_t)(b1[k] - b0[k]), (uint32_t)b, (uint32_t)(b >> 32));
      }
    }
    wp.count += total;
  }
}

// Top-down level of latency mode: 32 queue entries per warp slice (static
// first slice, then the cursor), warp-cooperative expansion as
// td_light_batch; no hub items (the graph has none).
template <typename OffT>
__device__ void td_phase_latency(const Params<OffT>& p, uint32_t depth, const uint4* qin,
                                 unsigned long long qlen, uint4* qout, WarpPush4& wp,
                                 LevelCnt* cnt, WarpTally& t) {
  // 4 slots: 32 vertices of a hub-free deep graph (degree ~4) fit one batch,
  // and the speculative offsets of 8 slots would spill.
  constexpr int K = 4;
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  const unsigned warps_total = gridDim.x * kWarps;
  // Slices narrower than 32 entries on a frontier smaller than one full
  // slice per warp, dealt round-robin over the CTAs (warp-major), so a ~4 K
  // level occupies every SM instead of the first few CTAs' warps.
  unsigned W = 32;
  while (PBFS_LAT_SPREAD && W > 1 && (unsigned long long)warps_total * (W / 2) >= qlen) W /= 2;
  const unsigned gwi = PBFS_LAT_SPREAD ? (threadIdx.x >> 5) * gridDim.x + blockIdx.x
                                       : blockIdx.x * kWarps + (threadIdx.x >> 5);
  unsigned long long base = (unsigned long long)gwi * W;
  while (base < qlen) {
    const unsigned long long i = base + lane;
    uint32_t deg = 0;
    unsigned long long beg = 0;
    if (lane < W && i < qlen) {
      const uint4 q = qin[i];
      deg = q.y;
      beg = (unsigned long long)q.z | ((unsigned long long)q.w << 32);
    }
    t.edges += deg;
    uint32_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    const uint32_t total = __shfl_sync(FULL, incl, 31);
    const uint32_t excl = incl - deg;
    if (total) {
      const unsigned nz = __ballot_sync(FULL, deg != 0);
      const unsigned long long b0 = __shfl_sync(FULL, beg, __ffs(nz) - 1);
      for (uint32_t e0 = 0; e0 < total; e0 += 32 * K) {
        uint32_t v[K];
        uint32_t okm = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t e = e0 + 32 * k + lane;
          int j = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t x = __shfl_sync(FULL, incl, j + step - 1);
            if (x <= e) j += step;
          }
          const unsigned long long ob = __shfl_sync(FULL, beg, j);
          const uint32_t oex = __shfl_sync(FULL, excl, j);
          const bool ok = e < total;
          okm |= (uint32_t)ok << k;
          v[k] = ld_stream(&p.col[ok ? ob + (e - oex) : b0]);
        }
        claim_latency<K>(p, nd, v, okm, qout, wp, cnt, t);
      }
    }
    if (qlen <= (unsigned long long)warps_total * W) break;
    unsigned int nb = 0;
    if (lane == 0) nb = atomicAdd(&cnt->td_cursor, 32u);
    base = (unsigned long long)warps_total * 32 + __shfl_sync(FULL, nb, 0);
  }
}

// ---- latency mode: several levels per grid barrier -----------------------------
// The mesh's ~3900 levels are each one dependent chain (queue -> col ->
// claim -> append) plus one grid barrier. A round runs kLatLevels levels per
// barrier: the warp that wins a vertex at level d+j < d+kLatLevels expands
// it itself right away (its row range is loaded in the shadow of the claim)
// instead of handing it to the next level through the queue and a barrier;
// only level d+kLatLevels goes to the next round's queue.
//  * Claims are atomicMin on dist. Level d+1 is exact (every vertex at
//    distance d+1 neighbours the complete level-d frontier); a claim at
//    d+j, j >= 2, can be premature -- a slower warp may still reach the
//    vertex at a lower level -- and is then lowered. The lowering warp owns
//    the vertex at its true level and expands it; every vertex at distance
//    d+j (j < kLatLevels) is therefore expanded at d+j exactly once within
//    the round (its parent is, by induction), and distances are exact.
//  * Bookkeeping keeps every per-level record equal to the level-synchronous
//    one: distinct size = wins - lowerings at that level; edges examined =
//    degrees expanded at that level minus those of vertices lowered from it
//    (their expansion was wasted). A vertex lowered from d+kLatLevels stays
//    in the next queue as a stale entry: expanded next round, every one of
//    its claims fails (its neighbours hold <= d+kLatLevels by then), and its
//    degree is taken off that level's count.
// Grid-bipartite meshes make premature claims rare (a vertex's neighbours
// sit one level up or down); the shortcut edges cause the few there are.
#ifndef PBFS_LAT_LEVELS
#define PBFS_LAT_LEVELS 5
#endif
constexpr int kLatLevels = PBFS_LAT_LEVELS;  // levels per grid barrier (1 = plain latency mode)
static_assert(kLatLevels >= 1 && kLatLevels <= 6, "PBFS_LAT_LEVELS must be 1..6");
// Dynamic shared memory of the latency kernel: kLatLevels buffers of 128
// 16 B entries per warp (LatRound).
constexpr size_t kLatSmem = kLatLevels >= 2 ? (size_t)kWarps * kLatLevels * 128 * 16 : 0;

// Round counters (Ctl::latk[round & 3], one 256 B row): index
//   kLkEdges0 (level d's expanded degrees), kLkCursor, kLkPush (next-queue
//   appends), kLkWins + j, kLkLow + j (lowered from d+j), kLkLowDeg + j,
//   kLkExp + j (degrees expanded at d+j), j = 1 .. kLatLevels.
constexpr int kLkEdges0 = 0, kLkCursor = 1, kLkPush = 2, kLkWins = 4, kLkLow = 11, kLkLowDeg = 18,
              kLkExp = 25;

template <typename OffT>
struct LatRound {
  static constexpr int K = 4;          // edge slots per lane
  // Entries per level buffer: one claim's winners, so each claim has a single
  // drain / flush site and the nested expansion's code stays linear in
  // kLatLevels. Buffers live in dynamic shared memory (kLatSmem per CTA).
  static constexpr int kCap = 32 * K;
  const Params<OffT>& p;
  uint32_t d;
  uint4* buf;                        // smem: level buffers 1 .. kLatLevels - 1, then the push buffer
  uint4* qout;
  unsigned long long* ctr;           // this round's counter row
  WarpPush4 wp;
  int lcount[kLatLevels + 1] = {};
  // Per-lane tallies, reduced per warp at the end of the round.
  unsigned long long edges0 = 0;
  unsigned long long wins[kLatLevels + 1] = {}, low[kLatLevels + 1] = {}, lowdeg[kLatLevels + 1] = {},
                     exp[kLatLevels + 1] = {};

  // Level j's buffer (j = kLatLevels: the push buffer).
  __device__ __forceinline__ uint4* level_buf(int j) { return buf + (j - 1) * kCap; }

  // Claims at level d+J of K edge slots (okm = live slots).
  template <int J>
  __device__ __forceinline__ void claim(const uint32_t (&v)[K], uint32_t okm) {
    const uint32_t nd = d + J;
    uint32_t old[K];
    OffT b0[K], b1[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      old[k] = nd;
      if ((okm >> k) & 1u) old[k] = atomicMin(&p.dist[v[k]], nd);
      b0[k] = ld_stream(&p.rowptr[v[k]]);  // dead slots hold a valid id
      b1[k] = ld_stream(&p.rowptr[v[k] + 1]);
    }
    uint32_t winmask = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool won = old[k] > nd;
      winmask |= (uint32_t)won << k;
      if constexpr (J < kLatLevels) {
        // A premature claim at d+i (J < i <= kLatLevels) is lowered.
        if (won && old[k] != kUnreached) {
          const uint32_t i = old[k] - d;
#pragma unroll
          for (int q = J + 1; q <= kLatLevels; ++q) {
            if (i == (uint32_t)q) {
              ++low[q];
              lowdeg[q] += (unsigned long long)(b1[k] - b0[k]);
            }
          }
        }
      }
    }
    wins[J] += __popc(winmask);
    const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(winmask));
    if (total == 0) return;
    uint4* out;
    int* cnt;
    if constexpr (J < kLatLevels) {
      if (lcount[J] + total > kCap) drain<J>();
      out = level_buf(J);
      cnt = &lcount[J];
    } else {
      if (wp.count + total > kCap) wp.flush(qout, &ctr[kLkPush], p.qcap, &p.ctl->overflow);
      out = wp.buf;
      cnt = &wp.count;
    }
    // Slot by slot: one ballot each, lanes in order.
    int pos = *cnt;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool w = (winmask >> k) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, w);
      if (w) {
        const unsigned long long b = (unsigned long long)b0[k];
        out[pos + __popc(m & lanemask_lt())] =
            make_uint4(v[k], (uint32_t)(b1[k] - b0[k]), (uint32_t)b, (uint32_t)(b >> 32));
      }
      pos += __popc(m);
    }
    *cnt = pos;
    __syncwarp();
  }

  // Warp-cooperative expansion of `count` row ranges {v, degree, beg lo, hi}
  // (32 at a time, as td_phase_latency); every edge slot is claimed at d+J.
  template <int J, class Load>
  __device__ __forceinline__ void expand(unsigned long long count, Load&& load, unsigned long long& edges) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lane = lane_id();
    for (unsigned long long base = 0; base < count; base += 32) {
      uint32_t deg = 0;
      unsigned long long beg = 0;
      if (base + lane < count) {
        const uint4 q = load(base + lane);
        deg = q.y;
        beg = (unsigned long long)q.z | ((unsigned long long)q.w << 32);
      }
      edges += deg;
      uint32_t incl = deg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(FULL, incl, o);
        if (lane >= (unsigned)o) incl += x;
      }
      const uint32_t total = __shfl_sync(FULL, incl, 31);
      const uint32_t excl = incl - deg;
      if (!total) continue;
      const unsigned nz = __ballot_sync(FULL, deg != 0);
      const unsigned long long b0 = __shfl_sync(FULL, beg, __ffs(nz) - 1);
      for (uint32_t e0 = 0; e0 < total; e0 += 32 * K) {
        uint32_t v[K];
        uint32_t okm = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t e = e0 + 32 * k + lane;
          int j = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t x = __shfl_sync(FULL, incl, j + step - 1);
            if (x <= e) j += step;
          }
          const unsigned long long ob = __shfl_sync(FULL, beg, j);
          const uint32_t oex = __shfl_sync(FULL, excl, j);
          const bool ok = e < total;
          okm |= (uint32_t)ok << k;
          v[k] = ld_stream(&p.col[ok ? ob + (e - oex) : b0]);
        }
        claim<J>(v, okm);
      }
    }
  }

  // Expands local level buffer J (its vertices' claims are at d+J+1).
  template <int J>
  __device__ __forceinline__ void drain() {
    if constexpr (J >= 1 && J < kLatLevels) {
      __syncwarp();
      const int n = lcount[J];
      lcount[J] = 0;
      // In place: this expansion's claims are at level J + 1 and append to
      // buffer J + 1 (draining it, and deeper ones, when full), never to J.
      uint4* lb = level_buf(J);
      expand<J + 1>((unsigned long long)n, [&](unsigned long long i) { return lb[i]; }, exp[J]);
      __syncwarp();
    }
  }
};

// One round (levels d .. d+kLatLevels-1) over the queue qin of qlen entries:
// slices as td_phase_latency (adaptive width, dealt over the CTAs, then a
// cursor), local levels drained in order at the end.
template <typename OffT>
__device__ void latency_round(const Params<OffT>& p, uint32_t d, const uint4* qin,
                              unsigned long long qlen, uint4* qout, uint4* sbuf,
                              unsigned long long* ctr) {
  using LR = LatRound<OffT>;
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  LR lr{p, d, sbuf, qout, ctr, WarpPush4{sbuf + (kLatLevels - 1) * LR::kCap, 0}};
  const unsigned warps_total = gridDim.x * kWarps;
  unsigned W = 32;
  while (W > 1 && (unsigned long long)warps_total * (W / 2) >= qlen) W /= 2;
  const unsigned gwi = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  unsigned long long base = (unsigned long long)gwi * W;
  while (base < qlen) {
    const unsigned long long n_here = qlen - base < W ? qlen - base : W;
    lr.template expand<1>(n_here, [&](unsigned long long i) { return qin[base + i]; }, lr.edges0);
    if (qlen <= (unsigned long long)warps_total * W) break;
    unsigned int nb = 0;
    if (lane == 0) nb = atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kLkCursor]), 32u);
    base = (unsigned long long)warps_total * 32 + __shfl_sync(FULL, nb, 0);
    W = 32;
  }
  // Local levels in order: draining level j only appends to levels > j.
  if constexpr (kLatLevels >= 2) lr.template drain<1>();
  if constexpr (kLatLevels >= 3) lr.template drain<2>();
  if constexpr (kLatLevels >= 4) lr.template drain<3>();
  if constexpr (kLatLevels >= 5) lr.template drain<4>();
  if constexpr (kLatLevels >= 6) lr.template drain<5>();
  lr.wp.flush(qout, &ctr[kLkPush], p.qcap, &p.ctl->overflow);
  // Warp-reduced tallies into the round's row.
  auto add = [&](int idx, unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    if (lane == 0 && x) atomicAdd(&ctr[idx], x);
  };
  add(kLkEdges0, lr.edges0);
#pragma unroll
  for (int j = 1; j <= kLatLevels; ++j) {
    add(kLkWins + j, lr.wins[j]);
    add(kLkLow + j, lr.low[j]);
    add(kLkLowDeg + j, lr.lowdeg[j]);
    if (j < kLatLevels) add(kLkExp + j, lr.exp[j]);
  }
}

// Bottom-up over all vertices (kernels.cpp:340-382), per warp task of one
// 32-word group (one visited word per lane), or of kBuSparseGroups groups
// with all loads in flight when few vertices are left unvisited (settled
// regions then cost a fraction of a round trip per group). Tasks after the first come from a cursor fetched
// one task ahead. A group's unvisited vertices are listed in shared memory
// (in rounds of kListCap) and resolved in two stages:
//  A. kBuSlots per lane at once: the first neighbour (dense first_nbr, a
//     coalesced read since the list ascends) and its frontier word. On RMAT
//     nearly every vertex with a frontier parent finds it here (hubs sort
//     first), without touching rowptr / col.
//  B. The misses, compacted in place, are scanned in chunks of 8 edges with
//     lane refill: a lane whose vertex is settled (parent found or list
//     exhausted) takes the next miss, so the warp is not held to its longest
//     scan (ER levels scan ~12 edges per vertex with a long geometric tail).
// Optional copies of the `next` words a bottom-up level produces (the
// multi-partition engine's peers' bitmaps at this partition's slice offset:
// the exchange fused into the level, pbfs_multi.cu).
struct NextPeers {
  uint32_t* const* dst;  // shared memory, n entries
  int n;
};

template <int GPT, typename OffT>
__device__ void bu_phase_t(const Params<OffT>& p, uint32_t depth, const uint32_t* front,
                           uint32_t* next, uint32_t* list, uint32_t* found, WarpTally& t,
                           unsigned int* cursor, VGrid vg, NextPeers peers = NextPeers{nullptr, 0}) {
  constexpr bool sparse = GPT > 1;
  constexpr int KB = kBuSlots;
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  const uint32_t nd = depth + 1;
  const unsigned warps_total = vg.ctas * kWarps;
  const unsigned gw = vg.cta * kWarps + (threadIdx.x >> 5);
  const uint32_t groups = (p.words + 31) / 32;
  constexpr uint32_t gpt = GPT;
  const uint32_t tasks = (groups + gpt - 1) / gpt;
  const bool beamer = p.policy == kPolicyBeamer;
  uint32_t task = gw;
  while (task < tasks) {
    // Next task index, fetched now so the cursor round trip overlaps this one.
    uint32_t nxt = 0;
    if (lane == 0) nxt = warps_total + atomicAdd(cursor, 1u);
    const uint32_t wbase = task * gpt * 32;  // first bitmap word of the task
    uint32_t visw[GPT];
#pragma unroll
    for (int j = 0; j < GPT; ++j) {
      const uint32_t w = wbase + j * 32 + lane;
      visw[j] = w < p.words ? p.visited[w] : 0xffffffffu;
    }
    // One id list for the whole task (padding bits are pre-set, so settled
    // words contribute nothing): a sparse task with a handful of unvisited
    // vertices over 8 groups costs one pass, not eight.
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < GPT; ++j) c += __popc(~visw[j]);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    const uint32_t total = __shfl_sync(FULL, incl, 31);
    if (total == 0 || sparse) {
      // Sparse tasks mark discoveries straight into next / visited (global
      // atomics; there are few), so their next words start zeroed. (The
      // multi-partition engine never runs sparse tasks: its peers' copies
      // are plain stores of whole words.)
#pragma unroll
      for (int j = 0; j < GPT; ++j) {
        const uint32_t w = wbase + j * 32 + lane;
        if (w < p.words) {
          next[w] = 0;
          for (int r = 0; r < peers.n; ++r) peers.dst[r][w] = 0;
        }
      }
      if (total == 0) {
        task = __shfl_sync(FULL, nxt, 0);
        continue;
      }
    } else {
      found[lane] = 0;
    }
    // Discovery of v: the group's shared-memory word (owner writes it back),
    // or directly into the global bitmaps on a sparse task.
    auto mark = [&](uint32_t v) {
      const uint32_t bit = 1u << (v & 31);
      if (sparse) {
        atomicOr(&next[v >> 5], bit);
        atomicOr(&p.visited[v >> 5], bit);
      } else {
        atomicOr(&found[(v >> 5) - wbase], bit);
      }
    };
    {
      for (uint32_t r0 = 0; r0 < total; r0 += kListCap) {
        // This round's slice [r0, r0 + kListCap) of the id list (lane-major,
        // ascending within a lane's words).
        __syncwarp();
        {
          uint32_t pos = incl - c;
#pragma unroll
          for (int j = 0; j < GPT; ++j) {
            uint32_t bits = ~visw[j];
            const uint32_t w = wbase + j * 32 + lane;
            while (bits && pos < r0 + kListCap) {
              const int b = __ffs(bits) - 1;
              bits &= bits - 1;
              if (pos >= r0) list[pos - r0] = w * 32 + b;
              ++pos;
            }
          }
        }
        __syncwarp();
        const uint32_t cnt = total - r0 < kListCap ? total - r0 : kListCap;
        // ---- stage A: first neighbours ----
        uint32_t nmiss = 0;  // warp-uniform; misses compact into list[0, nmiss)
        for (uint32_t k = 0; k < cnt; k += 32 * KB) {
          uint32_t v[KB], u0[KB], f0[KB];
          bool valid[KB];
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            const uint32_t idx = k + 32 * q + lane;
            valid[q] = idx < cnt;
            v[q] = list[valid[q] ? idx : 0];
            u0[q] = __ldg(&p.first_nbr[v[q]]);
          }
#pragma unroll
          for (int q = 0; q < KB; ++q) f0[q] = front[u0[q] >> 5];
          __syncwarp();  // every read of list[k, k + 32 KB) precedes the compaction
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            const bool hit = valid[q] && ((f0[q] >> (u0[q] & 31)) & 1u);
            const bool miss = valid[q] && !hit;
            if (hit) {
              // kernels.cpp:362-374: first frontier neighbour wins.
              p.dist[v[q]] = nd;
              mark(v[q]);
              ++t.produced;
              t.edges += 1;
              if (beamer) t.degree += (unsigned long long)(__ldg(&p.rowptr[v[q] + 1]) -
                                                           __ldg(&p.rowptr[v[q]]));
            }
            const unsigned mb = __ballot_sync(FULL, miss);
            if (miss) list[nmiss + __popc(mb & lanemask_lt())] = v[q];
            nmiss += __popc(mb);
          }
        }
        __syncwarp();
        // ---- stage B: windowed scans of the misses with lane refill ----
        // Each lane holds its current vertex plus a prefetched candidate
        // whose offsets load while the current window is in flight, so a
        // refill costs no extra round trip.
        uint32_t pos = 0;  // warp-uniform cursor into list[0, nmiss)
        bool active = false, cvalid = false;
        uint32_t v = 0, cv = 0;
        OffT e = 0, end = 0, beg0 = 0, cbeg = 0, cend = 0;
        unsigned long long scanned = 0;
        for (;;) {
          if (!active && cvalid) {
            v = cv;
            beg0 = cbeg;
            end = cend;
            e = beg0 + 1;  // the first neighbour was probed in stage A
            scanned = 1;
            cvalid = false;
            active = e < end;
            if (!active) t.edges += 1;  // degree 1 (isolated vertices are pre-visited)
          }
          if (pos < nmiss) {
            const unsigned need = __ballot_sync(FULL, !cvalid);
            if (!cvalid) {
              const uint32_t i = pos + __popc(need & lanemask_lt());
              if (i < nmiss) {
                cv = list[i];
                cbeg = __ldg(&p.rowptr[cv]);
                cend = __ldg(&p.rowptr[cv + 1]);
                cvalid = true;
              }
            }
            pos += __popc(need);
          }
          if (!__any_sync(FULL, active || cvalid)) break;
          if (active) {
            // Aligned kBuWin-entry windows (16 B loads, kBuWin / 8 sectors
            // per lane); out-of-range slots (other rows, or the allocation's
            // tail padding) issue no probe -- the probes' L1 tag lookups,
            // not bytes, bound this loop.
            const OffT wb = e & ~(OffT)(kBuWin - 1);
            const uint32_t lo = (uint32_t)(e - wb);
            const uint32_t hi = end - wb < (OffT)kBuWin ? (uint32_t)(end - wb) : (uint32_t)kBuWin;
            uint32_t x[kBuWin];
#pragma unroll
            for (int q4 = 0; q4 < kBuWin / 4; ++q4) {
              const uint4 a4 = __ldg(reinterpret_cast<const uint4*>(p.col + wb) + q4);
              x[4 * q4 + 0] = a4.x;
              x[4 * q4 + 1] = a4.y;
              x[4 * q4 + 2] = a4.z;
              x[4 * q4 + 3] = a4.w;
            }
            uint32_t fx[kBuWin];
#pragma unroll
            for (int c = 0; c < kBuWin; ++c) {
              const bool live = (uint32_t)c >= lo && (uint32_t)c < hi;
              fx[c] = ld_ca_if(live, &front[(live ? x[c] : 0u) >> 5], 0u);
            }
            unsigned hm = 0;
#pragma unroll
            for (int c = 0; c < kBuWin; ++c) hm |= ((fx[c] >> (x[c] & 31)) & 1u) << c;
            if (hm) {
              scanned += (unsigned long long)(__ffs(hm) - lo);
              t.edges += scanned;
              p.dist[v] = nd;
              mark(v);
              ++t.produced;
              if (beamer) t.degree += (unsigned long long)(end - beg0);
              active = false;
            } else {
              scanned += (unsigned long long)(hi - lo);
              e = wb + kBuWin;
              if (e >= end) {
                t.edges += scanned;
                active = false;
              }
            }
          }
        }
      }
    }
    __syncwarp();
    if (!sparse && wbase + lane < p.words) {
      const uint32_t f = found[lane];
      next[wbase + lane] = f;
      for (int r = 0; r < peers.n; ++r) peers.dst[r][wbase + lane] = f;
      if (f) p.visited[wbase + lane] = visw[0] | f;
    }
    task = __shfl_sync(FULL, nxt, 0);
  }
}

template <typename OffT>
__device__ __forceinline__ void bu_phase(const Params<OffT>& p, uint32_t depth,
                                         const uint32_t* front, uint32_t* next, uint32_t* list,
                                         uint32_t* found, WarpTally& t, unsigned int* cursor,
                                         bool sparse, VGrid vg = hw_grid(),
                                         NextPeers peers = NextPeers{nullptr, 0}) {
  if (sparse) {
    bu_phase_t<kBuSparseGroups>(p, depth, front, next, list, found, t, cursor, vg);
  } else {
    bu_phase_t<1>(p, depth, front, next, list, found, t, cursor, vg, peers);
  }
}

__device__ __forceinline__ void warp_flush_tally(LevelCnt* cnt, WarpTally& t, bool add_raw,
                                                 unsigned long long* viol = nullptr) {
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
    if (add_raw && t.raw) atomicAdd(&cnt->raw, t.raw);
    if (t.edges) atomicAdd(&cnt->edges, t.edges);
    if (t.degree) atomicAdd(&cnt->degree, t.degree);
    if (t.viol) atomicAdd(viol ? viol : &cnt->violations, t.viol);
  }
  t = WarpTally{};
}

// Bitmap -> queue (count_bitmap_slice / write_dense_slice, kernels.cpp:
// 225-241): each warp takes 8 x 32 words per step (all eight coalesced loads
// in flight), popcount-scans them and reserves its output range with one
// atomicAdd; optionally clears the words it consumed and zeroes the same
// words of a second bitmap. Latency-bound on sparse bitmaps: 8x fewer
// dependent round trips than one 32-word group per step.
template <int CW>
__device__ __forceinline__ void compact_bitmap_cw(uint32_t* nb, uint32_t* q, uint32_t words,
                                                  unsigned int* counter, bool clear,
                                                  uint32_t* zero_other, VGrid vg) {
  const unsigned lane = lane_id();
  const unsigned warps_total = vg.ctas * kWarps;
  const unsigned gw = vg.cta * kWarps + (threadIdx.x >> 5);
  for (uint32_t base = gw * 32 * CW; base < words; base += warps_total * 32 * CW) {
    uint32_t wd[CW];
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const uint32_t w = base + 32 * j + lane;
      wd[j] = w < words ? nb[w] : 0u;
    }
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const uint32_t w = base + 32 * j + lane;
      if (clear && wd[j]) nb[w] = 0;
      if (zero_other && w < words) zero_other[w] = 0;
      c += __popc(wd[j]);
    }
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += x;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (!total) continue;
    unsigned int off = 0;
    if (lane == 0) off = atomicAdd(counter, total);
    off = __shfl_sync(0xffffffffu, off, 0);
    uint32_t pos = off + incl - c;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      uint32_t bits = wd[j];
      const uint32_t w = base + 32 * j + lane;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        q[pos++] = w * 32 + b;
      }
    }
  }
}
// 8 words per lane only when that still gives every warp a step: on small
// bitmaps one word per lane keeps the bit extraction spread over the grid.
__device__ __forceinline__ void compact_bitmap(uint32_t* nb, uint32_t* q, uint32_t words,
                                               unsigned int* counter, bool clear,
                                               uint32_t* zero_other = nullptr, bool wide = false,
                                               VGrid vg = hw_grid()) {
  if (wide || words >= vg.ctas * kWarps * 32u * 8u) {
    compact_bitmap_cw<8>(nb, q, words, counter, clear, zero_other, vg);
  } else {
    compact_bitmap_cw<1>(nb, q, words, counter, clear, zero_other, vg);
  }
}

// Top-down -> bottom-up (kernels.cpp:191-213, "clear + mark"): the next
// frontier is exactly the vertices at distance nd, so its bitmap is one
// coalesced pass over dist (thread per word, 128 B per thread) instead of a
// red per discovery during the level. Bits past n stay clear.
// Words without a reached vertex (visited bits all pre-set isolated ones) need
// no dist read at all: on RMAT most high-id words are all isolated.
__device__ __forceinline__ void front_from_dist(const uint32_t* __restrict__ dist, uint32_t nd,
                                                uint32_t* out, uint32_t words,
                                                unsigned long long n, const uint32_t* visited,
                                                const uint32_t* init_mask, VGrid vg = hw_grid()) {
  const unsigned long long nthreads = (unsigned long long)vg.ctas * blockDim.x;
  for (unsigned long long w = (unsigned long long)vg.cta * blockDim.x + threadIdx.x;
       w < words; w += nthreads) {
    const unsigned long long base = w * 32;
    uint32_t bits = 0;
    const uint32_t reached = __ldcg(&visited[w]) & ~__ldg(&init_mask[w]);
    if (base < n && reached) {
      const uint4* d4 = reinterpret_cast<const uint4*>(dist + base);  // dist padded to 32
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 a = __ldcs(d4 + q);
        bits |= (uint32_t)(a.x == nd) << (4 * q) | (uint32_t)(a.y == nd) << (4 * q + 1) |
                (uint32_t)(a.z == nd) << (4 * q + 2) | (uint32_t)(a.w == nd) << (4 * q + 3);
      }
      bits &= reached;
    }
    out[w] = bits;
  }
}

// Plain-store top-down (kClaimPlain) keeps no visited bits: entering
// bottom-up, both come from dist in one coalesced pass -- visited = reached
// (or isolated / padding), frontier = dist == nd.
__device__ __forceinline__ void visited_front_from_dist(const uint32_t* __restrict__ dist, uint32_t nd,
                                                        uint32_t* visited, uint32_t* front,
                                                        uint32_t words, unsigned long long n,
                                                        const uint32_t* init_mask) {
  const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long w = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       w < words; w += nthreads) {
    const unsigned long long base = w * 32;
    uint32_t reached = 0, bits = 0;
    if (base < n) {
      const uint4* d4 = reinterpret_cast<const uint4*>(dist + base);  // dist padded to 32
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 a = __ldcs(d4 + q);
        reached |= (uint32_t)(a.x != kUnreached) << (4 * q) | (uint32_t)(a.y != kUnreached) << (4 * q + 1) |
                   (uint32_t)(a.z != kUnreached) << (4 * q + 2) | (uint32_t)(a.w != kUnreached) << (4 * q + 3);
        bits |= (uint32_t)(a.x == nd) << (4 * q) | (uint32_t)(a.y == nd) << (4 * q + 1) |
                (uint32_t)(a.z == nd) << (4 * q + 2) | (uint32_t)(a.w == nd) << (4 * q + 3);
      }
    }
    const uint32_t mask = __ldg(&init_mask[w]);
    visited[w] = reached | mask;
    front[w] = bits & ~mask;
  }
}

// kLat: latency mode (hub-free graphs run top-down only); kObs: observer
// snapshots (test instrumentation). Separate instantiations, so neither
// costs the general kernel registers.
template <int C, typename OffT, bool kLat, bool kObs>
__device__ __forceinline__ void bfs_traversal(const Params<OffT>& p) {
  __shared__ __align__(16) uint32_t s_list[kWarps][kListCap];  // BU id list / TD push buffer
  extern __shared__ __align__(16) uint4 s_lat[];  // latency mode: per-warp level buffers (kLatSmem)
  __shared__ uint32_t s_found[kWarps][kGroupWords];
  __shared__ unsigned long long s_snap[32];  // level-counter snapshots (GridBarrier)
  const unsigned warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  const unsigned long long tid = (unsigned long long)blockIdx.x * kThreads + threadIdx.x;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * kThreads;
  Ctl* ctl = p.ctl;
  GridBarrier bar{ctl, s_snap};
  WarpPush wp{s_list[warp], 0};
  // Trace records and the end-of-run summary come from the LAST CTA: CTA 0
  // holds the first frontier slices, the critical path of a small level.
  const bool leader = blockIdx.x == gridDim.x - 1 && threadIdx.x == 0;
  const CntSnap snap{s_snap};

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
      p.bm[1][w] = 0;
    }
    if (leader) {
      p.queue[0][0] = src;
      if (kLat) {
        const unsigned long long b = (unsigned long long)p.rowptr[src];
        p.lq[0][0] = make_uint4(src, (uint32_t)(p.rowptr[src + 1] - p.rowptr[src]), (uint32_t)b,
                                (uint32_t)(b >> 32));
      }
      for (int s = 0; s < 4; ++s) {
        LevelCnt z{};
        ctl->cnt[s] = z;
      }
      if (kLat) {
        for (int s = 0; s < 4 * 32; ++s) (&ctl->latk[0][0])[s] = 0;
      }
      ctl->overflow = 0;
      ctl->violations = 0;
      ctl->obs_count = 0;
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
  unsigned long long reached = 0, edges_total = 0;
  unsigned int bu_levels = 0;
  unsigned long long obs_pos = 0;  // observer log fill (identical in every CTA)
  unsigned long long t_start = leader ? globaltimer() : 0;
  bar.sync();

  // Bitmap bookkeeping (kClaimBitmap): fcur flips every level. A bottom-up
  // level reads bm[fcur] and writes every word of bm[fcur ^ 1]; a top-down
  // level touches no bitmap but `visited`, and the bitmap of its output is
  // built from dist only when bottom-up follows.
  uint32_t depth = 0;
  if constexpr (kLat && kLatLevels >= 2) {
    // ---- latency mode: kLatLevels levels per grid barrier (latency_round) ----

    unsigned long long carry = 0;  // degree of last round's lowered vertices (stale queue entries)
    for (unsigned r = 0;; ++r) {
      unsigned long long* ctr = ctl->latk[r & 3];
      if (leader) {
        // Round r + 2's row: its last readers finished before round r - 1's barrier.
        unsigned long long* z = ctl->latk[(r + 2) & 3];
        for (int i = 0; i < 32; ++i) z[i] = 0;
      }
      latency_round(p, depth, p.lq[qcur], qlen, p.lq[qcur ^ 1],
                    s_lat + warp * kLatLevels * LatRound<OffT>::kCap, ctr);
      bar.sync32(ctr);
      const unsigned long long* c = s_snap;
      // Per-level distinct sizes and edge counts of the round (see LatRound).
      unsigned long long dist_sz[kLatLevels + 1], edges[kLatLevels];
      dist_sz[0] = cur_distinct;
      edges[0] = c[kLkEdges0] - carry;
      for (int j = 1; j <= kLatLevels; ++j) dist_sz[j] = c[kLkWins + j] - c[kLkLow + j];
      for (int j = 1; j < kLatLevels; ++j) edges[j] = c[kLkExp + j] - c[kLkLowDeg + j];
      int levels_here = 1;
      while (levels_here < kLatLevels && dist_sz[levels_here] > 0) ++levels_here;
      if (leader) {
        const unsigned long long now = globaltimer();
        const long long span = (long long)(now - t_start) / levels_here;  // one round, split evenly
        for (int h = 0; h < levels_here && depth + h < p.rec_cap; ++h) {
          pbfs_level rec;
          rec.depth = depth + h;
          rec.phase = PBFS_TOP_DOWN;
          rec.frontier_size = rec.distinct_size = dist_sz[h];
          rec.duplicate_count = 0;
          rec.edges_examined = edges[h];
          rec.flush_events = 0;
          rec.elapsed_ns = span;
          p.records[depth + h] = rec;
        }
        t_start = now;
      }
      for (int h = 0; h < levels_here; ++h) {
        reached += dist_sz[h];
        edges_total += edges[h];
      }
      if (levels_here < kLatLevels || dist_sz[kLatLevels] == 0) {
        depth += levels_here - 1;  // the last level's index
        break;
      }
      carry = c[kLkLowDeg + kLatLevels];
      cur_distinct = dist_sz[kLatLevels];
      qlen = c[kLkPush] < p.qcap ? c[kLkPush] : p.qcap;
      qcur ^= 1;
      depth += kLatLevels;
    }
  } else
  for (;; ++depth) {
    LevelCnt* cnt = &ctl->cnt[depth & 3];
    if (leader) {
      LevelCnt z{};
      ctl->cnt[(depth + 2) & 3] = z;
    }
    WarpTally t;
    // Reduction claim (claim_batch): top-down levels of at least red_minq
    // frontier vertices set the next frontier with no-return reds instead of
    // returning claim atomics; the bitmap is counted and compacted after the
    // level (the next queue for top-down, the bitmap itself for bottom-up).
    uint32_t* red = nullptr;
    if constexpr (C == kClaimBitmap && !kLat && !kObs) {
      if (td && p.red_minq && qlen >= p.red_minq && p.policy != kPolicyBeamer) red = p.bm[fcur ^ 1];
    }
#if PBFS_TIMELINE
    // Diagnostic build: CTA 0 thread 0's view of the level (it holds the
    // first frontier slices), packed into the record's flush_events as four
    // 16-bit ns offsets from the level start.
    const bool tl_cta = blockIdx.x == 0 && threadIdx.x == 0;
    const unsigned long long tl0 = tl_cta ? globaltimer() : 0;
    unsigned long long tl_pack = 0;
    auto tl_mark = [&](int slot) {
      if (tl_cta) {
        const unsigned long long d = globaltimer() - tl0;
        tl_pack |= (d < 65535 ? d : 65535ull) << (16 * slot);
        if (slot == 3 && depth < p.rec_cap) p.records[depth].flush_events = tl_pack;
      }
    };
#else
    auto tl_mark = [](int) {};
#endif
    if (kLat && td) {
      WarpPush4 wp4{reinterpret_cast<uint4*>(s_list[warp]), 0};
      td_phase_latency(p, depth, p.lq[qcur], qlen, p.lq[qcur ^ 1], wp4, cnt, t);
      wp4.flush(p.lq[qcur ^ 1], &cnt->raw, p.qcap, &ctl->overflow);
      tl_mark(0);
    } else if (td) {
      uint32_t* qout = p.queue[qcur ^ 1];
      // No next-bitmap marks during the level (see front_from_dist).
      uint32_t* mark = nullptr;
      if (red) {
        // The next frontier accumulates in the bitmap that becomes bm[fcur]
        // after this level's flip.
        for (unsigned long long w = tid; w < p.words; w += nthreads) red[w] = 0;
        bar.sync();
      }
      td_phase_light<C>(p, depth, p.queue[qcur], qlen, qout, wp, cnt, t, mark, nullptr, hw_grid(),
                        red);
      tl_mark(0);
      if (p.max_degree > p.heavy_deg) {
        bar.sync(cnt);
        // Bounded by the capacity (an overflow is reported after the run).
        const unsigned int items = (unsigned long long)snap.heavy_count() < p.heavy_cap
                                       ? snap.heavy_count()
                                       : (unsigned int)p.heavy_cap;
        if (items) td_phase_heavy<C>(p, depth, items, qout, wp, cnt, t, mark, hw_grid(), red);
      }
      wp.flush(qout, &cnt->raw, p.qcap, &ctl->overflow);
    } else {
      // Unvisited non-isolated vertices left (every CTA tracks the same sums).
      const unsigned long long seen = reached + cur_distinct, live = p.n - p.isolated;
      const unsigned long long unv = live > seen ? live - seen : 0;
      // Sparse tasks only where they still give every warp one.
      const bool sparse =
          (p.force & kForceSparseBu) ||
          (unv * 64 < p.n && p.words >= gridDim.x * kWarps * 32u * (uint32_t)kBuSparseGroups);
      bu_phase(p, depth, p.bm[fcur], p.bm[fcur ^ 1], s_list[warp], s_found[warp], t,
               &cnt->bu_cursor, sparse);
      tl_mark(0);
    }
    warp_flush_tally(cnt, t, C == kClaimPlain, &ctl->violations);
    tl_mark(1);
    bar.sync(cnt);
    tl_mark(2);
    if (C == kClaimPlain && td) {
      // BFS-NonAtomic / plain-store hybrid: the marks collapse into the
      // distinct next frontier (the reference counts it with its seen_ scan,
      // kernels.cpp:409-420).
      compact_bitmap(p.bm[1], p.queue[qcur ^ 1], p.words, &cnt->conv_count, true, nullptr,
                     p.force & kForceWideCompact);
      bar.sync(cnt);
    }
    if (red) {
      // The distinct next frontier: count it and write it as the next queue.
      compact_bitmap(red, p.queue[qcur ^ 1], p.words, &cnt->conv_count, false, nullptr,
                     p.force & kForceWideCompact);
      bar.sync(cnt);
    }
    if (C == kClaimBitmap || !td) fcur ^= 1;  // this level's bitmap is the latest

    // ---- single section (kernels.cpp:384-464), evaluated by every CTA ----
    const unsigned long long produced =
        (C == kClaimPlain && td) || red ? (unsigned long long)snap.conv_count() : snap.produced();
    const unsigned long long raw = td && !red ? snap.raw() : produced;
    const unsigned long long edges = snap.edges();
    const unsigned long long pdeg = snap.degree();
    tl_mark(3);
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
        r.flush_events = 0;  // no local-buffer flushes to report on the GPU
        r.elapsed_ns = (long long)(now - t_start);
#if PBFS_TIMELINE
        pbfs_level* d = &p.records[depth];  // flush_events belongs to CTA 0 here
        d->depth = r.depth;
        d->phase = r.phase;
        d->frontier_size = r.frontier_size;
        d->distinct_size = r.distinct_size;
        d->duplicate_count = r.duplicate_count;
        d->edges_examined = r.edges_examined;
        d->elapsed_ns = r.elapsed_ns;
#else
        p.records[depth] = r;
#endif
      }
      t_start = now;
    }
    reached += cur_distinct;
    edges_total += edges;
    bu_levels += td ? 0 : 1;
    if (kObs && produced > 0) {
      // Observer snapshot of the frontier this level produced (emit_snapshot,
      // kernels.cpp:466-481): the next queue as pushed (top-down; the claims
      // are exclusive, or for plain stores collapsed into the distinct set),
      // or the produced bitmap's ids (bottom-up; the host sorts them
      // ascending). Entries land at obs_pos, which every CTA tracks
      // identically; ctl->obs_count follows it (bottom-up appends reserve
      // through it).
      if (obs_pos + produced > p.obs_cap) {
        if (leader) atomicExch(&ctl->overflow, 1u);
      } else if (td) {
        const uint32_t* qn = p.queue[qcur ^ 1];
        for (unsigned long long i = tid; i < produced; i += nthreads) p.obs[obs_pos + i] = qn[i];
        if (leader) ctl->obs_count = (unsigned int)(obs_pos + produced);
      } else {
        compact_bitmap(p.bm[fcur], p.obs, p.words, &ctl->obs_count, false);
        bar.sync();  // before any conversion clears the bitmap
      }
      obs_pos += produced;
    }
    if (raw == 0) break;
    unvisited_edges -= pdeg;
    const unsigned long long consumed = cur_distinct;
    const bool next_td = decide(td, produced, pdeg, consumed, unvisited_edges);
    if (td && next_td) {
      // Bounded by the queue capacity (an overflow is reported after the run).
      qlen = C == kClaimPlain ? produced : raw;
      if (qlen > p.qcap) qlen = p.qcap;
      qcur ^= 1;
    } else if (!td && next_td) {
      // Entering top-down: a queue from the produced bitmap
      // (count_bitmap_slice / write_dense_slice, kernels.cpp:225-241).
      // Plain-store top-down marks into bm[1] and needs it zero: this pass
      // clears the consumed bitmap and zeroes the other one.
      compact_bitmap(p.bm[fcur], p.queue[qcur], p.words, &cnt->conv_count, C == kClaimPlain,
                     C == kClaimPlain ? p.bm[fcur ^ 1] : nullptr, p.force & kForceWideCompact);
      bar.sync(cnt);
      qlen = snap.conv_count();
    } else if (C == kClaimBitmap && td && !next_td && !red) {
      // Entering bottom-up: the frontier bitmap from this level's distances
      // (a reduction-claim level left it in bm[fcur] already).
      front_from_dist(p.dist, depth + 1, p.bm[fcur], p.words, p.n, p.visited, p.init_mask);
      bar.sync();
    } else if (C == kClaimPlain && td && !next_td) {
      // Entering bottom-up after plain-store top-down levels (no visited
      // bits kept): visited and the frontier bitmap from dist.
      visited_front_from_dist(p.dist, depth + 1, p.visited, p.bm[fcur], p.words, p.n, p.init_mask);
      bar.sync();
    }
    // bottom-up -> bottom-up: nothing to convert.
    td = next_td;
    cur_raw = raw;
    cur_distinct = produced;
  }

  // Narrow copy of the distances for a batch's host transfer: 1 B per vertex
  // when every level fits (0xFF = unreached), else 2 B. No barrier needed:
  // the loop ended on one, after the last level's stores.
  if (p.pack) {
    const uint32_t bits = pack_bits(depth + 1, p.pack_min_bits);
    const uint32_t width = bits / 8;
    const uint4* d4 = reinterpret_cast<const uint4*>(p.dist);
    if (bits == 4) {
      // 32 vertices per 16 B: vertex v in byte v / 2, low nibble for even v.
      uint4* o = reinterpret_cast<uint4*>(p.pack);
      for (unsigned long long i = tid; i < (p.n + 31) / 32; i += nthreads) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 a = __ldcs(d4 + 8 * i + 2 * q);  // dist is padded to 32 entries
          const uint4 b = __ldcs(d4 + 8 * i + 2 * q + 1);
          w[q] = (a.x & 0xF) | (a.y & 0xF) << 4 | (a.z & 0xF) << 8 | (a.w & 0xF) << 12 |
                 (b.x & 0xF) << 16 | (b.y & 0xF) << 20 | (b.z & 0xF) << 24 | (b.w & 0xF) << 28;
        }
        o[i] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else if (width == 1) {
      uint4* o = reinterpret_cast<uint4*>(p.pack);
      for (unsigned long long i = tid; i < (p.n + 15) / 16; i += nthreads) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 a = __ldcs(d4 + 4 * i + q);  // dist is padded to 16 entries
          w[q] = (a.x & 0xFF) | (a.y & 0xFF) << 8 | (a.z & 0xFF) << 16 | (a.w & 0xFF) << 24;
        }
        o[i] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else if (width == 2) {
      uint2* o = reinterpret_cast<uint2*>(p.pack);
      for (unsigned long long i = tid; i < (p.n + 3) / 4; i += nthreads) {
        const uint4 a = __ldcs(d4 + i);
        o[i] = make_uint2((a.x & 0xFFFF) | a.y << 16, (a.z & 0xFFFF) | a.w << 16);
      }
    }
  }
  if (leader) {
    ctl->levels = depth + 1;
    ctl->bu_levels = bu_levels;
    ctl->reached = reached;
    ctl->edges = edges_total;
  }
}

template <int C, typename OffT, bool kLat = false, bool kObs = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks) bfs_persistent(Params<OffT> p) {
  bfs_traversal<C, OffT, kLat, kObs>(p);
}

// Latency mode runs one CTA per SM (g->lat_grid): the round's nested
// expansion gets the register file instead of spilling at the 3-CTA budget.
template <typename OffT>
__global__ void __launch_bounds__(kThreads, 1) bfs_latency(Params<OffT> p) {
  bfs_traversal<kClaimBitmap, OffT, true, false>(p);
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

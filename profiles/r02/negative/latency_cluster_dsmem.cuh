// Latency mode on ONE 16-CTA thread-block cluster with the visited set in
// distributed shared memory (Blackwell CGA + DSMEM).
//
// A deep hub-free graph run top-down only (config 3's mesh: ~3900 levels of
// ~4 K vertices) is bound by one level's dependent chain plus the level
// barrier, not by bytes. On 148 CTAs the chain's claim is an L2 atomic and
// the barrier a flip-bit word in L2 (~1.5 us). Here the whole traversal runs
// on one cluster of 16 CTAs x 1024 threads:
//   * the visited bitmap (n/8 bytes: 2 MiB for 2^24 vertices) is split over
//     the 16 CTAs' shared memory, so a claim is one atom.shared::cluster.or
//     on the owning CTA's slice (~200 cycles, against an L2 atomic);
//   * the level barrier is barrier.cluster (cluster.sync, ~380 cycles);
//   * everything else is the latency-mode path of pbfs_kernels.cuh: 16 B
//     queue entries {v, degree, row offset} in global memory, per-warp
//     flushes, warp-cooperative expansion.
// Used when the bitmap slice fits a CTA's shared memory and the device can
// place a 16-CTA cluster (cudaOccupancyMaxActiveClusters); else the
// 148-CTA latency kernel runs. Distances / records are identical.
#pragma once

#include <cooperative_groups.h>

#include "pbfs_kernels.cuh"

namespace pbfs {
namespace dev {

constexpr int kClusterCtas = 16;
constexpr int kClThreads = 1024;
constexpr int kClWarps = kClThreads / 32;
constexpr int kClPush = 64;  // 16 B entries per warp flush buffer

__device__ __forceinline__ uint32_t dsmem_atom_or(uint32_t local_saddr, uint32_t rank, uint32_t bit) {
  uint32_t raddr, old;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(local_saddr), "r"(rank));
  asm volatile("atom.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(raddr), "r"(bit) : "memory");
  return old;
}

// The cluster-wide level barrier: barrier.cluster.arrive.release +
// wait.acquire (global and distributed-shared writes of the level ordered
// before any read of the next), then thread 0 snapshots the level counters.
__device__ __forceinline__ void cluster_level_sync(const void* src, unsigned long long* snap) {
  cooperative_groups::this_cluster().sync();
  if (src && threadIdx.x == 0) {
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
    const ulonglong2 a = __ldcg(s2), b = __ldcg(s2 + 1), c = __ldcg(s2 + 2), d = __ldcg(s2 + 3);
    snap[0] = a.x; snap[1] = a.y; snap[2] = b.x; snap[3] = b.y;
    snap[4] = c.x; snap[5] = c.y; snap[6] = d.x; snap[7] = d.y;
  }
  __syncthreads();
}

template <int K, typename OffT>
__device__ __forceinline__ void claim_cluster(const Params<OffT>& p, uint32_t nd, const uint32_t (&v)[K],
                                              uint32_t okm, uint32_t bm_saddr, uint32_t wpc,
                                              uint4* qout, uint4* buf, int& count, LevelCnt* cnt,
                                              WarpTally& t) {
  uint32_t w[K];
  OffT b0[K], b1[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t word = v[k] >> 5;
    const uint32_t bit = 1u << (v[k] & 31);
    w[k] = 0xffffffffu;
    if ((okm >> k) & 1u) w[k] = dsmem_atom_or(bm_saddr + 4u * (word % wpc), word / wpc, bit);
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
  static_assert(kClPush >= 16 * K, "cluster latency discovery buffer");
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
    if (count + total > kClPush) {
      WarpPush4 wp{buf, count};
      wp.flush(qout, &cnt->raw, p.qcap, &p.ctl->overflow);
      count = 0;
    }
    uint32_t pos = count + incl - c;
#pragma unroll
    for (int k = h * K / 2; k < (h + 1) * K / 2; ++k) {
      if ((winmask >> k) & 1u) {
        const unsigned long long b = (unsigned long long)b0[k];
        buf[pos++] = make_uint4(v[k], (uint32_t)(b1[k] - b0[k]), (uint32_t)b, (uint32_t)(b >> 32));
      }
    }
    count += total;
  }
}

template <typename OffT>
__global__ void __launch_bounds__(kClThreads, 1) bfs_cluster_latency(Params<OffT> p, uint32_t wpc) {
  extern __shared__ uint32_t s_bm[];  // this CTA's slice of the visited bitmap: wpc words
  __shared__ __align__(16) uint4 s_push[kClWarps][kClPush];
  __shared__ unsigned long long s_snap[8];
  const unsigned rank = cooperative_groups::this_cluster().block_rank();
  const unsigned warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  const unsigned FULL = 0xffffffffu;
  const unsigned long long tid = (unsigned long long)rank * kClThreads + threadIdx.x;
  const unsigned long long nthreads = (unsigned long long)kClusterCtas * kClThreads;
  const unsigned warps_total = kClusterCtas * kClWarps;
  Ctl* ctl = p.ctl;
  const bool leader = rank == kClusterCtas - 1 && threadIdx.x == 0;
  const uint32_t bm_saddr = (uint32_t)__cvta_generic_to_shared(s_bm);
  const CntSnap snap{s_snap};

  // ---- init (kernels.cpp:72-102,144-163) --------------------------------
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
    const unsigned long long w0 = (unsigned long long)rank * wpc;
    for (unsigned long long i = threadIdx.x; i < wpc; i += kClThreads) {
      const unsigned long long w = w0 + i;
      uint32_t m = w < p.words ? p.init_mask[w] : 0xffffffffu;
      if (w == (src >> 5)) m |= 1u << (src & 31);
      s_bm[i] = m;
    }
    if (leader) {
      const unsigned long long b = (unsigned long long)p.rowptr[src];
      p.lq[0][0] = make_uint4(src, (uint32_t)(p.rowptr[src + 1] - p.rowptr[src]), (uint32_t)b,
                              (uint32_t)(b >> 32));
      for (int s = 0; s < 4; ++s) {
        LevelCnt z{};
        ctl->cnt[s] = z;
      }
      ctl->overflow = 0;
      ctl->violations = 0;
      ctl->obs_count = 0;
    }
  }
  int qcur = 0;
  unsigned long long qlen = 1, cur_raw = 1, reached = 0, edges_total = 0;
  unsigned long long t_start = leader ? globaltimer() : 0;
  cluster_level_sync(nullptr, s_snap);

  uint32_t depth = 0;
  for (;; ++depth) {
    LevelCnt* cnt = &ctl->cnt[depth & 3];
    if (leader) {
      LevelCnt z{};
      ctl->cnt[(depth + 2) & 3] = z;
    }
    WarpTally t;
    uint4* buf = s_push[warp];
    int count = 0;
    const uint4* qin = p.lq[qcur];
    uint4* qout = p.lq[qcur ^ 1];
    const uint32_t nd = depth + 1;
    // Top-down over the queue (td_phase_latency): 32-entry slices per warp,
    // static first slice, then the cursor.
    // Adaptive slice width and warp-major dealing over the 16 CTAs (as
    // td_phase_latency), so a small level spreads over every SM.
    unsigned W = 32;
    while (W > 1 && (unsigned long long)warps_total * (W / 2) >= qlen) W /= 2;
    unsigned long long base = (unsigned long long)(warp * kClusterCtas + rank) * W;
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
        constexpr int K = 4;
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
          claim_cluster<K>(p, nd, v, okm, bm_saddr, wpc, qout, buf, count, cnt, t);
        }
      }
      if (qlen <= (unsigned long long)warps_total * W) break;
      unsigned int nb = 0;
      if (lane == 0) nb = atomicAdd(&cnt->td_cursor, 32u);
      base = (unsigned long long)warps_total * 32 + __shfl_sync(FULL, nb, 0);
    }
    {
      WarpPush4 wp{buf, count};
      wp.flush(qout, &cnt->raw, p.qcap, &ctl->overflow);
    }
    warp_flush_tally(cnt, t, false, &ctl->violations);
    cluster_level_sync(cnt, s_snap);

    // ---- single section (kernels.cpp:384-464), every CTA ----------------
    const unsigned long long raw = snap.raw();
    const unsigned long long edges = snap.edges();
    if (leader) {
      const unsigned long long now = globaltimer();
      if (depth < p.rec_cap) {
        pbfs_level r;
        r.depth = depth;
        r.phase = PBFS_TOP_DOWN;
        r.frontier_size = cur_raw;
        r.distinct_size = cur_raw;
        r.duplicate_count = 0;
        r.edges_examined = edges;
        r.flush_events = 0;
        r.elapsed_ns = (long long)(now - t_start);
        p.records[depth] = r;
      }
      t_start = now;
    }
    reached += cur_raw;
    edges_total += edges;
    if (raw == 0) break;
    qlen = raw < p.qcap ? raw : p.qcap;
    qcur ^= 1;
    cur_raw = raw;
  }
  // Narrow copy of the distances for a batch / pageable host transfer (as
  // bfs_persistent; the loop ended on a cluster barrier).
  if (p.pack) {
    const uint32_t width = pack_width(depth + 1);
    const uint4* d4 = reinterpret_cast<const uint4*>(p.dist);
    if (width == 1) {
      uint4* o = reinterpret_cast<uint4*>(p.pack);
      for (unsigned long long i = tid; i < (p.n + 15) / 16; i += nthreads) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 a = __ldcs(d4 + 4 * i + q);
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
    ctl->bu_levels = 0;
    ctl->reached = reached;
    ctl->edges = edges_total;
  }
}

}  // namespace dev
}  // namespace pbfs

// Internal: the per-rank partition handle of the 1D vertex-partitioned
// engines (pbfs_part.cu: per-level launches + a caller-run allgather;
// pbfs_multi.cu: one persistent launch per device with the exchange fused
// into the level kernels over peer memory).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "pbfs_internal.h"
#include "pbfs_kernels.cuh"

namespace pbfs {
namespace part {

// ---- relabel pi on [0, 2^k) ---------------------------------------------------
struct Relabel {
  uint32_t k = 0;       // n_pad = 2^k when hashed
  uint32_t hashed = 0;  // 0: identity
  uint64_t mask = 0;
  uint64_t a = 0, b = 0;
  uint32_t h = 0;
};


inline Relabel make_relabel(uint32_t k, bool hashed) {
  Relabel r;
  r.k = k;
  r.hashed = hashed && k >= 2;
  r.mask = k >= 64 ? ~0ull : ((1ull << k) - 1);
  r.a = 0x9E3779B97F4A7C15ull & r.mask;
  r.b = 0xC2B2AE3D27D4EB4Full & r.mask;
  r.a |= 1;
  r.b |= 1;
  r.h = (k + 1) / 2;  // 2h >= k: x ^= x >> h is its own inverse
  return r;
}

__host__ __device__ __forceinline__ uint64_t pi_fwd(const Relabel& r, uint64_t v) {
  if (!r.hashed) return v;
  uint64_t x = (v * r.a) & r.mask;
  x ^= x >> r.h;
  return (x * r.b) & r.mask;
}

constexpr uint32_t kPartRecCap = 1u << 16;  // device level records kept per traversal

struct PartState {
  unsigned long long qlen;          // current top-down queue length
  unsigned long long distinct;      // popcount of the gathered next bitmap
  unsigned long long cur_distinct;  // current frontier size
  unsigned int td, fcur, depth, done, compact;
  unsigned int pad[3];
};


}  // namespace part
}  // namespace pbfs

struct pbfs_part {
  int device = 0;
  uint32_t rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  pbfs::part::Relabel rl;
  uint64_t n = 0, npad = 0, nloc = 0, lo = 0;
  uint64_t words_total = 0, lwords = 0;
  uint64_t m_loc = 0;
  uint32_t offb = 8;
  bool shared = false;
  int grid = 0;
  // row slice (bottom-up)
  unsigned long long* rowloc = nullptr;  // nloc + 1
  uint32_t* colrow = nullptr;            // m_loc, global pi-ids
  uint32_t* first = nullptr;             // nloc + 1: first row-slice neighbour
  // order-preserving numbering (k_owner_gid): vertex -> gid, gid -> vertex
  uint32_t* gid = nullptr;               // n
  uint32_t* inv = nullptr;               // npad (0xFFFFFFFF = padding)
  std::vector<uint32_t> gid_host;        // lazily copied for pbfs_part_unrelabel_host
  // column slice (top-down)
  unsigned long long* colptr = nullptr;  // npad + 1
  uint32_t* colcol = nullptr;            // m_loc, local ids
  uint64_t col_maxdeg = 0, heavy_cap = 0;
  size_t persist = 0;  // persisting-L2 set-aside available to the level kernels
  // traversal state
  uint32_t* dist = nullptr;      // nloc
  uint32_t* visited = nullptr;   // lwords
  uint32_t* mask = nullptr;      // lwords
  uint32_t* bm[2] = {nullptr, nullptr};  // full bitmaps (own or shared)
  int fcur = 0;                  // bm[fcur] = current frontier, bm[fcur^1] = next
  uint32_t* queue[2] = {nullptr, nullptr};
  pbfs::dev::HeavyItem* heavy = nullptr;
  pbfs::dev::Ctl* ctl = nullptr;
  pbfs::part::PartState* st = nullptr;
  pbfs::part::PartState* st_host = nullptr;  // pinned mirror
  std::vector<void*> allocs;
  pbfs_level* recs = nullptr;    // device, kPartRecCap level records
  // host mirror of the level state (identical on every rank)
  uint32_t issued = 0;           // levels enqueued since begin
  uint32_t depth = 0;
  bool td = true;
  int policy = pbfs::dev::kPolicyFraction;
  double threshold = 0.05;
};


namespace pbfs {
namespace part {

// Builds one rank's partition (row + column slices, gid maps, scratch) on
// `device` from a resident full CSR (pbfs_part.cu).
pbfs_status create(uint64_t n, bool symmetric, int device, const void* rowptr, const uint32_t* col,
                   uint32_t offb, const pbfs_part_options* opt, pbfs_part** out);
void release(pbfs_part* g);
// Level-kernel views of a partition: column slice (top-down), row slice
// (bottom-up).
pbfs::dev::Params<unsigned long long> td_params(const pbfs_part* g);
pbfs::dev::Params<unsigned long long> bu_params(const pbfs_part* g);

}  // namespace part
}  // namespace pbfs

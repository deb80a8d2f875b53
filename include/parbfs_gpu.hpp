// parbfs_gpu.hpp — the reference `parbfs` C++ API served by the B200 C ABI.
//
// Header-only adapter a maintainer adds next to the reference's
// core/include/parbfs headers. It keeps the reference's
// types and signatures:
//   parbfs::gpu::run_bfs(const CsrGraph&, VertexId, const KernelConfig&,
//                        const GraphStats&)            ~ kernels.hpp:80-81
//   parbfs::gpu::bfs(const CsrGraph&, VertexId, const KernelConfig&)
//                                                      ~ kernels.hpp:34-75
//   parbfs::gpu::kernel_fn()  -> parbfs::KernelFn      ~ timing.hpp:17-18
// and rethrows C-ABI statuses as the reference exception classes
// (types.hpp:25-68). The CsrGraph is borrowed zero-copy (its u64 offsets and
// u32 columns are exactly pbfs_csr's layout); one device handle is cached per
// graph identity (address, n, m, device) so a KernelFn called per source does
// not re-upload.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "parbfs/graph_stats.hpp"
#include "parbfs/kernels.hpp"
#include "parbfs/timing.hpp"
#include "pbfs.h"

namespace parbfs::gpu {

inline void throw_status(pbfs_status st) {
  if (st == PBFS_OK) return;
  const std::string msg = pbfs_last_error();
  switch (st) {
    case PBFS_E_INPUT: throw InputError(msg);
    case PBFS_E_CONFIG: throw ConfigError(msg);
    case PBFS_E_FORMAT: throw FormatError(msg);
    case PBFS_E_CAPACITY: throw CapacityError(msg);
    case PBFS_E_METRIC: throw MetricError(msg);
    case PBFS_E_CORRECTNESS: throw CorrectnessError(msg);
    default: throw Error(msg);
  }
}

inline pbfs_config to_c(const KernelConfig& c) {
  pbfs_config out;
  pbfs_config_init(&out);
  out.variant = static_cast<uint32_t>(c.variant);
  out.worker_count = c.worker_count;
  out.hybrid_threshold_fraction = c.hybrid_threshold_fraction;
  out.alpha = c.alpha;
  out.beta = c.beta;
  out.flush_capacity = c.flush_capacity;
  out.force_top_down_only = c.force_top_down_only ? 1u : 0u;
  out.validate_same_value_stores = c.validate_same_value_stores ? 1u : 0u;
  out.racy_visited_claim = c.racy_visited_claim ? 1u : 0u;
  return out;
}

// One resident device graph per (CsrGraph address, n, m, device).
class DeviceGraphCache {
 public:
  static DeviceGraphCache& instance() {
    static DeviceGraphCache cache;
    return cache;
  }
  pbfs_graph* get(const CsrGraph& g, int device) {
    const auto key = std::make_tuple(static_cast<const void*>(&g), g.vertex_count, g.edge_count,
                                     device);
    std::lock_guard<std::mutex> lock(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) return it->second;
    pbfs_csr csr{};
    csr.vertex_count = g.vertex_count;
    csr.edge_count = g.edge_count;
    csr.row_offsets = g.row_offsets.data();
    csr.column_indices = g.column_indices.data();
    csr.offset_bytes = sizeof(EdgeOffset);
    csr.symmetric = g.symmetric ? 1u : 0u;
    pbfs_graph_options opt{device, 0};
    pbfs_graph* h = nullptr;
    throw_status(pbfs_graph_create(&csr, &opt, &h));
    map_.emplace(key, h);
    return h;
  }
  // Call when a CsrGraph is destroyed or mutated (identity is by address).
  void evict(const CsrGraph& g) {
    std::lock_guard<std::mutex> lock(mu_);
    for (auto it = map_.begin(); it != map_.end();) {
      if (std::get<0>(it->first) == static_cast<const void*>(&g)) {
        pbfs_graph_destroy(it->second);
        it = map_.erase(it);
      } else {
        ++it;
      }
    }
  }
  ~DeviceGraphCache() {
    for (auto& kv : map_) pbfs_graph_destroy(kv.second);
  }

 private:
  std::mutex mu_;
  std::map<std::tuple<const void*, std::uint64_t, std::uint64_t, int>, pbfs_graph*> map_;
};

// bfs_conventional / bfs_nonatomic / bfs_hybrid / bfs_hybrid_beamer /
// bfs_visited_bitmap(inline) by config.variant, on the GPU.
inline BfsResult bfs(const CsrGraph& g, VertexId source, const KernelConfig& config,
                     int device = 0) {
  validate(config);
  if (source >= g.vertex_count) {
    throw InputError("source vertex " + std::to_string(source) +
                     " is out of range for a graph with " + std::to_string(g.vertex_count) +
                     " vertices");
  }
  pbfs_graph* h = DeviceGraphCache::instance().get(g, device);
  const pbfs_config c = to_c(config);
  BfsResult r;
  r.distances.resize(g.vertex_count);
  std::vector<pbfs_level> levels(
      static_cast<std::size_t>(std::min<std::uint64_t>(g.vertex_count + 1, 1u << 20)));
  pbfs_run_info info{};
  throw_status(pbfs_bfs(h, source, &c, r.distances.data(), levels.data(),
                        static_cast<uint32_t>(levels.size()), &info));
  r.trace.variant = config.variant;
  r.trace.worker_count = config.worker_count;
  r.trace.source = source;
  r.trace.same_value_violations = info.same_value_violations;
  r.trace.total_elapsed =
      std::chrono::nanoseconds(static_cast<std::int64_t>(info.device_ms * 1e6));
  for (std::uint32_t i = 0; i < info.levels && i < levels.size(); ++i) {
    LevelRecord rec;
    rec.depth = levels[i].depth;
    rec.phase = levels[i].phase ? TraversalPhase::BottomUp : TraversalPhase::TopDown;
    rec.frontier_size = levels[i].frontier_size;
    rec.distinct_size = levels[i].distinct_size;
    rec.duplicate_count = levels[i].duplicate_count;
    rec.edges_examined = levels[i].edges_examined;
    rec.flush_events = levels[i].flush_events;
    rec.elapsed = std::chrono::nanoseconds(levels[i].elapsed_ns);
    r.trace.records.push_back(rec);
  }
  return r;
}

// kernels.cpp:657-691 semantics: large-diameter graphs run top-down only.
inline BfsResult run_bfs(const CsrGraph& g, VertexId source, const KernelConfig& config,
                         const GraphStats& stats, int device = 0) {
  KernelConfig effective = config;
  if (stats.category == GraphCategory::LargeDiameter) effective.force_top_down_only = true;
  return bfs(g, source, effective, device);
}

// The plugin slot: time_run(graph, src, cfg, trials, warmups, gpu::kernel_fn()).
inline KernelFn kernel_fn(int device = 0) {
  return [device](const CsrGraph& g, VertexId s, const KernelConfig& c) {
    return run_bfs(g, s, c, compute_stats(g), device);
  };
}

}  // namespace parbfs::gpu

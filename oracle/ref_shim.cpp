// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// A C-ABI shim over the UNMODIFIED reference library (`parbfs`, built from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load it. It exposes exactly the reference entry points the
// parity checks need:
//   generate()            proj/core/src/generator.cpp:41-92
//   build_csr()           proj/core/src/csr_graph.cpp:11-55
//   bfs_serial()          proj/core/src/kernels.cpp:19-41
//   run_bfs() / bfs_*()   proj/core/src/kernels.cpp:586-691
//   compute_stats()       proj/core/src/graph_stats.cpp:9-25
// Exceptions are mapped onto integer codes that mirror include/pbfs.h.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "parbfs/csr_graph.hpp"
#include "parbfs/generator.hpp"
#include "parbfs/graph_stats.hpp"
#include "parbfs/kernel_config.hpp"
#include "parbfs/kernels.hpp"
#include "parbfs/types.hpp"

namespace {
thread_local std::string g_err;

int map_exception() {
  try {
    throw;
  } catch (const parbfs::InputError& e) {
    g_err = e.what();
    return 1;
  } catch (const parbfs::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const parbfs::FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const parbfs::CapacityError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}
}  // namespace

extern "C" {

struct ref_graph {
  parbfs::CsrGraph g;
};

struct ref_level {
  uint32_t depth;
  uint32_t phase;  // 0 top-down, 1 bottom-up
  uint64_t frontier_size;
  uint64_t distinct_size;
  uint64_t duplicate_count;
  uint64_t edges_examined;
  uint64_t flush_events;
  int64_t elapsed_ns;
};

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_graph_generate(int kind, uint32_t scale, uint32_t edge_factor,
                       uint64_t seed, ref_graph** out) {
  try {
    parbfs::GeneratorSpec spec;
    spec.kind = kind == 1 ? parbfs::GeneratorKind::Kronecker
                          : parbfs::GeneratorKind::UniformRandom;
    spec.scale = scale;
    spec.edge_factor = edge_factor;
    spec.seed = seed;
    *out = new ref_graph{parbfs::generate(spec)};
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_graph_build(const uint32_t* pairs, uint64_t npairs, uint64_t n,
                    int symmetrize, ref_graph** out) {
  try {
    std::vector<parbfs::EdgePair> e(npairs);
    for (uint64_t i = 0; i < npairs; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
    *out = new ref_graph{parbfs::build_csr(e, n, symmetrize != 0)};
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Wraps an existing CSR (offsets widened to u64 by the caller) without
// rebuilding it, so the reference kernels run on exactly our graph.
int ref_graph_from_csr(uint64_t n, uint64_t m, const uint64_t* offsets,
                       const uint32_t* col, int symmetric, ref_graph** out) {
  try {
    auto* r = new ref_graph;
    r->g.vertex_count = n;
    r->g.edge_count = m;
    r->g.row_offsets.assign(offsets, offsets + n + 1);
    r->g.column_indices.assign(col, col + m);
    r->g.symmetric = symmetric != 0;
    *out = r;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

void ref_graph_info(const ref_graph* r, uint64_t* n, uint64_t* m,
                    int* symmetric) {
  *n = r->g.vertex_count;
  *m = r->g.edge_count;
  *symmetric = r->g.symmetric ? 1 : 0;
}

void ref_graph_export(const ref_graph* r, uint64_t* offsets, uint32_t* col) {
  std::memcpy(offsets, r->g.row_offsets.data(),
              r->g.row_offsets.size() * sizeof(uint64_t));
  std::memcpy(col, r->g.column_indices.data(),
              r->g.column_indices.size() * sizeof(uint32_t));
}

void ref_graph_free(ref_graph* r) { delete r; }

int ref_bfs_serial(const ref_graph* r, uint32_t source, uint32_t* dist) {
  try {
    auto d = parbfs::bfs_serial(r->g, source);
    std::memcpy(dist, d.data(), d.size() * sizeof(uint32_t));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_stats(const ref_graph* r, double threshold, double* avg_degree,
              uint64_t* max_degree, int* large_diameter) {
  try {
    auto s = parbfs::compute_stats(r->g, threshold);
    *avg_degree = s.average_degree;
    *max_degree = s.max_degree;
    *large_diameter = s.category == parbfs::GraphCategory::LargeDiameter;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// variant: parbfs::KernelVariant numbering (Serial=0 ... PeriodicFlush=7).
// dispatch != 0 routes through run_bfs with compute_stats (the category
// dispatcher, kernels.cpp:657-691); otherwise the bfs_* entry is called
// directly like test_kernels.cpp:18-41. wall_ns receives the call's
// steady-clock duration (the reference's own time_run clock).
int ref_run(const ref_graph* r, uint32_t source, int variant, uint32_t workers,
            double threshold, double alpha, double beta, int force_td,
            int dispatch, uint32_t* dist, ref_level* levels, uint32_t cap,
            uint32_t* nlevels, int64_t* wall_ns) {
  try {
    parbfs::KernelConfig cfg;
    cfg.variant = static_cast<parbfs::KernelVariant>(variant);
    cfg.worker_count = workers;
    cfg.hybrid_threshold_fraction = threshold;
    cfg.alpha = alpha;
    cfg.beta = beta;
    cfg.force_top_down_only = force_td != 0;
    parbfs::BfsResult res;
    const auto t0 = std::chrono::steady_clock::now();
    if (dispatch) {
      res = parbfs::run_bfs(r->g, source, cfg, parbfs::compute_stats(r->g));
    } else {
      switch (cfg.variant) {
        case parbfs::KernelVariant::Serial:
          res.distances = parbfs::bfs_serial(r->g, source);
          break;
        case parbfs::KernelVariant::Conventional:
          res = parbfs::bfs_conventional(r->g, source, cfg);
          break;
        case parbfs::KernelVariant::NonAtomic:
          res = parbfs::bfs_nonatomic(r->g, source, cfg);
          break;
        case parbfs::KernelVariant::Hybrid:
          res = parbfs::bfs_hybrid(r->g, source, cfg);
          break;
        case parbfs::KernelVariant::HybridBeamer:
          res = parbfs::bfs_hybrid_beamer(r->g, source, cfg);
          break;
        case parbfs::KernelVariant::VisitedBitmapInline:
          res = parbfs::bfs_visited_bitmap(r->g, source, cfg, false);
          break;
        case parbfs::KernelVariant::VisitedBitmapDeferred:
          res = parbfs::bfs_visited_bitmap(r->g, source, cfg, true);
          break;
        case parbfs::KernelVariant::TopDownPeriodicFlush:
          res = parbfs::bfs_topdown_periodic_flush(r->g, source, cfg);
          break;
      }
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_ns) {
      *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0)
                     .count();
    }
    if (dist) {
      std::memcpy(dist, res.distances.data(),
                  res.distances.size() * sizeof(uint32_t));
    }
    const auto& rec = res.trace.records;
    if (nlevels) *nlevels = static_cast<uint32_t>(rec.size());
    if (levels) {
      for (size_t i = 0; i < rec.size() && i < cap; ++i) {
        levels[i].depth = rec[i].depth;
        levels[i].phase =
            rec[i].phase == parbfs::TraversalPhase::BottomUp ? 1 : 0;
        levels[i].frontier_size = rec[i].frontier_size;
        levels[i].distinct_size = rec[i].distinct_size;
        levels[i].duplicate_count = rec[i].duplicate_count;
        levels[i].edges_examined = rec[i].edges_examined;
        levels[i].flush_events = rec[i].flush_events;
        levels[i].elapsed_ns = rec[i].elapsed.count();
      }
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"

// TEST DRIVER for the C++ drop-in (include/parbfs_gpu.hpp), compiled against
// the UNMODIFIED reference headers and linked with the reference library
// (oracle/_ref/libparbfs_ref.so) plus libpbfs.so by `make -C oracle adapter`
// in the container that has /root/reference; the binary travels to the GPU
// box (oracle/_ref/ is git-ignored, not gpurun-ignored). Modes:
//   criterion1      acceptance.cpp:112-147 through gpu::run_bfs: 200
//                   generated graphs x 5 sources x the GPU variants against
//                   the reference's bfs_serial. Every graph is a fresh
//                   `const CsrGraph` in the same stack slot -- the pattern
//                   the device cache must not confuse.
//   timerun         the reference's own oracle-checked time_run over
//                   gpu::kernel_fn(); two equal-sized graphs rebuilt at one
//                   address; the LevelObserver through the adapter.
//   multi           the same calls over a device list (the graph partitioned
//                   over {0,0} and {0,0,0}: loopback partitions on one GPU
//                   through the multi-GPU exchange code): criterion-1 graphs
//                   against bfs_serial, time_run over gpu::kernel_fn(devices).
//   percall FILE N  plugin-slot e2e: read a CSR1 file into a CsrGraph,
//                   call gpu::kernel_fn() once per source
//                   (bfsbench pick_sources rule, seed 1) and print GTEPS per
//                   call (steady clock around the KernelFn, i.e. including
//                   the BfsResult's host distance array).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "parbfs/generator.hpp"
#include "parbfs/graph_io.hpp"
#include "parbfs/graph_stats.hpp"
#include "parbfs/kernels.hpp"
#include "parbfs/timing.hpp"
#include "parbfs_gpu.hpp"

using namespace parbfs;

namespace {

std::vector<VertexId> sources_of(const CsrGraph& g, std::size_t count, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<VertexId> out;
  while (out.size() < count) {
    const auto v = static_cast<VertexId>(rng() % g.vertex_count);
    if (g.degree(v) > 0) out.push_back(v);
  }
  return out;
}

int criterion1() {
  const KernelVariant variants[] = {KernelVariant::Conventional, KernelVariant::NonAtomic,
                                    KernelVariant::Hybrid, KernelVariant::HybridBeamer,
                                    KernelVariant::VisitedBitmapInline};
  std::uint64_t runs = 0;
  for (int i = 0; i < 200; ++i) {
    GeneratorSpec spec;
    spec.kind = (i % 2 == 0) ? GeneratorKind::UniformRandom : GeneratorKind::Kronecker;
    spec.scale = 4 + static_cast<std::uint32_t>(i % 9);
    spec.edge_factor = 1 + static_cast<std::uint32_t>((i * 5) % 16);
    spec.seed = 7000 + static_cast<std::uint64_t>(i);
    const CsrGraph g = generate(spec);
    const GraphStats stats = compute_stats(g);
    for (const VertexId src : sources_of(g, 5, static_cast<std::uint64_t>(i))) {
      const DistanceArray want = bfs_serial(g, src);
      for (const KernelVariant v : variants) {
        KernelConfig cfg;
        cfg.variant = v;
        const BfsResult got = gpu::run_bfs(g, src, cfg, stats);
        ++runs;
        if (got.distances != want) {
          std::printf("FAIL criterion1 graph %d (%s) variant %s source %u\n", i,
                      to_string(spec).c_str(), to_string(v).c_str(), src);
          return 1;
        }
      }
    }
  }
  std::printf("OK criterion1 %llu runs through gpu::run_bfs, cache holds %zu graphs\n",
              static_cast<unsigned long long>(runs), gpu::DeviceGraphCache::instance().size());
  return 0;
}

CsrGraph star_or_path(bool star) {
  std::vector<std::pair<VertexId, VertexId>> e;
  for (VertexId v = 1; v < 5; ++v) e.emplace_back(star ? 0 : v - 1, v);
  return build_csr(e, 5, true);
}

int timerun() {
  const CsrGraph g = generate({GeneratorKind::Kronecker, 12, 16, 3});
  KernelConfig cfg;
  cfg.variant = KernelVariant::Hybrid;
  const TimingReport rep = time_run(g, 0, cfg, 3, 1, gpu::kernel_fn());
  std::printf("time_run median %lld ns\n", static_cast<long long>(rep.median.count()));
  // Same stack slot, same n and m (5 vertices, 8 arcs), different graphs.
  for (int round = 0; round < 4; ++round) {
    const CsrGraph h = star_or_path(round % 2 == 0);
    const BfsResult r = gpu::run_bfs(h, 4, cfg, compute_stats(h));
    if (r.distances != bfs_serial(h, 4)) {
      std::printf("FAIL stale device copy for round %d\n", round);
      return 1;
    }
  }
  // LevelObserver through the adapter: every reached vertex exactly once, at
  // its distance, seed first.
  std::map<std::uint32_t, std::multiset<VertexId>> seen;
  KernelConfig obs = cfg;
  obs.level_observer = [&](const LevelSnapshot& s) {
    seen[s.depth].insert(s.entries.begin(), s.entries.end());
  };
  const VertexId src = sources_of(g, 1, 9)[0];
  const BfsResult r = gpu::run_bfs(g, src, obs, compute_stats(g));
  const DistanceArray want = bfs_serial(g, src);
  std::uint64_t total = 0;
  for (const auto& [d, set] : seen) {
    for (VertexId v : set) {
      if (want[v] != d) {
        std::printf("FAIL observer: vertex %u snapshot at depth %u, distance %u\n", v, d, want[v]);
        return 1;
      }
    }
    total += set.size();
  }
  const auto reached = static_cast<std::uint64_t>(
      std::count_if(want.begin(), want.end(), [](std::uint32_t x) { return x != kUnreached; }));
  if (total != reached || r.distances != want || seen[0] != std::multiset<VertexId>{src}) {
    std::printf("FAIL observer totals %llu vs %llu\n", static_cast<unsigned long long>(total),
                static_cast<unsigned long long>(reached));
    return 1;
  }
  std::printf("OK timerun + cache identity + observer (%zu snapshots)\n", seen.size());
  return 0;
}

int multi() {
  std::uint64_t runs = 0;
  for (const std::vector<std::int32_t>& devs :
       {std::vector<std::int32_t>{0, 0}, std::vector<std::int32_t>{0, 0, 0}}) {
    for (int i = 0; i < 40; ++i) {
      GeneratorSpec spec;
      spec.kind = (i % 2 == 0) ? GeneratorKind::UniformRandom : GeneratorKind::Kronecker;
      spec.scale = 4 + static_cast<std::uint32_t>(i % 9);
      spec.edge_factor = 1 + static_cast<std::uint32_t>((i * 5) % 16);
      spec.seed = 9000 + static_cast<std::uint64_t>(i);
      const CsrGraph g = generate(spec);
      const GraphStats stats = compute_stats(g);
      KernelConfig cfg;
      cfg.variant = KernelVariant::Hybrid;
      for (const VertexId src : sources_of(g, 3, static_cast<std::uint64_t>(i))) {
        const BfsResult got = gpu::run_bfs(g, src, cfg, stats, devs);
        ++runs;
        if (got.distances != bfs_serial(g, src)) {
          std::printf("FAIL multi graph %d (%s) on %zu partitions source %u\n", i,
                      to_string(spec).c_str(), devs.size(), src);
          return 1;
        }
      }
    }
    const CsrGraph g = generate({GeneratorKind::Kronecker, 12, 16, 3});
    KernelConfig cfg;
    cfg.variant = KernelVariant::Hybrid;
    const TimingReport rep = time_run(g, 0, cfg, 3, 1, gpu::kernel_fn(devs));
    std::printf("time_run over %zu partitions: median %lld ns\n", devs.size(),
                static_cast<long long>(rep.median.count()));
  }
  std::printf("OK multi %llu runs through gpu::run_bfs over device lists\n",
              static_cast<unsigned long long>(runs));
  return 0;
}

// The CSR1 file (graph_io.hpp layout) read straight into a CsrGraph: the
// reference's own load_binary_csr parses it element by element (minutes at
// RMAT-26). The file comes from the symmetric generator.
CsrGraph fast_load_csr1(const char* path) {
  CsrGraph g;
  FILE* f = std::fopen(path, "rb");
  char magic[4];
  std::uint64_t n = 0, m = 0;
  if (!f || std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CSR1", 4) != 0 ||
      std::fread(&n, 8, 1, f) != 1 || std::fread(&m, 8, 1, f) != 1) {
    throw FormatError(std::string("cannot read CSR1 header: ") + path);
  }
  g.vertex_count = n;
  g.edge_count = m;
  g.row_offsets.resize(n + 1);
  g.column_indices.resize(m);
  const bool ok = std::fread(g.row_offsets.data(), 8, n + 1, f) == n + 1 &&
                  std::fread(g.column_indices.data(), 4, m, f) == m;
  std::fclose(f);
  if (!ok) throw FormatError(std::string("truncated CSR1 file: ") + path);
  g.symmetric = true;
  return g;
}

int percall(const char* path, std::size_t nsrc) {
  const auto t0 = std::chrono::steady_clock::now();
  const CsrGraph g = fast_load_csr1(path);
  const auto t1 = std::chrono::steady_clock::now();
  const KernelFn fn = gpu::kernel_fn();
  KernelConfig cfg;
  cfg.variant = KernelVariant::Hybrid;
  const auto srcs = sources_of(g, nsrc, 1);
  fn(g, srcs[0], cfg);  // upload + warm-up (not timed)
  const auto t2 = std::chrono::steady_clock::now();
  double inv = 0.0;
  for (const VertexId s : srcs) {
    const auto a = std::chrono::steady_clock::now();
    const BfsResult r = fn(g, s, cfg);
    const auto b = std::chrono::steady_clock::now();
    std::uint64_t arcs = 0;
    for (VertexId v = 0; v < g.vertex_count; ++v) {
      if (r.distances[v] != kUnreached) arcs += g.degree(v);
    }
    const double secs = std::chrono::duration<double>(b - a).count();
    inv += secs / (arcs / 2.0 / 1e9);
  }
  std::printf("{\"plugin_per_call_gteps\": %.3f, \"sources\": %zu, \"load_s\": %.2f, "
              "\"upload_and_warmup_s\": %.2f}\n",
              static_cast<double>(srcs.size()) / inv, srcs.size(),
              std::chrono::duration<double>(t1 - t0).count(),
              std::chrono::duration<double>(t2 - t1).count());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "criterion1";
  try {
    if (mode == "criterion1") return criterion1();
    if (mode == "timerun") return timerun();
    if (mode == "multi") return multi();
    if (mode == "percall" && argc > 3) return percall(argv[2], std::strtoull(argv[3], nullptr, 10));
  } catch (const Error& e) {
    std::printf("ERROR %s\n", e.what());
    return std::strstr(e.what(), "no CUDA device") ? 3 : 1;
  }
  std::printf("usage: adapter_check criterion1|timerun|multi|percall FILE N\n");
  return 2;
}

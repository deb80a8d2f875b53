// Internal helpers shared by the host graph library and the device runtime.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "pbfs.h"

namespace pbfs {

// Thread-local message behind pbfs_last_error(); every failing entry point
// sets it before returning its status.
pbfs_status fail(pbfs_status st, const std::string& msg);
void clear_error();

// Host CSR owned by the library. Raw arrays (no value-initialisation) so a
// multi-GB graph is not zero-filled before the builder overwrites it.
struct FreeDeleter {
  void operator()(void* p) const { std::free(p); }
};

struct HostCsr {
  uint64_t n = 0;
  uint64_t m = 0;
  std::unique_ptr<uint64_t[]> offsets;  // n + 1
  // malloc'd: the builder compacts the columns inside its key buffer and
  // shrinks it with realloc instead of holding a second m-sized array.
  std::unique_ptr<uint32_t[], FreeDeleter> col;  // m
  bool symmetric = false;
};

unsigned resolve_threads(uint32_t requested);

// Runs f(t) for t in [0, threads) on threads-1 spawned threads plus the caller.
template <typename F>
void parallel_for_threads(unsigned threads, F&& f) {
  std::vector<std::thread> pool;
  pool.reserve(threads ? threads - 1 : 0);
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back([&f, t] { f(t); });
  f(0u);
  for (auto& th : pool) th.join();
}

// Offset at index i of a borrowed CSR view (4- or 8-byte offsets).
inline uint64_t csr_offset(const pbfs_csr* c, uint64_t i) {
  return c->offset_bytes == 8 ? static_cast<const uint64_t*>(c->row_offsets)[i]
                              : static_cast<const uint32_t*>(c->row_offsets)[i];
}

// Level codes of `bits` = 4 (vertex v in byte v / 2, low nibble for even v;
// 0xF = unreached) or 8 (0xFF = unreached) bits per vertex -> uint32 distances
// for entries [b, e), with whole-cache-line non-temporal stores where the host
// has AVX-512 (pbfs_graph.cpp; runtime dispatch). Returns false when the host
// lacks it (the caller's SSE2 loop runs instead). dst + b must be 64 B aligned
// and b even.
bool widen_codes_avx512(const uint8_t* src, uint32_t* dst, uint64_t b, uint64_t e, uint32_t bits);

// Structural validation of a borrowed CSR (validate_csr, csr_graph.cpp:68-113).
pbfs_status validate_csr_view(const pbfs_csr* c, unsigned threads);

}  // namespace pbfs

struct pbfs_host_csr {
  pbfs::HostCsr g;
};

// Device runtime behind include/pbfs.h: graph residency in HBM, the
// persistent traversal launch, trace/result copies, error mapping.
//
// Replaces, per reference file:
//   kernels.cpp:72-126  Engine ctor/run   -> pbfs_graph_create (once per graph)
//                                            + one cooperative launch per BFS
//   kernels.cpp:562-577 check_source/check_symmetric -> pbfs_bfs prologue
//   kernels.cpp:586-655 bfs_* wrappers     -> variant -> (claim, policy) map
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <emmintrin.h>
#include <deque>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <new>
#include <string>
#include <vector>

#include "pbfs_internal.h"
#include "pbfs_kernels.cuh"

namespace pbfs {
const char* last_error_cstr();
}

using namespace pbfs;
using namespace pbfs::dev;

namespace {

constexpr uint64_t kPackMinVertices = uint64_t{1} << 25;
// Narrow-transfer slots of pbfs_bfs_batch: traversal i may run while the
// widening of i - 1 .. i - (slots - 1) is still queued on the host, so the
// host-bound widening (~2.3 ms per RMAT-26 array with the transfers landing
// alongside) and the traversal time (0.8 - 5.8 ms per source) average out
// over sources instead of pairwise (RMAT-26 e2e: 2 slots 317, 4 slots 346,
// 6 or 8 no better).
constexpr int kMaxBatchSlots = 8;
constexpr int kBatchSlots = 4;

// Host threads of the widening pool (PBFS_WIDEN_THREADS overrides for A/B runs).
unsigned widen_threads() {
  // Every hardware thread (RMAT-26 e2e, 16-core host: 16 threads 346, 14
  // threads 343 GTEPS -- within run-to-run noise).
  unsigned t = std::max(1u, std::thread::hardware_concurrency());
  if (const char* e = std::getenv("PBFS_WIDEN_THREADS")) t = std::max(1, std::atoi(e));
  return t;
}

// Host-side widening of packed distances (4-bit, 1 B or 2 B codes, all-ones =
// unreached) into the caller's uint32 arrays, on a persistent pool. Jobs are
// numbered by the caller (0, 1, 2, ...), submitted in order and run one at a
// time, each split across every worker.
class Widener {
 public:
  struct Job {
    const void* src = nullptr;
    uint32_t* dst = nullptr;
    uint64_t n = 0;
    uint32_t width = 0;  // code width in BITS (4, 8 or 16); 0 = nothing to widen (bookkeeping only)
    uint64_t id = 0;
    Widener* owner = nullptr;
  };
  explicit Widener(unsigned threads) : T_(std::max(1u, threads)) {
    for (unsigned t = 0; t < T_; ++t) th_.emplace_back([this, t] { run(t); });
  }
  ~Widener() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_work_.notify_all();
    for (auto& t : th_) t.join();
  }
  void reset() {  // start a new batch numbering (no job may be pending)
    std::lock_guard<std::mutex> l(mu_);
    done_ = 0;
  }
  // cudaLaunchHostFunc callback: the transfer for this job has landed.
  static void CUDART_CB submit_cb(void* arg) {
    Job* j = static_cast<Job*>(arg);
    j->owner->submit(*j);
  }
  void submit(const Job& j) {
    std::lock_guard<std::mutex> l(mu_);
    q_.push_back(j);
    publish_locked();
  }
  // Blocks until jobs 0 .. id have completed.
  void wait(uint64_t id) {
    std::unique_lock<std::mutex> l(mu_);
    cv_done_.wait(l, [&] { return done_ > id; });
  }

 private:
  void publish_locked() {
    if (busy_ || q_.empty()) return;
    cur_ = q_.front();
    q_.pop_front();
    ++seq_;
    pending_ = T_;
    busy_ = true;
    cv_work_.notify_all();
  }
  void run(unsigned t) {
    uint64_t last = 0;
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_work_.wait(l, [&] { return stop_ || (busy_ && seq_ != last); });
        if (stop_) return;
        j = cur_;
        last = seq_;
      }
      // Workers split the job in 64-entry-aligned chunks; small jobs use
      // fewer workers (one per 1 Mi entries) so a wake-up is not the cost.
      const uint64_t parts = std::min<uint64_t>(T_, std::max<uint64_t>(1, j.n >> 20));
      if (t < parts && j.width) {
        const uint64_t b = (j.n * t / parts) & ~63ull;
        const uint64_t e = t + 1 == parts ? j.n : (j.n * (t + 1) / parts) & ~63ull;
        widen(j, b, e);
      }
      std::lock_guard<std::mutex> l(mu_);
      if (--pending_ == 0) {
        busy_ = false;
        done_ = j.id + 1;
        cv_done_.notify_all();
        publish_locked();
      }
    }
  }
  // dst[b, e) from the packed source. SSE2 with non-temporal stores (no
  // read-for-ownership of the 4 B/vertex destination): unpacking against the
  // all-ones mask turns 0xFF / 0xFFFF into 0xFFFFFFFF and zero-extends the
  // rest.
  static void widen(const Job& j, uint64_t b, uint64_t e) {
    uint64_t i = b;  // a multiple of 64 (even: nibble codes pair up)
    auto scalar = [&](uint64_t k) {
      if (j.width == 4) {
        const uint32_t x = (static_cast<const uint8_t*>(j.src)[k >> 1] >> ((k & 1) * 4)) & 0xFu;
        j.dst[k] = x == 0xF ? 0xFFFFFFFFu : x;
      } else if (j.width == 8) {
        const uint8_t x = static_cast<const uint8_t*>(j.src)[k];
        j.dst[k] = x == 0xFF ? 0xFFFFFFFFu : x;
      } else {
        const uint16_t x = static_cast<const uint16_t*>(j.src)[k];
        j.dst[k] = x == 0xFFFF ? 0xFFFFFFFFu : x;
      }
    };
    while (i < e && ((reinterpret_cast<uintptr_t>(j.dst + i) & 63) || (i & 1))) scalar(i++);
    // Whole-line stores where the host has AVX-512 (pbfs_graph.cpp).
    if (j.width <= 8 && i < e &&
        widen_codes_avx512(static_cast<const uint8_t*>(j.src), j.dst, i, e, j.width)) return;
    const __m128i ones = _mm_set1_epi32(-1);
    // 16 one-byte codes x (m = their unreached mask) -> 16 uint32 at d.
    auto expand16 = [&](__m128i x, __m128i m, __m128i* d) {
      const __m128i lo = _mm_unpacklo_epi8(x, m), hi = _mm_unpackhi_epi8(x, m);
      const __m128i mlo = _mm_unpacklo_epi8(m, m), mhi = _mm_unpackhi_epi8(m, m);
      _mm_stream_si128(d + 0, _mm_unpacklo_epi16(lo, mlo));
      _mm_stream_si128(d + 1, _mm_unpackhi_epi16(lo, mlo));
      _mm_stream_si128(d + 2, _mm_unpacklo_epi16(hi, mhi));
      _mm_stream_si128(d + 3, _mm_unpackhi_epi16(hi, mhi));
    };
    if (j.width == 4) {
      const uint8_t* s = static_cast<const uint8_t*>(j.src);
      const __m128i nib = _mm_set1_epi8(0x0F);
      for (; i + 16 <= e; i += 16) {
        const __m128i x = _mm_loadl_epi64(reinterpret_cast<const __m128i*>(s + (i >> 1)));
        const __m128i lo = _mm_and_si128(x, nib), hi = _mm_and_si128(_mm_srli_epi16(x, 4), nib);
        const __m128i y = _mm_unpacklo_epi8(lo, hi);  // vertex order: even = low nibble
        // 0x0F -> 0xFF under its own mask, so the byte expansion's all-ones rule applies
        const __m128i m = _mm_cmpeq_epi8(y, nib);
        expand16(_mm_or_si128(y, m), m, reinterpret_cast<__m128i*>(j.dst + i));
      }
    } else if (j.width == 8) {
      const uint8_t* s = static_cast<const uint8_t*>(j.src);
      for (; i + 16 <= e; i += 16) {
        const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        expand16(x, _mm_cmpeq_epi8(x, ones), reinterpret_cast<__m128i*>(j.dst + i));
      }
    } else {
      const uint16_t* s = static_cast<const uint16_t*>(j.src);
      for (; i + 8 <= e; i += 8) {
        const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        const __m128i m = _mm_cmpeq_epi16(x, ones);
        __m128i* d = reinterpret_cast<__m128i*>(j.dst + i);
        _mm_stream_si128(d + 0, _mm_unpacklo_epi16(x, m));
        _mm_stream_si128(d + 1, _mm_unpackhi_epi16(x, m));
      }
    }
    while (i < e) scalar(i++);
    _mm_sfence();
  }
  unsigned T_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_work_, cv_done_;
  std::deque<Job> q_;
  Job cur_;
  uint64_t seq_ = 0, done_ = 0;
  unsigned pending_ = 0;
  bool busy_ = false, stop_ = false;
};

}  // namespace

struct pbfs_graph {
  std::mutex mu;
  // Multi-GPU placement (pbfs_graph_options.devices): every traversal entry
  // point forwards to the multi-partition engine (pbfs_multi.cu).
  pbfs_multi* multi = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // Recorded right after every traversal launch on whatever stream it used;
  // every later launch (or reset, or read of the handle's buffers) waits on
  // it first. All traversals share the handle's ctl (grid-barrier word), bitmaps
  // and dist, so two launches must never overlap, whichever streams the callers
  // pass (pbfs_bfs_async) -- without holding on to a caller's stream handle.
  cudaEvent_t order_ev = nullptr;
  uint64_t n = 0, m = 0, max_degree = 0;
  uint32_t offb = 8;
  bool symmetric = false;
  uint32_t words = 0;
  void* rowptr = nullptr;
  uint32_t* col = nullptr;
  uint32_t* init_mask = nullptr;
  uint32_t* first_nbr = nullptr;
  uint32_t* dist = nullptr;
  uint32_t* visited = nullptr;
  uint32_t* bm[2] = {nullptr, nullptr};
  uint32_t* queue[2] = {nullptr, nullptr};
  uint4* lq[2] = {nullptr, nullptr};  // latency-mode queues (hub-free graphs only)
  int lat_grid = 0;                   // latency-mode grid (one CTA per SM)
  HeavyItem* heavy = nullptr;
  Ctl* ctl = nullptr;
  pbfs_level* records = nullptr;
  unsigned long long* comp = nullptr;
  uint32_t rec_cap = 0;
  uint64_t qcap = 0, heavy_cap = 0;
  uint32_t heavy_deg = kHeavyDeg, chunk_log2 = 0;
  uint64_t isolated = 0;  // zero-degree vertices (symmetric graphs), pre-set in init_mask
  uint32_t force = 0;     // kForce* test hooks
  int grid = 0;
  size_t bitmap_bytes = 0;
  size_t persist_bytes = 0;  // L2 set-aside granted for the bitmap window
  uint64_t device_bytes = 0;
  std::vector<void*> allocs;
  bool poisoned = false;  // a launch failed; ctl must be reset
  // pbfs_bfs_batch state, created on first use.
  uint32_t* dist2 = nullptr;
  uint32_t* obs = nullptr;  // observer log (allocated on the first observed run)
  // Single calls into pageable host memory (the C++ KernelFn's std::vector):
  // packed device copy + pinned staging + the widening pool.
  void* pack1 = nullptr;
  void* stage1 = nullptr;
  uint64_t obs_cap = 0;
  cudaStream_t copy_stream = nullptr;
  int batch_slots = 0;
  cudaEvent_t kern_done[kMaxBatchSlots] = {}, copy_done[kMaxBatchSlots] = {};
  void* pack[kMaxBatchSlots] = {};   // device: packed distances (<= 2 B per vertex)
  void* stage[kMaxBatchSlots] = {};  // pinned host: their landing buffers
  std::unique_ptr<Widener> widener;
  Ctl* ctl_host = nullptr;  // pinned, ctl_host_cap entries
  uint32_t ctl_host_cap = 0;
  std::vector<cudaEvent_t> run_ev;  // per-source start/end events (2 per source)
  uint32_t red_minq = 0;  // reduction-claim frontier length (bfs_persistent), 0 = off
  uint32_t pack_min_bits = 4;  // narrowest packed transfer code (PBFS_PACK_MIN_BITS=8: no 4-bit codes)
};

namespace {

pbfs_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky non-fatal state
  return fail(PBFS_E_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PBFS_CUDA(call, what)                 \
  do {                                        \
    cudaError_t _e = (call);                  \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

template <typename T>
pbfs_status dalloc(pbfs_graph* g, T** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PBFS_E_CAPACITY, "cudaMalloc of " + std::to_string(bytes) +
                                     " bytes failed: " + cudaGetErrorString(e));
  }
  g->allocs.push_back(q);
  g->device_bytes += bytes;
  *p = static_cast<T*>(q);
  return PBFS_OK;
}

void release(pbfs_graph* g) {
  if (!g) return;
  if (g->multi) {
    pbfs_multi_destroy(g->multi);
    delete g;
    return;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  for (void* p : g->allocs) cudaFree(p);
  g->widener.reset();
  if (g->ctl_host) cudaFreeHost(g->ctl_host);
  for (void* h : g->stage) if (h) cudaFreeHost(h);
  if (g->stage1) cudaFreeHost(g->stage1);
  for (cudaEvent_t e : g->run_ev) cudaEventDestroy(e);
  for (int i = 0; i < kMaxBatchSlots; ++i) {
    if (g->kern_done[i]) cudaEventDestroy(g->kern_done[i]);
    if (g->copy_done[i]) cudaEventDestroy(g->copy_done[i]);
  }
  if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->order_ev) cudaEventDestroy(g->order_ev);
  if (g->stream) cudaStreamDestroy(g->stream);
  cudaSetDevice(prev);
  delete g;
}

struct Launch {
  int claim;
  int policy;
};

pbfs_status map_variant(const pbfs_config* c, bool* hybrid_like, Launch* out) {
  switch (c->variant) {
    case PBFS_CONVENTIONAL:
      *out = {kClaimCas, kPolicyTopDown};
      *hybrid_like = false;
      return PBFS_OK;
    case PBFS_NONATOMIC:
      *out = {kClaimPlain, kPolicyTopDown};
      *hybrid_like = false;
      return PBFS_OK;
    case PBFS_HYBRID:
    case PBFS_VISITED_INLINE:
      *out = {kClaimBitmap, c->force_top_down_only ? kPolicyTopDown : kPolicyFraction};
      *hybrid_like = true;
      return PBFS_OK;
    case PBFS_HYBRID_BEAMER:
      *out = {kClaimBitmap, c->force_top_down_only ? kPolicyTopDown : kPolicyBeamer};
      *hybrid_like = true;
      return PBFS_OK;
    case PBFS_HYBRID_PLAIN:
      *out = {kClaimPlain, c->force_top_down_only ? kPolicyTopDown : kPolicyFraction};
      *hybrid_like = true;
      return PBFS_OK;
    case PBFS_SERIAL:
      return fail(PBFS_E_CONFIG, "the serial variant is the CPU oracle, not a GPU kernel");
    case PBFS_VISITED_DEFERRED:
    case PBFS_PERIODIC_FLUSH:
      return fail(PBFS_E_CONFIG,
                  "visited-deferred and periodic-flush are CPU cache/memory artefacts "
                  "with no GPU kernel (SURVEY.md §2)");
    default:
      return fail(PBFS_E_CONFIG, "unknown kernel variant");
  }
}

// Latency mode (pbfs_kernels.cuh: td_phase_latency): the visited-bitmap
// claim run top-down only on a graph without hubs. PBFS_LATENCY=0 disables it.
bool latency_mode(const pbfs_graph* g, int claim, int policy, bool observe) {
  const char* e = std::getenv("PBFS_LATENCY");
  const bool off = e && e[0] == '0';
  return !off && !observe && g->lq[0] && claim == kClaimBitmap && policy == kPolicyTopDown;
}

template <int C, typename OffT>
cudaError_t launch_typed(pbfs_graph* g, uint32_t source, const pbfs_config* cfg, int policy,
                         cudaStream_t s, uint32_t* dist, void* pack) {
  Params<OffT> p;
  p.pack = pack;
  p.rowptr = static_cast<const OffT*>(g->rowptr);
  p.col = g->col;
  p.dist = dist;
  p.visited = g->visited;
  p.bm[0] = g->bm[0];
  p.bm[1] = g->bm[1];
  p.init_mask = g->init_mask;
  p.first_nbr = g->first_nbr;
  p.queue[0] = g->queue[0];
  p.queue[1] = g->queue[1];
  p.lq[0] = g->lq[0];
  p.lq[1] = g->lq[1];
  p.latency = latency_mode(g, C, policy, cfg->observe_frontiers != 0) ? 1 : 0;
  p.obs = cfg->observe_frontiers ? g->obs : nullptr;
  p.obs_cap = g->obs_cap;
  p.heavy = g->heavy;
  p.ctl = g->ctl;
  p.records = g->records;
  p.qcap = g->qcap;
  p.heavy_cap = g->heavy_cap;
  p.heavy_deg = g->heavy_deg;
  p.isolated = g->isolated;
  p.chunk_log2 = g->chunk_log2;
  p.small_chunks = 1;
  p.force = g->force;
  p.n = g->n;
  p.m = g->m;
  p.max_degree = g->max_degree;
  p.words = g->words;
  p.rec_cap = g->rec_cap;
  p.source = source;
  p.policy = policy;
  p.validate = cfg->validate_same_value_stores ? 1 : 0;
  p.threshold = cfg->hybrid_threshold_fraction;
  p.alpha = cfg->alpha;
  p.beta = cfg->beta;
  p.red_minq = g->red_minq;
  p.pack_min_bits = g->pack_min_bits;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(p.latency ? g->lat_grid : g->grid);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = 0;
  lc.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  int nattr = 1;
  if (g->persist_bytes) {
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = g->visited;
    attr[1].val.accessPolicyWindow.num_bytes = g->bitmap_bytes;
    attr[1].val.accessPolicyWindow.hitRatio =
        std::min(1.0f, static_cast<float>(g->persist_bytes) / static_cast<float>(g->bitmap_bytes));
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    nattr = 2;
  }
  lc.attrs = attr;
  lc.numAttrs = nattr;
  if (p.obs) return cudaLaunchKernelEx(&lc, bfs_persistent<C, OffT, false, true>, p);
  if constexpr (C == kClaimBitmap) {
    if (p.latency) {
      lc.dynamicSmemBytes = kLatSmem;
      // Per launch: function attributes belong to the current device.
      const cudaError_t ae = cudaFuncSetAttribute(bfs_latency<OffT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(kLatSmem));
      if (ae != cudaSuccess) return ae;
      return cudaLaunchKernelEx(&lc, bfs_latency<OffT>, p);
    }
  }
  return cudaLaunchKernelEx(&lc, bfs_persistent<C, OffT>, p);
}

cudaError_t launch(pbfs_graph* g, uint32_t source, const pbfs_config* cfg, const Launch& l,
                   cudaStream_t s, uint32_t* dist = nullptr, void* pack = nullptr) {
  const bool wide = g->offb == 8;
  if (!dist) dist = g->dist;
  switch (l.claim) {
    case kClaimCas:
      return wide ? launch_typed<kClaimCas, unsigned long long>(g, source, cfg, l.policy, s, dist, pack)
                  : launch_typed<kClaimCas, uint32_t>(g, source, cfg, l.policy, s, dist, pack);
    case kClaimPlain:
      return wide ? launch_typed<kClaimPlain, unsigned long long>(g, source, cfg, l.policy, s, dist, pack)
                  : launch_typed<kClaimPlain, uint32_t>(g, source, cfg, l.policy, s, dist, pack);
    default:
      return wide ? launch_typed<kClaimBitmap, unsigned long long>(g, source, cfg, l.policy, s, dist, pack)
                  : launch_typed<kClaimBitmap, uint32_t>(g, source, cfg, l.policy, s, dist, pack);
  }
}

template <typename OffT>
int occupancy_for(int claim) {
  int blocks = 0;
  const void* fn = claim == kClaimCas     ? reinterpret_cast<const void*>(&bfs_persistent<kClaimCas, OffT>)
                   : claim == kClaimPlain ? reinterpret_cast<const void*>(&bfs_persistent<kClaimPlain, OffT>)
                                          : reinterpret_cast<const void*>(&bfs_persistent<kClaimBitmap, OffT>);
  // Smallest shared-memory carveout that fits kMinBlocks resident CTAs: the
  // rest of the SM's 256 KB stays L1, which caches the visited-bitmap probes
  // (profiles/r01_ab.txt: 16 KB more per CTA, L1 192 -> 124 KB, cost 17 %).
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, fn);
  const size_t per_sm = static_cast<size_t>(kMinBlocks) * (fa.sharedSizeBytes + 1024);
  const int pct = static_cast<int>((per_sm * 100 + 228 * 1024 - 1) / (228 * 1024));
  cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, std::min(100, pct));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, 0);
  return blocks;
}

// Orders stream s after the handle's last launch (see pbfs_graph::order_ev).
pbfs_status order_after_last(pbfs_graph* g, cudaStream_t s) {
  PBFS_CUDA(cudaStreamWaitEvent(s, g->order_ev, 0), "order after the last traversal");
  return PBFS_OK;
}
pbfs_status mark_launch(pbfs_graph* g, cudaStream_t s) {
  PBFS_CUDA(cudaEventRecord(g->order_ev, s), "order event");
  return PBFS_OK;
}

pbfs_status prologue(pbfs_graph* g, uint32_t source, const pbfs_config* cfg, Launch* l,
                     cudaStream_t s) {
  if (!g || !cfg) return fail(PBFS_E_INPUT, "null argument");
  pbfs_status st = pbfs_config_validate(cfg);
  if (st != PBFS_OK) return st;
  bool hybrid_like = false;
  st = map_variant(cfg, &hybrid_like, l);
  if (st != PBFS_OK) return st;
  if (source >= g->n) {
    return fail(PBFS_E_INPUT, "source vertex " + std::to_string(source) +
                                  " is out of range for a graph with " + std::to_string(g->n) +
                                  " vertices");
  }
  if (hybrid_like && !cfg->force_top_down_only && !g->symmetric) {
    return fail(PBFS_E_INPUT,
                "direction-switching traversal reads each adjacency list as in-edges, which "
                "requires a symmetric graph; symmetrize the input or force the top-down-only "
                "path");
  }
  PBFS_CUDA(cudaSetDevice(g->device), "cudaSetDevice");
  if ((st = order_after_last(g, s)) != PBFS_OK) return st;
  if (cfg->observe_frontiers && !g->obs) {
    // Every vertex is produced once (distinct snapshots): n entries suffice.
    g->obs_cap = g->n + 64;
    if ((st = dalloc(g, &g->obs, g->obs_cap * 4)) != PBFS_OK) return st;
  }
  if (g->poisoned) {
    // On the launching stream, after the previous launch: never under a
    // running traversal.
    PBFS_CUDA(cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), s), "reset control block");
    g->poisoned = false;
  }
  return PBFS_OK;
}

}  // namespace

extern "C" {

uint32_t pbfs_abi_version(void) { return PBFS_ABI_VERSION; }
const char* pbfs_last_error(void) { return pbfs::last_error_cstr(); }

const char* pbfs_status_string(pbfs_status s) {
  switch (s) {
    case PBFS_OK: return "ok";
    case PBFS_E_INPUT: return "input error";
    case PBFS_E_CONFIG: return "config error";
    case PBFS_E_FORMAT: return "format error";
    case PBFS_E_CAPACITY: return "capacity error";
    case PBFS_E_DEVICE: return "device error";
    case PBFS_E_COMM: return "communication error";
    case PBFS_E_METRIC: return "metric error";
    case PBFS_E_CORRECTNESS: return "correctness error";
  }
  return "unknown status";
}

void pbfs_config_init(pbfs_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->variant = PBFS_CONVENTIONAL;
  c->worker_count = 1;
  c->hybrid_threshold_fraction = 0.05;
  c->alpha = 15.0;
  c->beta = 18.0;
  c->flush_capacity = 4096;
}

// kernel_config.cpp:9-26
pbfs_status pbfs_config_validate(const pbfs_config* c) {
  if (!c) return fail(PBFS_E_INPUT, "null config");
  if (c->worker_count < 1) return fail(PBFS_E_CONFIG, "worker count must be at least 1");
  if (!(c->hybrid_threshold_fraction > 0.0) || c->hybrid_threshold_fraction > 1.0) {
    return fail(PBFS_E_CONFIG, "hybrid threshold fraction must be in (0, 1]");
  }
  if (!(c->alpha > 0.0)) return fail(PBFS_E_CONFIG, "alpha must be positive");
  if (!(c->beta > 0.0)) return fail(PBFS_E_CONFIG, "beta must be positive");
  if (c->flush_capacity < 1) return fail(PBFS_E_CONFIG, "flush capacity must be at least 1");
  return PBFS_OK;
}

pbfs_status pbfs_graph_create(const pbfs_csr* csr, const pbfs_graph_options* opt,
                              pbfs_graph** out) {
  if (!csr || !out) return fail(PBFS_E_INPUT, "null argument");
  const unsigned threads = resolve_threads(0);
  pbfs_status st = validate_csr_view(csr, threads);
  if (st != PBFS_OK) return st;
  const uint64_t n = csr->vertex_count, m = csr->edge_count;
  uint32_t offb = opt ? opt->device_offset_bytes : 0;
  if (offb == 0) offb = m < (1ull << 31) ? 4 : 8;
  if (offb != 4 && offb != 8) return fail(PBFS_E_CONFIG, "device offset width must be 0, 4 or 8");
  if (offb == 4 && m > 0x7fffffffULL) {
    return fail(PBFS_E_CAPACITY, "edge count " + std::to_string(m) + " needs 64-bit offsets");
  }
  int device = opt ? opt->device : 0;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(PBFS_E_DEVICE, "no CUDA device available: the BFS kernels need a B200 "
                               "(there is no CPU fallback)");
  }
  if (device < 0 || device >= ndev) return fail(PBFS_E_CONFIG, "device ordinal out of range");

  auto* g = new (std::nothrow) pbfs_graph;
  if (!g) return fail(PBFS_E_CAPACITY, "host allocation failed");
  g->device = device;
  g->n = n;
  g->m = m;
  g->offb = offb;
  g->symmetric = csr->symmetric != 0;
  if (opt && opt->devices && opt->num_devices > 1) {
    // Partitioned over several devices: the handle is a pbfs_multi.
    g->device = opt->devices[0];
    g->offb = 8;
    for (uint64_t v = 0; v < n; ++v) {
      g->max_degree = std::max<uint64_t>(g->max_degree, csr_offset(csr, v + 1) - csr_offset(csr, v));
    }
    st = pbfs_multi_create(csr, opt->devices, opt->num_devices, &g->multi);
    if (st != PBFS_OK) {
      delete g;
      return st;
    }
    pbfs_multi_info mi;
    pbfs_multi_get_info(g->multi, &mi);
    g->grid = static_cast<int>(mi.ctas_per_partition * mi.partitions);
    *out = g;
    return PBFS_OK;
  }
  // Host-side per-graph facts: max degree, heavy-item capacity, the
  // zero-degree mask that lets bottom-up skip isolated vertices.
  // Whole 32-word groups: bottom-up takes 16-word groups, the merge and
  // compaction passes 32-word warp groups.
  g->words = static_cast<uint32_t>(((n + 31) / 32 + 31) / 32 * 32);
  if (g->words == 0) g->words = kGroupWords;
  std::vector<uint32_t> mask(g->words, 0);
  // PBFS_FORCE_MODES (test hook, a kForce* bitmask) forces the size-gated
  // paths on any graph so small-graph parity tests cover them.
  if (const char* fm = std::getenv("PBFS_FORCE_MODES")) g->force = static_cast<uint32_t>(std::strtoul(fm, nullptr, 0));
  const bool big = static_cast<unsigned long long>(g->m) >= kBigArcs || (g->force & kForceBigSplit);
  g->heavy_deg = big ? kHeavyDegBig : kHeavyDeg;
  const uint64_t chunk = big ? kChunkBig : kChunk;
  static_assert((kChunk & (kChunk - 1)) == 0, "PBFS_CHUNK must be a power of two");
  while ((1ull << g->chunk_log2) < chunk) ++g->chunk_log2;
  {
    std::vector<uint64_t> mx(threads, 0), hc(threads, 0);
    std::vector<std::vector<uint64_t>> hubs(threads);
    parallel_for_threads(threads, [&](unsigned t) {
      const uint64_t b = n * t / threads, en = n * (t + 1) / threads;
      for (uint64_t v = b; v < en; ++v) {
        const uint64_t d = csr_offset(csr, v + 1) - csr_offset(csr, v);
        mx[t] = std::max(mx[t], d);
        if (d > g->heavy_deg) {
          hc[t] += (d + chunk - 1) / chunk;
          hubs[t].push_back(d);
        }
      }
    });
    for (unsigned t = 0; t < threads; ++t) {
      g->max_degree = std::max(g->max_degree, mx[t]);
      g->heavy_cap += hc[t];
    }
    // Small frontiers (<= kSmallFrontier vertices) split hubs into
    // 2^kSmallChunkLog2-edge items so a few hubs still spread over the grid;
    // their item count is bounded by the kSmallFrontier largest degrees.
    std::vector<uint64_t> all;
    for (auto& h : hubs) all.insert(all.end(), h.begin(), h.end());
    const size_t top = std::min<size_t>(all.size(), kSmallFrontier);
    std::nth_element(all.begin(), all.begin() + top, all.end(), std::greater<uint64_t>());
    uint64_t small_items = 0;
    for (size_t i = 0; i < top; ++i) small_items += (all[i] + (1ull << kSmallChunkLog2) - 1) >> kSmallChunkLog2;
    g->heavy_cap = std::max(g->heavy_cap, small_items);
    if (g->symmetric) {
      for (uint64_t v = 0; v < n; ++v) {
        if (csr_offset(csr, v + 1) == csr_offset(csr, v)) {
          mask[v >> 5] |= 1u << (v & 31);
          ++g->isolated;
        }
      }
    }
    for (uint64_t v = n; v < static_cast<uint64_t>(g->words) * 32; ++v) mask[v >> 5] |= 1u << (v & 31);
  }
  g->qcap = n + g->max_degree;
  // Test hooks: shrink the frontier queue / hub-item capacities so the
  // device-side overflow -> PBFS_E_CAPACITY path (frontier.hpp:88-93) runs.
  if (const char* q = std::getenv("PBFS_TEST_QCAP")) g->qcap = std::min<uint64_t>(g->qcap, std::strtoull(q, nullptr, 0));
  if (const char* h = std::getenv("PBFS_TEST_HEAVY_CAP")) {
    g->heavy_cap = std::min<uint64_t>(g->heavy_cap, std::strtoull(h, nullptr, 0));
  }
  g->rec_cap = static_cast<uint32_t>(std::min<uint64_t>(n + 1, 1u << 20));

  int prev = 0;
  cudaGetDevice(&prev);
  auto bail = [&](pbfs_status s2) {
    release(g);
    cudaSetDevice(prev);
    return s2;
  };
  if ((e = cudaSetDevice(device)) != cudaSuccess) return bail(cuda_fail(e, "cudaSetDevice"));
  if ((e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaStreamCreate"));
  if ((e = cudaEventCreate(&g->ev0)) != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
  if ((e = cudaEventCreate(&g->ev1)) != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
  if ((e = cudaEventCreateWithFlags(&g->order_ev, cudaEventDisableTiming)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaEventCreate"));
  // Never recorded yet: waiting on it is a no-op until the first launch.

  const size_t wbytes = static_cast<size_t>(g->words) * 4;
  if ((st = dalloc(g, &g->rowptr, (n + 1) * offb)) != PBFS_OK) return bail(st);
  // Padded to whole 16 B vectors: hub chunks are read with uint4 loads.
  // Whole 64 B windows past the end: bottom-up scans read aligned 16-entry windows.
  if ((st = dalloc(g, &g->col, ((m + 15) / 16) * 64 + 64)) != PBFS_OK) return bail(st);
  if ((st = dalloc(g, &g->init_mask, wbytes)) != PBFS_OK) return bail(st);
  if ((st = dalloc(g, &g->first_nbr, (n + 1) * 4)) != PBFS_OK) return bail(st);
  // Whole 32-entry groups: front_from_dist reads 128 B per bitmap word and
  // the batch path's pack pass 64 B at a time.
  if ((st = dalloc(g, &g->dist, ((n + 31) / 32) * 128)) != PBFS_OK) return bail(st);
  // visited | frontier | next bitmaps in one block: the probe-heavy working
  // set (3 n/8 bytes) sits under one persisting L2 access-policy window so
  // the multi-GB `col` stream cannot evict it.
  if ((st = dalloc(g, &g->visited, 3 * wbytes)) != PBFS_OK) return bail(st);
  g->bm[0] = g->visited + g->words;
  g->bm[1] = g->visited + 2 * static_cast<size_t>(g->words);
  g->bitmap_bytes = 3 * wbytes;
  if ((st = dalloc(g, &g->queue[0], g->qcap * 4)) != PBFS_OK) return bail(st);
  if ((st = dalloc(g, &g->queue[1], g->qcap * 4)) != PBFS_OK) return bail(st);
  if (g->max_degree <= g->heavy_deg) {
    // Hub-free graph: 16 B queue entries for the latency-mode top-down path.
    if ((st = dalloc(g, &g->lq[0], g->qcap * sizeof(uint4))) != PBFS_OK) return bail(st);
    if ((st = dalloc(g, &g->lq[1], g->qcap * sizeof(uint4))) != PBFS_OK) return bail(st);
  }
  if ((st = dalloc(g, &g->heavy, std::max<uint64_t>(g->heavy_cap, 1) * sizeof(HeavyItem))) != PBFS_OK)
    return bail(st);
  if ((st = dalloc(g, &g->ctl, sizeof(Ctl))) != PBFS_OK) return bail(st);
  if ((st = dalloc(g, &g->records, static_cast<size_t>(g->rec_cap) * sizeof(pbfs_level))) != PBFS_OK)
    return bail(st);
  if ((st = dalloc(g, &g->comp, 2 * sizeof(unsigned long long))) != PBFS_OK) return bail(st);

  // Offsets: upload as-is when the widths match, else narrow on the host.
  if (offb == csr->offset_bytes) {
    if ((e = cudaMemcpy(g->rowptr, csr->row_offsets, (n + 1) * offb, cudaMemcpyHostToDevice)) != cudaSuccess)
      return bail(cuda_fail(e, "upload offsets"));
  } else {
    std::vector<uint8_t> tmp((n + 1) * offb);
    for (uint64_t v = 0; v <= n; ++v) {
      const uint64_t o = csr_offset(csr, v);
      if (offb == 4) {
        reinterpret_cast<uint32_t*>(tmp.data())[v] = static_cast<uint32_t>(o);
      } else {
        reinterpret_cast<uint64_t*>(tmp.data())[v] = o;
      }
    }
    if ((e = cudaMemcpy(g->rowptr, tmp.data(), tmp.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return bail(cuda_fail(e, "upload offsets"));
  }
  if (m && (e = cudaMemcpy(g->col, csr->column_indices, m * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
    return bail(cuda_fail(e, "upload columns"));
  if ((e = cudaMemcpy(g->init_mask, mask.data(), wbytes, cudaMemcpyHostToDevice)) != cudaSuccess)
    return bail(cuda_fail(e, "upload mask"));
  {
    // First neighbour of every vertex, read coalesced by bottom-up: on RMAT
    // almost every unvisited vertex finds its parent there (hubs sort first),
    // so rowptr / col are touched only for the rest.
    std::vector<uint32_t> first(n + 1, 0);
    parallel_for_threads(threads, [&](unsigned t) {
      const uint64_t b = n * t / threads, en = n * (t + 1) / threads;
      for (uint64_t v = b; v < en; ++v) {
        const uint64_t o = csr_offset(csr, v);
        first[v] = o < csr_offset(csr, v + 1) ? csr->column_indices[o] : 0u;
      }
    });
    if ((e = cudaMemcpy(g->first_nbr, first.data(), (n + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
      return bail(cuda_fail(e, "upload first neighbours"));
  }
  if ((e = cudaMemset(g->ctl, 0, sizeof(Ctl))) != cudaSuccess) return bail(cuda_fail(e, "memset ctl"));

  // Persistent grid: every SM x resident CTAs of the widest instantiation.
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return bail(cuda_fail(e, "props"));
  int occ = 1 << 30;
  for (int c = 0; c < 3; ++c) {
    occ = std::min(occ, offb == 8 ? occupancy_for<unsigned long long>(c) : occupancy_for<uint32_t>(c));
  }
  if (occ < 1) return bail(fail(PBFS_E_DEVICE, "traversal kernel cannot be resident"));
  g->grid = prop.multiProcessorCount * occ;
  if (const char* e = std::getenv("PBFS_GRID")) {  // A/B knob: a smaller persistent grid
    g->grid = std::max(1, std::min(g->grid, std::atoi(e)));
  }
  // Latency mode: one CTA per SM halves nothing of a small level's work but
  // a quarter of its grid-barrier time (tools/ubench_barrier.cu: 1.5 vs 2.0 us).
  g->lat_grid = prop.multiProcessorCount;
  if (const char* e = std::getenv("PBFS_LATENCY_GRID")) {
    g->lat_grid = std::max(1, std::min(g->grid, std::atoi(e)));
  }
  // Persisting L2 set-aside for the bitmap block (process-wide device limit;
  // only ever raised). PBFS_NO_L2_PERSIST=1 disables it for A/B runs.
  const char* no_persist = std::getenv("PBFS_NO_L2_PERSIST");
  if (prop.persistingL2CacheMaxSize > 0 && prop.accessPolicyMaxWindowSize > 0 &&
      !(no_persist && no_persist[0] == '1')) {
    // The window covers all three bitmaps when they fit the set-aside; else
    // only `visited` (the top-down probe target): a window larger than the
    // set-aside thrashes its own lines (RMAT-28: 96 MB of bitmaps, 79 MB
    // set-aside). PBFS_L2_WINDOW=all|visited overrides for A/B runs.
    const char* win = std::getenv("PBFS_L2_WINDOW");
    const size_t vis_bytes = static_cast<size_t>(g->words) * 4;
    bool all = g->bitmap_bytes <= static_cast<size_t>(prop.persistingL2CacheMaxSize);
    if (win && std::strcmp(win, "all") == 0) all = true;
    if (win && std::strcmp(win, "visited") == 0) all = false;
    if (!all) g->bitmap_bytes = vis_bytes;
    g->bitmap_bytes = std::min<size_t>(g->bitmap_bytes, prop.accessPolicyMaxWindowSize);
    const size_t want = std::min<size_t>(g->bitmap_bytes, prop.persistingL2CacheMaxSize);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
      cudaGetLastError();
    } else {
      g->persist_bytes = want;
    }
  }
  // Reduction claim: only where visited + both frontier bitmaps fit the
  // persisting-L2 set-aside. Its reds go to two bitmaps instead of one, and
  // on RMAT-28 (96 MB of bitmaps against 79 MB) they miss L2 and cost more
  // than the claim round trips they save: 423 GTEPS with it, 448 without
  // (RMAT-26, 25 MB: 491 with, 476 without; profiles/r02/ab.txt).
  const size_t red_fit = prop.persistingL2CacheMaxSize > 0
                             ? static_cast<size_t>(prop.persistingL2CacheMaxSize)
                             : (64u << 20);
  g->red_minq = 3 * wbytes <= red_fit ? kRedMinQ : 0;
  if (const char* q = std::getenv("PBFS_RED_MINQ")) g->red_minq = static_cast<uint32_t>(std::strtoul(q, nullptr, 0));
  if (const char* b = std::getenv("PBFS_PACK_MIN_BITS")) g->pack_min_bits = std::atoi(b) >= 8 ? 8u : 4u;
  cudaSetDevice(prev);
  *out = g;
  return PBFS_OK;
}

pbfs_status pbfs_graph_destroy(pbfs_graph* g) {
  release(g);
  return PBFS_OK;
}

pbfs_status pbfs_graph_get_info(const pbfs_graph* g, pbfs_graph_info* info) {
  if (!g || !info) return fail(PBFS_E_INPUT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->vertex_count = g->n;
  info->edge_count = g->m;
  info->max_degree = g->max_degree;
  info->device_bytes = g->device_bytes;
  info->device_offset_bytes = g->offb;
  info->symmetric = g->symmetric;
  info->device = g->device;
  info->grid_blocks = static_cast<uint32_t>(g->grid);
  info->block_threads = kThreads;
  if (g->multi) {
    pbfs_multi_info mi;
    pbfs_multi_get_info(g->multi, &mi);
    info->partitions = mi.partitions;
  } else {
    info->partitions = 1;
  }
  return PBFS_OK;
}

}  // extern "C"

namespace {
pbfs_status pbfs_bfs_locked(pbfs_graph* g, uint32_t source, const pbfs_config* cfg,
                            uint32_t* dist_host, pbfs_level* levels, uint32_t levels_cap,
                            pbfs_run_info* info) {
  Launch l;
  pbfs_status st = prologue(g, source, cfg, &l, g->stream);
  if (st != PBFS_OK) return st;
  cudaError_t e;
  // A large PAGEABLE destination (e.g. a std::vector behind the reference's
  // KernelFn) would take the driver's staged pageable copy at 4 B/vertex:
  // instead the kernel also writes level codes (4 bits to 2 B per vertex),
  // those land in pinned staging, and the widening pool expands them into the
  // caller's array on every host core (faulting its pages in parallel too).
  // A PINNED destination takes the same path only from 2^27 vertices: a lone
  // call wakes an idle pool, whose widening of a 256 MB array takes ~4 ms
  // (1.8 ms back to back) and gives back what the shorter transfer saves
  // (RMAT-26: 146 packed, 150 GTEPS plain), but at 1 GB per array it wins
  // (RMAT-28: 199 against 141-150; profiles/r02/ab.txt).
  // PBFS_PINNED_PACKED_MIN=N overrides the vertex count (A/B knob).
  bool packed = false;
  if (dist_host && (g->n >= kPackMinVertices || (g->force & kForcePack))) {
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, dist_host) == cudaSuccess &&
                        pa.type != cudaMemoryTypeUnregistered;
    cudaGetLastError();
    uint64_t pinned_min = uint64_t{1} << 27;
    if (const char* pm = std::getenv("PBFS_PINNED_PACKED_MIN")) pinned_min = std::strtoull(pm, nullptr, 0);
    if (!pinned || g->n >= pinned_min) {
      const uint64_t pbytes = ((g->n + 15) / 16) * 32;
      if (!g->pack1 && (st = dalloc(g, &g->pack1, pbytes)) != PBFS_OK) return st;
      if (!g->stage1) PBFS_CUDA(cudaHostAlloc(&g->stage1, pbytes, cudaHostAllocDefault), "pinned staging");
      if (!g->widener) g->widener.reset(new Widener(widen_threads()));
      packed = true;
    }
  }
  PBFS_CUDA(cudaEventRecord(g->ev0, g->stream), "event record");
  if ((e = launch(g, source, cfg, l, g->stream, nullptr, packed ? g->pack1 : nullptr)) != cudaSuccess) {
    g->poisoned = true;
    return cuda_fail(e, "traversal launch");
  }
  PBFS_CUDA(cudaEventRecord(g->ev1, g->stream), "event record");
  if ((st = mark_launch(g, g->stream)) != PBFS_OK) return st;
  Ctl ctl;
  PBFS_CUDA(cudaMemcpyAsync(&ctl, g->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, g->stream), "read control");
  if ((e = cudaStreamSynchronize(g->stream)) != cudaSuccess) {
    g->poisoned = true;
    return cuda_fail(e, "traversal");
  }
  if (ctl.overflow) {
    g->poisoned = true;
    return fail(PBFS_E_CAPACITY, "dense frontier overflow");
  }
  if (dist_host) {
    const uint32_t bits = packed ? pack_bits(ctl.levels, g->pack_min_bits) : 32u;
    if (bits < 32) {
      PBFS_CUDA(cudaMemcpy(g->stage1, g->pack1, packed_bytes(g->n, bits), cudaMemcpyDeviceToHost),
                "read distances");
      Widener& wd = *g->widener;
      wd.reset();
      Widener::Job job{g->stage1, dist_host, g->n, bits, 0, &wd};
      wd.submit(job);
      wd.wait(0);
    } else {
      PBFS_CUDA(cudaMemcpy(dist_host, g->dist, g->n * 4, cudaMemcpyDeviceToHost), "read distances");
    }
  }
  const uint32_t nrec = std::min<uint32_t>(ctl.levels, g->rec_cap);
  if (levels && levels_cap) {
    const uint32_t k = std::min(nrec, levels_cap);
    PBFS_CUDA(cudaMemcpy(levels, g->records, k * sizeof(pbfs_level), cudaMemcpyDeviceToHost), "read trace");
  }
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->levels = ctl.levels;
    info->bottom_up_levels = ctl.bu_levels;
    info->reached = ctl.reached;
    info->same_value_violations = ctl.violations;
    info->edges_examined = ctl.edges;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g->ev0, g->ev1);
    info->device_ms = ms;
  }
  if (ctl.levels > g->rec_cap && levels && levels_cap > g->rec_cap) {
    // Deeper than the device record buffer (min(n + 1, 2^20) levels): grow it
    // to the depth just seen and run the traversal again, so any depth is
    // recorded (the reference records every level, trace.hpp:37-48).
    pbfs_level* bigger = nullptr;
    PBFS_CUDA(cudaMalloc(&bigger, static_cast<size_t>(ctl.levels) * sizeof(pbfs_level)),
              "grow the trace buffer");
    for (auto& a : g->allocs) {
      if (a == g->records) a = bigger;
    }
    cudaFree(g->records);
    g->device_bytes += static_cast<uint64_t>(ctl.levels - g->rec_cap) * sizeof(pbfs_level);
    g->records = bigger;
    g->rec_cap = ctl.levels;
    return pbfs_bfs_locked(g, source, cfg, dist_host, levels, levels_cap, info);
  }
  return PBFS_OK;
}

}  // namespace

extern "C" {

pbfs_status pbfs_bfs(pbfs_graph* g, uint32_t source, const pbfs_config* cfg, uint32_t* dist_host,
                     pbfs_level* levels, uint32_t levels_cap, pbfs_run_info* info) {
  if (!g) return fail(PBFS_E_INPUT, "null graph");
  if (g->multi) return pbfs_multi_bfs(g->multi, source, cfg, dist_host, levels, levels_cap, info);
  std::lock_guard<std::mutex> lock(g->mu);
  return pbfs_bfs_locked(g, source, cfg, dist_host, levels, levels_cap, info);
}

pbfs_status pbfs_bfs_batch(pbfs_graph* g, const uint32_t* sources, uint32_t count,
                           const pbfs_config* cfg, uint32_t* const* dist_host,
                           pbfs_run_info* infos) {
  if (!g) return fail(PBFS_E_INPUT, "null graph");
  if (count && (!sources || !dist_host)) return fail(PBFS_E_INPUT, "null argument");
  if (g->multi) {
    for (uint32_t i = 0; i < count; ++i) {
      pbfs_status st = pbfs_multi_bfs(g->multi, sources[i], cfg, dist_host[i], nullptr, 0,
                                      infos ? &infos[i] : nullptr);
      if (st != PBFS_OK) return st;
      if (infos) infos[i].transfer_width = 4;
    }
    return PBFS_OK;
  }
  std::lock_guard<std::mutex> lock(g->mu);
  Launch l;
  for (uint32_t i = 0; i < count; ++i) {
    pbfs_status st = prologue(g, sources[i], cfg, &l, g->stream);
    if (st != PBFS_OK) return st;
  }
  if (count == 0) return PBFS_OK;
  PBFS_CUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaError_t e;
  const uint64_t n = g->n;
  if (!g->copy_stream) {
    PBFS_CUDA(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    g->batch_slots = kBatchSlots;
    if (const char* es = std::getenv("PBFS_BATCH_SLOTS")) {
      g->batch_slots = std::max(2, std::min(kMaxBatchSlots, std::atoi(es)));
    }
    for (int i = 0; i < g->batch_slots; ++i) {
      PBFS_CUDA(cudaEventCreateWithFlags(&g->kern_done[i], cudaEventDisableTiming), "cudaEventCreate");
      PBFS_CUDA(cudaEventCreateWithFlags(&g->copy_done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    const uint64_t pbytes = ((n + 15) / 16) * 32;  // 2 B per vertex, whole 16-vertex groups
    for (int i = 0; i < g->batch_slots; ++i) {
      pbfs_status st = dalloc(g, &g->pack[i], pbytes);
      if (st != PBFS_OK) return st;
      PBFS_CUDA(cudaHostAlloc(&g->stage[i], pbytes, cudaHostAllocDefault), "pinned staging");
    }
    g->widener.reset(new Widener(widen_threads()));
  }
  if (!g->dist2) {
    pbfs_status st = dalloc(g, &g->dist2, ((n + 31) / 32) * 128);
    if (st != PBFS_OK) return st;
  }
  if (g->ctl_host_cap < count) {
    if (g->ctl_host) cudaFreeHost(g->ctl_host);
    g->ctl_host = nullptr;
    g->ctl_host_cap = 0;
    PBFS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->ctl_host), count * sizeof(Ctl),
                            cudaHostAllocDefault), "pinned control snapshots");
    g->ctl_host_cap = count;
  }
  while (g->run_ev.size() < 2ull * count) {
    cudaEvent_t ev;
    PBFS_CUDA(cudaEventCreate(&ev), "cudaEventCreate");
    g->run_ev.push_back(ev);
  }
  // Pipeline per source i (slot = i % S; dist buffer i & 1):
  //   compute stream: traversal i into dist/pack[slot] (+ a narrow copy of
  //                   the distances at the end), control snapshot;
  //   copy stream:    pack[slot] -> pinned stage[slot] (4 bits, 1 B or 2 B per vertex,
  //                   chosen from the level count), then a host callback
  //                   hands it to the widener pool, which writes dist_host[i];
  //   host:           enqueues traversal i+1 before it waits for traversal i.
  // PCIe then moves n/2 .. 2n B per source instead of 4n B, overlapped with the
  // next traversal, and the widening runs on the host cores in parallel.
  uint32_t* buf[2] = {g->dist, g->dist2};
  // Narrow transfers pay off once the 4 B/vertex copy outlasts the traversal
  // and the host-side widening (measured: RMAT-26 4.84 -> 3.47 ms per source;
  // ER-24 and smaller are faster with the plain copy).
  const bool packed = n >= kPackMinVertices || (g->force & kForcePack);
  // Plain copies read the dist buffers themselves: two slots.
  const uint32_t S = packed ? static_cast<uint32_t>(g->batch_slots) : 2u;
  std::vector<uint8_t> reads_dist(count, packed ? 0 : 1);  // transfer j copies buf[j & 1]
  Widener& wd = *g->widener;
  wd.reset();
  std::vector<Widener::Job> jobs(count);
  std::unordered_map<const uint32_t*, int64_t> last_use;  // output buffer -> last job writing it
  auto finish = [&](uint32_t j) -> cudaError_t {
    const uint32_t slot = j % S;
    cudaError_t ce;
    if (!packed) {
      // Plain 4 B/vertex copy, stream-ordered: no host wait at all.
      if ((ce = cudaStreamWaitEvent(g->copy_stream, g->kern_done[slot], 0)) != cudaSuccess) return ce;
      if ((ce = cudaMemcpyAsync(dist_host[j], buf[j & 1], n * 4, cudaMemcpyDeviceToHost,
                                g->copy_stream)) != cudaSuccess) return ce;
      return cudaEventRecord(g->copy_done[slot], g->copy_stream);
    }
    ce = cudaEventSynchronize(g->kern_done[slot]);
    if (ce != cudaSuccess) return ce;
    const Ctl& c = g->ctl_host[j];
    const uint32_t bits = packed ? pack_bits(c.levels, g->pack_min_bits) : 32u;
    const uint32_t width = bits < 32 ? 1u : 4u;  // below: < 4 = codes + widening, 4 = the plain copy
    Widener::Job& job = jobs[j];
    job = Widener::Job{g->stage[slot], dist_host[j], n, bits < 32 ? bits : 0, j, &wd};
    // stage[slot] was last read by job j-S. dist_host[j] may alias an earlier
    // output (rotating buffers): the pool runs jobs in order, so only a DMA
    // straight into dist_host (the 4 B fallback) waits for that job.
    int64_t need = j >= S ? static_cast<int64_t>(j) - S : -1;
    auto it = last_use.find(dist_host[j]);
    if (width >= 4 && it != last_use.end()) need = std::max<int64_t>(need, it->second);
    if (need >= 0) wd.wait(static_cast<uint64_t>(need));
    last_use[dist_host[j]] = j;
    if ((ce = cudaStreamWaitEvent(g->copy_stream, g->kern_done[slot], 0)) != cudaSuccess) return ce;
    if (width < 4) {
      ce = cudaMemcpyAsync(g->stage[slot], g->pack[slot], packed_bytes(n, bits), cudaMemcpyDeviceToHost,
                           g->copy_stream);
    } else {
      reads_dist[j] = 1;  // > 65534 levels: the full 4 B copy of the dist buffer
      ce = cudaMemcpyAsync(dist_host[j], buf[j & 1], n * 4, cudaMemcpyDeviceToHost, g->copy_stream);
    }
    if (ce != cudaSuccess) return ce;
    if ((ce = cudaLaunchHostFunc(g->copy_stream, Widener::submit_cb, &job)) != cudaSuccess) return ce;
    return cudaEventRecord(g->copy_done[slot], g->copy_stream);
  };
  for (uint32_t i = 0; i <= count; ++i) {
    if (i < count) {
      const uint32_t slot = i % S;
      // pack/stage[slot] are free once transfer i-S has landed; dist buffer
      // i & 1 once transfer i-2 has, if that transfer read it.
      if (i >= S && (e = cudaStreamWaitEvent(g->stream, g->copy_done[slot], 0)) != cudaSuccess) break;
      if (i >= 2 && S > 2 && reads_dist[i - 2] &&
          (e = cudaStreamWaitEvent(g->stream, g->copy_done[(i - 2) % S], 0)) != cudaSuccess) break;
      if ((e = cudaEventRecord(g->run_ev[2 * i], g->stream)) != cudaSuccess) break;
      if ((e = launch(g, sources[i], cfg, l, g->stream, buf[i & 1],
                      packed ? g->pack[slot] : nullptr)) != cudaSuccess) {
        g->poisoned = true;
        break;
      }
      if ((e = cudaEventRecord(g->run_ev[2 * i + 1], g->stream)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(&g->ctl_host[i], g->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost,
                               g->stream)) != cudaSuccess) break;
      if ((e = cudaEventRecord(g->kern_done[slot], g->stream)) != cudaSuccess) break;
    }
    if (i >= 1 && (e = finish(i - 1)) != cudaSuccess) break;
  }
  if (e == cudaSuccess) e = cudaEventRecord(g->order_ev, g->stream);
  cudaError_t e1 = cudaStreamSynchronize(g->stream);
  cudaError_t e2 = cudaStreamSynchronize(g->copy_stream);
  // Every callback that fired has submitted its job; wait for those.
  if (packed && e == cudaSuccess && e1 == cudaSuccess && e2 == cudaSuccess) wd.wait(count - 1);
  if (e != cudaSuccess || e1 != cudaSuccess || e2 != cudaSuccess) {
    g->poisoned = true;
    // Jobs whose callbacks ran may still be widening: drain the pool first.
    g->widener.reset(new Widener(widen_threads()));
    return cuda_fail(e != cudaSuccess ? e : e1 != cudaSuccess ? e1 : e2, "traversal batch");
  }
  // The handle's dist keeps meaning "the last traversal" (device_dist, component).
  if ((count - 1) & 1) std::swap(g->dist, g->dist2);
  for (uint32_t i = 0; i < count; ++i) {
    const Ctl& c = g->ctl_host[i];
    if (c.overflow) {
      g->poisoned = true;
      return fail(PBFS_E_CAPACITY, "dense frontier overflow");
    }
    if (infos) {
      pbfs_run_info* info = &infos[i];
      std::memset(info, 0, sizeof(*info));
      info->levels = c.levels;
      info->bottom_up_levels = c.bu_levels;
      info->reached = c.reached;
      info->same_value_violations = c.violations;
      info->edges_examined = c.edges;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, g->run_ev[2 * i], g->run_ev[2 * i + 1]);
      info->device_ms = ms;
      info->transfer_width = packed ? pack_width(c.levels) : 4u;
    }
  }
  return PBFS_OK;
}

pbfs_status pbfs_bfs_async(pbfs_graph* g, uint32_t source, const pbfs_config* cfg, void* stream) {
  if (!g) return fail(PBFS_E_INPUT, "null graph");
  if (g->multi) {
    // The launches go to the engine's own per-device streams; the caller's
    // stream then waits for the traversal on every device.
    pbfs_status st = pbfs_multi_bfs_async(g->multi, source, cfg);
    if (st != PBFS_OK || !stream) return st;
    return pbfs_multi_join(g->multi, stream);
  }
  std::lock_guard<std::mutex> lock(g->mu);
  Launch l;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  pbfs_status st = prologue(g, source, cfg, &l, s);
  if (st != PBFS_OK) return st;
  cudaError_t e = launch(g, source, cfg, l, s);
  if (e != cudaSuccess) {
    g->poisoned = true;
    return cuda_fail(e, "traversal launch");
  }
  return mark_launch(g, s);
}

pbfs_status pbfs_graph_sync(pbfs_graph* g, void* stream) {
  if (!g) return fail(PBFS_E_INPUT, "null graph");
  if (g->multi) return pbfs_multi_sync(g->multi, nullptr);
  std::lock_guard<std::mutex> lock(g->mu);
  PBFS_CUDA(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  cudaError_t e = cudaStreamSynchronize(s);
  // Also the handle's last traversal, if it went to another stream.
  if (e == cudaSuccess) e = cudaEventSynchronize(g->order_ev);
  if (e != cudaSuccess) {
    g->poisoned = true;
    return cuda_fail(e, "traversal");
  }
  unsigned int overflow = 0;
  PBFS_CUDA(cudaMemcpy(&overflow, &g->ctl->overflow, sizeof(overflow), cudaMemcpyDeviceToHost),
            "read control");
  if (overflow) {
    g->poisoned = true;
    return fail(PBFS_E_CAPACITY, "dense frontier overflow");
  }
  return PBFS_OK;
}

pbfs_status pbfs_graph_device_arrays(const pbfs_graph* g, const void** row_offsets,
                                     const uint32_t** column_indices, uint32_t* offset_bytes) {
  if (!g || !row_offsets || !column_indices || !offset_bytes) {
    return fail(PBFS_E_INPUT, "null argument");
  }
  if (g->multi) return fail(PBFS_E_CONFIG, "a multi-device handle holds partitions, not the full CSR");
  *row_offsets = g->rowptr;
  *column_indices = g->col;
  *offset_bytes = g->offb;
  return PBFS_OK;
}

pbfs_status pbfs_graph_trace(pbfs_graph* g, pbfs_level* levels, uint32_t levels_cap,
                             uint32_t* count) {
  if (!g || !count || (levels_cap && !levels)) return fail(PBFS_E_INPUT, "null argument");
  if (g->multi) return pbfs_multi_trace(g->multi, levels, levels_cap, count);
  std::lock_guard<std::mutex> lock(g->mu);
  PBFS_CUDA(cudaSetDevice(g->device), "cudaSetDevice");
  PBFS_CUDA(cudaEventSynchronize(g->order_ev), "traversal");
  unsigned int nlev = 0;
  PBFS_CUDA(cudaMemcpy(&nlev, &g->ctl->levels, sizeof(nlev), cudaMemcpyDeviceToHost), "read control");
  const uint32_t k = std::min<uint32_t>(std::min<uint32_t>(nlev, g->rec_cap), levels_cap);
  if (k) {
    PBFS_CUDA(cudaMemcpy(levels, g->records, k * sizeof(pbfs_level), cudaMemcpyDeviceToHost),
              "read trace");
  }
  *count = k;
  if (nlev > g->rec_cap) {
    return fail(PBFS_E_CAPACITY, "the last traversal was deeper than the device trace buffer");
  }
  return PBFS_OK;
}

pbfs_status pbfs_graph_observed(pbfs_graph* g, uint32_t* out, uint64_t cap, uint64_t* count) {
  if (!g || !count || (cap && !out)) return fail(PBFS_E_INPUT, "null argument");
  if (g->multi) return fail(PBFS_E_CONFIG, "frontier observation runs on single-device handles");
  std::lock_guard<std::mutex> lock(g->mu);
  PBFS_CUDA(cudaSetDevice(g->device), "cudaSetDevice");
  PBFS_CUDA(cudaEventSynchronize(g->order_ev), "traversal");
  if (!g->obs) return fail(PBFS_E_CONFIG, "no traversal ran with observe_frontiers");
  unsigned int total = 0;
  PBFS_CUDA(cudaMemcpy(&total, &g->ctl->obs_count, sizeof(total), cudaMemcpyDeviceToHost),
            "read control");
  const uint64_t k = std::min<uint64_t>(total, cap);
  if (k) PBFS_CUDA(cudaMemcpy(out, g->obs, k * 4, cudaMemcpyDeviceToHost), "read observed frontiers");
  *count = total;
  return PBFS_OK;
}

pbfs_status pbfs_graph_device_dist(pbfs_graph* g, uint32_t** dist_dev) {
  if (!g || !dist_dev) return fail(PBFS_E_INPUT, "null argument");
  if (g->multi) {
    return fail(PBFS_E_CONFIG, "a multi-device handle keeps distances in its partitions: "
                               "read them with pbfs_bfs (dist_host)");
  }
  *dist_dev = g->dist;
  return PBFS_OK;
}

pbfs_status pbfs_graph_component(pbfs_graph* g, uint64_t* n_reached, uint64_t* arcs_reached) {
  if (!g || !n_reached || !arcs_reached) return fail(PBFS_E_INPUT, "null argument");
  if (g->multi) return pbfs_multi_component(g->multi, n_reached, arcs_reached);
  std::lock_guard<std::mutex> lock(g->mu);
  PBFS_CUDA(cudaSetDevice(g->device), "cudaSetDevice");
  pbfs_status st = order_after_last(g, g->stream);
  if (st != PBFS_OK) return st;
  PBFS_CUDA(cudaMemsetAsync(g->comp, 0, 2 * sizeof(unsigned long long), g->stream), "memset");
  if (g->offb == 8) {
    component_kernel<unsigned long long><<<g->grid, kThreads, 0, g->stream>>>(
        static_cast<const unsigned long long*>(g->rowptr), g->dist, g->n, g->comp);
  } else {
    component_kernel<uint32_t><<<g->grid, kThreads, 0, g->stream>>>(
        static_cast<const uint32_t*>(g->rowptr), g->dist, g->n, g->comp);
  }
  PBFS_CUDA(cudaGetLastError(), "component launch");
  unsigned long long h[2];
  PBFS_CUDA(cudaMemcpyAsync(h, g->comp, sizeof(h), cudaMemcpyDeviceToHost, g->stream), "read");
  PBFS_CUDA(cudaStreamSynchronize(g->stream), "component");
  *n_reached = h[0];
  *arcs_reached = h[1];
  return PBFS_OK;
}

pbfs_status pbfs_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(PBFS_E_INPUT, "null argument");
  PBFS_CUDA(cudaMallocHost(out, bytes ? bytes : 16), "cudaMallocHost");
  return PBFS_OK;
}

pbfs_status pbfs_host_free(void* p) {
  if (p) PBFS_CUDA(cudaFreeHost(p), "cudaFreeHost");
  return PBFS_OK;
}

}  // extern "C"

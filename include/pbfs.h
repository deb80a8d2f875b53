/* pbfs.h — C ABI of the B200-native level-synchronous BFS (arXiv 2503.00430).
 *
 * This is the drop-in boundary the reference's C++ entry points reach the GPU
 * through. Plain C types only: pointers, sizes, status codes. No torch, no
 * C++ types. Every entry point cites the reference interface it replaces
 * (paths relative to the reference's proj/ directory).
 *
 * Threading: a pbfs_graph is immutable after creation; pbfs_bfs* calls on one
 * handle are serialised by a per-handle mutex (its traversal scratch lives in
 * the handle); distinct handles may run concurrently ("safe to
 * invoke concurrently on distinct output buffers").
 *
 * Errors: every call returns a pbfs_status; pbfs_last_error() holds a
 * thread-local message. The status values map one-to-one onto the reference
 * exception classes (core/include/parbfs/types.hpp:25-68).
 */
#ifndef PBFS_H
#define PBFS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBFS_ABI_VERSION 2u
#define PBFS_UNREACHED 0xFFFFFFFFu /* == parbfs::kUnreached (types.hpp:19) == int32 -1 */

typedef enum pbfs_status {
  PBFS_OK = 0,
  PBFS_E_INPUT = 1,       /* parbfs::InputError    (types.hpp:33-36) */
  PBFS_E_CONFIG = 2,      /* parbfs::ConfigError   (types.hpp:39-42) */
  PBFS_E_FORMAT = 3,      /* parbfs::FormatError   (types.hpp:45-48) */
  PBFS_E_CAPACITY = 4,    /* parbfs::CapacityError (types.hpp:53-56) */
  PBFS_E_DEVICE = 5,      /* CUDA runtime failure  -> parbfs::Error  */
  PBFS_E_COMM = 6,        /* collective failure    -> parbfs::Error  */
  PBFS_E_METRIC = 7,      /* parbfs::MetricError   (types.hpp:65-68) */
  PBFS_E_CORRECTNESS = 8  /* parbfs::CorrectnessError (types.hpp:59-62) */
} pbfs_status;

/* parbfs::KernelVariant (core/include/parbfs/kernel_config.hpp:13-22),
 * same numbering. The GPU implements CONVENTIONAL, NONATOMIC, HYBRID,
 * HYBRID_BEAMER and VISITED_INLINE; SERIAL, VISITED_DEFERRED and
 * PERIODIC_FLUSH are CPU-only artefacts and are rejected with PBFS_E_CONFIG. */
typedef enum pbfs_variant {
  PBFS_SERIAL = 0,
  PBFS_CONVENTIONAL = 1,     /* top-down, atomicCAS claim on dist (kernels.cpp:282-290) */
  PBFS_NONATOMIC = 2,        /* top-down, plain same-value dist stores (kernels.cpp:291-301) */
  PBFS_HYBRID = 3,           /* TD/BU by the 5 % frontier-size rule (kernels.cpp:494-497) */
  PBFS_HYBRID_BEAMER = 4,    /* TD/BU by Beamer alpha/beta (kernels.cpp:498-511) */
  PBFS_VISITED_INLINE = 5,   /* hybrid, visited-bitmap claim, inline dist (kernels.cpp:302-320) */
  PBFS_VISITED_DEFERRED = 6,
  PBFS_PERIODIC_FLUSH = 7,
  /* GPU addition: the reference's own Hybrid claim discipline -- top-down
   * with PlainStore (probe dist, plain same-value store, no atomic; racing
   * writers may all push, kernels.cpp:291-301) and bottom-up, 5 % rule
   * (kernels.cpp:606-616). PBFS_HYBRID runs the visited-bitmap claim. */
  PBFS_HYBRID_PLAIN = 8
} pbfs_variant;

typedef enum pbfs_phase { PBFS_TOP_DOWN = 0, PBFS_BOTTOM_UP = 1 } pbfs_phase;

/* Borrowed host view of a CSR graph, layout-compatible with parbfs::CsrGraph
 * (core/include/parbfs/csr_graph.hpp:20-46): row_offsets has vertex_count+1
 * entries of offset_bytes (8 = parbfs::EdgeOffset, or 4), column_indices has
 * edge_count u32 entries sorted per row. Only read during the call. */
typedef struct pbfs_csr {
  uint64_t vertex_count;
  uint64_t edge_count;
  const void* row_offsets;
  const uint32_t* column_indices;
  uint32_t offset_bytes;
  uint32_t symmetric;
} pbfs_csr;

/* parbfs::KernelConfig (kernel_config.hpp:38-70). worker_count and
 * flush_capacity are validated exactly like parbfs::validate
 * (kernel_config.cpp:9-26) but have no GPU meaning. */
typedef struct pbfs_config {
  uint32_t variant;
  uint32_t worker_count;
  double hybrid_threshold_fraction; /* (0, 1], default 0.05 */
  double alpha;                     /* > 0, default 15 */
  double beta;                      /* > 0, default 18 */
  uint64_t flush_capacity;          /* >= 1, default 4096 */
  uint32_t force_top_down_only;
  uint32_t validate_same_value_stores;
  uint32_t racy_visited_claim;
  /* Test instrumentation (KernelConfig::level_observer, kernel_config.hpp:
   * 26-36): record every produced frontier as it is formed on the device
   * (pbfs_graph_observed reads them back). Off in measurements. */
  uint32_t observe_frontiers;
} pbfs_config;

/* parbfs::LevelRecord (core/include/parbfs/trace.hpp:26-35). */
typedef struct pbfs_level {
  uint32_t depth;
  uint32_t phase; /* pbfs_phase */
  uint64_t frontier_size;
  uint64_t distinct_size;
  uint64_t duplicate_count;
  uint64_t edges_examined;
  uint64_t flush_events;
  int64_t elapsed_ns; /* device %globaltimer span of the iteration */
} pbfs_level;

/* Whole-run figures (parbfs::TraversalTrace, trace.hpp:37-48). */
typedef struct pbfs_run_info {
  uint32_t levels;                /* records produced (may exceed levels_cap) */
  uint32_t bottom_up_levels;
  uint64_t reached;               /* sum of distinct sizes = reachable set */
  uint64_t same_value_violations; /* under validate_same_value_stores */
  uint64_t edges_examined;
  float device_ms;                /* CUDA-event time of the traversal kernel */
  uint32_t transfer_width;        /* pbfs_bfs_batch: bytes per vertex moved device->host,
                                     rounded up (1 or 2 when packed -- 4-bit codes, used
                                     below 15 levels, report 1 -- else 4); 0 elsewhere */
} pbfs_run_info;

typedef struct pbfs_graph_options {
  int32_t device;               /* CUDA ordinal */
  uint32_t device_offset_bytes; /* 0 = auto (4 if edge_count < 2^31 else 8), 4 or 8 */
  /* Optional multi-GPU placement (SURVEY.md §8(b) "devices[], num_devices"):
   * with num_devices > 1 the handle partitions the graph over devices[0..n)
   * (one partition each; repeats place several partitions on one GPU) and
   * every traversal entry point runs the multi-partition engine
   * (pbfs_multi_*, below) -- so run_bfs / a KernelFn built on this handle
   * reach every GPU. num_devices <= 1 (or devices == NULL): one GPU,
   * `device`. */
  const int32_t* devices;
  uint32_t num_devices;
  uint32_t reserved;
} pbfs_graph_options;

typedef struct pbfs_graph_info {
  uint64_t vertex_count;
  uint64_t edge_count;
  uint64_t max_degree;
  uint64_t device_bytes; /* HBM held by the handle (graph + scratch) */
  uint32_t device_offset_bytes;
  uint32_t symmetric;
  int32_t device;
  uint32_t grid_blocks; /* persistent traversal grid (SMs x resident CTAs) */
  uint32_t block_threads;
  uint32_t partitions;  /* 1, or the multi-GPU placement's partition count */
} pbfs_graph_info;

typedef struct pbfs_graph pbfs_graph;

/* ---- version / errors --------------------------------------------------- */
uint32_t pbfs_abi_version(void);
const char* pbfs_last_error(void);
const char* pbfs_status_string(pbfs_status status);

/* Fills cfg with parbfs::KernelConfig{} defaults (kernel_config.hpp:38-70). */
void pbfs_config_init(pbfs_config* cfg);

/* parbfs::validate (kernel_config.cpp:9-26) plus the GPU variant check. */
pbfs_status pbfs_config_validate(const pbfs_config* cfg);

/* ---- device graph -------------------------------------------------------- */
/* Uploads a host CSR to HBM and allocates the per-handle traversal scratch.
 * Replaces the parbfs::Engine constructor's allocations (kernels.cpp:72-102),
 * paid once per graph instead of once per BFS. Validates the CSR invariants
 * (validate_csr, csr_graph.cpp:68-113): PBFS_E_FORMAT on a broken graph. */
pbfs_status pbfs_graph_create(const pbfs_csr* csr, const pbfs_graph_options* opt,
                              pbfs_graph** out);
pbfs_status pbfs_graph_destroy(pbfs_graph* g);
pbfs_status pbfs_graph_get_info(const pbfs_graph* g, pbfs_graph_info* info);

/* ---- traversal ----------------------------------------------------------- */
/* One BFS end to end: the reference's run_bfs / bfs_* call
 * (core/include/parbfs/kernels.hpp:34-81; kernels.cpp:586-691) with the
 * parbfs::BfsResult written into caller buffers.
 *   dist_host: vertex_count u32 (int32 -1 = unreached), may be NULL (results
 *              then stay on the device: pbfs_graph_device_dist).
 *   levels:    up to levels_cap parbfs::LevelRecord rows, may be NULL.
 *   info:      may be NULL.
 * Applies the reference's checks first: check_source (kernels.cpp:562-568,
 * PBFS_E_INPUT) and check_symmetric for direction-switching variants
 * (kernels.cpp:570-577, PBFS_E_INPUT). Frontier overflow -> PBFS_E_CAPACITY
 * (frontier.hpp:88-93). Synchronous. */
pbfs_status pbfs_bfs(pbfs_graph* g, uint32_t source, const pbfs_config* cfg,
                     uint32_t* dist_host, pbfs_level* levels, uint32_t levels_cap,
                     pbfs_run_info* info);

/* A batch of traversals (the reference's per-source loop in time_run /
 * bfsbench run, timing.cpp:74-76, bfsbench.cpp:458-460) with the distance
 * array of source i copied to dist_host[i] while source i+1 traverses: two
 * device distance buffers, the copies on a second stream. dist_host[i] may
 * repeat (e.g. two rotating buffers); it should be pinned (pbfs_host_alloc)
 * for the copies to overlap. infos: NULL or `count` entries (device_ms is the
 * traversal alone). Same checks and errors as pbfs_bfs, for every source
 * before any launch. Synchronous: returns when every copy has landed. */
pbfs_status pbfs_bfs_batch(pbfs_graph* g, const uint32_t* sources, uint32_t count,
                           const pbfs_config* cfg, uint32_t* const* dist_host,
                           pbfs_run_info* infos);

/* Enqueue-only traversal on a caller stream (cudaStream_t passed as void*,
 * NULL = the handle's stream); distances stay in HBM. No trace, no host sync.
 * For benchmark loops that keep inputs resident. pbfs_graph_sync() collects
 * the status (capacity overflow is reported there). */
pbfs_status pbfs_bfs_async(pbfs_graph* g, uint32_t source, const pbfs_config* cfg,
                           void* stream);
pbfs_status pbfs_graph_sync(pbfs_graph* g, void* stream);

/* The per-level records (parbfs::LevelRecord) of the handle's last traversal,
 * read back after the fact, so a caller can size its buffer to the depth the
 * run actually had (pbfs_run_info.levels) instead of to the worst case.
 * Copies min(levels, levels_cap) records; PBFS_E_CAPACITY if the traversal
 * was deeper than the device record buffer (pbfs_bfs with a large enough
 * levels_cap grows it). */
pbfs_status pbfs_graph_trace(pbfs_graph* g, pbfs_level* levels, uint32_t levels_cap,
                             uint32_t* count);

/* The frontiers the last traversal produced, recorded when it ran with
 * cfg.observe_frontiers: the snapshots of depths 1, 2, ... concatenated
 * (depth d's has levels[d].distinct_size entries; top-down levels in the
 * order the device produced them, bottom-up levels as a set, any order).
 * Copies min(total, cap) entries; *count = total. */
pbfs_status pbfs_graph_observed(pbfs_graph* g, uint32_t* out, uint64_t cap, uint64_t* count);

/* Device pointer of the distance array written by the last traversal. */
pbfs_status pbfs_graph_device_dist(pbfs_graph* g, uint32_t** dist_dev);

/* Reached-component figures of the last traversal, computed on the device:
 * N_r and A_r = sum of reached degrees (SURVEY.md §8(d) metric inputs). */
pbfs_status pbfs_graph_component(pbfs_graph* g, uint64_t* n_reached,
                                 uint64_t* arcs_reached);

/* Pinned host buffers for zero-staging device<->host copies. */
pbfs_status pbfs_host_alloc(size_t bytes, void** out);
pbfs_status pbfs_host_free(void* p);

/* ---- host graph construction (core/include/parbfs/{generator,csr_graph,
 *      graph_stats,graph_io}.hpp) -------------------------------------------- */
typedef struct pbfs_host_csr pbfs_host_csr; /* owns u64 offsets + u32 columns */

typedef enum pbfs_gen_kind {
  PBFS_GEN_UNIFORM = 0,   /* GeneratorKind::UniformRandom (generator.cpp:60-66) */
  PBFS_GEN_KRONECKER = 1, /* GeneratorKind::Kronecker     (generator.cpp:67-89) */
  PBFS_GEN_MESH = 2       /* config-3 road-like mesh (new) */
} pbfs_gen_kind;

typedef struct pbfs_gen_spec {
  uint32_t kind;        /* pbfs_gen_kind */
  uint32_t scale;       /* n = 2^scale (uniform / Kronecker) */
  uint32_t edge_factor; /* samples = edge_factor * n */
  uint32_t drop_self_loops; /* 1 = BASELINE semantics, 0 = reference semantics */
  uint64_t seed;
  uint32_t mesh_side;      /* mesh: side x side grid */
  uint32_t mesh_radius;    /* mesh: shortcut Manhattan radius (32) */
  double mesh_keep;        /* mesh: edge keep probability (0.9) */
  uint64_t mesh_shortcuts; /* mesh: shortcut count (round(0.001 n)) */
  uint32_t threads;        /* host threads for the builder, 0 = all */
  uint32_t reserved;
} pbfs_gen_spec;

/* parbfs::generate (generator.cpp:41-92): the same mt19937_64 draw sequence
 * bit for bit, then build_csr(symmetrize=true). */
pbfs_status pbfs_generate(const pbfs_gen_spec* spec, pbfs_host_csr** out);

/* parbfs::build_csr (csr_graph.cpp:11-55): range check, optional symmetrize,
 * per-row sort + dedup; drop_self_loops applies BASELINE's removal. pairs is
 * npairs interleaved (src, dst) u32. Parallel 2-pass bucketed counting sort. */
pbfs_status pbfs_build_csr(const uint32_t* pairs, uint64_t npairs, uint64_t vertex_count,
                           uint32_t symmetrize, uint32_t drop_self_loops, uint32_t threads,
                           pbfs_host_csr** out);

/* View (borrowed for the lifetime of the handle) with 8-byte offsets. */
pbfs_status pbfs_host_csr_view(const pbfs_host_csr* h, pbfs_csr* view);
pbfs_status pbfs_host_csr_free(pbfs_host_csr* h);

/* parbfs::compute_stats (graph_stats.cpp:9-25). */
typedef struct pbfs_stats {
  uint64_t vertex_count;
  uint64_t edge_count;
  double average_degree;
  uint64_t max_degree;
  uint32_t large_diameter; /* GraphCategory::LargeDiameter iff avg < threshold */
  uint32_t reserved;
} pbfs_stats;
pbfs_status pbfs_compute_stats(const pbfs_csr* csr, double threshold, pbfs_stats* out);

/* bfsbench pick_sources (tools/bfsbench.cpp:206-235). */
pbfs_status pbfs_pick_sources(const pbfs_csr* csr, uint32_t count, uint64_t seed,
                              uint32_t* out);

/* CSR1 binary format (core/src/graph_io.cpp:70-119). */
pbfs_status pbfs_save_csr1(const pbfs_csr* csr, const char* path);
pbfs_status pbfs_load_csr1(const char* path, pbfs_host_csr** out);

/* ---- 1D vertex-partitioned multi-GPU BFS (new) ------------
 * One partition per rank/GPU built on the device from a resident full graph.
 * Ownership by a hashed bijection pi (rank = pi(v) / local_count, balanced
 * arcs on RMAT); numbering by gid(v) = rank * local_count + the number of
 * lower-numbered vertices with the same owner (order-preserving, so sorted
 * adjacency stays sorted and dense per partition). Row slice (bottom-up) +
 * column slice (top-down). Per
 * level: pbfs_part_step (local work, writes this rank's slice of `next`),
 * then the caller allgathers the slices of `next` in place (e.g. NCCL
 * all_gather with sendbuff = next + rank * words_local), then
 * pbfs_part_end_level (identical distinct count / direction / termination
 * on every rank). Partitions on one device may share `frontier`/`next`
 * (loopback: the allgather is then a no-op). Hybrid (5 % rule) only. */
typedef struct pbfs_part pbfs_part;

typedef struct pbfs_part_options {
  uint32_t rank;
  uint32_t world;
  uint32_t relabel;        /* 1: hashed pi when n is a power of two */
  uint32_t reserved;
  void* shared_frontier;   /* loopback: words_total u32 on the same device, or NULL */
  void* shared_next;
} pbfs_part_options;

typedef struct pbfs_part_info {
  uint64_t vertex_count;
  uint64_t padded_count;   /* gid space (power of two or multiple of 512*world) */
  uint64_t local_first;    /* first owned gid */
  uint64_t local_count;    /* owned gids */
  uint64_t local_arcs;     /* row-slice arcs (= column-slice arcs) */
  uint64_t words_total;    /* full bitmap words */
  uint64_t words_local;    /* this rank's slice: next + rank * words_local */
  uint32_t rank;
  uint32_t world;
  uint32_t relabel_hashed;
  uint32_t depth;
  uint32_t top_down;
  uint32_t reserved;
  uint32_t* frontier;      /* device, current frontier bitmap (full) */
  uint32_t* next;          /* device, next frontier bitmap (full; allgather target) */
  uint32_t* dist_local;    /* device, local_count entries, gid order */
} pbfs_part_info;

/* Device pointers of a resident graph (for building partitions). */
pbfs_status pbfs_graph_device_arrays(const pbfs_graph* g, const void** row_offsets,
                                     const uint32_t** column_indices, uint32_t* offset_bytes);
pbfs_status pbfs_part_create(const pbfs_graph* full, const pbfs_part_options* opt,
                             pbfs_part** out);
/* Same, from a device CSR view (row_offsets / column_indices are DEVICE
 * pointers on `device`, e.g. buffers received by a broadcast); only read
 * during the call. */
pbfs_status pbfs_part_create_device(const pbfs_csr* device_csr, int32_t device,
                                    const pbfs_part_options* opt, pbfs_part** out);
pbfs_status pbfs_part_destroy(pbfs_part* p);
/* This rank's share of the reached-component figures of the last traversal
 * (owned vertices only; sum over ranks = N_r, A_r). */
pbfs_status pbfs_part_component(pbfs_part* p, uint64_t* n_reached, uint64_t* arcs_reached);
pbfs_status pbfs_part_get_info(const pbfs_part* p, pbfs_part_info* info);
/* gid(v) (the id used by the bitmaps, queues and dist_local). */
pbfs_status pbfs_part_relabel(const pbfs_part* p, uint64_t v, uint64_t* pi_v);
pbfs_status pbfs_part_begin(pbfs_part* p, uint32_t source, const pbfs_config* cfg, void* stream);
/* One level = pbfs_part_step, the caller's allgather of info.next, then
 * pbfs_part_end_level_async. The level's direction, termination and queue
 * live on the device, so a caller may enqueue several levels ahead and
 * pbfs_part_poll (which synchronises) only now and then: levels enqueued past
 * the end are no-ops. info.next is the allgather target of the NEXT level to
 * be stepped (it alternates every level). */
pbfs_status pbfs_part_step(pbfs_part* p, void* stream);
pbfs_status pbfs_part_end_level_async(pbfs_part* p, void* stream);
/* done: the traversal has finished; levels: levels recorded so far. */
pbfs_status pbfs_part_poll(pbfs_part* p, void* stream, uint32_t* done, uint32_t* levels);
/* The device record of level `depth` (this rank's edges_examined). */
pbfs_status pbfs_part_level_record(pbfs_part* p, uint32_t depth, pbfs_level* rec);
/* end_level_async + poll + the level's record (one sync per level). */
pbfs_status pbfs_part_end_level(pbfs_part* p, void* stream, uint32_t* done, pbfs_level* rec);
pbfs_status pbfs_part_sync(pbfs_part* p, void* stream);
/* dist[v] = dist_pi[gid(v)] for v < vertex_count (dist_pi: padded_count
 * entries, the ranks' dist_local slices concatenated). */
pbfs_status pbfs_part_unrelabel(pbfs_part* p, const uint32_t* dist_pi, uint32_t* dist, void* stream);
/* Host-side helpers: copy this rank's dist_local (local_count u32) to host;
 * un-relabel a host gid-order array (padded_count entries) into dist (n). */
pbfs_status pbfs_part_copy_dist(pbfs_part* p, uint32_t* host_out);
pbfs_status pbfs_part_unrelabel_host(const pbfs_part* p, const uint32_t* dist_pi, uint32_t* dist);

/* ---- multi-partition engine: the exchange fused into the level kernels ----
 * The same 1D vertex partition, run as ONE persistent cooperative launch per
 * device for a whole traversal (pbfs_multi.cu). Partition i lives on
 * devices[i]; partitions on one device (listed contiguously) share that
 * device's launch, so devices = {0, 0, 0, 0} runs four partitions on one
 * GPU through exactly the exchange code that devices = {0, 1, 2, 3} runs over
 * NVLink. Per level every partition stores its discoveries (top-down: its
 * queue segment; bottom-up: its next-bitmap slice) straight into every
 * peer's buffers, then one flag round (a sequence-numbered slot per
 * partition in every partition's exchange block) replaces the allgather and
 * the host round trip; every partition applies the reference's 5 % rule to
 * the summed counts. Replaces, for several GPUs, what pbfs_graph + pbfs_bfs
 * do for one (run_bfs, kernels.hpp:80-81). Hybrid (5 % rule) and its
 * top-down-only dispatch. Peer access is enabled between distinct devices
 * (PBFS_E_DEVICE if a pair has no peer path). */
typedef struct pbfs_multi pbfs_multi;

typedef struct pbfs_multi_info {
  uint64_t vertex_count;
  uint64_t edge_count;
  uint64_t padded_count;      /* gid space */
  uint64_t local_arcs[8];     /* per partition (row slice = column slice arcs) */
  uint32_t partitions;
  uint32_t devices;           /* distinct devices (= launches per traversal) */
  uint32_t ctas_per_partition;
  uint32_t relabel_hashed;
} pbfs_multi_info;

/* Uploads the host CSR once per device, builds each partition there. */
pbfs_status pbfs_multi_create(const pbfs_csr* csr, const int32_t* devices,
                              uint32_t num_partitions, pbfs_multi** out);
pbfs_status pbfs_multi_destroy(pbfs_multi* m);
pbfs_status pbfs_multi_get_info(const pbfs_multi* m, pbfs_multi_info* info);
/* Synchronous traversal: distances gathered in vertex order into dist_host
 * (may be NULL), level records from partition 0, device_ms = first device's
 * start to the last device's end. Same checks and errors as pbfs_bfs. */
pbfs_status pbfs_multi_bfs(pbfs_multi* m, uint32_t source, const pbfs_config* cfg,
                           uint32_t* dist_host, pbfs_level* levels, uint32_t levels_cap,
                           pbfs_run_info* info);
/* Enqueue-only traversal (one launch per device); pbfs_multi_sync waits for
 * every device and reports the span (may be NULL) and any overflow. */
pbfs_status pbfs_multi_bfs_async(pbfs_multi* m, uint32_t source, const pbfs_config* cfg);
pbfs_status pbfs_multi_sync(pbfs_multi* m, float* device_ms);
/* The first device's stream (cudaStream_t as void*): every traversal joins
 * on it, so an event recorded there after pbfs_multi_bfs_async follows the
 * traversal on every device. */
pbfs_status pbfs_multi_stream(pbfs_multi* m, void** stream);
/* Reached-component figures of the last traversal (summed over partitions). */
pbfs_status pbfs_multi_component(pbfs_multi* m, uint64_t* n_reached, uint64_t* arcs_reached);
/* Makes `stream` (a cudaStream_t on any device) wait for the last traversal. */
pbfs_status pbfs_multi_join(pbfs_multi* m, void* stream);
/* Level records of the last traversal (partition 0's), as pbfs_graph_trace. */
pbfs_status pbfs_multi_trace(pbfs_multi* m, pbfs_level* levels, uint32_t levels_cap,
                             uint32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* PBFS_H */

/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the BFS hot path.
 *
 * A plain-C restatement of the reference `parbfs` algorithms, each function
 * citing the reference file:line it follows. Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may
 * load it; the product library never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * golden vectors in tests/golden/ that tests/golden/make_golden.py produced by
 * running the UNMODIFIED reference library (oracle/_ref) in the build
 * container, and against the reference's own hand-coded expectations
 * (test_graph_core.cpp:59-78, test_kernels.cpp:108-118).
 */
#ifndef PBFS_ORACLE_H
#define PBFS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 as specified by [rand.eng.mt] / [rand.predef]. */
typedef struct {
  uint64_t mt[312];
  uint32_t idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);

/* Edge-pair sampling of generator.cpp:41-89 (kind 0 uniform, 1 Kronecker).
 * Writes ef * 2^scale (src, dst) pairs interleaved into pairs[2*i], [2*i+1]. */
int orc_generate_pairs(int kind, uint32_t scale, uint32_t edge_factor,
                       uint64_t seed, uint32_t* pairs);

/* build_csr (csr_graph.cpp:11-55): optional symmetrize (reverse of every
 * non-loop pair), sort, unique. drop_self_loops=1 applies BASELINE's
 * self-loop removal. offsets: n+1 u64; col: capacity
 * 2*npairs. Returns the arc count, or UINT64_MAX on an out-of-range pair. */
uint64_t orc_build_csr(const uint32_t* pairs, uint64_t npairs, uint64_t n,
                       int symmetrize, int drop_self_loops, uint64_t* offsets,
                       uint32_t* col);

/* bfs_serial (kernels.cpp:19-41). dist: n entries, 0xFFFFFFFF = unreached. */
int orc_bfs_serial(uint64_t n, const uint64_t* offsets, const uint32_t* col,
                   uint32_t source, uint32_t* dist);

/* relaxation_distances (tests/support/graphs.hpp:138-156): the O(N*M)
 * Bellman-style fixpoint, independent of the queue BFS. */
int orc_relaxation(uint64_t n, const uint64_t* offsets, const uint32_t* col,
                   uint32_t source, uint32_t* dist);

/* pick_sources (tools/bfsbench.cpp:206-235): mt19937_64(seed), v = rng() % n,
 * keep v iff degree(v) > 0, with replacement. Returns 0, or -1 when no vertex
 * has positive degree. */
int orc_pick_sources(uint64_t n, const uint64_t* offsets, uint32_t count,
                     uint64_t seed, uint32_t* out);

/* simulate_phases (tests/support/graphs.hpp:177-215): the direction each
 * iteration must take, replayed over exact BFS layers. phases[d] = 0 top-down,
 * 1 bottom-up. Returns the number of iterations written (layers). */
uint32_t orc_simulate_phases(uint64_t n, uint64_t m, const uint64_t* offsets,
                             const uint32_t* dist, double threshold,
                             int beamer, double alpha, double beta,
                             uint8_t* phases, uint32_t cap);

/* compute_stats (graph_stats.cpp:9-25). */
void orc_stats(uint64_t n, uint64_t m, const uint64_t* offsets,
               double threshold, double* avg_degree, uint64_t* max_degree,
               int* large_diameter);

/* Config 3 mesh generator (new; specified in SURVEY.md §8(d) and DESIGN.md):
 * side x side grid, id = r*side + c; in row-major order each existing right
 * edge, then each existing down edge, is kept iff unit() < keep; then
 * shortcuts pairs: u = bounded(n), offsets (dr, dc) = bounded(2R+1)-R each,
 * redrawn until 1 <= |dr|+|dc| <= R and the target is inside the grid.
 * Writes pairs; returns the number written (<= 2*side*(side-1) + shortcuts). */
uint64_t orc_mesh_pairs(uint32_t side, double keep, uint64_t shortcuts,
                        uint32_t radius, uint64_t seed, uint32_t* pairs);

/* Reached-component figures used by the GTEPS / roofline arithmetic
 * (SURVEY §8(d)): N_r reached vertices and A_r = sum of their degrees. */
void orc_component(uint64_t n, const uint64_t* offsets, const uint32_t* dist,
                   uint64_t* n_reached, uint64_t* arcs_reached);

#ifdef __cplusplus
}
#endif
#endif

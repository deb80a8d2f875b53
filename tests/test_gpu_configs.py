"""BASELINE.json configs on the B200, every one at full size in the default
GPU run: config 1 (RMAT-20, int32 offsets) for all 64 seeded sources against
the oracle's serial BFS; configs 2-4 (ER 2^24, 4096^2 mesh, RMAT-26) on all
64 of the bench's seeded sources and config 5 (RMAT-28) on 4 of them, against
the reference's own parbfs::bfs_hybrid (oracle/_ref, all host threads) --
distances, per-level phases and distinct sizes; plus size-independent BFS
properties (checked vectorised over every arc). PBFS_TEST_LARGE=1 adds
RMAT-28 on 8 sources and the Beamer rule on 16 RMAT-26 sources."""
import os

import numpy as np
import pytest

import paper_2503_00430_b200 as pb

pytestmark = pytest.mark.gpu
UNREACHED = 0xFFFFFFFF


def bfs_properties(g, dist, source):
    """dist is a BFS layering of the component of `source`: dist[src] = 0,
    no arc crosses more than one level or leaves the reached set, and every
    reached vertex but the source has a neighbour one level closer."""
    assert dist[source] == 0
    deg = g.degrees()
    d64 = dist.astype(np.int64)
    d64[dist == UNREACHED] = -1
    src = np.repeat(np.arange(g.vertex_count, dtype=np.int64), deg)
    du, dv = d64[src], d64[g.column_indices]
    assert ((du < 0) == (dv < 0)).all(), "an arc leaves the reached set"
    both = du >= 0
    assert (np.abs(du[both] - dv[both]) <= 1).all(), "an arc skips a level"
    big = np.iinfo(np.int64).max
    nb = np.where(dv >= 0, dv, big)
    has = deg > 0
    mins = np.full(g.vertex_count, big, dtype=np.int64)
    mins[has] = np.minimum.reduceat(nb, g.row_offsets[:-1][has].astype(np.int64))
    reached = d64 > 0
    assert (mins[reached] == d64[reached] - 1).all(), "a vertex lacks a parent"


def config_graph(name):
    if name == "rmat20":
        return pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 20, 16, 1,
                                            drop_self_loops=True)), 4
    if name == "er24":
        return pb.generate(pb.GeneratorSpec(pb.GeneratorKind.UniformRandom, 24, 16, 1,
                                            drop_self_loops=True)), 8
    if name == "mesh4096":
        return pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Mesh, seed=1, mesh_side=4096,
                                            drop_self_loops=True)), 8
    if name in ("rmat26", "rmat28"):
        return pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, int(name[4:]), 16, 1,
                                            drop_self_loops=True)), 8
    raise KeyError(name)


def dispatch_config(g):
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    if pb.compute_stats(g).category == pb.GraphCategory.LargeDiameter:
        cfg.force_top_down_only = True
    return cfg


def test_config1_rmat20_all_64_sources(port):
    g, offb = config_graph("rmat20")
    dg = g.device(0, offb)
    assert dg.info["device_offset_bytes"] == 4
    cfg = dispatch_config(g)
    for i, s in enumerate(pb.pick_sources(g, 64, 1)):
        want = port.bfs_serial(g.row_offsets, g.column_indices, int(s))
        got = dg.bfs(int(s), cfg).distances
        assert np.array_equal(got, want), int(s)
        if i < 8:
            for v in (pb.KernelVariant.Conventional, pb.KernelVariant.NonAtomic,
                      pb.KernelVariant.HybridBeamer):
                assert np.array_equal(dg.bfs(int(s), pb.KernelConfig(variant=v)).distances,
                                      want)
    bfs_properties(g, got, int(s))


def _ref_graph(g):
    import oracle
    assert oracle.ref_available(), "oracle/_ref (the reference library) must travel with the repo"
    ref = oracle.ref()
    return ref, ref.from_csr(g.row_offsets.astype(np.uint64, copy=False), g.column_indices, True)


def _check_against_reference(g, dg, srcs, cfg, variant=3):
    """Distances, per-level phases and distinct sizes equal the reference's
    own parbfs::bfs_hybrid (variant 3) / bfs_hybrid_beamer (4) on all host
    threads -- acceptance.cpp:112-147's equivalence gate at full size."""
    ref, rg = _ref_graph(g)
    for i, s in enumerate(srcs):
        r = dg.bfs(s, cfg)
        want, recs, _ = ref.run(rg, s, variant, workers=os.cpu_count() or 1,
                                force_td=cfg.force_top_down_only)
        assert np.array_equal(r.distances, want), (i, s)
        assert [(x.depth, int(x.phase), x.distinct_size) for x in r.trace.records] == \
            [(x["depth"], x["phase"], x["distinct_size"]) for x in recs], (i, s)
    del rg


@pytest.fixture(scope="module")
def rmat26():
    g, offb = config_graph("rmat26")
    dg = g.device(0, offb)
    yield g, dg
    g.release_device()


def test_config4_rmat26_all_64_sources_vs_reference_hybrid(rmat26):
    # Every one of the bench's 64 seeded sources (pick_sources, seed 1): the
    # headline workload's distances, phases and distinct sizes (~80 s of
    # reference CPU time on the box's host cores).
    g, dg = rmat26
    cfg = dispatch_config(g)
    assert not cfg.force_top_down_only
    srcs = [int(s) for s in pb.pick_sources(g, 64, 1)]
    _check_against_reference(g, dg, srcs, cfg)


def test_config4_rmat26_beamer_vs_reference_beamer(rmat26):
    g, dg = rmat26
    srcs = [int(s) for s in pb.pick_sources(g, 64, 1)][16:20]
    _check_against_reference(g, dg, srcs, pb.KernelConfig(variant=pb.KernelVariant.HybridBeamer),
                             variant=4)


@pytest.mark.parametrize("name", ["er24", "mesh4096"])
def test_config2_config3_all_64_sources_vs_reference_hybrid(name):
    g, offb = config_graph(name)
    dg = g.device(0, offb)
    cfg = dispatch_config(g)
    if name == "mesh4096":
        assert cfg.force_top_down_only  # avg degree ~3.6 -> the dispatcher's TD-only path
    srcs = [int(s) for s in pb.pick_sources(g, 64, 1)]
    _check_against_reference(g, dg, srcs, cfg)
    bfs_properties(g, dg.bfs(srcs[-1], cfg).distances, srcs[-1])
    g.release_device()


def test_config5_rmat28_4_sources_vs_reference_hybrid():
    # 8.6 G arcs: generation (jump-ahead parallel), 38 GB resident on one
    # B200, four bench sources against the reference's bfs_hybrid.
    g, offb = config_graph("rmat28")
    dg = g.device(0, offb)
    cfg = dispatch_config(g)
    srcs = [int(s) for s in pb.pick_sources(g, 64, 1)][:4]
    _check_against_reference(g, dg, srcs, cfg)
    g.release_device()


@pytest.mark.skipif(os.environ.get("PBFS_TEST_LARGE") != "1", reason="set PBFS_TEST_LARGE=1")
def test_config4_rmat26_properties():
    g, offb = config_graph("rmat26")
    dg = g.device(0, offb)
    cfg = dispatch_config(g)
    for s in pb.pick_sources(g, 2, 1):
        r = dg.bfs(int(s), cfg)
        bfs_properties(g, r.distances, int(s))


@pytest.mark.skipif(os.environ.get("PBFS_TEST_LARGE") != "1", reason="set PBFS_TEST_LARGE=1")
@pytest.mark.parametrize("name", ["rmat28"])
def test_large_configs_all_64_sources_bit_exact(name, port):
    # RMAT-28 on the first 8 bench sources (configs 2-4 run all 64 in the
    # default GPU run above),
    # bit-exact against the reference's own parbfs::bfs_hybrid (oracle/_ref,
    # all host threads) on RMAT-26/28, against the C port's bfs_serial on
    # ER-24 and the mesh; the per-level phases and distinct frontier sizes
    # equal the reference's.
    import oracle
    g, offb = config_graph(name)
    dg = g.device(0, offb)
    cfg = dispatch_config(g)
    srcs = [int(s) for s in pb.pick_sources(g, 64, 1)]
    if name == "rmat28":
        srcs = srcs[:8]
    rg = None
    if name.startswith("rmat2"):
        assert oracle.ref_available()
        ref = oracle.ref()
        rg = ref.from_csr(g.row_offsets.astype(np.uint64, copy=False), g.column_indices, True)
    for i, s in enumerate(srcs):
        r = dg.bfs(s, cfg)
        if rg is not None:
            want, recs, _ = ref.run(rg, s, 3, workers=os.cpu_count() or 1,
                                    force_td=cfg.force_top_down_only)
            assert [(x.depth, int(x.phase), x.distinct_size) for x in r.trace.records] == \
                [(x["depth"], x["phase"], x["distinct_size"]) for x in recs], (name, s)
        else:
            want = port.bfs_serial(g.row_offsets, g.column_indices, s)
        assert np.array_equal(r.distances, want), (name, i, s)
    g.release_device()


@pytest.mark.skipif(os.environ.get("PBFS_TEST_LARGE") != "1", reason="set PBFS_TEST_LARGE=1")
def test_rmat26_beamer_matches_reference_beamer(port):
    # The Beamer-rule hybrid (kernels.cpp:498-511) at full size: distances and
    # the per-level phase / distinct-size sequence equal the reference's own
    # parbfs::bfs_hybrid_beamer on the first 16 bench sources.
    import oracle
    g, offb = config_graph("rmat26")
    dg = g.device(0, offb)
    ref = oracle.ref()
    rg = ref.from_csr(g.row_offsets.astype(np.uint64, copy=False), g.column_indices, True)
    cfg = pb.KernelConfig(variant=pb.KernelVariant.HybridBeamer)
    for s in [int(x) for x in pb.pick_sources(g, 16, 1)]:
        r = dg.bfs(s, cfg)
        want, recs, _ = ref.run(rg, s, 4, workers=os.cpu_count() or 1)
        assert np.array_equal(r.distances, want), s
        assert [(x.depth, int(x.phase), x.distinct_size) for x in r.trace.records] == \
            [(x["depth"], x["phase"], x["distinct_size"]) for x in recs], s
    g.release_device()

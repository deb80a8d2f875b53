"""GPU parity: every traversal runs on the B200 through the C ABI
(libpbfs.so) and is compared bit-exactly with the CPU oracle (serial BFS /
relaxation restated from the reference, pinned by tests/test_oracle.py) and
with the reference's own golden vectors. Mirrors test_kernels.cpp and
acceptance.cpp criteria 1, 2 and 4."""
import glob
import os

import numpy as np
import pytest

import paper_2503_00430_b200 as pb
from paper_2503_00430_b200.parbfs import DeviceGraph
from graphs import (from_edges, hand_suite, make_circulant, make_complete_bipartite,
                    make_clique, make_edgeless, make_path, make_star, random_graph)

pytestmark = pytest.mark.gpu
UNREACHED = 0xFFFFFFFF
V = pb.KernelVariant
GPU_VARIANTS = [V.Conventional, V.NonAtomic, V.Hybrid, V.HybridBeamer, V.VisitedBitmapInline,
                V.HybridPlainStore]
DIRECT = {V.Conventional: pb.bfs_conventional, V.NonAtomic: pb.bfs_nonatomic,
          V.Hybrid: pb.bfs_hybrid, V.HybridBeamer: pb.bfs_hybrid_beamer,
          V.HybridPlainStore: pb.bfs_hybrid_plain,
          V.VisitedBitmapInline: lambda g, s, c: pb.bfs_visited_bitmap(g, s, c, False)}


def run(variant, g, s, **kw):
    cfg = pb.KernelConfig(variant=variant, **kw)
    return DIRECT[variant](g, s, cfg)


def check_trace_shape(r, dist, source):
    # test_kernels.cpp:53-66
    assert r.trace.source == source
    total = 0
    for i, rec in enumerate(r.trace.records):
        assert rec.depth == i
        assert rec.frontier_size == rec.distinct_size + rec.duplicate_count
        total += rec.distinct_size
    assert total == int((dist != UNREACHED).sum())


def phases(r):
    return [int(rec.phase) for rec in r.trace.records]


@pytest.mark.parametrize("variant", GPU_VARIANTS, ids=lambda v: pb.to_string(v))
def test_hand_graphs_match_relaxation(variant, port):
    # test_kernels.cpp:129-166
    for name, g, s in hand_suite():
        want = port.relaxation(g.row_offsets, g.column_indices, s)
        r = run(variant, g, s)
        assert np.array_equal(r.distances, want), name
        assert r.trace.variant == variant
        check_trace_shape(r, r.distances, s)


@pytest.mark.parametrize("offset_bytes", [4, 8])
def test_acceptance_criterion_1_generated_graphs(offset_bytes, port):
    # acceptance.cpp:112-147: 200 graphs, 5 sources each, every GPU variant
    runs = 0
    for i in range(200):
        kind = pb.GeneratorKind.UniformRandom if i % 2 == 0 else pb.GeneratorKind.Kronecker
        spec = pb.GeneratorSpec(kind, 4 + i % 9, 1 + (i * 5) % 16, 7000 + i)
        g = pb.generate(spec)
        dg = g.device(0, offset_bytes)
        raw = port.mt64(i, 4096)
        deg = g.degrees()
        sources = [int(v) for v in (raw % np.uint64(g.vertex_count)) if deg[int(v)] > 0][:5]
        for s in sources:
            want = port.bfs_serial(g.row_offsets, g.column_indices, s)
            for variant in GPU_VARIANTS:
                r = dg.bfs(s, pb.KernelConfig(variant=variant))
                runs += 1
                assert np.array_equal(r.distances, want), (pb.to_string(spec), s, variant)
        g.release_device()
    assert runs >= 4500


def test_golden_vectors_from_reference(golden_dir):
    # distances and per-level phases produced by the reference library itself
    for path in sorted(glob.glob(os.path.join(golden_dir, "gen_*.npz"))):
        gold = np.load(path)
        kind, scale, ef, seed = os.path.basename(path)[4:-4].split("_")
        g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker if kind == "kron"
                                         else pb.GeneratorKind.UniformRandom,
                                         int(scale), int(ef), int(seed)))
        for s in gold["sources"]:
            s = int(s)
            if f"dist_{s}" not in gold:
                continue
            r = run(V.Hybrid, g, s)
            assert np.array_equal(r.distances, gold[f"dist_{s}"]), (path, s)
            assert phases(r) == gold[f"hybrid_phase_{s}"].tolist(), (path, s)
            assert [rec.distinct_size for rec in r.trace.records] == \
                gold[f"hybrid_distinct_{s}"].tolist()
            rb = run(V.HybridBeamer, g, s)
            assert np.array_equal(rb.distances, gold[f"dist_{s}"])
            assert phases(rb) == gold[f"beamer_phase_{s}"].tolist(), (path, s)
            rc = run(V.Conventional, g, s)
            assert np.array_equal(rc.distances, gold[f"dist_{s}"])


def test_star_frontier_series_and_edges():
    # test_kernels.cpp:168-184
    r = run(V.Conventional, make_star(64), 0)
    assert pb.frontier_size_series(r.trace) == [(0, 1), (1, 64)]
    assert [rec.duplicate_count for rec in r.trace.records] == [0, 0]
    assert [rec.edges_examined for rec in r.trace.records] == [64, 64]


def test_zero_degree_source_single_level():
    # test_kernels.cpp:186-197
    r = run(V.Conventional, make_edgeless(5), 3)
    assert r.distances.tolist() == [UNREACHED] * 3 + [0, UNREACHED]
    assert len(r.trace.records) == 1
    assert r.trace.records[0].frontier_size == 1 and r.trace.records[0].edges_examined == 0


def test_small_dense_graph_bottom_up_from_seed(port):
    # test_kernels.cpp:199-211
    g = make_star(16)
    r = run(V.Hybrid, g, 0)
    assert r.trace.records[0].phase == pb.TraversalPhase.BottomUp
    assert r.trace.level_count(pb.TraversalPhase.BottomUp) == len(r.trace.records)
    assert np.array_equal(r.distances, port.relaxation(g.row_offsets, g.column_indices, 0))


def test_threshold_one_keeps_hybrid_top_down():
    # test_kernels.cpp:213-232
    g = make_path(10)
    plain = run(V.NonAtomic, g, 0)
    hyb = run(V.Hybrid, g, 0, hybrid_threshold_fraction=1.0)
    assert hyb.trace.level_count(pb.TraversalPhase.BottomUp) == 0
    assert np.array_equal(hyb.distances, plain.distances)
    assert phases(hyb) == phases(plain)
    assert [r.distinct_size for r in hyb.trace.records] == \
        [r.distinct_size for r in plain.trace.records]


def test_long_path_stays_top_down(port):
    # test_kernels.cpp:234-242
    g = make_path(1000)
    r = run(V.Hybrid, g, 0)
    assert len(r.trace.records) == 1000
    assert r.trace.level_count(pb.TraversalPhase.BottomUp) == 0
    assert np.array_equal(r.distances, port.relaxation(g.row_offsets, g.column_indices, 0))


def test_phases_follow_replayed_rules(port):
    # test_kernels.cpp:244-283 (size fraction and edge count)
    items = [(make_circulant(100, [2, 3, 50]), 0), (make_complete_bipartite(8, 64), 0),
             (random_graph(200, 1400, 21), 0), (make_path(10), 0),
             (make_circulant(100, [2, 3, 50]), 7),
             (pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 10, 8, 77)), 0)]
    for g, s in items:
        if g.degree(s) == 0:
            s = int(np.argmax(g.degrees()))
        dist = port.bfs_serial(g.row_offsets, g.column_indices, s)
        r = run(V.Hybrid, g, s)
        assert phases(r) == port.simulate_phases(g.row_offsets, dist)
        rb = run(V.HybridBeamer, g, s)
        assert phases(rb) == port.simulate_phases(g.row_offsets, dist, beamer=True)
        assert np.array_equal(r.distances, dist) and np.array_equal(rb.distances, dist)


def test_beamer_policy_limits(port):
    # test_kernels.cpp:285-309
    g = make_circulant(100, [2, 3, 50])
    dist = port.bfs_serial(g.row_offsets, g.column_indices, 0)
    r = run(V.HybridBeamer, g, 0, alpha=1e-9)
    assert phases(r) == port.simulate_phases(g.row_offsets, dist, beamer=True, alpha=1e-9)
    assert all(p == 0 for p in phases(r)[:-1]) and phases(r)[-1] == 1
    r = run(V.HybridBeamer, g, 0, alpha=1e9)
    assert phases(r)[0] == 1
    assert phases(r) == port.simulate_phases(g.row_offsets, dist, beamer=True, alpha=1e9)


def test_hybrid_examines_fewer_edges_than_conventional(port):
    # test_kernels.cpp:311-326
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 12, 16, 3))
    src = int(np.argmax(g.degrees()))
    want = port.bfs_serial(g.row_offsets, g.column_indices, src)
    conv = run(V.Conventional, g, src)
    hyb = run(V.Hybrid, g, src)
    assert np.array_equal(conv.distances, want) and np.array_equal(hyb.distances, want)
    assert hyb.trace.level_count(pb.TraversalPhase.BottomUp) >= 1
    assert phases(hyb) == port.simulate_phases(g.row_offsets, want)
    assert hyb.trace.total_edges_examined() < conv.trace.total_edges_examined()


def test_symmetry_requirement_and_directed_top_down():
    # test_kernels.cpp:423-449
    chain = from_edges([(0, 1), (1, 2)], 3, symmetrize=False)
    assert not chain.symmetric
    for v in (V.Hybrid, V.HybridBeamer, V.VisitedBitmapInline):
        with pytest.raises(pb.InputError, match="symmetric"):
            run(v, chain, 0)
    r = run(V.Hybrid, chain, 0, force_top_down_only=True)
    assert r.distances.tolist() == [0, 1, 2]
    assert r.trace.level_count(pb.TraversalPhase.BottomUp) == 0
    assert run(V.Conventional, chain, 0).distances.tolist() == [0, 1, 2]
    assert run(V.NonAtomic, chain, 2).distances.tolist() == [UNREACHED, UNREACHED, 0]


def test_dispatcher_forces_sparse_graphs_top_down(port):
    # test_kernels.cpp:451-497
    edges = [(i, (i + 1) % 100) for i in range(100)] + [(i, i + 50) for i in range(33)]
    g = from_edges(edges, 100)
    st = pb.compute_stats(g)
    assert st.average_degree == pytest.approx(2.66)
    assert st.category == pb.GraphCategory.LargeDiameter
    cfg = pb.KernelConfig(variant=V.Hybrid)
    d = pb.run_bfs(g, 0, cfg, st)
    assert d.trace.level_count(pb.TraversalPhase.BottomUp) == 0
    assert np.array_equal(d.distances, port.relaxation(g.row_offsets, g.column_indices, 0))
    direct = pb.bfs_hybrid(g, 0, cfg)
    assert phases(direct) == port.simulate_phases(g.row_offsets, d.distances)
    star = make_star(40)
    forced = pb.run_bfs(star, 0, cfg, pb.compute_stats(star))
    assert forced.trace.level_count(pb.TraversalPhase.BottomUp) == 0
    free = pb.bfs_hybrid(star, 0, cfg)
    assert free.trace.level_count(pb.TraversalPhase.BottomUp) == 1
    dense = make_circulant(100, [2, 3, 4, 5, 6, 7, 50])
    r = pb.run_bfs(dense, 0, cfg, pb.compute_stats(dense))
    assert r.trace.level_count(pb.TraversalPhase.BottomUp) >= 1


def test_errors_map_to_reference_exceptions():
    # test_kernels.cpp:120-127; variants without a GPU form
    g = make_path(3)
    with pytest.raises(pb.InputError):
        run(V.Conventional, g, 99)
    with pytest.raises(pb.InputError):
        pb.run_bfs(g, 3, pb.KernelConfig(variant=V.Hybrid), pb.compute_stats(g))
    for v in (V.Serial, V.VisitedBitmapDeferred, V.TopDownPeriodicFlush):
        with pytest.raises(pb.ConfigError):
            pb.run_bfs(g, 0, pb.KernelConfig(variant=v), pb.compute_stats(g))
    with pytest.raises(pb.ConfigError):
        run(V.Hybrid, g, 0, hybrid_threshold_fraction=0.0)


def test_same_value_stores_and_duplicates(port):
    # acceptance.cpp:151-186, test_kernels.cpp:553-564
    for g in (random_graph(128, 700, 31), make_clique(24), make_complete_bipartite(16, 16)):
        r = run(V.NonAtomic, g, 0, validate_same_value_stores=True)
        assert r.trace.same_value_violations == 0
        assert np.array_equal(r.distances, port.relaxation(g.row_offsets, g.column_indices, 0))
        check_trace_shape(r, r.distances, 0)


def test_top_down_edges_equal_reached_degree_sum():
    # test_kernels.cpp:566-576
    g = random_graph(160, 900, 13)
    r = run(V.Conventional, g, 2)
    want = int(g.degrees()[r.distances != UNREACHED].sum())
    assert r.trace.total_edges_examined() == want


def test_repeated_and_interleaved_traversals_are_independent(port):
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 14, 16, 5,
                                     drop_self_loops=True))
    dg = g.device(0, 8)
    srcs = [int(s) for s in pb.pick_sources(g, 6, 2)]
    want = {s: port.bfs_serial(g.row_offsets, g.column_indices, s) for s in srcs}
    for _ in range(3):
        for s in srcs:
            for v in GPU_VARIANTS:
                assert np.array_equal(dg.bfs(s, pb.KernelConfig(variant=v)).distances, want[s])


def test_async_api_and_device_component(port):
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 14, 16, 1,
                                     drop_self_loops=True))
    dg = g.device(0, 4)
    s = int(pb.pick_sources(g, 1, 1)[0])
    dg.bfs_async(s, pb.KernelConfig(variant=V.Hybrid))
    dg.sync()
    nr, ar = dg.component()
    want = port.bfs_serial(g.row_offsets, g.column_indices, s)
    assert (nr, ar) == port.component(g.row_offsets, want)


@pytest.mark.parametrize("force,slots", [("0", "4"), ("8", "4"), ("8", "2"), ("8", "8")],
                         ids=["plain", "packed", "packed2", "packed8"])
def test_batch_api_overlapped_copies(force, slots, port, monkeypatch):
    # pbfs_bfs_batch: distances of source i land in outs[i] while later
    # traversals run; "packed" forces the narrow 1/2 B transfers + host
    # widening that the library uses from 2^25 vertices up, with 2, 4 (the
    # default) or 8 transfer slots in flight.
    monkeypatch.setenv("PBFS_FORCE_MODES", force)
    monkeypatch.setenv("PBFS_BATCH_SLOTS", slots)
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 15, 16, 3,
                                     drop_self_loops=True))
    dg = g.device(0, 8)
    srcs = [int(s) for s in pb.pick_sources(g, 7, 4)]
    want = {s: port.bfs_serial(g.row_offsets, g.column_indices, s) for s in srcs}
    for v in (V.Hybrid, V.Conventional, V.NonAtomic):
        cfg = pb.KernelConfig(variant=v)
        outs = [pb.parbfs.pinned_empty(g.vertex_count, np.uint32) for _ in srcs]
        widths = []
        ms = dg.bfs_batch(srcs, cfg, outs, widths)
        assert len(ms) == len(srcs) and all(t > 0 for t in ms)
        # packed: < 15 levels here, so 4-bit codes
        assert widths == [0.5 if force == "8" else 4] * len(srcs)
        for s, o in zip(srcs, outs):
            assert np.array_equal(o, want[s])
        # the handle's device distances are the last source's
        nr, ar = dg.component()
        assert (nr, ar) == port.component(g.row_offsets, want[srcs[-1]])
        # two rotating buffers: each ends with the last source written to it
        rot = [pb.parbfs.pinned_empty(g.vertex_count, np.uint32) for _ in range(2)]
        dg.bfs_batch(srcs, cfg, [rot[i % 2] for i in range(len(srcs))])
        assert np.array_equal(rot[(len(srcs) - 1) % 2], want[srcs[-1]])
        assert np.array_equal(rot[(len(srcs) - 2) % 2], want[srcs[-2]])
        # a single traversal after a batch still sees the right buffers
        assert np.array_equal(dg.bfs(srcs[0], cfg).distances, want[srcs[0]])
    with pytest.raises(pb.InputError, match="out of range"):
        dg.bfs_batch([0, g.vertex_count], pb.KernelConfig(variant=V.Hybrid),
                     [np.empty(g.vertex_count, np.uint32)] * 2)
    # transfer widths: 1 B (< 255 levels, above), 2 B (< 65535 levels) and the
    # full 4 B copy for deeper traversals; pageable outputs work too
    # transfer widths: 4-bit codes (< 15 levels, above), then ...
    for n in (100, 600, 70000):
        pg = make_path(n)
        pdg = pg.device(0, 8)
        srcs = [0, n - 1, n // 3]
        outs = [np.empty(n, np.uint32) for _ in srcs]
        widths = []
        pdg.bfs_batch(srcs, pb.KernelConfig(variant=V.Hybrid), outs, widths)
        for s, o, w in zip(srcs, outs, widths):
            want_s = port.bfs_serial(pg.row_offsets, pg.column_indices, s)
            assert np.array_equal(o, want_s)
            levels = int(want_s.max()) + 1  # a path is connected
            if force == "8":
                assert w == (0.5 if levels < 15 else 1 if levels < 255 else 2 if levels < 65535 else 4)
        pg.release_device()


@pytest.mark.parametrize("force", [1, 2, 4, 7])
def test_size_gated_paths_forced_on_small_graphs(force, port, monkeypatch):
    # Paths that only switch on at RMAT-26 scale (sparse bottom-up tasks, the
    # 8-words-per-lane compaction, the >= 2^30-arc hub split), forced through
    # the PBFS_FORCE_MODES test hook so they are parity-checked here too.
    monkeypatch.setenv("PBFS_FORCE_MODES", str(force))
    graphs = [pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 15, 16, 7,
                                           drop_self_loops=True)),
              pb.generate(pb.GeneratorSpec(pb.GeneratorKind.UniformRandom, 14, 8, 2,
                                           drop_self_loops=True)),
              random_graph(3000, 9000, 11)]
    for g in graphs:
        dg = g.device(0, 8)
        for s in [int(x) for x in pb.pick_sources(g, 3, 5)]:
            want = port.bfs_serial(g.row_offsets, g.column_indices, s)
            for v in (V.Hybrid, V.HybridBeamer, V.NonAtomic, V.Conventional):
                r = dg.bfs(s, pb.KernelConfig(variant=v))
                assert np.array_equal(r.distances, want), (force, v, s)
            r = dg.bfs(s, pb.KernelConfig(variant=V.Hybrid, hybrid_threshold_fraction=0.001))
            assert np.array_equal(r.distances, want)
        g.release_device()


@pytest.mark.parametrize("force", [0, 2, 4])
def test_reduction_claim_forced_on_small_graphs(force, port, monkeypatch):
    # Top-down levels of >= 65536 frontier vertices claim with no-return reds
    # and compact the next-frontier bitmap afterwards; forced onto every
    # top-down level here (PBFS_RED_MINQ=1), with the narrow and the wide
    # compaction and the >= 2^30-arc hub split (1024-edge items). Distances must equal the oracle's, and per-level records
    # the atomic-claim run's (phases, distinct sizes; raw == distinct).
    monkeypatch.setenv("PBFS_RED_MINQ", "1")
    monkeypatch.setenv("PBFS_FORCE_MODES", str(force))
    graphs = [(pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 15, 16, 7,
                                            drop_self_loops=True)), 8),
              (pb.generate(pb.GeneratorSpec(pb.GeneratorKind.UniformRandom, 14, 8, 2,
                                            drop_self_loops=True)), 4),
              (make_path(300), 8), (make_star(5000), 4), (random_graph(3000, 9000, 11), 8)]
    for g, ob in graphs:
        dg = DeviceGraph(g, 0, ob)
        monkeypatch.setenv("PBFS_RED_MINQ", "0")
        ref = DeviceGraph(g, 0, ob)
        monkeypatch.setenv("PBFS_RED_MINQ", "1")
        for s in [int(x) for x in pb.pick_sources(g, 3, 4)]:
            want = port.bfs_serial(g.row_offsets, g.column_indices, s)
            for v in (V.Hybrid, V.VisitedBitmapInline, V.HybridBeamer):
                for kw in ({}, {"force_top_down_only": True}, {"hybrid_threshold_fraction": 0.5}):
                    cfg = pb.KernelConfig(variant=v, **kw)
                    r = dg.bfs(s, cfg)
                    assert np.array_equal(r.distances, want), (v, s, kw)
                    base = ref.bfs(s, cfg)
                    assert ([(x.phase, x.distinct_size, x.frontier_size) for x in r.trace.records]
                            == [(x.phase, x.distinct_size, x.frontier_size)
                                for x in base.trace.records]), (v, s, kw)
        ref.close()
        dg.close()


def test_time_run_checks_every_run(port):
    # timing.cpp:33-69 and test_instrumentation.cpp:168-198 (fault injection)
    g = make_circulant(64, [3])
    want = port.bfs_serial(g.row_offsets, g.column_indices, 0)
    rep = pb.time_run(g, 0, pb.KernelConfig(variant=V.Hybrid), 3, 1, pb.compute_stats(g), want)
    assert len(rep.samples_ns) == 3 and rep.median_ns in rep.samples_ns

    def broken(gr, s, c):
        r = pb.bfs_hybrid(gr, s, c)
        r.distances = r.distances.copy()
        r.distances[5] += 1
        return r
    with pytest.raises(pb.CorrectnessError, match="vertex 5"):
        pb.time_run(g, 0, pb.KernelConfig(variant=V.Hybrid), 1, 0, broken, want)


@pytest.mark.parametrize("offset_bytes", [4, 8])
def test_latency_mode_matches_the_general_top_down(offset_bytes, port, monkeypatch):
    # Hub-free graphs run top-down only take the latency-mode kernel path
    # (16 B queue entries with row ranges, atom.or-only claims, one CTA per
    # SM); it must give the oracle's distances and the general path's trace.
    graphs = [pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Mesh, seed=3, mesh_side=96,
                                           drop_self_loops=True)),
              make_path(5000), make_circulant(4000, [1, 7, 33]),
              random_graph(3000, 6000, 5)]
    for g in graphs:
        assert int(g.degrees().max()) <= 128
        srcs = [int(x) for x in pb.pick_sources(g, 3, 2)]
        recs = {}
        for lat in ("1", "0"):
            monkeypatch.setenv("PBFS_LATENCY", lat)
            dg = g.device(0, offset_bytes)
            for s in srcs:
                want = port.bfs_serial(g.row_offsets, g.column_indices, s)
                r = dg.bfs(s, pb.KernelConfig(variant=V.Hybrid, force_top_down_only=True))
                assert np.array_equal(r.distances, want), (lat, s)
                recs[lat, s] = [(x.depth, x.phase, x.frontier_size, x.distinct_size,
                                 x.edges_examined) for x in r.trace.records]
            g.release_device()
        for s in srcs:
            assert recs["1", s] == recs["0", s]


def test_async_on_two_streams_is_ordered(port):
    # pbfs_bfs_async on caller streams: every launch waits for the handle's
    # previous one (they share ctl / bitmaps / dist), whichever streams the
    # callers pass; then pbfs_bfs on the handle's own stream and the
    # component read see the last traversal.
    import torch
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 16, 16, 2,
                                     drop_self_loops=True))
    dg = g.device(0, 8)
    srcs = [int(s) for s in pb.pick_sources(g, 6, 3)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    cfg = pb.KernelConfig(variant=V.Hybrid)
    for i, s in enumerate(srcs):
        dg.bfs_async(s, cfg, streams[i % 2].cuda_stream)
    # No host sync in between: the component read must follow the last launch.
    nr, ar = dg.component()
    want = port.bfs_serial(g.row_offsets, g.column_indices, srcs[-1])
    assert (nr, ar) == port.component(g.row_offsets, want)
    for i, s in enumerate(srcs):
        dg.bfs_async(s, cfg, streams[i % 2].cuda_stream)
        got = dg.bfs(srcs[0], cfg).distances
        assert np.array_equal(got, port.bfs_serial(g.row_offsets, g.column_indices, srcs[0]))
    dg.sync(streams[0].cuda_stream)


def test_trace_deeper_than_the_default_record_buffer(port):
    # A path of 2^20 + 40 vertices: more levels than the default device record
    # buffer (2^20); every level is still recorded (trace.hpp:37-48).
    n = (1 << 20) + 40
    off = np.zeros(n + 1, dtype=np.uint64)
    deg = np.full(n, 2, dtype=np.uint64)
    deg[0] = deg[-1] = 1
    off[1:] = np.cumsum(deg)
    col = np.empty(int(off[-1]), dtype=np.uint32)
    v = np.arange(n, dtype=np.int64)
    left = off[:-1].astype(np.int64)
    col[left[1:]] = v[1:] - 1                      # left neighbour first (ascending)
    col[left[:-1] + (v[:-1] > 0)] = v[:-1] + 1     # then the right one
    g = pb.CsrGraph(n, off, col, True)
    cfg = pb.KernelConfig(variant=V.Hybrid, force_top_down_only=True)
    r = g.device(0, 8).bfs(0, cfg)
    assert np.array_equal(r.distances, np.arange(n, dtype=np.uint32))
    assert len(r.trace.records) == n
    assert r.trace.records[-1].depth == n - 1 and r.trace.records[-1].distinct_size == 1


def test_single_call_into_pageable_memory_packed(port, monkeypatch):
    # pbfs_bfs into a PAGEABLE destination (numpy, or the C++ adapter's
    # std::vector) takes the packed 1-2 B/vertex transfer + host widening;
    # kForcePack (8) runs it on small graphs: 1 B codes, 2 B codes (a path of
    # 300 levels), and the plain 4 B copy past 65534 levels.
    monkeypatch.setenv("PBFS_FORCE_MODES", "8")
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 15, 16, 9,
                                     drop_self_loops=True))
    dg = g.device(0, 8)
    for s in pb.pick_sources(g, 4, 2):
        out = np.empty(g.vertex_count, dtype=np.uint32)  # pageable
        dg.bfs(int(s), pb.KernelConfig(variant=V.Hybrid), out=out)
        assert np.array_equal(out, port.bfs_serial(g.row_offsets, g.column_indices, int(s)))
    for n in (300, 70000):
        p = make_path(n)
        out = np.empty(n, dtype=np.uint32)
        p.device(0, 8).bfs(0, pb.KernelConfig(variant=V.Hybrid, force_top_down_only=True),
                           out=out, want_trace=False)
        assert np.array_equal(out, np.arange(n, dtype=np.uint32))
    # Code widths at ragged sizes (n not a multiple of the 32-vertex nibble
    # group or the 16-entry widening step), through a misaligned destination,
    # with unreached vertices: 4-bit codes (< 15 levels) and 1 B codes (a
    # 40-level path glued on), single calls and a batch.
    for n, m, tail in ((3001, 9000, 0), (4097, 20000, 0), (1531, 5000, 40)):
        rg = random_graph(n, m, seed=n)
        if tail:
            pairs = np.column_stack([np.repeat(np.arange(n, dtype=np.int64),
                                               np.diff(rg.row_offsets).astype(np.int64)),
                                     rg.column_indices.astype(np.int64)])
            chain = np.column_stack([np.arange(n - 1, n - 1 + tail), np.arange(n, n + tail)])
            rg = pb.build_csr(np.vstack([pairs, chain]), n + tail, True, drop_self_loops=True)
        rdg = rg.device(0, 8)
        srcs = [int(x) for x in pb.pick_sources(rg, 3, 5)]
        want = {s: port.bfs_serial(rg.row_offsets, rg.column_indices, s) for s in srcs}
        for s in srcs:
            backing = np.empty(rg.vertex_count + 2, dtype=np.uint32)
            out = backing[2:]  # 8 B past the allocation's alignment: a scalar prologue, then the vector loop
            rdg.bfs(s, pb.KernelConfig(variant=V.Hybrid), out=out, want_trace=False)
            assert np.array_equal(out, want[s]), (n, s)
        outs = [np.empty(rg.vertex_count, np.uint32) for _ in srcs]
        widths = []
        rdg.bfs_batch(srcs, pb.KernelConfig(variant=V.Hybrid), outs, widths)
        for s, o, w in zip(srcs, outs, widths):
            assert np.array_equal(o, want[s]), (n, s)
            levels = int(want[s][want[s] != 0xFFFFFFFF].max()) + 1
            assert w == (0.5 if levels < 15 else 1), (n, s, levels, w)

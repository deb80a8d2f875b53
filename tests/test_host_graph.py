"""Host graph layer of the product library (libpbfs.so, CPU side): generator,
builder, classifier, sources, CSR1 — checked against the reference's golden
vectors and its own unit-test expectations (test_graph_core.cpp)."""
import glob
import hashlib
import io
import os

import numpy as np
import pytest

import paper_2503_00430_b200 as pb
from graphs import make_circulant, make_path, random_graph


def spec_of(path):
    kind, scale, ef, seed = os.path.basename(path)[4:-4].split("_")
    return pb.GeneratorKind.Kronecker if kind == "kron" else pb.GeneratorKind.UniformRandom, \
        int(scale), int(ef), int(seed)


def test_generate_matches_reference_bit_for_bit(golden_dir):
    for path in sorted(glob.glob(os.path.join(golden_dir, "gen_*.npz"))):
        gold = np.load(path)
        kind, scale, ef, seed = spec_of(path)
        for threads in (1, 3):
            g = pb.generate(pb.GeneratorSpec(kind, scale, ef, seed), threads=threads)
            assert g.symmetric
            assert hashlib.sha256(g.row_offsets.tobytes()).hexdigest() == \
                str(gold["sha256_offsets"]), path
            assert hashlib.sha256(g.column_indices.tobytes()).hexdigest() == \
                str(gold["sha256_col"]), path


def test_generate_drop_self_loops_matches_oracle(port):
    for kind, scale, ef, seed in [(1, 10, 16, 1), (0, 9, 8, 4), (1, 14, 16, 2)]:
        g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind(kind), scale, ef, seed,
                                         drop_self_loops=True))
        off, col = port.build_csr(port.generate_pairs(kind, scale, ef, seed), 1 << scale,
                                  symmetrize=True, drop_self_loops=True)
        assert np.array_equal(g.row_offsets, off) and np.array_equal(g.column_indices, col)
        src = np.repeat(np.arange(g.vertex_count), g.degrees())
        assert not (src == g.column_indices).any()


def test_build_csr_golden_arrays():
    # test_graph_core.cpp:59-78
    edges = [(1, 0), (0, 1), (0, 1), (2, 2), (2, 0)]
    g = pb.build_csr(edges, 3, symmetrize=False)
    assert (g.vertex_count, g.edge_count) == (3, 4)
    assert g.row_offsets.tolist() == [0, 1, 2, 4] and g.column_indices.tolist() == [1, 0, 0, 2]
    assert not g.symmetric
    pb.validate_csr(g)
    g = pb.build_csr(edges, 3, symmetrize=True)
    assert g.row_offsets.tolist() == [0, 2, 3, 5] and g.column_indices.tolist() == [1, 2, 0, 0, 2]
    assert g.symmetric and pb.adjacency_is_symmetric(g)


def test_build_csr_parallel_equals_oracle(port):
    raw = port.mt64(99, 400000)
    pairs = (raw % np.uint64(5000)).astype(np.uint32).reshape(-1, 2)
    for sym in (True, False):
        off, col = port.build_csr(pairs, 5000, symmetrize=sym)
        for threads in (1, 2, 7):
            g = pb.build_csr(pairs, 5000, symmetrize=sym, threads=threads)
            assert np.array_equal(g.row_offsets, off) and np.array_equal(g.column_indices, col)


def test_build_csr_rejects_out_of_range():
    with pytest.raises(pb.InputError, match="references a vertex"):
        pb.build_csr([(0, 1), (2, 5)], 3, symmetrize=True)
    with pytest.raises(pb.InputError):
        pb.build_csr([(0, 1)], 2**31, symmetrize=True)


def test_generator_contract():
    # test_graph_core.cpp:257-303
    a = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 6, 4, 99))
    b = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 6, 4, 99))
    assert a.structurally_equal(b) and a.symmetric
    c = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 6, 4, 100))
    assert not c.structurally_equal(a)
    for scale in (4, 7, 10):
        g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.UniformRandom, scale, 2, scale))
        assert g.vertex_count == 1 << scale and g.edge_count <= 4 * g.vertex_count
        pb.validate_csr(g)
    with pytest.raises(pb.ConfigError):
        pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 0, 4, 1))
    with pytest.raises(pb.ConfigError):
        pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 5, 0, 1))
    with pytest.raises(pb.CapacityError):
        pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 31, 1, 1))
    assert pb.to_string(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 10, 15, 42)) == "kron:10:15:42"
    assert pb.to_string(pb.GeneratorKind.UniformRandom) == "uniform"


def test_mesh_generator_matches_oracle(port):
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Mesh, seed=3, mesh_side=128,
                                     drop_self_loops=True))
    pairs = port.mesh_pairs(128, 0.9, round(0.001 * 128 * 128), 32, 3)
    off, col = port.build_csr(pairs, 128 * 128, symmetrize=True, drop_self_loops=True)
    assert np.array_equal(g.row_offsets, off) and np.array_equal(g.column_indices, col)
    st = pb.compute_stats(g)
    assert 3.4 < st.average_degree < 3.8 and st.category == pb.GraphCategory.LargeDiameter


def test_stats_and_classifier():
    # test_graph_core.cpp:305-315
    s = pb.compute_stats(make_path(3))
    assert (s.vertex_count, s.edge_count, s.max_degree) == (3, 4, 2)
    assert s.average_degree == pytest.approx(4.0 / 3.0)
    assert s.category == pb.GraphCategory.LargeDiameter
    g = make_circulant(100, [2, 3, 50])
    s = pb.compute_stats(g)
    assert s.average_degree == pytest.approx(7.0) and s.max_degree == 7
    assert s.category == pb.GraphCategory.SmallDiameter
    assert pb.compute_stats(g, 7.5).category == pb.GraphCategory.LargeDiameter
    with pytest.raises(pb.InputError):
        pb.compute_stats(pb.build_csr(np.zeros((0, 2)), 0, True))


def test_pick_sources_matches_oracle(port):
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 12, 16, 1,
                                     drop_self_loops=True))
    assert np.array_equal(pb.pick_sources(g, 64, 1),
                          port.pick_sources(g.row_offsets, 64, 1))
    with pytest.raises(pb.ConfigError):
        pb.pick_sources(pb.build_csr(np.zeros((0, 2)), 5, True), 3, 1)


def test_csr1_golden_bytes(tmp_path):
    # test_graph_core.cpp:182-203
    p = tmp_path / "golden.csr"
    pb.save_binary_csr(make_path(3), str(p))
    expected = (b"CSR1" + (3).to_bytes(8, "little") + (4).to_bytes(8, "little")
                + b"".join(x.to_bytes(8, "little") for x in (0, 1, 3, 4))
                + b"".join(x.to_bytes(4, "little") for x in (1, 0, 2, 1)))
    assert p.read_bytes() == expected


def test_csr1_roundtrip_and_errors(tmp_path):
    g = random_graph(200, 600, 11)
    p = tmp_path / "round.csr"
    pb.save_binary_csr(g, str(p))
    back = pb.load_binary_csr(str(p))
    assert back.structurally_equal(g) and back.symmetric == g.symmetric
    raw = p.read_bytes()
    bad = tmp_path / "bad.csr"
    bad.write_bytes(b"CSR2" + raw[4:])
    with pytest.raises(pb.FormatError, match="missing CSR1 header"):
        pb.load_binary_csr(str(bad))
    bad.write_bytes(raw[:-3])
    with pytest.raises(pb.FormatError, match="truncated"):
        pb.load_binary_csr(str(bad))
    bad.write_bytes(raw + b"\0")
    with pytest.raises(pb.FormatError, match="trailing"):
        pb.load_binary_csr(str(bad))
    with pytest.raises(pb.InputError):
        pb.load_binary_csr(str(tmp_path / "missing.csr"))
    # A crafted edge count (m * 4 wraps 64 bits) is rejected from the file
    # size before any allocation.
    bad.write_bytes(raw[:12] + ((1 << 62) + 1).to_bytes(8, "little") + raw[20:])
    with pytest.raises(pb.FormatError, match="truncated"):
        pb.load_binary_csr(str(bad))
    # A huge interior offset is caught by the offsets-first pass, before any
    # column read.
    n = g.vertex_count
    offs = bytearray(raw[20:20 + 8 * (n + 1)])
    offs[8 * 5:8 * 6] = (1 << 40).to_bytes(8, "little")
    bad.write_bytes(raw[:20] + bytes(offs) + raw[20 + 8 * (n + 1):])
    with pytest.raises(pb.FormatError, match="decreases|exceeds"):
        pb.load_binary_csr(str(bad))


def test_validate_csr_errors():
    g = make_path(4)
    broken = pb.CsrGraph(4, g.row_offsets.copy(), g.column_indices.copy(), True)
    broken.column_indices[1] = 9
    with pytest.raises(pb.FormatError):
        pb.validate_csr(broken)
    broken = pb.CsrGraph(4, g.row_offsets.copy(), g.column_indices.copy(), True)
    broken.row_offsets[-1] = 99
    with pytest.raises(pb.FormatError, match="edge count"):
        pb.validate_csr(broken)


def test_config_validation_and_labels():
    # test_kernels.cpp:501-547
    pb.validate(pb.KernelConfig())
    for kw in [dict(worker_count=0), dict(hybrid_threshold_fraction=0.0),
               dict(hybrid_threshold_fraction=1.5), dict(alpha=0.0), dict(beta=-1.0),
               dict(flush_capacity=0)]:
        with pytest.raises(pb.ConfigError):
            pb.validate(pb.KernelConfig(**kw))
    pb.validate(pb.KernelConfig(hybrid_threshold_fraction=1.0))
    for v in pb.KernelVariant:
        assert pb.parse_kernel_variant(pb.to_string(v)) == v
    assert pb.to_string(pb.KernelVariant.HybridBeamer) == "hybrid-beamer"
    assert pb.to_string(pb.KernelVariant.TopDownPeriodicFlush) == "periodic-flush"
    assert pb.parse_kernel_variant("dfs") is None
    assert pb.to_string(pb.TraversalPhase.TopDown) == "top-down"
    assert pb.to_string(pb.TraversalPhase.BottomUp) == "bottom-up"


def test_trace_helpers():
    # trace.cpp:21-61 (test_instrumentation.cpp:99-118 frozen schema)
    t = pb.TraversalTrace(variant=pb.KernelVariant.Hybrid, source=3)
    with pytest.raises(pb.MetricError):
        pb.average_duplicate_percentage(t)
    t.records = [pb.LevelRecord(0, pb.TraversalPhase.TopDown, 1, 1, 0, 5, 0, 10),
                 pb.LevelRecord(1, pb.TraversalPhase.BottomUp, 4, 2, 2, 7, 0, 20),
                 pb.LevelRecord(2, pb.TraversalPhase.TopDown, 0, 0, 0, 0, 0, 5)]
    assert pb.average_duplicate_percentage(t) == pytest.approx(25.0)
    assert pb.frontier_size_series(t) == [(0, 1), (1, 4), (2, 0)]
    assert t.total_edges_examined() == 12 and t.level_count(pb.TraversalPhase.BottomUp) == 1
    out = io.StringIO()
    pb.write_trace_csv_header(out)
    pb.write_trace_csv(out, t, "r1")
    lines = out.getvalue().splitlines()
    assert lines[0] == ("run_id,variant,source,depth,phase,frontier_size,distinct_size,"
                        "duplicate_count,edges_examined,flush_events,elapsed_ns")
    assert lines[2] == "r1,hybrid,3,1,bottom-up,4,2,2,7,0,20"


@pytest.mark.parametrize("kind,scale,ef", [(pb.GeneratorKind.Kronecker, 17, 8),
                                           (pb.GeneratorKind.UniformRandom, 16, 16)])
def test_parallel_generation_equals_one_stream(kind, scale, ef):
    # The stream is cut into chunks whose start states come from mt19937_64
    # jump-ahead (pbfs_mt64.cpp); any thread count must give the graph the
    # single sequential stream gives (threads=1 never jumps), and the
    # reference's own generate() (pinned by the digests above).
    spec = pb.GeneratorSpec(kind, scale, ef, 77, drop_self_loops=True)
    one = pb.generate(spec, threads=1)
    for t in (2, 3, 8):
        g = pb.generate(spec, threads=t)
        assert np.array_equal(g.row_offsets, one.row_offsets), t
        assert np.array_equal(g.column_indices, one.column_indices), t

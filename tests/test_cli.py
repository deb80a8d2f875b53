"""bfsbench-compatible CLI (paper_2503_00430_b200.cli) and the edge-list
loader: subcommands, CSV schemas and exit codes of tools/bfsbench.cpp."""
import csv
import os

import numpy as np
import pytest

import paper_2503_00430_b200 as pb
from paper_2503_00430_b200 import cli


def test_stats_and_generate(tmp_path, capsys):
    assert cli.main(["stats", "--gen", "kron:10:15:1"]) == 0
    out = capsys.readouterr().out
    assert "vertices: 1024" in out and "category: small-diameter" in out
    f = tmp_path / "g.csr"
    assert cli.main(["generate", "--gen", "uniform:8:4:3", "--out", str(f)]) == 0
    g = pb.load_binary_csr(str(f))
    assert g.structurally_equal(pb.generate(pb.GeneratorSpec(pb.GeneratorKind.UniformRandom,
                                                              8, 4, 3)))
    assert cli.main(["stats", "--graph", str(f)]) == 0


def test_exit_codes(tmp_path):
    assert cli.main(["stats", "--gen", "kron:10:15"]) == 2          # ConfigError
    assert cli.main(["stats", "--gen", "dfs:10:15:1"]) == 2
    assert cli.main(["stats", "--graph", str(tmp_path / "nope")]) == 3  # InputError
    bad = tmp_path / "bad.csr"
    bad.write_bytes(b"CSR1" + b"\0" * 7)
    assert cli.main(["stats", "--graph", str(bad)]) == 3           # FormatError
    assert cli.main(["frobnicate"]) == 2
    assert cli.main(["generate", "--gen", "kron:4:4:1"]) == 2       # missing --out


def test_edge_list_loader(tmp_path):
    # edge_list.cpp:26-82
    f = tmp_path / "g.txt"
    f.write_text("% header\n# comment\n\n1 2 0.5\n2 3\n3 1 extra fields\n")
    g = pb.load_edge_list(str(f), one_based=True)
    assert g.vertex_count == 3 and g.symmetric
    assert g.row_offsets.tolist() == [0, 2, 4, 6]
    d = pb.load_edge_list(str(f), one_based=False, symmetrize=False, vertex_count_hint=6)
    assert d.vertex_count == 6 and not d.symmetric
    f.write_text("1 x\n")
    with pytest.raises(pb.InputError, match="expected two integer"):
        pb.load_edge_list(str(f))
    f.write_text("0 1\n")
    with pytest.raises(pb.InputError, match="below the index base"):
        pb.load_edge_list(str(f), one_based=True)
    with pytest.raises(pb.InputError, match="declared vertex count"):
        pb.load_edge_list(str(f), vertex_count_hint=1)


def test_layering_certificate_catches_faults():
    import oracle
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 10, 8, 5))
    s = int(pb.pick_sources(g, 1, 1)[0])
    d = oracle.port().bfs_serial(g.row_offsets, g.column_indices, s)
    assert cli.bfs_layering_ok(g, d, s)[0]
    for v in (s, int(np.nonzero(d == 2)[0][0]), int(np.nonzero(d == 1)[0][0])):
        bad = d.copy()
        bad[v] += 1
        assert not cli.bfs_layering_ok(g, bad, s)[0]


@pytest.mark.gpu
def test_verify_and_run_on_gpu(tmp_path, capsys):
    assert cli.main(["verify", "--gen", "kron:12:16:1", "--sources", "4"]) == 0
    assert "verification passed" in capsys.readouterr().out
    assert cli.main(["verify", "--gen", "kron:12:16:1", "--sources", "2",
                     "--inject-fault"]) == 1
    out = tmp_path / "out"
    assert cli.main(["run", "--gen", "kron:12:16:1", "--sources", "3", "--trials", "2",
                     "--warmups", "1", "--variants", "conventional,hybrid",
                     "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out / "results.csv")))
    assert len(rows) == 6 and set(rows[0]) == {
        "graph", "variant", "worker_count", "source", "trials", "median_ns", "min_ns",
        "max_ns", "total_edges_examined", "avg_duplicate_pct", "bu_levels", "td_levels"}
    assert any(int(r["bu_levels"]) > 0 for r in rows if r["variant"] == "hybrid")
    traces = list(csv.DictReader(open(out / "traces.csv")))
    assert traces and traces[0]["run_id"].startswith("kron:12:16:1/")


@pytest.mark.gpu
def test_level_observer_snapshots(port):
    # kernel_config.hpp:26-36; test_kernels.cpp:213-232 compares level sets
    from graphs import make_path, make_star
    sets = {}
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid, hybrid_threshold_fraction=1.0,
                          level_observer=lambda snap: sets.__setitem__(
                              snap.depth, sorted(snap.entries.tolist())))
    pb.bfs_hybrid(make_path(10), 0, cfg)
    assert sets == {d: [d] for d in range(10)}
    seen = []
    cfg = pb.KernelConfig(variant=pb.KernelVariant.NonAtomic,
                          level_observer=lambda snap: seen.append(
                              (snap.depth, snap.produced_by, snap.entries.tolist())))
    pb.bfs_nonatomic(make_star(8), 0, cfg)
    assert seen == [(0, pb.TraversalPhase.TopDown, [0]),
                    (1, pb.TraversalPhase.TopDown, list(range(1, 9)))]

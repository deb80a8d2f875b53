"""Pins the CPU oracle (oracle/pbfs_oracle.c) before it is trusted: against
the golden vectors the reference library produced (tests/golden/*.npz, made
by tests/golden/make_golden.py) and against the reference's own hand-coded
expectations."""
import glob
import hashlib
import os

import numpy as np
import pytest

UNREACHED = 0xFFFFFFFF


def golden_files(golden_dir):
    return sorted(glob.glob(os.path.join(golden_dir, "gen_*.npz")))


def spec_of(path):
    kind, scale, ef, seed = os.path.basename(path)[4:-4].split("_")
    return (1 if kind == "kron" else 0), int(scale), int(ef), int(seed)


def test_mt19937_64_known_answer(port):
    # [rand.predef]: the 10000th output of a default-constructed
    # mt19937_64 (seed 5489) is 9981545732273789042.
    vals = port.mt64(5489, 10000)
    assert int(vals[-1]) == 9981545732273789042
    assert int(vals[0]) == 14514284786278117030


def test_build_csr_hand_golden(port):
    # test_graph_core.cpp:59-78
    pairs = np.array([[1, 0], [0, 1], [0, 1], [2, 2], [2, 0]], dtype=np.uint32)
    off, col = port.build_csr(pairs, 3, symmetrize=False)
    assert off.tolist() == [0, 1, 2, 4] and col.tolist() == [1, 0, 0, 2]
    off, col = port.build_csr(pairs, 3, symmetrize=True)
    assert off.tolist() == [0, 2, 3, 5] and col.tolist() == [1, 2, 0, 0, 2]
    off, col = port.build_csr(pairs, 3, symmetrize=True, drop_self_loops=True)
    assert off.tolist() == [0, 2, 3, 4] and col.tolist() == [1, 2, 0, 0]
    with pytest.raises(ValueError):
        port.build_csr(np.array([[0, 3]], dtype=np.uint32), 3)


def test_generator_matches_reference_golden(port, golden_dir):
    files = golden_files(golden_dir)
    assert len(files) >= 7
    for path in files:
        g = np.load(path)
        kind, scale, ef, seed = spec_of(path)
        off, col = port.build_csr(port.generate_pairs(kind, scale, ef, seed), 1 << scale,
                                  symmetrize=True)
        assert int(g["m"]) == col.size, path
        assert hashlib.sha256(off.tobytes()).hexdigest() == str(g["sha256_offsets"]), path
        assert hashlib.sha256(col.tobytes()).hexdigest() == str(g["sha256_col"]), path
        if "col" in g:
            assert np.array_equal(off, g["offsets"]) and np.array_equal(col, g["col"])


def test_serial_bfs_and_phases_match_reference_golden(port, golden_dir):
    for path in golden_files(golden_dir):
        g = np.load(path)
        kind, scale, ef, seed = spec_of(path)
        off, col = port.build_csr(port.generate_pairs(kind, scale, ef, seed), 1 << scale)
        for s in g["sources"]:
            key = f"dist_{int(s)}"
            if key not in g:
                continue
            dist = port.bfs_serial(off, col, int(s))
            assert np.array_equal(dist, g[key]), (path, s)
            assert port.simulate_phases(off, dist) == g[f"hybrid_phase_{int(s)}"].tolist()
            assert port.simulate_phases(off, dist, beamer=True) == \
                g[f"beamer_phase_{int(s)}"].tolist()
            # distinct sizes per level == exact layer sizes (trace.hpp:14-24)
            sizes = np.bincount(dist[dist != UNREACHED]).tolist()
            assert sizes == g[f"hybrid_distinct_{int(s)}"].tolist()


def test_stats_match_reference_golden(port, golden_dir):
    for path in golden_files(golden_dir):
        g = np.load(path)
        kind, scale, ef, seed = spec_of(path)
        off, _ = port.build_csr(port.generate_pairs(kind, scale, ef, seed), 1 << scale)
        avg, mx, large = port.stats(off)
        assert (avg, mx, large) == (g["stats"][0], int(g["stats"][1]), bool(g["stats"][2]))


def test_relaxation_equals_serial(port):
    # test_kernels.cpp:108-118: serial BFS vs the independent relaxation oracle
    for seed in (5, 6, 7):
        raw = port.mt64(seed, 2000)
        pairs = (raw % np.uint64(256)).astype(np.uint32).reshape(-1, 2)
        off, col = port.build_csr(pairs, 256)
        assert np.array_equal(port.bfs_serial(off, col, 0), port.relaxation(off, col, 0))


def test_serial_marks_unreachable(port):
    # test_kernels.cpp:105-109
    off, col = port.build_csr(np.array([[0, 1]], dtype=np.uint32), 4)
    assert port.bfs_serial(off, col, 0).tolist() == [0, 1, UNREACHED, UNREACHED]
    with pytest.raises(ValueError):
        port.bfs_serial(off, col, 4)


def test_pick_sources_rule(port):
    # bfsbench.cpp:229-233: rng() % n with replacement, degree-0 rejected
    off, col = port.build_csr(port.generate_pairs(1, 10, 4, 1), 1 << 10)
    got = port.pick_sources(off, 64, 1)
    raw = port.mt64(1, 4096)
    deg = np.diff(off)
    want = [int(v) for v in (raw % np.uint64(1 << 10)) if deg[int(v)] > 0][:64]
    assert got.tolist() == want
    with pytest.raises(ValueError):
        port.pick_sources(np.zeros(5, dtype=np.uint64), 1, 1)


def test_mesh_generator_shape(port):
    pairs = port.mesh_pairs(64, keep=0.9, shortcuts=4, radius=32, seed=1)
    n = 64 * 64
    grid = pairs[:-4]
    assert ((grid[:, 1] - grid[:, 0] == 1) | (grid[:, 1] - grid[:, 0] == 64)).all()
    assert 0.85 * 2 * 64 * 63 < grid.shape[0] < 0.95 * 2 * 64 * 63
    sc = pairs[-4:].astype(np.int64)
    man = np.abs(sc[:, 0] // 64 - sc[:, 1] // 64) + np.abs(sc[:, 0] % 64 - sc[:, 1] % 64)
    assert ((man >= 1) & (man <= 32)).all() and (sc < n).all()

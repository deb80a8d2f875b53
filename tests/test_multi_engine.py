"""The multi-partition engine (pbfs_multi.cu): the 1D vertex partition with
the frontier exchange fused into one persistent launch per device -- queue
segments / bitmap slices stored straight into every partition's buffers and
one sequence-numbered flag round per level. On one B200 the partitions share
one launch ("loopback": devices = [0] * P), running exactly the exchange
code a multi-GPU box runs over NVLink; every traversal must equal the
oracle's distances and take the reference's phase sequence."""
import numpy as np
import pytest

import paper_2503_00430_b200 as pb
from graphs import make_path, make_star, random_graph

pytestmark = pytest.mark.gpu
UNREACHED = 0xFFFFFFFF


def check(port, g, mg, srcs, cfg, phases=True):
    for s in srcs:
        want = port.bfs_serial(g.row_offsets, g.column_indices, int(s))
        r = mg.bfs(int(s), cfg)
        assert np.array_equal(r.distances, want), int(s)
        recs = r.trace.records
        assert [x.distinct_size for x in recs] == np.bincount(want[want != UNREACHED]).tolist()
        if phases:
            want_ph = port.simulate_phases(g.row_offsets, want) if not cfg.force_top_down_only \
                else [0] * len(recs)
            assert [int(x.phase) for x in recs] == want_ph, int(s)
        # top-down edges_examined = reached-degree sum of the level's frontier
        deg = np.diff(g.row_offsets.astype(np.int64))
        for x in recs:
            if int(x.phase) == 0:
                assert x.edges_examined == int(deg[want == x.depth].sum())


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("scope", ["gpu", "sys"])
def test_loopback_partitions_rmat(parts, scope, port, monkeypatch):
    # scope=sys: the system-scope exchange a multi-GPU placement uses
    # (PBFS_MULTI_SYS_SCOPE test hook), run on one GPU.
    monkeypatch.setenv("PBFS_MULTI_SYS_SCOPE", "1" if scope == "sys" else "0")
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 16, 16, 1,
                                     drop_self_loops=True))
    mg = g.multi_device([0] * parts)
    assert mg.info["partitions"] == parts and mg.info["devices"] == 1
    assert sum(mg.info["local_arcs"]) == g.edge_count
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    check(port, g, mg, pb.pick_sources(g, 6, 3), cfg)
    mg.close()


@pytest.mark.parametrize("parts", [2, 5])
def test_loopback_uniform_and_top_down_only(parts, port):
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.UniformRandom, 15, 8, 4,
                                     drop_self_loops=True))
    mg = g.multi_device([0] * parts)
    srcs = pb.pick_sources(g, 4, 2)
    check(port, g, mg, srcs, pb.KernelConfig(variant=pb.KernelVariant.Hybrid))
    check(port, g, mg, srcs, pb.KernelConfig(variant=pb.KernelVariant.Hybrid,
                                             force_top_down_only=True))


def test_loopback_hand_graphs_and_padding(port):
    # n not a power of two (identity relabel + padding), a star that goes
    # bottom-up from the seed, a path that stays top-down for 3000 levels.
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    for g, s in [(random_graph(5000, 40000, 9), 17), (make_star(40), 0), (make_path(3000), 0)]:
        for parts in (2, 3):
            mg = g.multi_device([0] * parts)
            check(port, g, mg, [s], cfg)
            mg.close()


def test_repeated_runs_and_async_component(port):
    # Exchange sequence numbers carry the run number: back-to-back traversals
    # must never read a previous run's flags.
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 14, 16, 7,
                                     drop_self_loops=True))
    mg = g.multi_device([0, 0, 0, 0])
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    srcs = [int(s) for s in pb.pick_sources(g, 5, 9)]
    for _ in range(3):
        for s in srcs:
            mg.bfs_async(s, cfg)
    mg.sync()
    assert mg.component() == port.component(
        g.row_offsets, port.bfs_serial(g.row_offsets, g.column_indices, srcs[-1]))
    check(port, g, mg, srcs, cfg)


def test_rejects_unsupported_configs():
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 10, 8, 1, drop_self_loops=True))
    mg = g.multi_device([0, 0])
    with pytest.raises(pb.ConfigError):
        mg.bfs(1, pb.KernelConfig(variant=pb.KernelVariant.Conventional))
    with pytest.raises(pb.InputError):
        mg.bfs(g.vertex_count, pb.KernelConfig(variant=pb.KernelVariant.Hybrid))
    with pytest.raises(pb.ConfigError):
        g.multi_device([0] * 9)


def test_run_bfs_reaches_the_multi_engine_through_graph_options(port):
    # pbfs_graph_options.devices: run_bfs (kernels.cpp:657-691) on a handle
    # partitioned over a device list, the path a KernelFn takes.
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 14, 16, 3,
                                     drop_self_loops=True))
    stats = pb.compute_stats(g)
    for s in pb.pick_sources(g, 3, 5):
        want = port.bfs_serial(g.row_offsets, g.column_indices, int(s))
        r = pb.run_bfs(g, int(s), pb.KernelConfig(variant=pb.KernelVariant.Hybrid), stats,
                       device=[0, 0, 0])
        assert np.array_equal(r.distances, want)
        assert [int(x.phase) for x in r.trace.records] == port.simulate_phases(g.row_offsets, want)
    dg = g.device([0, 0, 0])
    assert dg.info["partitions"] == 3
    dg.bfs_async(int(pb.pick_sources(g, 1, 5)[0]), pb.KernelConfig(variant=pb.KernelVariant.Hybrid))
    dg.sync()
    assert dg.component()[0] > 0

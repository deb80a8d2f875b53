"""Multi-GPU (1D vertex partition).

CPU: two gloo ranks run the partition protocol (relabel, row/column slices,
in-place allgather of next-frontier bitmap slices, identical per-rank
decisions) on a numpy model and must reproduce the oracle's distances and
phases. GPU (-m gpu): the device engine (pbfs_part.cu) with G partitions on
one B200 sharing the full bitmaps (loopback) is bit-exact against the oracle
and takes the single-GPU hybrid's phase sequence.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import partition_model as pm

UNREACHED = 0xFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, scale, out):
    import torch
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_lib = oracle.port()
    off, col = port_lib.build_csr(port_lib.generate_pairs(1, scale, 8, 5), 1 << scale,
                                  symmetrize=True, drop_self_loops=True)
    n = 1 << scale
    part = pm.build_partition(off, col.astype(np.int64), n, rank, world)
    nloc = part["nloc"]

    def allgather(local):
        t = torch.from_numpy(local.astype(np.uint8))
        full = torch.empty(nloc * world, dtype=torch.uint8)
        dist.all_gather_into_tensor(full, t)
        return full.numpy().astype(bool)

    deg = np.diff(off)
    src = int(np.nonzero(deg)[0][7])
    d_loc, phases = pm.bfs_rank(part, src, 0.05, allgather)
    gathered = [None] * world
    dist.all_gather_object(gathered, (d_loc.tolist(), phases, len(part["rows"]),
                                      int(sum(len(r) for r in part["rows"]))))
    if rank == 0:
        dist_pi = np.concatenate([np.array(g[0], dtype=np.uint64) for g in gathered])
        got = dist_pi[part["pi"]]
        want = port_lib.bfs_serial(off, col, src)
        out.put((bool(np.array_equal(got.astype(np.uint32), want)),
                 [g[1] for g in gathered], port_lib.simulate_phases(off, want),
                 [g[3] for g in gathered]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_partition_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 12, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    equal, phases, want_phases, arcs = res
    assert equal, "partitioned distances differ from the oracle"
    assert all(p == phases[0] for p in phases), "ranks took different directions"
    assert phases[0] == want_phases
    share = np.array(arcs) / sum(arcs)
    assert (abs(share - 1 / world) < 0.1).all(), share  # hashed relabel balances arcs


def test_relabel_is_a_bijection():
    for n, world in [(1 << 14, 2), (1 << 16, 8), (5000, 4), (1 << 14, 3), (1 << 16, 6)]:
        rl = pm.Relabel(n, world)
        img = rl.fwd(np.arange(n, dtype=np.uint64))
        assert len(np.unique(img)) == n and int(img.max()) < rl.npad
        assert rl.npad % (512 * world) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_loopback_partitions_match_oracle(world, port):
    import paper_2503_00430_b200 as pb
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 16, 16, 1,
                                     drop_self_loops=True))
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    parts = None
    for s in pb.pick_sources(g, 6, 3):
        want = port.bfs_serial(g.row_offsets, g.column_indices, int(s))
        got, recs, parts = pb.bfs_partitioned_loopback(g, int(s), cfg, world, parts=parts)
        assert np.array_equal(got, want), (world, int(s))
        assert [int(r.phase) for r in recs] == port.simulate_phases(g.row_offsets, want)
        assert [r.distinct_size for r in recs] == np.bincount(want[want != UNREACHED]).tolist()
    info = parts[0].info()
    assert info["relabel_hashed"] == 1
    arcs = [p.info()["local_arcs"] for p in parts]
    assert sum(arcs) == g.edge_count
    if world > 1:
        assert max(arcs) / min(arcs) < 1.15  # hashed relabel balances the arcs


@pytest.mark.gpu
def test_loopback_identity_relabel_and_padding(port):
    # n not a power of two: identity relabel, padded to a multiple of 512*world
    import paper_2503_00430_b200 as pb
    from graphs import random_graph
    g = random_graph(5000, 40000, 9)
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    for world in (2, 3):
        got, _, parts = pb.bfs_partitioned_loopback(g, 17, cfg, world)
        assert parts[0].info()["relabel_hashed"] == 0
        assert np.array_equal(got, port.bfs_serial(g.row_offsets, g.column_indices, 17))
    # top-down-only dispatch also runs partitioned
    cfg.force_top_down_only = True
    got, recs, _ = pb.bfs_partitioned_loopback(g, 17, cfg, 2)
    assert all(int(r.phase) == 0 for r in recs)
    assert np.array_equal(got, port.bfs_serial(g.row_offsets, g.column_indices, 17))


def test_gid_map_is_order_preserving_and_balanced():
    for n, world in [(1 << 14, 2), (1 << 16, 8), (5000, 4), (1 << 14, 3), (1 << 14, 7)]:
        rl, nloc, gid = pm.gid_map(n, world)
        assert len(np.unique(gid)) == n and int(gid.max()) < rl.npad
        owner = gid // nloc
        for r in range(world):
            mine = np.nonzero(owner == r)[0]          # ascending vertex ids
            assert (np.diff(gid[mine]) == 1).all()   # consecutive, same order
        if rl.hashed:
            assert (np.bincount(owner, minlength=world) == nloc).all()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [3, 6])
def test_loopback_non_power_of_two_world_on_kronecker(world, port):
    # n = 2^14 is a power of two but world is not: the partition must fall
    # back to identity + padding (the hashed ranges would not tile 2^k).
    import paper_2503_00430_b200 as pb
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 14, 16, 1,
                                     drop_self_loops=True))
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    parts = None
    for s in pb.pick_sources(g, 3, 1):
        want = port.bfs_serial(g.row_offsets, g.column_indices, int(s))
        got, _, parts = pb.bfs_partitioned_loopback(g, int(s), cfg, world, parts=parts)
        assert np.array_equal(got, want), (world, int(s))
    info = parts[0].info()
    assert info["relabel_hashed"] == 0 and info["padded_count"] % (512 * world) == 0
    assert sum(p.info()["local_arcs"] for p in parts) == g.edge_count


@pytest.mark.gpu
def test_device_relabel_matches_model():
    import ctypes
    import paper_2503_00430_b200 as pb
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 14, 4, 2))
    p = pb.PartitionedGraph(g.device(0, 8), 1, 4)
    _, _, gid = pm.gid_map(g.vertex_count, 4)
    out = ctypes.c_uint64()
    for v in [0, 1, 2, 777, g.vertex_count - 1]:
        pb.parbfs._check(pb.parbfs.lib.pbfs_part_relabel(p.h, v, ctypes.byref(out)))
        assert out.value == int(gid[v])


class _DevView:
    """Zero-copy torch view of library-owned device memory (int32 words)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _cuda_engine_worker(rank, world, port, out):
    # One rank of the per-level partitioned engine (pbfs_part.cu, the real
    # CUDA kernels) per process, both on cuda:0; the per-level exchange is a
    # gloo allgather of the next-bitmap slices staged through host memory
    # (bench.py's PBFS_DIST_BACKEND=gloo mode). Kernels of the two ranks never
    # wait on each other: the ranks meet only in the host collective.
    import torch
    import oracle
    import paper_2503_00430_b200 as pb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = pb.generate(pb.GeneratorSpec(pb.GeneratorKind.Kronecker, 15, 16, 2,
                                     drop_self_loops=True))
    part = pb.PartitionedGraph(g.device(0, 8), rank, world)
    info = part.info()
    wl, wt = info["words_local"], info["words_total"]
    cfg = pb.KernelConfig(variant=pb.KernelVariant.Hybrid)
    port_lib = oracle.port()
    ok, phases_ok = True, True
    for s in [int(x) for x in pb.pick_sources(g, 4, 6)]:
        part.begin(s, cfg)
        recs = []
        while True:
            part.step()
            part.sync()
            nxt = part.info()["next"]
            view = torch.as_tensor(_DevView(nxt, wt), device="cuda")  # the full next bitmap
            mine = view[rank * wl:(rank + 1) * wl].cpu()
            gathered = torch.empty(wt, dtype=torch.int32)
            dist.all_gather_into_tensor(gathered, mine)
            view.copy_(gathered)
            torch.cuda.synchronize()
            done, rec = part.end_level()
            recs.append(int(rec.phase))
            if done:
                break
        local = part.local_distances()
        allp = [None] * world
        dist.all_gather_object(allp, local.tolist())
        if rank == 0:
            dist_pi = np.concatenate([np.array(a, dtype=np.uint32) for a in allp])
            got = part.unrelabel_host(dist_pi)
            want = port_lib.bfs_serial(g.row_offsets, g.column_indices, s)
            ok &= bool(np.array_equal(got, want))
            phases_ok &= recs == port_lib.simulate_phases(g.row_offsets, want)
    if rank == 0:
        out.put((ok, phases_ok))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_cuda_partition_engine_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_engine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, phases_ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok, "2-process partitioned distances differ from the oracle"
    assert phases_ok, "2-process partitioned phases differ from the reference rule"

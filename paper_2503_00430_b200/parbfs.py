"""Host-side mirror of the reference ``parbfs`` C++ API over the GPU C ABI.

Same names, argument meanings and error behaviour as the reference library
(``proj/core/include/parbfs/*.hpp``); every traversal runs on the B200 through
``include/pbfs.h`` -- there is no CPU traversal in this module.

Reference interface -> here:
  types.hpp:12-68         VertexId/Distance/kUnreached, Error hierarchy
  csr_graph.hpp:20-63     CsrGraph, build_csr, adjacency check, validate_csr
  generator.hpp:17-28     GeneratorKind, GeneratorSpec, generate
  graph_stats.hpp:14-29   GraphCategory, GraphStats, compute_stats
  kernel_config.hpp:13-78 KernelVariant, TraversalPhase, KernelConfig, validate,
                          to_string, parse_kernel_variant
  trace.hpp:26-63         LevelRecord, TraversalTrace, average_duplicate_percentage,
                          frontier_size_series, write_trace_csv(_header)
  kernels.hpp:15-81       BfsResult, bfs_conventional/nonatomic/hybrid/
                          hybrid_beamer/visited_bitmap, run_bfs
  timing.hpp:17-34        KernelFn, TimingReport, time_run
  graph_io.hpp:26-37      save_binary_csr, load_binary_csr
  bfsbench.cpp:206-235    pick_sources
"""
from __future__ import annotations

import ctypes
import enum
import os
import time
import weakref
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib as L

lib = L.lib

UNREACHED = 0xFFFFFFFF  # parbfs::kUnreached (types.hpp:19) == int32 -1
MAX_VERTEX_COUNT = 0x7FFFFFFF  # types.hpp:21
DEFAULT_DEGREE_THRESHOLD = 7.0  # graph_stats.hpp:24


# ---- errors (types.hpp:25-68) ------------------------------------------------
class Error(RuntimeError):
    pass


class InputError(Error):
    pass


class ConfigError(Error):
    pass


class FormatError(Error):
    pass


class CapacityError(Error):
    pass


class CorrectnessError(Error):
    pass


class MetricError(Error):
    pass


_STATUS = {1: InputError, 2: ConfigError, 3: FormatError, 4: CapacityError, 5: Error,
           6: Error, 7: MetricError, 8: CorrectnessError}


def _check(status: int) -> None:
    if status != 0:
        msg = (lib.pbfs_last_error() or b"").decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


# ---- enums (kernel_config.hpp:13-24, generator.hpp:11, graph_stats.hpp:14) ----
class KernelVariant(enum.IntEnum):
    Serial = 0
    Conventional = 1
    NonAtomic = 2
    Hybrid = 3
    HybridBeamer = 4
    VisitedBitmapInline = 5
    VisitedBitmapDeferred = 6
    TopDownPeriodicFlush = 7
    # GPU addition (pbfs.h PBFS_HYBRID_PLAIN): the reference Hybrid's own
    # PlainStore top-down claim (no atomic) with the 5 % switch.
    HybridPlainStore = 8


class TraversalPhase(enum.IntEnum):
    TopDown = 0
    BottomUp = 1


class GeneratorKind(enum.IntEnum):
    UniformRandom = 0
    Kronecker = 1
    Mesh = 2  # config 3 (new)


class GraphCategory(enum.IntEnum):
    SmallDiameter = 0
    LargeDiameter = 1


_VARIANT_TOKENS = {
    KernelVariant.Serial: "serial", KernelVariant.Conventional: "conventional",
    KernelVariant.NonAtomic: "nonatomic", KernelVariant.Hybrid: "hybrid",
    KernelVariant.HybridBeamer: "hybrid-beamer",
    KernelVariant.VisitedBitmapInline: "visited-inline",
    KernelVariant.VisitedBitmapDeferred: "visited-deferred",
    KernelVariant.TopDownPeriodicFlush: "periodic-flush",
    KernelVariant.HybridPlainStore: "hybrid-plain",
}


def to_string(x) -> str:
    """kernel_config.cpp:28-52, graph_stats.cpp:27-35, generator.cpp:94-107."""
    if isinstance(x, KernelVariant):
        return _VARIANT_TOKENS[x]
    if isinstance(x, TraversalPhase):
        return "top-down" if x == TraversalPhase.TopDown else "bottom-up"
    if isinstance(x, GraphCategory):
        return "small-diameter" if x == GraphCategory.SmallDiameter else "large-diameter"
    if isinstance(x, GeneratorKind):
        return {0: "uniform", 1: "kron", 2: "mesh"}[int(x)]
    if isinstance(x, GeneratorSpec):
        return f"{to_string(x.kind)}:{x.scale}:{x.edge_factor}:{x.seed}"
    raise TypeError(type(x))


def parse_kernel_variant(token: str) -> Optional[KernelVariant]:
    """kernel_config.cpp:54-64."""
    for v, t in _VARIANT_TOKENS.items():
        if t == token:
            return v
    return None


# ---- config (kernel_config.hpp:38-70) -----------------------------------------
@dataclass
class KernelConfig:
    variant: KernelVariant = KernelVariant.Conventional
    worker_count: int = 1
    hybrid_threshold_fraction: float = 0.05
    alpha: float = 15.0
    beta: float = 18.0
    flush_capacity: int = 4096
    force_top_down_only: bool = False
    validate_same_value_stores: bool = False
    racy_visited_claim: bool = False
    # kernel_config.hpp:26-36: called once per frontier (the seed, then every
    # produced level) with a LevelSnapshot. Test instrumentation only.
    level_observer: Optional[Callable] = None

    def _c(self) -> L.Config:
        c = L.Config()
        c.variant = int(self.variant)
        c.worker_count = max(0, int(self.worker_count))
        c.hybrid_threshold_fraction = float(self.hybrid_threshold_fraction)
        c.alpha = float(self.alpha)
        c.beta = float(self.beta)
        c.flush_capacity = max(0, int(self.flush_capacity))
        c.force_top_down_only = int(bool(self.force_top_down_only))
        c.validate_same_value_stores = int(bool(self.validate_same_value_stores))
        c.racy_visited_claim = int(bool(self.racy_visited_claim))
        c.observe_frontiers = int(self.level_observer is not None)
        return c


def validate(config: KernelConfig) -> None:
    """kernel_config.cpp:9-26 (raises ConfigError)."""
    c = config._c()
    _check(lib.pbfs_config_validate(ctypes.byref(c)))


# ---- graph (csr_graph.hpp:20-63) ------------------------------------------------
class CsrGraph:
    """Canonical CSR: per-row sorted, deduplicated adjacency (csr_graph.hpp:20-46).

    ``row_offsets`` is uint64 (parbfs::EdgeOffset) unless built otherwise;
    ``column_indices`` is uint32. Arrays produced by the native builder are
    zero-copy views of library-owned memory kept alive by this object.
    """

    def __init__(self, vertex_count: int, row_offsets: np.ndarray, column_indices: np.ndarray,
                 symmetric: bool, _owner=None):
        self.vertex_count = int(vertex_count)
        self.row_offsets = row_offsets
        self.column_indices = column_indices
        self.edge_count = int(column_indices.size)
        self.symmetric = bool(symmetric)
        self._owner = _owner
        self._device = {}  # (device, offset bytes) -> DeviceGraph (handle cache)

    def neighbors(self, u: int) -> np.ndarray:
        return self.column_indices[int(self.row_offsets[u]):int(self.row_offsets[u + 1])]

    def degree(self, u: int) -> int:
        return int(self.row_offsets[u + 1] - self.row_offsets[u])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets.astype(np.int64))

    def structurally_equal(self, other: "CsrGraph") -> bool:
        return (self.vertex_count == other.vertex_count and self.edge_count == other.edge_count
                and np.array_equal(self.row_offsets.astype(np.uint64),
                                   other.row_offsets.astype(np.uint64))
                and np.array_equal(self.column_indices, other.column_indices))

    def _view(self) -> L.Csr:
        if self.row_offsets.dtype not in (np.uint64, np.int64, np.uint32, np.int32):
            raise FormatError("row offsets must be 32- or 64-bit integers")
        self.row_offsets = np.ascontiguousarray(self.row_offsets)
        self.column_indices = np.ascontiguousarray(self.column_indices, dtype=np.uint32)
        c = L.Csr()
        c.vertex_count = self.vertex_count
        c.edge_count = self.edge_count
        c.row_offsets = self.row_offsets.ctypes.data
        c.column_indices = self.column_indices.ctypes.data if self.edge_count else None
        c.offset_bytes = self.row_offsets.dtype.itemsize
        c.symmetric = int(self.symmetric)
        return c

    def device(self, device=0, offset_bytes: int = 0) -> "DeviceGraph":
        """The resident device copy (created once per graph/device/offset
        width). `device` may be a list of CUDA ordinals: the graph is then
        partitioned over them (pbfs_graph_options.devices, the
        multi-partition engine) behind the same DeviceGraph interface."""
        key = (tuple(device) if isinstance(device, (list, tuple)) else device, offset_bytes)
        g = self._device.get(key)
        if g is None:
            g = DeviceGraph(self, device=device, offset_bytes=offset_bytes)
            self._device[key] = g
        return g

    def release_device(self) -> None:
        for g in self._device.values():
            g.close()
        self._device.clear()

    def multi_device(self, devices) -> "MultiDeviceGraph":
        """The graph partitioned over `devices` (one partition per entry;
        repeats = several partitions on one GPU) for the multi-partition
        engine (pbfs_multi_create)."""
        return MultiDeviceGraph(self, devices)


def _from_host_handle(h: ctypes.c_void_p) -> CsrGraph:
    view = L.Csr()
    _check(lib.pbfs_host_csr_view(h, ctypes.byref(view)))
    n, m = view.vertex_count, view.edge_count

    class _Owner:
        def __init__(self, handle):
            self.h = handle

        def __del__(self):
            try:
                lib.pbfs_host_csr_free(self.h)
            except Exception:
                pass

    owner = _Owner(h)
    off = np.ctypeslib.as_array(ctypes.cast(view.row_offsets, ctypes.POINTER(ctypes.c_uint64)),
                                shape=(n + 1,))
    if m:
        col = np.ctypeslib.as_array(
            ctypes.cast(view.column_indices, ctypes.POINTER(ctypes.c_uint32)), shape=(m,))
    else:
        col = np.zeros(0, dtype=np.uint32)
    return CsrGraph(n, off, col, bool(view.symmetric), _owner=owner)


def build_csr(edge_pairs, vertex_count: int, symmetrize: bool, drop_self_loops: bool = False,
              threads: int = 0) -> CsrGraph:
    """csr_graph.cpp:11-55. ``drop_self_loops`` applies BASELINE's removal
    (the reference keeps self-loops)."""
    pairs = np.ascontiguousarray(np.asarray(edge_pairs, dtype=np.int64).reshape(-1, 2))
    if pairs.size and (pairs.min() < 0 or pairs.max() > 0xFFFFFFFF):
        bad = np.nonzero((pairs < 0).any(axis=1) | (pairs > 0xFFFFFFFF).any(axis=1))[0][0]
        raise InputError(f"edge ({pairs[bad, 0]}, {pairs[bad, 1]}) references a vertex >= "
                         f"{vertex_count}")
    p32 = np.ascontiguousarray(pairs.astype(np.uint32))
    h = ctypes.c_void_p()
    _check(lib.pbfs_build_csr(p32.ctypes.data if p32.size else None, p32.shape[0],
                              int(vertex_count), int(symmetrize), int(drop_self_loops),
                              int(threads), ctypes.byref(h)))
    return _from_host_handle(h)


def adjacency_is_symmetric(graph: CsrGraph) -> bool:
    """csr_graph.cpp:57-66 (re-derived by rebuilding without symmetrize)."""
    deg = graph.degrees()
    src = np.repeat(np.arange(graph.vertex_count, dtype=np.uint32), deg)
    fwd = (src.astype(np.uint64) << 32) | graph.column_indices.astype(np.uint64)
    rev = (graph.column_indices.astype(np.uint64) << 32) | src.astype(np.uint64)
    return bool(np.array_equal(np.sort(fwd), np.sort(rev)))


def validate_csr(graph: CsrGraph) -> None:
    """csr_graph.cpp:68-113: the same checks the C ABI applies at upload."""
    off = graph.row_offsets
    if graph.vertex_count > MAX_VERTEX_COUNT:
        raise FormatError(f"vertex count {graph.vertex_count} exceeds the supported maximum")
    if off.size != graph.vertex_count + 1:
        raise FormatError(f"offset array has {off.size} entries, expected vertex count + 1 = "
                          f"{graph.vertex_count + 1}")
    if int(off[0]) != 0:
        raise FormatError("offset array must start at 0")
    if int(off[-1]) != graph.edge_count:
        raise FormatError(f"offset array ends at {int(off[-1])} but edge count is "
                          f"{graph.edge_count}")
    d = np.diff(off.astype(np.int64))
    if (d < 0).any():
        raise FormatError(f"offset array decreases at vertex {int(np.argmax(d < 0))}")
    col = graph.column_indices
    if col.size and int(col.max()) >= graph.vertex_count:
        raise FormatError("a neighbor lies outside the graph")
    if col.size > 1:
        row_start = np.zeros(col.size, dtype=bool)
        row_start[off[:-1][d > 0].astype(np.int64)] = True
        bad = (np.diff(col.astype(np.int64)) <= 0) & ~row_start[1:]
        if bad.any():
            raise FormatError("an adjacency list is not strictly increasing")


@dataclass
class GeneratorSpec:
    """generator.hpp:17-22 plus the config-3 mesh parameters."""
    kind: GeneratorKind = GeneratorKind.UniformRandom
    scale: int = 1
    edge_factor: int = 1
    seed: int = 0
    drop_self_loops: bool = False
    mesh_side: int = 0
    mesh_keep: float = 0.9
    mesh_shortcuts: Optional[int] = None
    mesh_radius: int = 32


def generate(spec: GeneratorSpec, threads: int = 0) -> CsrGraph:
    """generator.cpp:41-92: identical mt19937_64 draw sequence, then
    build_csr(symmetrize=true)."""
    s = L.GenSpec()
    s.kind = int(spec.kind)
    s.scale = int(spec.scale)
    s.edge_factor = int(spec.edge_factor)
    s.drop_self_loops = int(bool(spec.drop_self_loops))
    s.seed = int(spec.seed) & 0xFFFFFFFFFFFFFFFF
    s.mesh_side = int(spec.mesh_side)
    s.mesh_radius = int(spec.mesh_radius)
    s.mesh_keep = float(spec.mesh_keep)
    n = spec.mesh_side * spec.mesh_side
    s.mesh_shortcuts = int(round(0.001 * n)) if spec.mesh_shortcuts is None else int(
        spec.mesh_shortcuts)
    s.threads = int(threads)
    h = ctypes.c_void_p()
    _check(lib.pbfs_generate(ctypes.byref(s), ctypes.byref(h)))
    return _from_host_handle(h)


# ---- stats (graph_stats.hpp:14-29) ------------------------------------------------
@dataclass
class GraphStats:
    vertex_count: int = 0
    edge_count: int = 0
    average_degree: float = 0.0
    max_degree: int = 0
    category: GraphCategory = GraphCategory.SmallDiameter


def compute_stats(graph: CsrGraph, threshold: float = DEFAULT_DEGREE_THRESHOLD) -> GraphStats:
    """graph_stats.cpp:9-25."""
    out = L.Stats()
    v = graph._view()
    _check(lib.pbfs_compute_stats(ctypes.byref(v), float(threshold), ctypes.byref(out)))
    return GraphStats(out.vertex_count, out.edge_count, out.average_degree, out.max_degree,
                      GraphCategory.LargeDiameter if out.large_diameter
                      else GraphCategory.SmallDiameter)


def pick_sources(graph: CsrGraph, count: int, seed: int = 1) -> np.ndarray:
    """bfsbench.cpp:206-235: mt19937_64(seed), v = rng() % n, keep iff degree > 0."""
    out = np.empty(max(int(count), 0), dtype=np.uint32)
    v = graph._view()
    _check(lib.pbfs_pick_sources(ctypes.byref(v), int(count), int(seed),
                                 out.ctypes.data if out.size else None))
    return out


def load_edge_list(path: str, one_based: bool = False, symmetrize: bool = True,
                   vertex_count_hint: Optional[int] = None) -> CsrGraph:
    """edge_list.cpp:26-82: whitespace "u v" lines, '#'/'%' comments and blank
    lines skipped, trailing fields ignored, one-based ids shifted, vertex
    count = max id + 1 unless a (larger) hint is given."""
    pairs = []
    max_seen = -1
    try:
        fh = open(path)
    except OSError:
        raise InputError(f"cannot open edge list file: {path}")
    with fh:
        for line_no, line in enumerate(fh, 1):
            stripped = line.strip(" \t\r\n")
            if not stripped or stripped[0] in "#%":
                continue
            fields = stripped.split()
            try:
                a, b = int(fields[0]), int(fields[1])
            except (ValueError, IndexError):
                raise InputError(f"{path}:{line_no}: expected two integer vertex ids")
            if one_based:
                a, b = a - 1, b - 1
            if a < 0 or b < 0:
                raise InputError(f"{path}:{line_no}: vertex id below the index base")
            if a > MAX_VERTEX_COUNT or b > MAX_VERTEX_COUNT:
                raise InputError(f"{path}:{line_no}: vertex id exceeds the supported maximum")
            pairs.append((a, b))
            max_seen = max(max_seen, a, b)
    n = max_seen + 1
    if vertex_count_hint is not None:
        if vertex_count_hint < n:
            raise InputError(f"{path}: declared vertex count {vertex_count_hint} is smaller "
                             f"than the largest referenced vertex + 1 ({n})")
        n = vertex_count_hint
    return build_csr(np.array(pairs, dtype=np.int64).reshape(-1, 2), n, symmetrize)


def save_binary_csr(graph: CsrGraph, path: str) -> None:
    """graph_io.cpp:70-85."""
    v = graph._view()
    _check(lib.pbfs_save_csr1(ctypes.byref(v), str(path).encode()))


def load_binary_csr(path: str) -> CsrGraph:
    """graph_io.cpp:87-119."""
    h = ctypes.c_void_p()
    _check(lib.pbfs_load_csr1(str(path).encode(), ctypes.byref(h)))
    return _from_host_handle(h)


# ---- trace (trace.hpp:26-63) -------------------------------------------------------
@dataclass
class LevelRecord:
    depth: int = 0
    phase: TraversalPhase = TraversalPhase.TopDown
    frontier_size: int = 0
    distinct_size: int = 0
    duplicate_count: int = 0
    edges_examined: int = 0
    flush_events: int = 0
    elapsed_ns: int = 0


@dataclass
class TraversalTrace:
    records: list = field(default_factory=list)
    total_elapsed_ns: int = 0
    variant: KernelVariant = KernelVariant.Serial
    worker_count: int = 1
    source: int = 0
    same_value_violations: int = 0
    device_ms: float = 0.0

    def total_edges_examined(self) -> int:
        return sum(r.edges_examined for r in self.records)

    def level_count(self, phase: TraversalPhase) -> int:
        return sum(1 for r in self.records if r.phase == phase)


def average_duplicate_percentage(trace: TraversalTrace) -> float:
    """trace.cpp:21-35."""
    vals = [100.0 * r.duplicate_count / r.frontier_size for r in trace.records
            if r.frontier_size]
    if not vals:
        raise MetricError("average duplicate percentage is undefined: no non-empty frontier")
    return sum(vals) / len(vals)


def frontier_size_series(trace: TraversalTrace):
    """trace.cpp:37-45."""
    return [(r.depth, r.frontier_size) for r in trace.records]


def write_trace_csv_header(out) -> None:
    """trace.cpp:47-50 (frozen schema)."""
    out.write("run_id,variant,source,depth,phase,frontier_size,distinct_size,"
              "duplicate_count,edges_examined,flush_events,elapsed_ns\n")


def write_trace_csv(out, trace: TraversalTrace, run_id: str) -> None:
    """trace.cpp:52-61."""
    for r in trace.records:
        out.write(f"{run_id},{to_string(trace.variant)},{trace.source},{r.depth},"
                  f"{to_string(r.phase)},{r.frontier_size},{r.distinct_size},"
                  f"{r.duplicate_count},{r.edges_examined},{r.flush_events},{r.elapsed_ns}\n")


@dataclass
class BfsResult:
    """kernels.hpp:15-20: uint32 distances (kUnreached = 0xFFFFFFFF = int32 -1)."""
    distances: np.ndarray
    trace: TraversalTrace
    # Device-recorded frontiers (cfg.level_observer set), for _emit_snapshots.
    _observed: Optional[np.ndarray] = None


# ---- device graph + traversal -------------------------------------------------------
class MultiDeviceGraph:
    """pbfs_multi: the 1D vertex partition with the frontier exchange fused
    into one persistent launch per device (see include/pbfs.h)."""

    def __init__(self, graph: "CsrGraph", devices):
        devs = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        v = graph._view()
        h = ctypes.c_void_p()
        _check(lib.pbfs_multi_create(ctypes.byref(v), devs, len(devices), ctypes.byref(h)))
        self.h = h
        self.vertex_count = graph.vertex_count
        self.devices = list(devices)
        i = L.MultiInfo()
        _check(lib.pbfs_multi_get_info(h, ctypes.byref(i)))
        self.info = {k: (list(getattr(i, k)) if k == "local_arcs" else getattr(i, k))
                     for k, _ in L.MultiInfo._fields_}
        self.info["local_arcs"] = self.info["local_arcs"][:len(devices)]

    def close(self) -> None:
        if getattr(self, "h", None):
            lib.pbfs_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bfs(self, source: int, config: KernelConfig, want_distances: bool = True,
            want_trace: bool = True, out: Optional[np.ndarray] = None) -> BfsResult:
        c = config._c()
        dist = None
        if want_distances:
            dist = out if out is not None else np.empty(self.vertex_count, dtype=np.uint32)
        cap = min(self.vertex_count + 1, 1 << 16) if want_trace else 0
        levels = (L.Level * cap)() if cap else None
        info = L.RunInfo()
        t0 = time.perf_counter_ns()
        _check(lib.pbfs_multi_bfs(self.h, int(source) & 0xFFFFFFFF, ctypes.byref(c),
                                  dist.ctypes.data if dist is not None else None, levels, cap,
                                  ctypes.byref(info)))
        t1 = time.perf_counter_ns()
        trace = TraversalTrace(variant=KernelVariant(config.variant),
                               worker_count=config.worker_count, source=int(source),
                               total_elapsed_ns=t1 - t0, device_ms=float(info.device_ms))
        for i in range(min(info.levels, cap)):
            r = levels[i]
            trace.records.append(LevelRecord(r.depth, TraversalPhase(r.phase), r.frontier_size,
                                             r.distinct_size, r.duplicate_count,
                                             r.edges_examined, r.flush_events, r.elapsed_ns))
        return BfsResult(dist, trace)

    def bfs_async(self, source: int, config: KernelConfig) -> None:
        c = config._c()
        _check(lib.pbfs_multi_bfs_async(self.h, int(source) & 0xFFFFFFFF, ctypes.byref(c)))

    def sync(self) -> float:
        ms = ctypes.c_float()
        _check(lib.pbfs_multi_sync(self.h, ctypes.byref(ms)))
        return ms.value

    def stream(self) -> int:
        s = ctypes.c_void_p()
        _check(lib.pbfs_multi_stream(self.h, ctypes.byref(s)))
        return s.value or 0

    def component(self):
        nr = ctypes.c_uint64()
        ar = ctypes.c_uint64()
        _check(lib.pbfs_multi_component(self.h, ctypes.byref(nr), ctypes.byref(ar)))
        return nr.value, ar.value


class DeviceGraph:
    """A graph resident in HBM (pbfs_graph handle) with its traversal scratch."""

    def __init__(self, graph: CsrGraph, device=0, offset_bytes: int = 0):
        opt = L.GraphOptions()
        if isinstance(device, (list, tuple)):
            devs = (ctypes.c_int32 * len(device))(*[int(d) for d in device])
            self._devs = devs
            opt.device = int(device[0])
            opt.devices = ctypes.cast(devs, ctypes.c_void_p)
            opt.num_devices = len(device)
        else:
            opt.device = int(device)
        opt.device_offset_bytes = int(offset_bytes)
        v = graph._view()
        h = ctypes.c_void_p()
        _check(lib.pbfs_graph_create(ctypes.byref(v), ctypes.byref(opt), ctypes.byref(h)))
        self.h = h
        self.vertex_count = graph.vertex_count
        info = L.GraphInfo()
        _check(lib.pbfs_graph_get_info(h, ctypes.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in L.GraphInfo._fields_}

    def close(self) -> None:
        if getattr(self, "h", None):
            lib.pbfs_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bfs(self, source: int, config: KernelConfig, want_distances: bool = True,
            want_trace: bool = True, out: Optional[np.ndarray] = None) -> BfsResult:
        c = config._c()
        dist = None
        if want_distances:
            dist = out if out is not None else np.empty(self.vertex_count, dtype=np.uint32)
        cap = min(self.vertex_count + 1, 1 << 20) if want_trace else 0
        levels = (L.Level * cap)() if cap else None
        info = L.RunInfo()
        t0 = time.perf_counter_ns()
        _check(lib.pbfs_bfs(self.h, int(source) & 0xFFFFFFFF, ctypes.byref(c),
                            dist.ctypes.data if dist is not None else None, levels, cap,
                            ctypes.byref(info)))
        if cap and info.levels > cap:
            # Deeper than the default record buffer: ask again for every level
            # (the library grows its device trace buffer and re-runs).
            cap = int(info.levels)
            levels = (L.Level * cap)()
            _check(lib.pbfs_bfs(self.h, int(source) & 0xFFFFFFFF, ctypes.byref(c),
                                dist.ctypes.data if dist is not None else None, levels, cap,
                                ctypes.byref(info)))
        t1 = time.perf_counter_ns()
        observed = None
        if config.level_observer is not None:
            total = ctypes.c_uint64()
            _check(lib.pbfs_graph_observed(self.h, None, 0, ctypes.byref(total)))
            observed = np.empty(total.value, dtype=np.uint32)
            _check(lib.pbfs_graph_observed(self.h, observed.ctypes.data, observed.size,
                                           ctypes.byref(total)))
        trace = TraversalTrace(variant=KernelVariant(config.variant),
                               worker_count=config.worker_count, source=int(source),
                               same_value_violations=int(info.same_value_violations),
                               total_elapsed_ns=t1 - t0, device_ms=float(info.device_ms))
        if cap:
            for i in range(min(info.levels, cap)):
                r = levels[i]
                trace.records.append(LevelRecord(r.depth, TraversalPhase(r.phase), r.frontier_size,
                                                 r.distinct_size, r.duplicate_count,
                                                 r.edges_examined, r.flush_events, r.elapsed_ns))
        return BfsResult(dist, trace, observed)

    def bfs_batch(self, sources, config: KernelConfig, outs,
                  widths: Optional[list] = None) -> List[float]:
        """pbfs_bfs_batch: traversal i+1 overlaps the host copy of distances i.
        `outs[i]` receives source i's distances (entries may repeat, e.g. two
        rotating pinned buffers). Returns per-source device ms; `widths`, if
        given, receives the bytes per vertex each transfer moved (0.5 for
        4-bit codes)."""
        srcs = np.ascontiguousarray(np.asarray(sources, dtype=np.uint32))
        k = int(srcs.size)
        if len(outs) != k:
            raise ConfigError("bfs_batch needs one output buffer per source")
        for o in outs:
            if o.dtype != np.uint32 or o.size != self.vertex_count or not o.flags.c_contiguous:
                raise ConfigError("bfs_batch outputs must be contiguous uint32[vertex_count]")
        c = config._c()
        ptrs = (ctypes.c_void_p * k)(*[o.ctypes.data for o in outs])
        infos = (L.RunInfo * k)()
        _check(lib.pbfs_bfs_batch(self.h, srcs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                  k, ctypes.byref(c), ptrs, infos))
        if widths is not None:
            # transfer_width is in whole bytes, rounded up: a packed traversal
            # of fewer than 15 levels moves 4-bit codes (pack_bits).
            nibble = os.environ.get("PBFS_PACK_MIN_BITS", "4") != "8"
            widths[:] = [0.5 if nibble and infos[i].transfer_width == 1 and infos[i].levels < 15
                         else int(infos[i].transfer_width) for i in range(k)]
        return [float(infos[i].device_ms) for i in range(k)]

    def bfs_async(self, source: int, config: KernelConfig, stream: int = 0) -> None:
        c = config._c()
        _check(lib.pbfs_bfs_async(self.h, int(source) & 0xFFFFFFFF, ctypes.byref(c),
                                  ctypes.c_void_p(stream) if stream else None))

    def sync(self, stream: int = 0) -> None:
        _check(lib.pbfs_graph_sync(self.h, ctypes.c_void_p(stream) if stream else None))

    def device_arrays(self) -> dict:
        """Device CSR view (pointers into this handle's HBM copy)."""
        r = ctypes.c_void_p()
        c = ctypes.c_void_p()
        ob = ctypes.c_uint32()
        _check(lib.pbfs_graph_device_arrays(self.h, ctypes.byref(r), ctypes.byref(c),
                                            ctypes.byref(ob)))
        return dict(vertex_count=self.info["vertex_count"], edge_count=self.info["edge_count"],
                    row_offsets=r.value, column_indices=c.value, offset_bytes=ob.value,
                    symmetric=self.info["symmetric"])

    def device_distances_ptr(self) -> int:
        p = ctypes.c_void_p()
        _check(lib.pbfs_graph_device_dist(self.h, ctypes.byref(p)))
        return int(p.value or 0)

    def component(self):
        nr = ctypes.c_uint64()
        ar = ctypes.c_uint64()
        _check(lib.pbfs_graph_component(self.h, ctypes.byref(nr), ctypes.byref(ar)))
        return nr.value, ar.value


def pinned_empty(count: int, dtype=np.uint32) -> np.ndarray:
    """A page-locked host array (cudaMallocHost) for full-bandwidth D2H copies."""
    dtype = np.dtype(dtype)
    nbytes = max(int(count) * dtype.itemsize, 1)
    p = ctypes.c_void_p()
    _check(lib.pbfs_host_alloc(nbytes, ctypes.byref(p)))
    buf = (ctypes.c_uint8 * nbytes).from_address(p.value)
    weakref.finalize(buf, lib.pbfs_host_free, ctypes.c_void_p(p.value))
    return np.frombuffer(buf, dtype=dtype, count=int(count))


@dataclass
class LevelSnapshot:
    """kernel_config.hpp:26-33."""
    depth: int
    produced_by: TraversalPhase
    entries: np.ndarray


def _emit_snapshots(result: BfsResult, observer: Callable) -> None:
    """LevelObserver parity (kernels.cpp:158-161,466-481): one snapshot for the
    seed frontier, then one per produced level, in depth order, carrying the
    frontier the DEVICE produced (recorded with cfg.observe_frontiers,
    pbfs_graph_observed): top-down levels as the device pushed them (its
    order), bottom-up levels as ascending ids (the reference scans its byte
    bitmap in id order)."""
    recs = result.trace.records
    log = result._observed
    observer(LevelSnapshot(0, TraversalPhase.TopDown,
                           np.array([result.trace.source], dtype=np.uint32)))
    pos = 0
    for depth in range(1, len(recs)):
        k = recs[depth].distinct_size
        entries = log[pos:pos + k]
        pos += k
        phase = recs[depth - 1].phase
        if phase == TraversalPhase.BottomUp:
            entries = np.sort(entries)
        observer(LevelSnapshot(depth, phase, entries))
    if pos != log.size:
        raise CorrectnessError(f"observed {log.size} frontier entries, the trace accounts "
                               f"for {pos}")


def _gpu_run(graph: CsrGraph, source: int, config: KernelConfig, variant: KernelVariant,
             device: int = 0) -> BfsResult:
    cfg = KernelConfig(**{**config.__dict__, "variant": variant})
    validate(cfg)
    if not (0 <= int(source) < graph.vertex_count):
        raise InputError(f"source vertex {source} is out of range for a graph with "
                         f"{graph.vertex_count} vertices")
    res = graph.device(device).bfs(source, cfg)
    if config.level_observer is not None:
        _emit_snapshots(res, config.level_observer)
    return res


def bfs_conventional(graph: CsrGraph, source: int, config: KernelConfig) -> BfsResult:
    """kernels.cpp:586-594: top-down, atomicCAS claim on the distance slot."""
    return _gpu_run(graph, source, config, KernelVariant.Conventional)


def bfs_nonatomic(graph: CsrGraph, source: int, config: KernelConfig) -> BfsResult:
    """kernels.cpp:596-604: top-down, plain same-value distance stores."""
    return _gpu_run(graph, source, config, KernelVariant.NonAtomic)


def bfs_hybrid(graph: CsrGraph, source: int, config: KernelConfig) -> BfsResult:
    """kernels.cpp:606-616: direction switch by the frontier-size fraction."""
    return _gpu_run(graph, source, config, KernelVariant.Hybrid)


def bfs_hybrid_plain(graph: CsrGraph, source: int, config: KernelConfig) -> BfsResult:
    """kernels.cpp:606-616 with the reference Hybrid's own claim discipline:
    PlainStore top-down (no atomic, kernels.cpp:291-301) + bottom-up, 5 %
    switch (GPU variant PBFS_HYBRID_PLAIN)."""
    return _gpu_run(graph, source, config, KernelVariant.HybridPlainStore)


def bfs_hybrid_beamer(graph: CsrGraph, source: int, config: KernelConfig) -> BfsResult:
    """kernels.cpp:618-627: direction switch by Beamer's alpha/beta rules."""
    return _gpu_run(graph, source, config, KernelVariant.HybridBeamer)


def bfs_visited_bitmap(graph: CsrGraph, source: int, config: KernelConfig,
                       deferred: bool) -> BfsResult:
    """kernels.cpp:629-644. Deferred mode has no GPU form (ConfigError)."""
    return _gpu_run(graph, source, config,
                    KernelVariant.VisitedBitmapDeferred if deferred
                    else KernelVariant.VisitedBitmapInline)


def bfs_topdown_periodic_flush(graph: CsrGraph, source: int, config: KernelConfig) -> BfsResult:
    """kernels.cpp:646-655: no GPU form (ConfigError)."""
    return _gpu_run(graph, source, config, KernelVariant.TopDownPeriodicFlush)


def run_bfs(graph: CsrGraph, source: int, config: KernelConfig, stats: GraphStats,
            device=0) -> BfsResult:
    """kernels.cpp:657-691: large-diameter graphs run top-down only.
    `device` may be a list of CUDA ordinals (the graph partitioned over
    them, the multi-partition engine)."""
    effective = KernelConfig(**config.__dict__)
    if stats.category == GraphCategory.LargeDiameter:
        effective.force_top_down_only = True
    validate(effective)
    if not (0 <= int(source) < graph.vertex_count):
        raise InputError(f"source vertex {source} is out of range for a graph with "
                         f"{graph.vertex_count} vertices")
    res = graph.device(device).bfs(source, effective)
    if config.level_observer is not None:
        _emit_snapshots(res, config.level_observer)
    return res


# ---- timing (timing.hpp:17-34, timing.cpp:33-77) -------------------------------------
KernelFn = Callable[[CsrGraph, int, KernelConfig], BfsResult]


@dataclass
class TimingReport:
    median_ns: int = 0
    samples_ns: list = field(default_factory=list)
    median_trace: Optional[TraversalTrace] = None


def _check_against(expected: np.ndarray, got: np.ndarray) -> None:
    """timing.cpp:16-29."""
    if got is None or got.size != expected.size:
        raise CorrectnessError(f"kernel returned {0 if got is None else got.size} distances, "
                               f"expected {expected.size}")
    diff = np.nonzero(got != expected)[0]
    if diff.size:
        v = int(diff[0])
        raise CorrectnessError(f"distance mismatch at vertex {v}: expected {int(expected[v])}, "
                               f"got {int(got[v])}")


def time_run(graph: CsrGraph, source: int, config: KernelConfig, trials: int, warmups: int,
             kernel, expected: np.ndarray) -> TimingReport:
    """timing.cpp:33-69. ``kernel`` is a KernelFn or a GraphStats (then run_bfs).

    The reference computes its serial oracle inside time_run; this library
    contains no CPU traversal, so the caller passes the expected distance
    array (tests and bench take it from the oracle). Every run, warm-ups
    included, is checked; the reported median is the lower median.
    """
    if trials < 1:
        raise ConfigError("timing needs at least one trial")
    if isinstance(kernel, GraphStats):
        stats = kernel
        kernel = lambda g, s, c: run_bfs(g, s, c, stats)  # noqa: E731
    for _ in range(warmups):
        _check_against(expected, kernel(graph, source, config).distances)
    samples, traces = [], []
    for _ in range(trials):
        t0 = time.perf_counter_ns()
        r = kernel(graph, source, config)
        t1 = time.perf_counter_ns()
        _check_against(expected, r.distances)
        samples.append(t1 - t0)
        traces.append(r.trace)
    order = sorted(range(trials), key=lambda i: samples[i])
    mid = order[(trials - 1) // 2]
    return TimingReport(samples[mid], samples, traces[mid])


# ---- 1D vertex-partitioned multi-GPU traversal ------------------------
class PartitionedGraph:
    """One rank's partition of a resident graph (pbfs_part handle).

    Per level: ``step()`` (local work), then the caller exchanges the slices
    of ``info()['next']`` (an in-place allgather of ``words_local`` uint32
    words per rank, e.g. NCCL over NVLink), then ``end_level()``.
    """

    def __init__(self, dgraph, rank: int, world: int, relabel: bool = True,
                 shared: Optional["PartitionedGraph"] = None, device: int = 0):
        """dgraph: a DeviceGraph, or a device CSR view dict(vertex_count,
        edge_count, row_offsets=<device ptr>, column_indices=<device ptr>,
        offset_bytes, symmetric) on `device`."""
        opt = L.PartOptions()
        opt.rank, opt.world, opt.relabel = int(rank), int(world), int(bool(relabel))
        if shared is not None:
            si = shared.info()
            opt.shared_frontier, opt.shared_next = si["frontier"], si["next"]
        h = ctypes.c_void_p()
        if isinstance(dgraph, DeviceGraph):
            _check(lib.pbfs_part_create(dgraph.h, ctypes.byref(opt), ctypes.byref(h)))
        else:
            c = L.Csr()
            c.vertex_count = int(dgraph["vertex_count"])
            c.edge_count = int(dgraph["edge_count"])
            c.row_offsets = int(dgraph["row_offsets"])
            c.column_indices = int(dgraph["column_indices"])
            c.offset_bytes = int(dgraph["offset_bytes"])
            c.symmetric = int(bool(dgraph["symmetric"]))
            _check(lib.pbfs_part_create_device(ctypes.byref(c), int(device), ctypes.byref(opt),
                                               ctypes.byref(h)))
        self.h = h
        self._keep = (dgraph, shared)

    def component(self):
        nr = ctypes.c_uint64()
        ar = ctypes.c_uint64()
        _check(lib.pbfs_part_component(self.h, ctypes.byref(nr), ctypes.byref(ar)))
        return nr.value, ar.value

    def close(self):
        if getattr(self, "h", None):
            lib.pbfs_part_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = L.PartInfo()
        _check(lib.pbfs_part_get_info(self.h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in L.PartInfo._fields_}

    def begin(self, source: int, config: KernelConfig, stream: int = 0) -> None:
        c = config._c()
        _check(lib.pbfs_part_begin(self.h, int(source), ctypes.byref(c),
                                   ctypes.c_void_p(stream) if stream else None))

    def step(self, stream: int = 0) -> None:
        _check(lib.pbfs_part_step(self.h, ctypes.c_void_p(stream) if stream else None))

    def end_level(self, stream: int = 0):
        done = ctypes.c_uint32()
        rec = L.Level()
        _check(lib.pbfs_part_end_level(self.h, ctypes.c_void_p(stream) if stream else None,
                                       ctypes.byref(done), ctypes.byref(rec)))
        return bool(done.value), LevelRecord(rec.depth, TraversalPhase(rec.phase),
                                             rec.frontier_size, rec.distinct_size,
                                             rec.duplicate_count, rec.edges_examined, 0, 0)

    def end_level_async(self, stream: int = 0) -> None:
        """Enqueue the level's decision on the device (no sync)."""
        _check(lib.pbfs_part_end_level_async(self.h, ctypes.c_void_p(stream) if stream else None))

    def poll(self, stream: int = 0):
        """Synchronise; (done, levels recorded so far)."""
        done = ctypes.c_uint32()
        levels = ctypes.c_uint32()
        _check(lib.pbfs_part_poll(self.h, ctypes.c_void_p(stream) if stream else None,
                                  ctypes.byref(done), ctypes.byref(levels)))
        return bool(done.value), int(levels.value)

    def level_record(self, depth: int) -> LevelRecord:
        rec = L.Level()
        _check(lib.pbfs_part_level_record(self.h, int(depth), ctypes.byref(rec)))
        return LevelRecord(rec.depth, TraversalPhase(rec.phase), rec.frontier_size,
                           rec.distinct_size, rec.duplicate_count, rec.edges_examined, 0, 0)

    def sync(self, stream: int = 0) -> None:
        _check(lib.pbfs_part_sync(self.h, ctypes.c_void_p(stream) if stream else None))

    def local_distances(self) -> np.ndarray:
        out = np.empty(self.info()["local_count"], dtype=np.uint32)
        _check(lib.pbfs_part_copy_dist(self.h, out.ctypes.data))
        return out

    def unrelabel_host(self, dist_pi: np.ndarray) -> np.ndarray:
        dist_pi = np.ascontiguousarray(dist_pi, dtype=np.uint32)
        out = np.empty(self.info()["vertex_count"], dtype=np.uint32)
        _check(lib.pbfs_part_unrelabel_host(self.h, dist_pi.ctypes.data, out.ctypes.data))
        return out

    def unrelabel(self, dist_pi_dev: int, dist_dev: int, stream: int = 0) -> None:
        _check(lib.pbfs_part_unrelabel(self.h, ctypes.c_void_p(dist_pi_dev),
                                       ctypes.c_void_p(dist_dev),
                                       ctypes.c_void_p(stream) if stream else None))


def bfs_partitioned_loopback(graph: CsrGraph, source: int, config: KernelConfig, world: int,
                             device: int = 0, relabel: bool = True, parts=None):
    """G-way partitioned traversal with all partitions on one device sharing
    the full frontier bitmaps (the per-level allgather becomes a no-op).
    Returns (distances in original ids, per-level records, partitions)."""
    if parts is None:
        dg = graph.device(device, 8)
        p0 = PartitionedGraph(dg, 0, world, relabel)
        parts = [p0] + [PartitionedGraph(dg, r, world, relabel, shared=p0)
                        for r in range(1, world)]
    for p in parts:
        p.begin(source, config)
    records = []
    while True:
        for p in parts:
            p.step()
        for p in parts:
            p.sync()
        results = [p.end_level() for p in parts]
        done = results[0][0]
        assert all(r[0] == done for r in results), "ranks disagree on termination"
        rec = results[0][1]
        rec.edges_examined = sum(r[1].edges_examined for r in results)
        records.append(rec)
        if done:
            break
    dist_pi = np.concatenate([p.local_distances() for p in parts])
    return parts[0].unrelabel_host(dist_pi), records, parts

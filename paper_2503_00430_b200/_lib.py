"""ctypes binding of ``include/pbfs.h`` (the C ABI of ``libpbfs.so``).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2503_00430_b200/csrc``). There is no fallback: if the shared object is
missing or does not load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PBFS_LIB overrides the library path (A/B builds of the same ABI).
LIB_PATH = os.environ.get("PBFS_LIB", os.path.join(HERE, "libpbfs.so"))

c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class Csr(ctypes.Structure):
    _fields_ = [("vertex_count", c_u64), ("edge_count", c_u64), ("row_offsets", c_vp),
                ("column_indices", c_vp), ("offset_bytes", c_u32), ("symmetric", c_u32)]


class Config(ctypes.Structure):
    _fields_ = [("variant", c_u32), ("worker_count", c_u32),
                ("hybrid_threshold_fraction", c_dbl), ("alpha", c_dbl), ("beta", c_dbl),
                ("flush_capacity", c_u64), ("force_top_down_only", c_u32),
                ("validate_same_value_stores", c_u32), ("racy_visited_claim", c_u32),
                ("observe_frontiers", c_u32)]


class Level(ctypes.Structure):
    _fields_ = [("depth", c_u32), ("phase", c_u32), ("frontier_size", c_u64),
                ("distinct_size", c_u64), ("duplicate_count", c_u64),
                ("edges_examined", c_u64), ("flush_events", c_u64), ("elapsed_ns", c_i64)]


class RunInfo(ctypes.Structure):
    _fields_ = [("levels", c_u32), ("bottom_up_levels", c_u32), ("reached", c_u64),
                ("same_value_violations", c_u64), ("edges_examined", c_u64),
                ("device_ms", ctypes.c_float), ("transfer_width", c_u32)]


class GraphOptions(ctypes.Structure):
    _fields_ = [("device", c_i32), ("device_offset_bytes", c_u32), ("devices", c_vp),
                ("num_devices", c_u32), ("reserved", c_u32)]


class GraphInfo(ctypes.Structure):
    _fields_ = [("vertex_count", c_u64), ("edge_count", c_u64), ("max_degree", c_u64),
                ("device_bytes", c_u64), ("device_offset_bytes", c_u32), ("symmetric", c_u32),
                ("device", c_i32), ("grid_blocks", c_u32), ("block_threads", c_u32),
                ("partitions", c_u32)]


class GenSpec(ctypes.Structure):
    _fields_ = [("kind", c_u32), ("scale", c_u32), ("edge_factor", c_u32),
                ("drop_self_loops", c_u32), ("seed", c_u64), ("mesh_side", c_u32),
                ("mesh_radius", c_u32), ("mesh_keep", c_dbl), ("mesh_shortcuts", c_u64),
                ("threads", c_u32), ("reserved", c_u32)]


class Stats(ctypes.Structure):
    _fields_ = [("vertex_count", c_u64), ("edge_count", c_u64), ("average_degree", c_dbl),
                ("max_degree", c_u64), ("large_diameter", c_u32), ("reserved", c_u32)]


class PartOptions(ctypes.Structure):
    _fields_ = [("rank", c_u32), ("world", c_u32), ("relabel", c_u32), ("reserved", c_u32),
                ("shared_frontier", c_vp), ("shared_next", c_vp)]


class PartInfo(ctypes.Structure):
    _fields_ = [("vertex_count", c_u64), ("padded_count", c_u64), ("local_first", c_u64),
                ("local_count", c_u64), ("local_arcs", c_u64), ("words_total", c_u64),
                ("words_local", c_u64), ("rank", c_u32), ("world", c_u32),
                ("relabel_hashed", c_u32), ("depth", c_u32), ("top_down", c_u32),
                ("reserved", c_u32), ("frontier", c_vp), ("next", c_vp), ("dist_local", c_vp)]


class MultiInfo(ctypes.Structure):
    _fields_ = [("vertex_count", c_u64), ("edge_count", c_u64), ("padded_count", c_u64),
                ("local_arcs", c_u64 * 8), ("partitions", c_u32), ("devices", c_u32),
                ("ctas_per_partition", c_u32), ("relabel_hashed", c_u32)]


P = ctypes.POINTER

# (name, restype, argtypes) for every symbol include/pbfs.h declares.
SIGNATURES = [
    ("pbfs_abi_version", c_u32, []),
    ("pbfs_last_error", ctypes.c_char_p, []),
    ("pbfs_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("pbfs_config_init", None, [P(Config)]),
    ("pbfs_config_validate", ctypes.c_int, [P(Config)]),
    ("pbfs_graph_create", ctypes.c_int, [P(Csr), P(GraphOptions), P(c_vp)]),
    ("pbfs_graph_destroy", ctypes.c_int, [c_vp]),
    ("pbfs_graph_get_info", ctypes.c_int, [c_vp, P(GraphInfo)]),
    ("pbfs_bfs", ctypes.c_int, [c_vp, c_u32, P(Config), c_vp, P(Level), c_u32, P(RunInfo)]),
    ("pbfs_bfs_batch", ctypes.c_int, [c_vp, P(c_u32), c_u32, P(Config), P(c_vp), P(RunInfo)]),
    ("pbfs_bfs_async", ctypes.c_int, [c_vp, c_u32, P(Config), c_vp]),
    ("pbfs_graph_sync", ctypes.c_int, [c_vp, c_vp]),
    ("pbfs_graph_trace", ctypes.c_int, [c_vp, P(Level), c_u32, P(c_u32)]),
    ("pbfs_graph_observed", ctypes.c_int, [c_vp, c_vp, c_u64, P(c_u64)]),
    ("pbfs_graph_device_dist", ctypes.c_int, [c_vp, P(c_vp)]),
    ("pbfs_graph_component", ctypes.c_int, [c_vp, P(c_u64), P(c_u64)]),
    ("pbfs_host_alloc", ctypes.c_int, [ctypes.c_size_t, P(c_vp)]),
    ("pbfs_host_free", ctypes.c_int, [c_vp]),
    ("pbfs_generate", ctypes.c_int, [P(GenSpec), P(c_vp)]),
    ("pbfs_build_csr", ctypes.c_int, [c_vp, c_u64, c_u64, c_u32, c_u32, c_u32, P(c_vp)]),
    ("pbfs_host_csr_view", ctypes.c_int, [c_vp, P(Csr)]),
    ("pbfs_host_csr_free", ctypes.c_int, [c_vp]),
    ("pbfs_compute_stats", ctypes.c_int, [P(Csr), c_dbl, P(Stats)]),
    ("pbfs_pick_sources", ctypes.c_int, [P(Csr), c_u32, c_u64, c_vp]),
    ("pbfs_save_csr1", ctypes.c_int, [P(Csr), ctypes.c_char_p]),
    ("pbfs_load_csr1", ctypes.c_int, [ctypes.c_char_p, P(c_vp)]),
    ("pbfs_graph_device_arrays", ctypes.c_int, [c_vp, P(c_vp), P(c_vp), P(c_u32)]),
    ("pbfs_part_create", ctypes.c_int, [c_vp, P(PartOptions), P(c_vp)]),
    ("pbfs_part_create_device", ctypes.c_int, [P(Csr), c_i32, P(PartOptions), P(c_vp)]),
    ("pbfs_part_destroy", ctypes.c_int, [c_vp]),
    ("pbfs_part_component", ctypes.c_int, [c_vp, P(c_u64), P(c_u64)]),
    ("pbfs_part_get_info", ctypes.c_int, [c_vp, P(PartInfo)]),
    ("pbfs_part_relabel", ctypes.c_int, [c_vp, c_u64, P(c_u64)]),
    ("pbfs_part_begin", ctypes.c_int, [c_vp, c_u32, P(Config), c_vp]),
    ("pbfs_part_step", ctypes.c_int, [c_vp, c_vp]),
    ("pbfs_part_end_level", ctypes.c_int, [c_vp, c_vp, P(c_u32), P(Level)]),
    ("pbfs_part_end_level_async", ctypes.c_int, [c_vp, c_vp]),
    ("pbfs_part_poll", ctypes.c_int, [c_vp, c_vp, P(c_u32), P(c_u32)]),
    ("pbfs_part_level_record", ctypes.c_int, [c_vp, c_u32, P(Level)]),
    ("pbfs_part_sync", ctypes.c_int, [c_vp, c_vp]),
    ("pbfs_part_unrelabel", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("pbfs_part_copy_dist", ctypes.c_int, [c_vp, c_vp]),
    ("pbfs_part_unrelabel_host", ctypes.c_int, [c_vp, c_vp, c_vp]),
    ("pbfs_multi_create", ctypes.c_int, [P(Csr), P(c_i32), c_u32, P(c_vp)]),
    ("pbfs_multi_destroy", ctypes.c_int, [c_vp]),
    ("pbfs_multi_get_info", ctypes.c_int, [c_vp, P(MultiInfo)]),
    ("pbfs_multi_bfs", ctypes.c_int, [c_vp, c_u32, P(Config), c_vp, P(Level), c_u32, P(RunInfo)]),
    ("pbfs_multi_bfs_async", ctypes.c_int, [c_vp, c_u32, P(Config)]),
    ("pbfs_multi_sync", ctypes.c_int, [c_vp, P(ctypes.c_float)]),
    ("pbfs_multi_stream", ctypes.c_int, [c_vp, P(c_vp)]),
    ("pbfs_multi_component", ctypes.c_int, [c_vp, P(c_u64), P(c_u64)]),
    ("pbfs_multi_join", ctypes.c_int, [c_vp, c_vp]),
    ("pbfs_multi_trace", ctypes.c_int, [c_vp, P(Level), c_u32, P(c_u32)]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

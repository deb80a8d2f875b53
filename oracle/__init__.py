"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the BFS hot path.

Python ctypes front for the two checkers built by ``oracle/Makefile``:

* ``port`` — ``liboracle_port.so``, our plain-C restatement of the reference
  algorithms (``pbfs_oracle.c``; every function cites the reference file:line).
* ``ref``  — ``_ref/libparbfs_ref.so``, the UNMODIFIED reference library
  compiled from ``/root/reference/proj/core/src`` plus our C shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libparbfs_ref.so")
REF_ROOT = "/root/reference/proj/core"
UNREACHED = 0xFFFFFFFF

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference (when its sources exist)."""
    targets = ["port"]
    if ref and os.path.isdir(REF_ROOT):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class _Port:
    def __init__(self):
        if not os.path.exists(PORT_SO):
            build(ref=False)
        lib = ctypes.CDLL(PORT_SO)
        lib.orc_generate_pairs.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_uint64, _u32p]
        lib.orc_build_csr.restype = ctypes.c_uint64
        lib.orc_build_csr.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                      ctypes.c_int, _u64p, _u32p]
        lib.orc_bfs_serial.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_uint32, _u32p]
        lib.orc_relaxation.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_uint32, _u32p]
        lib.orc_pick_sources.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_uint32,
                                         ctypes.c_uint64, _u32p]
        lib.orc_simulate_phases.restype = ctypes.c_uint32
        lib.orc_simulate_phases.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u32p,
                                            ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_double, _u8p, ctypes.c_uint32]
        lib.orc_stats.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_double,
                                  ctypes.POINTER(ctypes.c_double), _u64p,
                                  ctypes.POINTER(ctypes.c_int)]
        lib.orc_mesh_pairs.restype = ctypes.c_uint64
        lib.orc_mesh_pairs.argtypes = [ctypes.c_uint32, ctypes.c_double, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_uint64, _u32p]
        lib.orc_component.argtypes = [ctypes.c_uint64, _u64p, _u32p, _u64p, _u64p]
        lib.orc_mt64_seed.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        lib.orc_mt64_next.restype = ctypes.c_uint64
        lib.orc_mt64_next.argtypes = [ctypes.c_void_p]
        self.lib = lib

    def mt64(self, seed: int, count: int) -> np.ndarray:
        state = ctypes.create_string_buffer(312 * 8 + 8)
        self.lib.orc_mt64_seed(state, seed)
        return np.array([self.lib.orc_mt64_next(state) for _ in range(count)], dtype=np.uint64)

    def generate_pairs(self, kind: int, scale: int, edge_factor: int, seed: int) -> np.ndarray:
        pairs = np.empty(2 * (edge_factor << scale), dtype=np.uint32)
        if self.lib.orc_generate_pairs(kind, scale, edge_factor, seed, _ptr(pairs, _u32p)) != 0:
            raise ValueError("bad generator spec")
        return pairs.reshape(-1, 2)

    def build_csr(self, pairs: np.ndarray, n: int, symmetrize: bool = True,
                  drop_self_loops: bool = False):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
        npairs = pairs.size // 2
        offsets = np.zeros(n + 1, dtype=np.uint64)
        col = np.empty(max(1, 2 * npairs), dtype=np.uint32)
        m = self.lib.orc_build_csr(_ptr(pairs, _u32p), npairs, n, int(symmetrize),
                                   int(drop_self_loops), _ptr(offsets, _u64p), _ptr(col, _u32p))
        if m == 2**64 - 1:
            raise ValueError("edge references a vertex >= n")
        return offsets, col[:m].copy()

    def bfs_serial(self, offsets: np.ndarray, col: np.ndarray, source: int) -> np.ndarray:
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        col = np.ascontiguousarray(col, dtype=np.uint32)
        n = offsets.size - 1
        dist = np.empty(n, dtype=np.uint32)
        if self.lib.orc_bfs_serial(n, _ptr(offsets, _u64p), _ptr(col, _u32p), source,
                                   _ptr(dist, _u32p)) != 0:
            raise ValueError("source out of range")
        return dist

    def relaxation(self, offsets: np.ndarray, col: np.ndarray, source: int) -> np.ndarray:
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        col = np.ascontiguousarray(col, dtype=np.uint32)
        n = offsets.size - 1
        dist = np.empty(n, dtype=np.uint32)
        if self.lib.orc_relaxation(n, _ptr(offsets, _u64p), _ptr(col, _u32p), source,
                                   _ptr(dist, _u32p)) != 0:
            raise ValueError("source out of range")
        return dist

    def pick_sources(self, offsets: np.ndarray, count: int, seed: int) -> np.ndarray:
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        out = np.empty(count, dtype=np.uint32)
        if self.lib.orc_pick_sources(offsets.size - 1, _ptr(offsets, _u64p), count, seed,
                                     _ptr(out, _u32p)) != 0:
            raise ValueError("graph has no vertex with positive degree")
        return out

    def simulate_phases(self, offsets, dist, threshold=0.05, beamer=False, alpha=15.0,
                        beta=18.0) -> list[int]:
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        dist = np.ascontiguousarray(dist, dtype=np.uint32)
        n = offsets.size - 1
        cap = int(dist[dist != UNREACHED].max()) + 1 if n else 0
        phases = np.zeros(max(cap, 1), dtype=np.uint8)
        k = self.lib.orc_simulate_phases(n, int(offsets[-1]), _ptr(offsets, _u64p),
                                         _ptr(dist, _u32p), threshold, int(beamer), alpha, beta,
                                         _ptr(phases, _u8p), cap)
        return [int(p) for p in phases[:k]]

    def stats(self, offsets, threshold=7.0):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        avg = ctypes.c_double()
        mx = ctypes.c_uint64()
        large = ctypes.c_int()
        self.lib.orc_stats(offsets.size - 1, int(offsets[-1]), _ptr(offsets, _u64p), threshold,
                           ctypes.byref(avg), ctypes.byref(mx), ctypes.byref(large))
        return avg.value, mx.value, bool(large.value)

    def mesh_pairs(self, side, keep=0.9, shortcuts=None, radius=32, seed=1) -> np.ndarray:
        n = side * side
        if shortcuts is None:
            shortcuts = int(round(0.001 * n))
        pairs = np.empty(2 * (2 * side * (side - 1) + shortcuts), dtype=np.uint32)
        k = self.lib.orc_mesh_pairs(side, keep, shortcuts, radius, seed, _ptr(pairs, _u32p))
        return pairs[: 2 * k].reshape(-1, 2)

    def component(self, offsets, dist):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        dist = np.ascontiguousarray(dist, dtype=np.uint32)
        nr = ctypes.c_uint64()
        ar = ctypes.c_uint64()
        self.lib.orc_component(offsets.size - 1, _ptr(offsets, _u64p), _ptr(dist, _u32p),
                               ctypes.byref(nr), ctypes.byref(ar))
        return nr.value, ar.value


class RefLevel(ctypes.Structure):
    _fields_ = [("depth", ctypes.c_uint32), ("phase", ctypes.c_uint32),
                ("frontier_size", ctypes.c_uint64), ("distinct_size", ctypes.c_uint64),
                ("duplicate_count", ctypes.c_uint64), ("edges_examined", ctypes.c_uint64),
                ("flush_events", ctypes.c_uint64), ("elapsed_ns", ctypes.c_int64)]


class RefGraph:
    """A graph held by the reference library (parbfs::CsrGraph)."""

    def __init__(self, ref: "_Ref", handle):
        self._ref = ref
        self.h = handle
        n = ctypes.c_uint64()
        m = ctypes.c_uint64()
        sym = ctypes.c_int()
        ref.lib.ref_graph_info(handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(sym))
        self.n, self.m, self.symmetric = n.value, m.value, bool(sym.value)

    def export(self):
        offsets = np.empty(self.n + 1, dtype=np.uint64)
        col = np.empty(max(self.m, 1), dtype=np.uint32)
        self._ref.lib.ref_graph_export(self.h, _ptr(offsets, _u64p), _ptr(col, _u32p))
        return offsets, col[: self.m]

    def __del__(self):
        try:
            self._ref.lib.ref_graph_free(self.h)
        except Exception:
            pass


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Ref:
    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        lib = ctypes.CDLL(REF_SO)
        vp = ctypes.c_void_p
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_graph_generate.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_uint64, ctypes.POINTER(vp)]
        lib.ref_graph_build.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.POINTER(vp)]
        lib.ref_graph_from_csr.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u32p,
                                           ctypes.c_int, ctypes.POINTER(vp)]
        lib.ref_graph_info.argtypes = [vp, _u64p, _u64p, ctypes.POINTER(ctypes.c_int)]
        lib.ref_graph_export.argtypes = [vp, _u64p, _u32p]
        lib.ref_graph_free.argtypes = [vp]
        lib.ref_bfs_serial.argtypes = [vp, ctypes.c_uint32, _u32p]
        lib.ref_stats.argtypes = [vp, ctypes.c_double, ctypes.POINTER(ctypes.c_double), _u64p,
                                  ctypes.POINTER(ctypes.c_int)]
        lib.ref_run.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32,
                                ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                ctypes.c_int, _u32p, ctypes.POINTER(RefLevel), ctypes.c_uint32,
                                _u32p, ctypes.POINTER(ctypes.c_int64)]
        self.lib = lib

    def _check(self, rc: int):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def generate(self, kind: int, scale: int, edge_factor: int, seed: int) -> RefGraph:
        h = ctypes.c_void_p()
        self._check(self.lib.ref_graph_generate(kind, scale, edge_factor, seed, ctypes.byref(h)))
        return RefGraph(self, h)

    def build(self, pairs: np.ndarray, n: int, symmetrize: bool) -> RefGraph:
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
        h = ctypes.c_void_p()
        self._check(self.lib.ref_graph_build(_ptr(pairs, _u32p), pairs.size // 2, n,
                                             int(symmetrize), ctypes.byref(h)))
        return RefGraph(self, h)

    def from_csr(self, offsets: np.ndarray, col: np.ndarray, symmetric: bool = True) -> RefGraph:
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        col = np.ascontiguousarray(col, dtype=np.uint32)
        h = ctypes.c_void_p()
        self._check(self.lib.ref_graph_from_csr(offsets.size - 1, col.size, _ptr(offsets, _u64p),
                                                _ptr(col, _u32p), int(symmetric),
                                                ctypes.byref(h)))
        return RefGraph(self, h)

    def bfs_serial(self, g: RefGraph, source: int) -> np.ndarray:
        dist = np.empty(g.n, dtype=np.uint32)
        self._check(self.lib.ref_bfs_serial(g.h, source, _ptr(dist, _u32p)))
        return dist

    def stats(self, g: RefGraph, threshold: float = 7.0):
        avg = ctypes.c_double()
        mx = ctypes.c_uint64()
        large = ctypes.c_int()
        self._check(self.lib.ref_stats(g.h, threshold, ctypes.byref(avg), ctypes.byref(mx),
                                       ctypes.byref(large)))
        return avg.value, mx.value, bool(large.value)

    def run(self, g: RefGraph, source: int, variant: int, workers: int = 1,
            threshold: float = 0.05, alpha: float = 15.0, beta: float = 18.0,
            force_td: bool = False, dispatch: bool = False, want_dist: bool = True):
        """Runs a reference kernel; returns (dist or None, levels, wall_ns)."""
        dist = np.empty(g.n, dtype=np.uint32) if want_dist else None
        cap = 1 << 16
        levels = (RefLevel * cap)()
        nlev = ctypes.c_uint32()
        wall = ctypes.c_int64()
        self._check(self.lib.ref_run(g.h, source, variant, workers, threshold, alpha, beta,
                                     int(force_td), int(dispatch),
                                     _ptr(dist, _u32p) if want_dist else None, levels, cap,
                                     ctypes.byref(nlev), ctypes.byref(wall)))
        recs = [dict(depth=levels[i].depth, phase=levels[i].phase,
                     frontier_size=levels[i].frontier_size,
                     distinct_size=levels[i].distinct_size,
                     duplicate_count=levels[i].duplicate_count,
                     edges_examined=levels[i].edges_examined,
                     elapsed_ns=levels[i].elapsed_ns) for i in range(min(nlev.value, cap))]
        return dist, recs, wall.value


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_ROOT)

"""B200-native level-synchronous BFS (arXiv 2503.00430) behind the reference
``parbfs`` API. See DESIGN.md; the C ABI is include/pbfs.h."""
from .parbfs import *  # noqa: F401,F403
from .parbfs import (BfsResult, CsrGraph, DeviceGraph, GeneratorKind, GeneratorSpec,  # noqa: F401
                     GraphCategory, GraphStats, KernelConfig, KernelVariant, LevelRecord,
                     TraversalPhase, TraversalTrace, UNREACHED, build_csr, compute_stats,
                     generate, pick_sources, run_bfs)

__all__ = [n for n in dir() if not n.startswith("_")]

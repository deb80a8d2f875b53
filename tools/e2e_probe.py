#!/usr/bin/env python3
"""pbfs_bfs_batch over the 64 seeded sources: wall time vs summed device time
(is the e2e bound host-side?)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "rmat26"
g = bench.build_graph(w)
cfg, _ = bench.kernel_config(g)
dg = g.device(0, bench.WORKLOADS[w][3])
srcs = [int(s) for s in pb.pick_sources(g, 64, 1)]
host = [pb.parbfs.pinned_empty(g.vertex_count, np.uint32) for _ in range(2)]
outs = [host[i % 2] for i in range(len(srcs))]
dg.bfs_batch(srcs[:2], cfg, outs[:2])
for rep in range(3):
    t0 = time.perf_counter()
    ms = dg.bfs_batch(srcs, cfg, outs)
    wall = (time.perf_counter() - t0) * 1e3
    print(f"batch wall {wall:.1f} ms, device sum {sum(ms):.1f} ms, per source {wall/64:.3f} / {sum(ms)/64:.3f}")
dg.release() if hasattr(dg, "release") else None
g.release_device()

#!/usr/bin/env python3
"""Per-level timeline of CTA 0 (diagnostic build, PBFS_TIMELINE=1): where a
level's latency goes. Build: make -C paper_2503_00430_b200/csrc ab NAME=tl
DEFS=-DPBFS_TIMELINE=1, then PBFS_LIB=build/ab/libpbfs_tl.so tools/timeline.py."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="mesh4096")
ap.add_argument("--sources", type=int, default=2)
ap.add_argument("--per-level", action="store_true")
args = ap.parse_args()
g = bench.build_graph(args.workload)
cfg, _ = bench.kernel_config(g)
dg = g.device(0, bench.WORKLOADS[args.workload][3])
names = ["phase work", "flush+tally", "barrier", "counters"]
for s in pb.pick_sources(g, args.sources, 1):
    dg.bfs(int(s), cfg, want_trace=False)
    r = dg.bfs(int(s), cfg)
    recs = r.trace.records
    marks = np.array([[(rec.flush_events >> (16 * k)) & 0xFFFF for k in range(4)] for rec in recs],
                     dtype=np.float64)
    el = np.array([rec.elapsed_ns for rec in recs], dtype=np.float64)
    print(f"source {s}: {len(recs)} levels, device {r.trace.device_ms:.3f} ms, "
          f"mean level {el.mean()/1e3:.2f} us")
    if args.per_level:
        for i, rec in enumerate(recs):
            mk = " ".join(f"{nm}={marks[i][k]/1e3:.1f}" for k, nm in enumerate(names))
            print(f"  d={rec.depth:3d} {pb.to_string(rec.phase):9s} frontier={rec.frontier_size:10d} "
                  f"edges={rec.edges_examined:12d} span={el[i]/1e3:8.1f} us | {mk}")
        continue
    sel = slice(2, len(recs) - 1)
    m = marks[sel].mean(axis=0)
    prev = 0.0
    for k, nm in enumerate(names):
        print(f"  {nm:12s} ends at {m[k]/1e3:6.2f} us  (+{(m[k]-prev)/1e3:5.2f})")
        prev = m[k]
    print(f"  level span (record to record) {el[sel].mean()/1e3:6.2f} us")

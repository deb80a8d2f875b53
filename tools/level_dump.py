#!/usr/bin/env python3
"""Every level of the hybrid traversal from each of the 64 seeded sources as
CSV (source, depth, phase, frontier, next frontier, edges, us): the input of
the per-regime time breakdowns in DESIGN.md."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat26")
ap.add_argument("--sources", type=int, default=64)
args = ap.parse_args()
g = bench.build_graph(args.workload)
cfg, _ = bench.kernel_config(g)
dg = g.device(0, bench.WORKLOADS[args.workload][3])
print("source,depth,phase,frontier,next,edges,us")
for s in pb.pick_sources(g, args.sources, 1):
    dg.bfs(int(s), cfg, want_trace=False)  # warm
    recs = dg.bfs(int(s), cfg).trace.records
    for i, r in enumerate(recs):
        nxt = recs[i + 1].distinct_size if i + 1 < len(recs) else 0
        print(f"{s},{r.depth},{pb.to_string(r.phase)},{r.frontier_size},{nxt},"
              f"{r.edges_examined},{r.elapsed_ns / 1e3:.2f}")

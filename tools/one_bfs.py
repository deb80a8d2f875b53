#!/usr/bin/env python3
"""Repeated traversals from one seeded source (for ncu captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat20")
ap.add_argument("--source-index", type=int, default=0)
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--variant", default="hybrid")
ap.add_argument("--td-only", action="store_true")
args = ap.parse_args()
g = bench.build_graph(args.workload)
cfg, _ = bench.kernel_config(g)
cfg.variant = pb.parse_kernel_variant(args.variant)
cfg.force_top_down_only = cfg.force_top_down_only or args.td_only
dg = g.device(0, bench.WORKLOADS[args.workload][3])
s = int(pb.pick_sources(g, args.source_index + 1, 1)[args.source_index])
for _ in range(args.repeat):
    r = dg.bfs(s, cfg)
print(f"source {s}: {r.trace.device_ms:.3f} ms, {len(r.trace.records)} levels")

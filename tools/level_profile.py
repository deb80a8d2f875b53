#!/usr/bin/env python3
"""Per-level device trace (parbfs::LevelRecord fields + %globaltimer span) of
the hybrid traversal for a few seeded sources — where the time goes."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat26")
ap.add_argument("--sources", type=int, default=3)
ap.add_argument("--variant", default="hybrid")
args = ap.parse_args()
g = bench.build_graph(args.workload)
cfg, _ = bench.kernel_config(g)
cfg.variant = pb.parse_kernel_variant(args.variant)
dg = g.device(0, bench.WORKLOADS[args.workload][3])
for s in pb.pick_sources(g, min(args.sources, 3), 1):
    dg.bfs(int(s), cfg, want_trace=False)  # warm
    r = dg.bfs(int(s), cfg)
    t = r.trace
    print(f"source {s}: device {t.device_ms:.3f} ms, levels {len(t.records)}")
    for rec in t.records:
        print(f"  d={rec.depth:3d} {pb.to_string(rec.phase):9s} frontier={rec.frontier_size:10d} "
              f"distinct={rec.distinct_size:10d} edges={rec.edges_examined:12d} "
              f"t={rec.elapsed_ns/1e3:9.1f} us")

if args.sources >= 16:
    # Aggregate: where does the time go across sources (by phase and size).
    import collections
    agg = collections.Counter()
    times = []
    for s in pb.pick_sources(g, args.sources, 1):
        r = dg.bfs(int(s), cfg)
        times.append(r.trace.device_ms)
        for rec in r.trace.records:
            big = rec.edges_examined > 1e7 or rec.frontier_size > 1e6
            key = f"{pb.to_string(rec.phase)}-{'big' if big else 'small'}"
            agg[key] += rec.elapsed_ns / 1e6
    times.sort()
    print("per-source ms: min %.3f p50 %.3f p90 %.3f max %.3f sum %.1f" % (
        times[0], times[len(times) // 2], times[int(len(times) * 0.9)], times[-1], sum(times)))
    for k, v in sorted(agg.items()):
        print(f"  {k:18s} {v:9.2f} ms total")

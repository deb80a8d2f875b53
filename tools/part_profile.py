#!/usr/bin/env python3
"""Per-level device time of the partitioned engine with G loopback
partitions on one GPU (each partition's step timed with CUDA events), next
to the single-GPU persistent kernel's level trace -- where the partitioned
path loses per-GPU efficiency."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat26")
ap.add_argument("--partitions", type=int, default=2)
ap.add_argument("--sources", type=int, default=2)
ap.add_argument("--identity", action="store_true", help="contiguous split, no hashed relabel")
args = ap.parse_args()
g = bench.build_graph(args.workload)
cfg, _ = bench.kernel_config(g)
dg = g.device(0, 8)
G = args.partitions
rl = not args.identity
parts = [pb.PartitionedGraph(dg, 0, G, relabel=rl)]
parts += [pb.PartitionedGraph(dg, r, G, relabel=rl, shared=parts[0]) for r in range(1, G)]
print("local arcs", [p.info()["local_arcs"] for p in parts])
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
sptr = stream.cuda_stream
for s in pb.pick_sources(g, args.sources, 1):
    s = int(s)
    r = dg.bfs(s, cfg)
    print(f"source {s}: single-GPU kernel {r.trace.device_ms:.3f} ms")
    for rec in r.trace.records:
        print(f"   d={rec.depth} {pb.to_string(rec.phase):9s} edges={rec.edges_examined:12d} "
              f"{rec.elapsed_ns/1e3:9.1f} us")
    for rep in range(2):
        for p in parts:
            p.begin(s, cfg, sptr)
        rows = []
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        t_all0.record(stream)
        while True:
            ev = []
            for p in parts:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                p.step(sptr)
                b.record(stream)
                ev.append((a, b))
            c0 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            res = [p.end_level(sptr) for p in parts]
            c1 = torch.cuda.Event(enable_timing=True)
            c1.record(stream)
            c1.synchronize()
            rows.append((res[0][1], [a.elapsed_time(b) for a, b in ev], c0.elapsed_time(c1)))
            if res[0][0]:
                break
        t_all1.record(stream)
        t_all1.synchronize()
    print(f"   partitioned x{G}: {t_all0.elapsed_time(t_all1):.3f} ms (a sync every level)")
    for look in (4, 8):
        for rep in range(2):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for p in parts:
                p.begin(s, cfg, sptr)
            while True:
                for _ in range(look):
                    for p in parts:
                        p.step(sptr)
                    for p in parts:
                        p.end_level_async(sptr)
                if parts[0].poll(sptr)[0]:
                    break
            b.record(stream)
            b.synchronize()
        print(f"   partitioned x{G}, {look} levels per poll: {a.elapsed_time(b):.3f} ms")
    for rec, steps, endt in rows:
        print(f"   d={rec.depth} {pb.to_string(rec.phase):9s} step ms per partition "
              f"{[round(x, 3) for x in steps]} end_level {endt:.3f} ms")

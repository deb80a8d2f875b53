#!/usr/bin/env python3
"""Experiment: does a degree-ordered vertex numbering (hubs first, isolated
vertices last) speed the traversal kernels up? Builds the relabelled CSR on
the host, runs the unchanged kernels on both graphs from the same (mapped)
sources, checks the distances agree through the permutation, and prints
per-level-class times for both. Measurement tool, not product code."""
import argparse
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402
from paper_2503_00430_b200 import parbfs as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat26")
ap.add_argument("--sources", type=int, default=16)
ap.add_argument("--variant", default="hybrid")
ap.add_argument("--order", default="degree", choices=["degree", "degree-blocked"])
args = ap.parse_args()

g = bench.build_graph(args.workload)
n, m = g.vertex_count, g.edge_count
off = np.asarray(g.row_offsets)
col = np.asarray(g.column_indices)
deg = np.diff(off).astype(np.int64)
t0 = time.time()
order = np.argsort(-deg, kind="stable").astype(np.uint32)  # order[new] = old
perm = np.empty(n, dtype=np.uint32)
perm[order] = np.arange(n, dtype=np.uint32)
pairs = np.empty((m, 2), dtype=np.uint32)
pairs[:, 0] = np.repeat(perm, deg)
np.take(perm, col, out=pairs[:, 1])
print(f"[relabel] permuted pairs in {time.time()-t0:.1f}s", file=sys.stderr)
t0 = time.time()
h = ctypes.c_void_p()
P._check(P.lib.pbfs_build_csr(pairs.ctypes.data, m, n, 0, 0, 0, ctypes.byref(h)))
del pairs
g2 = P._from_host_handle(h)
print(f"[relabel] rebuilt CSR in {time.time()-t0:.1f}s: m={g2.edge_count}", file=sys.stderr)
assert g2.edge_count == m

cfg, _ = bench.kernel_config(g)
cfg.variant = pb.parse_kernel_variant(args.variant)
offb = bench.WORKLOADS[args.workload][3]
srcs = [int(s) for s in pb.pick_sources(g, args.sources, 1)]


def run(graph, sources, label):
    dg = graph.device(0, offb)
    out = []
    for s in sources:
        dg.bfs(s, cfg, want_trace=False)
        r = dg.bfs(s, cfg)
        out.append((r.distances.copy() if len(out) < 2 else None, r.trace))
    dg.close()
    return out


a = run(g, srcs, "original")
b = run(g2, [int(perm[s]) for s in srcs], "degree-ordered")
for i in range(2):
    assert np.array_equal(a[i][0], b[i][0][perm]), "distances differ through the permutation"
print("parity through the permutation: ok (2 sources)")


def classes(tr):
    c = {"td_big": 0.0, "td_mid": 0.0, "td_small": 0.0, "bu": 0.0}
    for r in tr.records:
        us = r.elapsed_ns / 1e3
        if pb.to_string(r.phase).startswith("bottom"):
            c["bu"] += us
        elif r.edges_examined > 1e8:
            c["td_big"] += us
        elif r.edges_examined > 1e7:
            c["td_mid"] += us
        else:
            c["td_small"] += us
    return c


tot = {"orig": {}, "new": {}}
ms = {"orig": [], "new": []}
for (_, ta), (_, tb) in zip(a, b):
    for k, tr in (("orig", ta), ("new", tb)):
        ms[k].append(tr.device_ms)
        for kk, v in classes(tr).items():
            tot[k][kk] = tot[k].get(kk, 0.0) + v
for k in ("orig", "new"):
    print(k, f"mean {np.mean(ms[k]):.4f} ms/BFS over {len(srcs)} sources;",
          {kk: round(v / len(srcs) / 1e3, 4) for kk, v in tot[k].items()}, "(ms per BFS by class)")
print("per-source ms orig:", [round(x, 3) for x in ms["orig"]])
print("per-source ms new :", [round(x, 3) for x in ms["new"]])

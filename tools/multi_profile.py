"""Per-traversal and per-level cost of the fused multi-partition engine
(pbfs_multi) against the single-GPU engine, on one B200 with loopback
partitions. Per level the fused engine adds one partition barrier, the
system-scope release and one flag round; on a deep graph (the mesh, ~3900
levels run top-down) the difference per level is that exchange cost.

  python tools/multi_profile.py [workload ...]
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2503_00430_b200 as pb  # noqa: E402


def main():
    names = sys.argv[1:] or ["rmat20", "mesh4096", "rmat26"]
    for name in names:
        g = bench.build_graph(name)
        cfg, _ = bench.kernel_config(g)
        cfg.variant = pb.KernelVariant.Hybrid
        srcs = [int(s) for s in pb.pick_sources(g, 8, 1)]
        dg = g.device(0, 8)
        single = []
        for s in srcs:
            r = dg.bfs(s, cfg)
            single.append((r.trace.device_ms, len(r.trace.records)))
        want = {s: dg.bfs(s, cfg, want_trace=False).distances.copy() for s in srcs[:2]}
        g.release_device()
        ms1 = statistics.mean(x[0] for x in single)
        lev = statistics.mean(x[1] for x in single)
        print(f"{name}: single-GPU engine {ms1:.3f} ms/BFS, {lev:.0f} levels "
              f"({1e3 * ms1 / lev:.2f} us/level)", flush=True)
        for parts in (1, 2, 4, 8):
            mg = g.multi_device([0] * parts)
            for s in srcs[:2]:
                assert np.array_equal(mg.bfs(s, cfg, want_trace=False).distances, want[s])
            rows = []
            for s in srcs:
                mg.bfs_async(s, cfg)
                ms = mg.sync()
                r = mg.bfs(s, cfg)
                rows.append((ms, len(r.trace.records)))
            msp = statistics.mean(x[0] for x in rows)
            levp = statistics.mean(x[1] for x in rows)
            print(f"  fused, {parts} loopback partition(s) x {mg.info['ctas_per_partition']} CTAs: "
                  f"{msp:.3f} ms/BFS, {1e3 * msp / levp:.2f} us/level "
                  f"(+{1e3 * (msp - ms1) / levp:.2f} us/level vs single)", flush=True)
            mg.close()


if __name__ == "__main__":
    main()

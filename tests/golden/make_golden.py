#!/usr/bin/env python3
"""Generates the golden fixtures in tests/golden/ by running the UNMODIFIED
reference library (oracle/_ref/libparbfs_ref.so, compiled from
/root/reference/proj/core/src by oracle/Makefile). Run in the build container
(the only place /root/reference exists); the .npz files are committed and
travel to the GPU box.

Contents per fixture (all produced by reference calls, none by our code):
  generate()        proj/core/src/generator.cpp:41-92  -> offsets, col (self-loops kept)
  bfs_serial()      proj/core/src/kernels.cpp:19-41    -> distances for listed sources
  bfs_hybrid()      proj/core/src/kernels.cpp:606-616  -> per-level phase / distinct size
  bfs_hybrid_beamer kernels.cpp:618-627                -> per-level phases
  compute_stats()   proj/core/src/graph_stats.cpp:9-25 -> avg degree, max degree, category
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

# (kind, scale, edge_factor, seed, sources) — kind 0 uniform, 1 Kronecker.
SPECS = [
    (1, 6, 4, 99, [0, 1, 5]),      # test_graph_core.cpp:257-266 determinism spec
    (0, 8, 4, 3, [0, 7, 100]),
    (1, 10, 8, 77, [0, 3, 512]),   # test_kernels.cpp:269 beamer-phase graph
    (1, 10, 15, 1, [0, 17]),       # test_graph_core.cpp:317-325 shallow-category graph
    (1, 12, 16, 3, [0, 1, 2]),     # test_kernels.cpp:312 hybrid-vs-conventional graph
    (0, 12, 2, 12, [5, 77]),
    (1, 16, 16, 1, [0, 1, 4242]),  # larger RMAT at BASELINE's edge factor / seed
]
VARIANT_HYBRID = 3
VARIANT_BEAMER = 4


def main():
    ref = oracle.ref()
    manifest = []
    for kind, scale, ef, seed, sources in SPECS:
        g = ref.generate(kind, scale, ef, seed)
        off, col = g.export()
        avg, mx, large = ref.stats(g)
        data = {"stats": np.array([avg, mx, large], dtype=np.float64),
                "sources": np.array(sources, dtype=np.uint32),
                "n": np.array(g.n, dtype=np.uint64), "m": np.array(g.m, dtype=np.uint64),
                "sha256_offsets": np.array(hashlib.sha256(off.astype(np.uint64).tobytes())
                                           .hexdigest()),
                "sha256_col": np.array(hashlib.sha256(col.astype(np.uint32).tobytes())
                                       .hexdigest())}
        if scale <= 12:  # small graphs carry the arrays themselves
            data["offsets"] = off.astype(np.uint64)
            data["col"] = col.astype(np.uint32)
        for s in sources:
            if off[s + 1] == off[s]:
                continue
            data[f"dist_{s}"] = ref.bfs_serial(g, s)
            _, recs, _ = ref.run(g, s, VARIANT_HYBRID, workers=2, want_dist=False)
            data[f"hybrid_phase_{s}"] = np.array([r["phase"] for r in recs], dtype=np.uint8)
            data[f"hybrid_distinct_{s}"] = np.array([r["distinct_size"] for r in recs],
                                                    dtype=np.uint64)
            _, recs, _ = ref.run(g, s, VARIANT_BEAMER, workers=2, want_dist=False)
            data[f"beamer_phase_{s}"] = np.array([r["phase"] for r in recs], dtype=np.uint8)
        name = f"gen_{'kron' if kind else 'uniform'}_{scale}_{ef}_{seed}.npz"
        np.savez_compressed(os.path.join(HERE, name), **data)
        digest = hashlib.sha256(off.tobytes() + col.tobytes()).hexdigest()[:16]
        manifest.append(f"{name} n={g.n} m={g.m} sha256[:16]={digest}")
        print(manifest[-1])
    with open(os.path.join(HERE, "MANIFEST.txt"), "w") as f:
        f.write("# produced by tests/golden/make_golden.py from the reference library\n")
        f.write("\n".join(manifest) + "\n")


if __name__ == "__main__":
    main()

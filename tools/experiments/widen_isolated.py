#!/usr/bin/env python3
"""The widening pool alone (no GPU activity) on the buffers the batch uses:
pinned destination (huge pages / 4 KB pages by PBFS_PINNED_HUGE) and a
pageable numpy destination. Diagnostic for the batch e2e."""
import ctypes, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
import paper_2503_00430_b200 as pb
from paper_2503_00430_b200 import parbfs as P
g = bench.build_graph("rmat26")
cfg, _ = bench.kernel_config(g)
dg = g.device(0, 8)
srcs = [int(s) for s in pb.pick_sources(g, 4, 1)]
host = [P.pinned_empty(g.vertex_count, np.uint32) for _ in range(2)]
dg.bfs_batch(srcs, cfg, [host[i % 2] for i in range(4)])
L = ctypes.CDLL(os.environ.get("PBFS_LIB", os.path.join(ROOT, "paper_2503_00430_b200", "libpbfs.so")))
L.pbfs_debug_widen.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_double)]
ms = ctypes.c_double()
handle = dg.h
for name, dst in (("pinned", host[0]), ("pageable", np.empty(g.vertex_count, np.uint32))):
    dst[:] = 0
    for rep in range(3):
        rc = L.pbfs_debug_widen(handle, dst.ctypes.data, 10, ctypes.byref(ms))
        print(name, "rc", rc, f"{ms.value:.3f} ms per 256 MB array")

# Interference: the same widening while (a) 64 MB D2H copies run back to back,
# (b) traversals run back to back (no copies), (c) both.
import threading
import torch
stop = False
dev_codes = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
pin_codes = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
def copier():
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        while not stop:
            pin_codes.copy_(dev_codes, non_blocking=True)
            st.synchronize()
def runner():
    i = 0
    while not stop:
        dg.bfs_async(srcs[i % 4], cfg)
        dg.sync()
        i += 1
for label, fns in (("copies", [copier]), ("kernels", [runner]), ("copies+kernels", [copier, runner])):
    stop = False
    th = [threading.Thread(target=f) for f in fns]
    for t in th: t.start()
    time.sleep(0.2)
    for rep in range(3):
        L.pbfs_debug_widen(handle, host[0].ctypes.data, 20, ctypes.byref(ms))
        print(label, f"{ms.value:.3f} ms per 256 MB array")
    stop = True
    for t in th: t.join()

"""TEST MODEL of the 1D vertex-partition protocol (csrc/pbfs_part.cu), in numpy:
same ownership (hashed pi) and order-preserving gid numbering, same
row/column slices, same per-level allgather of the next-frontier bitmap
slices. Used by the gloo world-size-2 CPU tests to
check the host-side partition logic and the exchange protocol without a GPU.
"""
import numpy as np

A64 = 0x9E3779B97F4A7C15
B64 = 0xC2B2AE3D27D4EB4F
UNREACHED = 0xFFFFFFFF


def inv_odd(a, mask):
    x = a
    for _ in range(6):
        x = (x * (2 - a * x)) & ((1 << 64) - 1)
    return x & mask


class Relabel:
    """pi on [0, 2^k): v*a, xor-shift by ceil(k/2), *b (mod 2^k)."""

    def __init__(self, n, world, hashed=True):
        k = max(1, (n - 1).bit_length())
        quantum = 512 * world
        world_pow2 = world & (world - 1) == 0
        if (1 << k) == n and world_pow2 and hashed and n >= quantum and k >= 2:
            self.hashed, self.npad = True, n
        else:
            self.hashed, self.npad = False, (n + quantum - 1) // quantum * quantum
        self.k, self.mask = k, (1 << k) - 1
        self.a, self.b = (A64 & self.mask) | 1, (B64 & self.mask) | 1
        self.h = (k + 1) // 2

    def fwd(self, v):
        v = np.asarray(v, dtype=np.uint64)
        if not self.hashed:
            return v
        m = np.uint64(self.mask)
        x = (v * np.uint64(self.a)) & m
        x ^= x >> np.uint64(self.h)
        return (x * np.uint64(self.b)) & m


def gid_map(n, world, hashed=True):
    """gid(v) = owner * nloc + rank of v among its owner's vertices (original
    order), owner = pi(v) // nloc."""
    rl = Relabel(n, world, hashed)
    nloc = rl.npad // world
    owner = rl.fwd(np.arange(n, dtype=np.uint64)).astype(np.int64) // nloc
    order = np.argsort(owner, kind="stable")
    counts = np.bincount(owner, minlength=world)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    gid = np.empty(n, dtype=np.int64)
    gid[order] = owner[order] * nloc + (np.arange(n) - starts[owner[order]])
    return rl, nloc, gid


def build_partition(offsets, col, n, rank, world, hashed=True):
    rl, nloc, pi = gid_map(n, world, hashed)
    lo = rank * nloc
    inv = np.full(rl.npad, -1, dtype=np.int64)
    inv[pi] = np.arange(n)
    rows = []
    for i in range(nloc):
        v = inv[lo + i]
        rows.append(pi[col[offsets[v]:offsets[v + 1]]] if v >= 0 else np.zeros(0, np.int64))
    # column slice: for every global u, owned neighbours as local ids
    cols = [[] for _ in range(rl.npad)]
    for i, r in enumerate(rows):
        for u in r:
            cols[int(u)].append(i)
    return dict(rl=rl, nloc=nloc, lo=lo, rows=rows, cols=cols, pi=pi)


def bfs_rank(part, source, threshold, allgather):
    """One rank's traversal; `allgather(local_words) -> full_words`."""
    rl, nloc, lo = part["rl"], part["nloc"], part["lo"]
    npad = rl.npad
    spi = int(part["pi"][source])
    dist = np.full(nloc, UNREACHED, dtype=np.uint64)
    visited = np.zeros(nloc, dtype=bool)
    if lo <= spi < lo + nloc:
        dist[spi - lo] = 0
        visited[spi - lo] = True
    frontier = np.zeros(npad, dtype=bool)
    frontier[spi] = True
    n = len(part["pi"])
    td = 1.0 < threshold * n
    depth = 0
    phases = []
    while True:
        nxt = np.zeros(nloc, dtype=bool)
        if td:
            for u in np.nonzero(frontier)[0]:
                for i in part["cols"][u]:
                    if not visited[i]:
                        visited[i] = True
                        dist[i] = depth + 1
                        nxt[i] = True
        else:
            for i in range(nloc):
                if visited[i] or len(part["rows"][i]) == 0:
                    continue
                if frontier[part["rows"][i]].any():
                    visited[i] = True
                    dist[i] = depth + 1
                    nxt[i] = True
        phases.append(0 if td else 1)
        full = allgather(nxt)
        produced = int(full.sum())
        if produced == 0:
            break
        td = produced < threshold * n
        frontier = full
        depth += 1
    return dist, phases

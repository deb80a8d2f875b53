"""Hand-built graph factories mirroring the reference's test fixtures
(proj/tests/support/graphs.hpp:23-134), built through our public build_csr."""
import numpy as np

import paper_2503_00430_b200 as pb


def from_edges(edges, n, symmetrize=True):
    return pb.build_csr(np.array(edges, dtype=np.int64).reshape(-1, 2), n, symmetrize)


def make_path(n):  # graphs.hpp:29-33
    return from_edges([(i, i + 1) for i in range(n - 1)], n)


def make_star(leaves):  # graphs.hpp:36-40
    return from_edges([(0, i) for i in range(1, leaves + 1)], leaves + 1)


def make_complete_bipartite(a, b):  # graphs.hpp:43-49
    return from_edges([(i, a + j) for i in range(a) for j in range(b)], a + b)


def _clique_edges(first, count):
    return [(i, j) for i in range(first, first + count) for j in range(i + 1, first + count)]


def make_clique(n):  # graphs.hpp:60-64
    return from_edges(_clique_edges(0, n), n)


def make_lollipop(clique_n, tail_n):  # graphs.hpp:68-78
    edges = _clique_edges(0, clique_n)
    prev = 0
    for i in range(tail_n):
        v = clique_n + i
        edges.append((prev, v))
        prev = v
    return from_edges(edges, clique_n + tail_n)


def make_wide_tail_lollipop(clique_n, tail_pairs):  # graphs.hpp:83-100
    edges = _clique_edges(0, clique_n)
    pa, pb_ = 0, 1
    for k in range(tail_pairs):
        a = clique_n + 2 * k
        b = a + 1
        edges += [(pa, a), (pa, b), (pb_, a), (pb_, b)]
        pa, pb_ = a, b
    return from_edges(edges, clique_n + 2 * tail_pairs)


def make_circulant(n, offsets):  # graphs.hpp:105-116
    edges = [(i, (i + 1) % n) for i in range(n)]
    for d in offsets:
        count = n // 2 if 2 * d == n else n
        edges += [(i, (i + d) % n) for i in range(count)]
    return from_edges(edges, n)


def make_edgeless(n):  # graphs.hpp:118-120
    return from_edges(np.zeros((0, 2), dtype=np.int64), n)


def random_graph(n, edge_count, seed):
    """graphs.hpp:124-134 draw rule (mt19937_64, rng() % n per endpoint)."""
    import oracle
    raw = oracle.port().mt64(seed, 2 * edge_count)
    pairs = (raw % np.uint64(n)).astype(np.int64).reshape(-1, 2)
    return from_edges(pairs, n)


def hand_suite():
    """The 11 (graph, source) pairs of test_kernels.cpp:135-147."""
    return [
        ("path17", make_path(17), 0),
        ("path17-mid", make_path(17), 8),
        ("star16", make_star(16), 0),
        ("star16-leaf", make_star(16), 5),
        ("bipartite", make_complete_bipartite(5, 9), 0),
        ("clique8", make_clique(8), 3),
        ("lollipop", make_lollipop(8, 8), 15),
        ("wide-tail", make_wide_tail_lollipop(6, 5), 0),
        ("circulant", make_circulant(48, [2, 5]), 7),
        ("random96", random_graph(96, 400, 11), 1),
        ("two-components", from_edges([(0, 1), (2, 3), (3, 4)], 6), 0),
    ]

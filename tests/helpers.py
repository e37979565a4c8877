"""Shared fixtures-as-functions for the parity tests (test infrastructure)."""
import numpy as np

from oracle.bindings import csr_from_pairs

# T4: triangle 0-1-2 plus pendant 3 (generators.cpp:74-78)
T4_PAIRS = np.array([[0, 1], [0, 2], [1, 0], [1, 2], [2, 0], [2, 1], [2, 3], [3, 2]], dtype=np.uint32)


def undirected(n, edges, orc):
    """gbtest::make_graph (test_support.hpp:12-16) via the restated normalize."""
    e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
    nn, pairs = orc.normalize(e, n)
    return nn, pairs


def csr(n, pairs):
    return csr_from_pairs(n, np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))


def star(n_leaves):
    return [(0, v) for v in range(1, n_leaves + 1)]


def complete(n):
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def members(mask):
    return set(np.nonzero(np.asarray(mask))[0].tolist())


PR_PATHS = ["rows", "tiled"]


def pagerank_on(gbg, g, path, *args):
    """gbg.pagerank through one of the two device paths: "rows" (the
    one-shot path a fresh container uses) or "tiled" (the source-sorted
    index gbg_pagerank_prepare builds, used by every later call)."""
    if path == "tiled":
        gbg.pagerank_prepare(g)
    return gbg.pagerank(g, *args)

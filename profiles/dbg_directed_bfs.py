"""Debug helper: per-level trace of the device BFS against the reference on
a seeded directed graph with sinks (tests/test_gpu_edge_cases.py case)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import Ref, csr_from_pairs  # noqa: E402

rng = np.random.default_rng(0)
n, p = 300, 0.02
a = rng.random((n, n)) < p
np.fill_diagonal(a, False)
a[rng.random(n) < 0.3, :] = False
s, d = np.nonzero(a)
pairs = np.stack([s, d], 1).astype(np.uint32)
off, nbr = csr_from_pairs(n, pairs)
ref = Ref()
rg = ref.csr(n, off, nbr)
want = rg.bfs(0)
print("ref trace", rg.bfs_trace(0))
g = gbg.CsrGraph.build(n, pairs)
r = gbg.bfs(g, 0)
print("gpu modes", r.modes, "sizes", r.frontier_sizes)
bad = np.nonzero(r.depth != want)[0]
print("mismatch", bad.tolist()[:20], "gpu", r.depth[bad][:20].tolist(), "ref", want[bad][:20].tolist())
deg = np.diff(off.astype(np.int64))
print("deg of mismatched", deg[bad][:20].tolist())
indeg = np.bincount(nbr, minlength=n)
print("indeg of mismatched", indeg[bad][:20].tolist())

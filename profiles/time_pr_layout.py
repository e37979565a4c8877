"""PageRank layout build time (cached per graph) and the pipelined end-to-end
create + 20 iterations from pinned host CSR, at the given R-MAT scales."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

for S in [int(x) for x in (sys.argv[1:] or ["24"])]:
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    n, m = g.num_vertices(), g.num_edges()
    print(f"s{S}: layout build {gbg.pagerank_prepare(g):.2f} ms", flush=True)
    off, nbr = g.to_csr()
    off_h = torch.from_numpy(off.view(np.int64)).pin_memory().numpy().view(np.uint64)
    nbr_h = torch.from_numpy(nbr.view(np.int32)).pin_memory().numpy().view(np.uint32)
    ranks = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    del g
    for r in range(3):
        t0 = time.perf_counter()
        h = gbg.CsrGraph.from_csr(off_h, nbr_h, prepare_pagerank=True)
        t1 = time.perf_counter()
        gbg.pagerank(h, 0.85, 20, 1e-300, out=ranks)
        t2 = time.perf_counter()
        del h
        print(f"s{S}: e2e create {1e3 * (t1 - t0):.1f} ms + pagerank {1e3 * (t2 - t1):.1f} ms = {1e3 * (t2 - t0):.1f} ms",
              flush=True)

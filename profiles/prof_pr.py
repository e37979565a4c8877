"""PageRank at one scale for ncu: index build, then `iters` iterations
(default 3); capture the per-iteration kernel with -k regex:pr_tile_k -s 1 -c 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
gbg.pagerank_prepare(g)
out = torch.empty(g.num_vertices(), dtype=torch.float64, device="cuda")
gbg.pagerank_device(g, out.data_ptr(), 0.85, iters, 1e-300)
torch.cuda.synchronize()
print("ok", float(out.sum()))

"""PageRank (20 fp64 iterations, device-resident) at the given R-MAT scales,
CUDA events on the library stream, mean of 10 calls after 3 warm-ups."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

for S in [int(x) for x in (sys.argv[1:] or ["20", "24"])]:
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    n, m = g.num_vertices(), g.num_edges()
    gbg.pagerank_prepare(g)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.ExternalStream(g.stream())
    for _ in range(3):
        gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, 1e-300)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(10):
        gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, 1e-300)
    e1.record(s)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"s{S}: pagerank 20 iterations {t:.2f} ms = {20 * m / t / 1e6:.1f} GTEPS", flush=True)
    del g

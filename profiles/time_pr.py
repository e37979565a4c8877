"""PageRank (20 fp64 iterations, device-resident) at the given R-MAT scales,
CUDA events on the library stream, mean of 10 calls after 3 warm-ups; the
index build time, and (with --check) the full vector against the reference
library's gb::pagerank."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

check = "--check" in sys.argv
scales = [int(x) for x in sys.argv[1:] if not x.startswith("--")] or [20, 24]
for S in scales:
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    n, m = g.num_vertices(), g.num_edges()
    build = gbg.pagerank_prepare(g)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.ExternalStream(g.stream())
    for _ in range(3):
        gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, 1e-300)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for iters in (20, 1):
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(10):
            gbg.pagerank_device(g, out.data_ptr(), 0.85, iters, 1e-300)
        e1.record(s)
        e1.synchronize()
        res[iters] = e0.elapsed_time(e1) / 10
    t = res[20]
    it = (res[20] - res[1]) / 19
    bpr = 8 * (n + 1) + 4 * m + 16 * n
    print(f"s{S}: pagerank 20 iterations {t:.3f} ms = {20 * m / t / 1e6:.1f} GTEPS; per iteration {it:.4f} ms "
          f"({bpr / it / 1e6:.0f} GB/s model); index build {build:.1f} ms", flush=True)
    if check:
        from oracle.bindings import Ref

        ref = Ref()
        ref.set_threads(os.cpu_count() or 1)
        off, nbr = g.to_csr()
        t0 = time.time()
        want = ref.csr(n, off, nbr).pagerank(0.85, 20, np.finfo(np.float64).tiny)
        got = gbg.pagerank(g, 0.85, 20, np.finfo(np.float64).tiny)
        rel = np.abs(got - want).sum() / np.abs(want).sum()
        print(f"   parity vs gb::pagerank: rel L1 {rel:.3e}, max rel {np.max(np.abs(got - want) / want):.3e} "
              f"(ref {time.time() - t0:.1f} s)", flush=True)
    del g

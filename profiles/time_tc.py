"""Triangle counting at R-MAT s20 / s24 on the device (run on the GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

for S in [int(x) for x in (sys.argv[1:] or ["20", "24"])]:
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    gbg.triangle_count(g)
    t = time.perf_counter()
    tri = gbg.triangle_count(g)
    print(f"s{S} tc: {(time.perf_counter() - t) * 1e3:.2f} ms triangles={tri}", flush=True)

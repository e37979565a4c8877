"""Compressed container at R-MAT s24 (run on the GPU box): encode time,
bytes per arc, and BFS / CC on the compressed handle (which decode it into
a transient CSR per call) against the plain CSR handle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402


def wall(fn, reps=3):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return (time.perf_counter() - t) / reps * 1e3, out


for S in (20, 24):
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    m = g.num_edges()
    t_enc, z = wall(lambda: gbg.CompressedGraph.from_graph(g))
    zb, cb = z.memory_bytes(), g.memory_bytes()
    src = int(np.argmax(g.degrees()))
    t_bfs_c, _ = wall(lambda: gbg.bfs(g, src))
    t_bfs_z, _ = wall(lambda: gbg.bfs(z, src))
    t_cc_c, _ = wall(lambda: gbg.cc(g))
    t_cc_z, _ = wall(lambda: gbg.cc(z))
    print(f"s{S}: m={m} encode {t_enc:.2f} ms ({m / t_enc / 1e6:.2f} Garcs/s); "
          f"compressed {zb / m:.2f} B/arc vs CSR {cb / m:.2f} B/arc; "
          f"bfs csr {t_bfs_c:.2f} ms / compressed {t_bfs_z:.2f} ms; cc csr {t_cc_c:.2f} / compressed {t_cc_z:.2f} ms",
          flush=True)

"""Capacity check at R-MAT scale 26 (67M vertices, ~2.1G arcs) on one B200:
device generation, PageRank (20 fp64 iterations), BFS and CC timed."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
t = time.perf_counter()
g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
n, m = g.num_vertices(), g.num_edges()
print(f"s{S}: n={n} m={m} generated in {time.perf_counter() - t:.2f} s; device memory "
      f"{torch.cuda.mem_get_info()[1] / 2**30 - torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB used", flush=True)
ms = gbg.pagerank_prepare(g)
out = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.ExternalStream(g.stream())
gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, 1e-300)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, 1e-300)
e1.record(s)
e1.synchronize()
pr = e0.elapsed_time(e1)
print(f"s{S}: pagerank layout {ms:.1f} ms, 20 iterations {pr:.1f} ms = {20 * m / pr / 1e6:.1f} GTEPS, "
      f"sum={out.sum().item():.12f}", flush=True)
deg = g.degrees()
src = int(np.argmax(deg))
gbg.bfs(g, src)
t = time.perf_counter()
r = gbg.bfs(g, src)
print(f"s{S}: bfs {1e3 * (time.perf_counter() - t):.2f} ms (host API incl. depth copy), levels {r.modes}, "
      f"reached {r.reached}", flush=True)
t = time.perf_counter()
lab = gbg.cc(g)
print(f"s{S}: cc {1e3 * (time.perf_counter() - t):.2f} ms (host API), components {np.unique(lab).size}", flush=True)

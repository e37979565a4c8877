"""BFS at R-MAT s16 / s24 (device-resident depths), CUDA events; per-level
device times from the library's stats.  GBG_COOP=0 forces the
launch-per-level path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

for S in [int(x) for x in (sys.argv[1:] or ["16", "24"])]:
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    src = int(np.argmax(g.degrees()))
    depth = torch.empty(g.num_vertices(), dtype=torch.int32, device="cuda")
    s = torch.cuda.ExternalStream(g.stream())
    for _ in range(3):
        st = gbg.bfs_device(g, src, depth.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(10):
        st = gbg.bfs_device(g, src, depth.data_ptr())
    e1.record(s)
    e1.synchronize()
    ts = e0.elapsed_time(e1) / 10
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(10):
        gbg.bfs_device(g, src, depth.data_ptr(), stats=False)  # NULL stats: asynchronous
    e1.record(s)
    e1.synchronize()
    os.environ["GBG_BFS_LEVEL_TIMES"] = "1"  # one untimed, instrumented call
    st = gbg.bfs_device(g, src, depth.data_ptr())
    os.environ.pop("GBG_BFS_LEVEL_TIMES")
    print(f"s{S}: bfs {e0.elapsed_time(e1) / 10:.3f} ms (with stats {ts:.3f}) levels {st['modes']} level_ms "
          f"{[round(x, 4) for x in st['level_ms']]}", flush=True)

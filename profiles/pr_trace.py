"""Per-tile timing trace of pr_tile_k (analysis build with -DGBG_PR_TRACE):
one 1-iteration call on the prepared s24 index, then per CTA the tiles it
took (block, arcs, group phase, finalize phase).  Prints summaries by block
class.  Analysis only."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
lib = C.CDLL(os.path.join(os.path.dirname(gbg.__file__), "libgbg.so"))
g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
gbg.pagerank_prepare(g)
out = torch.empty(g.num_vertices(), dtype=torch.float64, device="cuda")
buf = np.zeros(148 * 64 * 6, dtype=np.uint64)
cnt = np.zeros(148, dtype=np.uint32)
for it in range(3):
    gbg.pagerank_device(g, out.data_ptr(), 0.85, 1, 1e-300)
    torch.cuda.synchronize()
    lib.gbg_debug_pr_trace(buf.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p))
tr = buf.reshape(148, 64, 6).astype(np.int64)
rows = []
for c in range(148):
    for k in range(min(64, cnt[c])):
        rows.append((c, *tr[c, k]))
a = np.array(rows)
t0 = a[:, 3].min()
blk, arcs, ts, tg, tf = a[:, 1], a[:, 2], a[:, 3] - t0, a[:, 4] - t0, a[:, 5] - t0
print(f"tiles traced {len(a)}; kernel span {tf.max() / 1e3:.1f} us; CTAs' last finish min {np.array([tf[a[:,0]==c].max() for c in range(148)]).min()/1e3:.1f} us")
grp = tg - ts
fin = tf - tg
print(f"group phase total {grp.sum()/1e3:.0f} us-CTA, finalize/flush phase {fin.sum()/1e3:.0f} us-CTA, gaps "
      f"{(148 * tf.max() - grp.sum() - fin.sum())/1e3:.0f} us-CTA")
for lo, hi in [(0, 1), (1, 4), (4, 16), (16, 64), (64, 256), (256, 1100)]:
    sel = (blk >= lo) & (blk < hi)
    if sel.sum() == 0:
        continue
    print(f"blocks [{lo},{hi}): tiles {sel.sum()}, arcs {arcs[sel].sum()/1e6:.1f}M, group {grp[sel].sum()/1e3:.0f} us-CTA "
          f"({arcs[sel].sum()/grp[sel].sum():.1f} arcs/ns/CTA), finalize {fin[sel].sum()/1e3:.0f} us-CTA "
          f"({fin[sel].mean()/1e3:.2f} us/tile)")

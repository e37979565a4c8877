"""Wall-clock timing of the host-API kcore / coloring / mis / ldd calls at R-MAT
s20 and s24 (run on the GPU box: python profiles/time_greedy.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np
import paper_2405_11671_b200.graph as gbg
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C
for S in (20, 24):
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    for name, fn in (("kcore", lambda: gbg.kcore(g)), ("coloring", lambda: gbg.coloring(g)), ("mis", lambda: gbg.mis(g, 1)),
                     ("ldd", lambda: gbg.ldd(g, 0.2, 1)[0])):
        fn()
        t = time.perf_counter(); o = fn(); dt = time.perf_counter() - t
        print(f"s{S} {name}: {dt*1e3:.1f} ms max={int(o.max())} sum={int(o.astype(np.int64).sum())}", flush=True)

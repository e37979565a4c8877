import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2405_11671_b200.graph as gbg
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C
for S in (24, 24, 22, 22):
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    print(f"s{S}: layout build {gbg.pagerank_prepare(g):.2f} ms", flush=True)
    del g

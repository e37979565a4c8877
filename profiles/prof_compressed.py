"""Decode one s24 compressed graph once (for an ncu capture of cz_decode_k)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

z = gbg.generate_rmat(24, 16 << 24, 1, RMAT_A, RMAT_B, RMAT_C, kind=gbg.KIND_COMPRESSED)
gbg.cc(z)
print("ok")

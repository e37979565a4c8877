"""Gather ceiling of the PageRank pull at R-MAT scale S (default 24).

Builds the degree-ordered arc sequence the pull gathers -- rows in (degree
desc, id asc) order, each list's sources renumbered to that order and sorted
-- and times (a) one 8-byte gather of a vertex-sized vector per arc with the
ids streamed (gather_k) and (b) a streaming read of the same bytes (stream_k),
CUDA events, mean of 10 launches after 2 warm-ups.  Prints one JSON line.
    python profiles/gather_ceiling.py [S]
"""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "_gather")
LIB = os.path.join(OUT, "libgather.so")
if not os.path.exists(LIB):
    os.makedirs(OUT, exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                    "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(ROOT, "profiles", "gather_ceiling.cu")], check=True)
lib = C.CDLL(LIB)
lib.gc_run.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_float)]

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
off_h, nbr_h = g.to_csr()
n, m = g.num_vertices(), g.num_edges()
del g
dev = "cuda"
off = torch.from_numpy(off_h.astype("int64")).to(dev)
nbr = torch.from_numpy(nbr_h.view("int32")).to(dev)
del off_h, nbr_h
deg = off[1:] - off[:-1]
key = (deg.max() - deg) * (n + 1) + torch.arange(n, device=dev)  # (degree desc, id asc)
ordr = torch.argsort(key)
del key
pos = torch.empty(n, dtype=torch.int64, device=dev)
pos[ordr] = torch.arange(n, device=dev)
deg_new = deg[ordr]
start_old = off[:-1][ordr]
off_new = torch.zeros(n + 1, dtype=torch.int64, device=dev)
off_new[1:] = torch.cumsum(deg_new, 0)
rows = torch.repeat_interleave(torch.arange(n, device=dev), deg_new)
idx = start_old[rows] + (torch.arange(m, device=dev) - off_new[rows])
del start_old
src = pos[nbr[idx].long()]
del idx, nbr
k = rows * (n + 1) + src  # sort each row's sources ascending
del rows
k, _ = torch.sort(k)
ids = (k % (n + 1)).to(torch.int32).contiguous()
del k, src
nz = int((deg > 0).sum())
T = torch.randint(0, 1 << 40, (max(n, m),), dtype=torch.int64, device=dev)  # >= m words for the stream kernel
out = torch.zeros(1, dtype=torch.int64, device=dev)
torch.cuda.synchronize()
res = {"scale": S, "n": n, "m": m, "rows_with_edges": nz}
for kind, name in ((0, "gather"), (1, "stream")):
    ms = C.c_float()
    rc = lib.gc_run(kind, ids.data_ptr(), m, T.data_ptr(), out.data_ptr(), 10, C.byref(ms))
    assert rc == 0, rc
    b = 12 * m
    res[name] = {"ms": ms.value, "arcs_per_s": m / ms.value * 1e3, "bytes": b, "GBps": b / ms.value / 1e6}
# the pull's §8(d) model bytes per iteration, and what the gather ceiling implies for it
bpr = 8 * (n + 1) + 4 * m + 16 * n
res["B_PR"] = bpr
res["B_PR_GBps_at_gather_ceiling"] = bpr / res["gather"]["ms"] / 1e6
print(json.dumps(res), flush=True)

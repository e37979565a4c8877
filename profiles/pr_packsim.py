"""Simulation of bank-packed rounds for the PageRank tiled index (analysis
only): for a few row blocks of the scale-24 index, runs (arcs of one source
in one block, in source order) are packed first-fit into rounds of 32 slots
whose rows fall in distinct shared-memory banks (row & 31), with W rounds
open at a time; runs of 32+ arcs fill whole rounds in (rank-in-bank, bank)
order and pack their remainder like a short run.  Reports slot fill, bank
conflict degree per round, and gathers (distinct runs) per round, against
the plain source-sorted rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
W = int(sys.argv[2]) if len(sys.argv) > 2 else 16
RB = 13
g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
off, nbr = g.to_csr()
n = g.num_vertices()
del g
dev = "cuda"
off = torch.from_numpy(off.astype("int64")).to(dev)
nbr = torch.from_numpy(nbr.astype("int64")).to(dev)
deg = off[1:] - off[:-1]
ordr = torch.argsort((-deg) * (1 << 30) + torch.arange(n, device=dev))
pos = torch.empty_like(ordr)
pos[ordr] = torch.arange(n, device=dev)
rowv = torch.repeat_interleave(torch.arange(n, device=dev), deg)
row = pos[rowv]
src = pos[nbr]
del rowv, nbr
k = ((row >> RB) << (RB + 25)) | (src << RB) | (row & ((1 << RB) - 1))
k, _ = torch.sort(k)
blk_all = (k >> (RB + 25)).cpu().numpy()
src_all = ((k >> RB) & ((1 << 25) - 1)).cpu().numpy()
rib_all = (k & ((1 << RB) - 1)).cpu().numpy()
bstart = np.searchsorted(blk_all, np.arange(blk_all[-1] + 2))


def plain_stats(rib, srcs):
    R = len(rib) // 32
    b = (rib[: R * 32] & 31).reshape(R, 32)
    conf = np.array([np.bincount(x, minlength=32).max() for x in b])
    s = srcs[: R * 32].reshape(R, 32)
    dist = 1 + (s[:, 1:] != s[:, :-1]).sum(1)
    return conf.mean(), dist.mean(), 1.0


def packed_stats(rib, srcs):
    # runs
    starts = np.flatnonzero(np.r_[True, srcs[1:] != srcs[:-1]])
    ends = np.r_[starts[1:], len(srcs)]
    rounds = []  # list of (rows list, run count)
    open_r = []  # [mask, rows, nruns]
    for a, e in zip(starts, ends):
        rows = rib[a:e]
        if len(rows) >= 32:
            bank = rows & 31
            order = np.lexsort((bank, np.argsort(np.argsort(bank, kind="stable"), kind="stable")))
            # rank within bank
            rk = np.zeros(len(rows), dtype=np.int64)
            for bb in range(32):
                idx = np.flatnonzero(bank == bb)
                rk[idx] = np.arange(len(idx))
            order = np.lexsort((bank, rk))
            rows = rows[order]
            full = len(rows) // 32 * 32
            for i in range(0, full, 32):
                rounds.append((rows[i:i + 32], 1))
            rows = rows[full:]
            if len(rows) == 0:
                continue
        m = 0
        for r in rows:
            m |= 1 << int(r & 31)
        placed = False
        for o in open_r:
            if (o[0] & m) == 0 and len(o[1]) + len(rows) <= 32:
                o[0] |= m
                o[1].extend(rows.tolist())
                o[2] += 1
                placed = True
                if len(o[1]) == 32:
                    rounds.append((np.array(o[1]), o[2]))
                    open_r.remove(o)
                break
        if not placed:
            if len(open_r) >= W:
                o = max(open_r, key=lambda x: len(x[1]))
                rounds.append((np.array(o[1]), o[2]))
                open_r.remove(o)
            open_r.append([m, rows.tolist(), 1])
    for o in open_r:
        rounds.append((np.array(o[1]), o[2]))
    conf = np.array([np.bincount(np.asarray(r) & 31, minlength=32).max() for r, _ in rounds])
    fill = np.mean([len(r) for r, _ in rounds]) / 32
    return conf.mean(), np.mean([c for _, c in rounds]), fill


for b in [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else "0,5,20,60,200,600".split(","))]:
    a, e = bstart[b], bstart[b + 1]
    mid = (a + e) // 2
    a, e = max(a, mid - 300000), min(e, mid + 300000)  # a 600K-arc slice from the middle of the block
    rib, srcs = rib_all[a:e], src_all[a:e]
    c0, d0, _ = plain_stats(rib, srcs)
    c1, d1, f1 = packed_stats(rib, srcs)
    print(f"block {b}: arcs {e - a}: plain conflict {c0:.2f} runs/round {d0:.2f} | packed(W={W}) conflict {c1:.2f} "
          f"runs/round {d1:.2f} fill {f1:.3f}", flush=True)

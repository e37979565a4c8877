"""Run / bank statistics of the PageRank tiled index at a given R-MAT scale
(GPU, torch): rows with edges renumbered by (degree desc, id asc), blocks of
8192 rows, each block's arcs sorted by (source, row).  Reports the run-length
distribution (arc-weighted), distinct runs per 32-arc round, and the shared-
memory bank-conflict degree of the row-sum atomics per round under several
within-run row orders.  Analysis only (no product code)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402
from oracle.bindings import RMAT_A, RMAT_B, RMAT_C  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
RB = 13
g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
off, nbr = g.to_csr()
n = g.num_vertices()
del g
dev = "cuda"
off = torch.from_numpy(off.astype("int64")).to(dev)
nbr = torch.from_numpy(nbr.astype("int64")).to(dev)
deg = off[1:] - off[:-1]
key = (-deg) * (1 << 30) + torch.arange(n, device=dev)
ordr = torch.argsort(key)
pos = torch.empty_like(ordr)
pos[ordr] = torch.arange(n, device=dev)
m = nbr.numel()
rowv = torch.repeat_interleave(torch.arange(n, device=dev), deg)  # row vertex of each arc
row = pos[rowv]
src = pos[nbr]
del rowv, nbr
blk = row >> RB
rib = row & ((1 << RB) - 1)
k = (blk << (RB + 25)) | (src << RB) | rib
k, _ = torch.sort(k)
blk = k >> (RB + 25)
src = (k >> RB) & ((1 << 25) - 1)
rib = k & ((1 << RB) - 1)
del k
bs = (blk << 25) | src
start = torch.ones(m, dtype=torch.bool, device=dev)
start[1:] = bs[1:] != bs[:-1]
rid = torch.cumsum(start.to(torch.int64), 0) - 1
nruns = int(rid[-1]) + 1
rlen = torch.bincount(rid, minlength=nruns)
print(f"s{S}: m={m} runs={nruns} runs/arc={nruns / m:.3f} blocks={int(blk[-1]) + 1}")
edges = [1, 2, 4, 8, 16, 32, 64, 256, 1024, 1 << 30]
alen = rlen[rid]
for lo, hi in zip(edges[:-1], edges[1:]):
    sel = (alen >= lo) & (alen < hi)
    print(f"  runs of length [{lo},{hi}): arcs {sel.float().mean().item():.3f}, runs "
          f"{((rlen >= lo) & (rlen < hi)).float().sum().item() / nruns:.3f}")
# rounds: 32 consecutive arcs in block order (groups restart at block starts in the real index; ignored here)
R = m // 32
rr = rid[: R * 32].view(R, 32)
dist = 1 + (rr[:, 1:] != rr[:, :-1]).sum(1)
print(f"  distinct runs per round: mean {dist.float().mean().item():.2f}")


rblk = blk[: R * 32].view(R, 32)[:, 0]


def conflicts(rows):
    b = (rows[: R * 32] & 31).view(R, 32)
    oh = torch.zeros(R, 32, dtype=torch.int32, device=dev)
    oh.scatter_add_(1, b, torch.ones_like(b, dtype=torch.int32))
    mx = oh.max(1).values.float()
    parts = []
    for lo, hi in [(0, 16), (16, 64), (64, 256), (256, 1 << 20)]:
        sel = (rblk >= lo) & (rblk < hi)
        parts.append(f"[{lo},{hi}) {mx[sel].mean().item():.2f}")
    return f"{mx.mean().item():.2f} (" + ", ".join(parts) + ")"


print(f"  bank conflict degree per round (rows ascending in a run): {conflicts(rib)}")
# interleaved order inside each run: sort by (run, rank within (run, bank), bank)
bank = rib & 31
kb = (rid << 18) | (bank << 13) | rib
kb, perm = torch.sort(kb)
rb_run = kb >> 18
rb_bank = (kb >> 13) & 31
seg = torch.ones(m, dtype=torch.bool, device=dev)
seg[1:] = (rb_run[1:] != rb_run[:-1]) | (rb_bank[1:] != rb_bank[:-1])
idx = torch.arange(m, device=dev)
segstart = torch.cummax(torch.where(seg, idx, torch.zeros_like(idx)), 0).values
rank = idx - segstart
k2 = (rb_run << 18) | (rank.clamp(max=8191) << 5) | rb_bank
k2, p2 = torch.sort(k2)
rib2 = (kb & 8191)[p2]
print(f"  bank conflict degree per round (interleaved banks in a run): {conflicts(rib2)}")
rand = torch.randint(0, 8192, (m,), device=dev)
print(f"  bank conflict degree per round (random rows): {conflicts(rand)}")

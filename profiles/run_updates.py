"""Minimal driver for profiling the batch-update path alone (configs[4]):
s22 blocked container, one device-resident 10^7-edge batch (base-disjoint),
`--reps` timed insert+delete pairs.  Used under ncu by profiles/capture.sh."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_11671_b200.graph as gbg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--size", type=int, default=10**7)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
RMAT = (0.57, 0.19, 0.19)
g = gbg.generate_rmat(a.scale, 16 << a.scale, 1, *RMAT, kind=gbg.KIND_BLOCKED)
buf = torch.empty(4 * a.size, dtype=torch.int32, device="cuda")
# the reference's batch seed (bench.cpp:161); small literal seeds replay a
# shifted window of the base graph's own draws (counter-based RNG)
from bench import _hash_combine  # noqa: E402

gbg.generate_update_batch_device(a.scale, a.size, _hash_combine(_hash_combine(2, a.size), 0), buf.data_ptr(), *RMAT)
present = torch.empty(2 * a.size, dtype=torch.uint8, device="cuda")
g.contains_device(buf.data_ptr(), 2 * a.size, present.data_ptr())
dev = buf.view(-1, 2)[present == 0].contiguous()
print(f"graph m={g.num_edges()} raw arcs={2 * a.size} present={int(present.sum())} fresh={dev.shape[0]}")
s = torch.cuda.ExternalStream(g.stream())
for r in range(a.reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record(s)
    ins = g.insert_batch_device(dev.data_ptr(), dev.shape[0])
    e1.record(s)
    dele = g.delete_batch_device(dev.data_ptr(), dev.shape[0])
    e2.record(s)
    e2.synchronize()
    print(f"rep {r}: insert {e0.elapsed_time(e1):.3f} ms ({ins} arcs), delete {e1.elapsed_time(e2):.3f} ms ({dele})")

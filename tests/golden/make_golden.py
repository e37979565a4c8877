"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference library (oracle/_ref/libgbref.so, built from /root/reference by
`make -C oracle ref`) on the BASELINE.json configs.  Run here, in the
container that has /root/reference; the GPU box only reads the JSON output.

    python tests/golden/make_golden.py 16 20          # seconds
    python tests/golden/make_golden.py 22 24          # ~15 min (s24 gen ~400 s)

Per scale S (R-MAT a=.57 b=c=.19, arcs = 16*2^S, seed 1):
  graph      n, m, digest(offsets u64[n+1]), digest(neighbors u32[m])
  bfs        source = lowest-id max-degree vertex; digest(int32 depth),
             reached, max depth, per-level (mode, |F|) trace of gb::edge_map
  pagerank   gb::pagerank(0.85, 20, DBL_MIN) -> sum, and exact values (hex)
             at 1024 fixed sample ids
  cc         digest(uint32 labels), component count
  tc         triangle count from the C restatement (the reference has none)
At S=22 also the config-5 update sequence on the reference "chunked_set"
container (see `updates()`).

    python tests/golden/make_golden.py --greedy 16 20 24
    python tests/golden/make_golden.py --updates 22   # config 5, reps 0..2

adds (in place) the priority-order consumers of §8(f) row 3:
  kcore      digest(uint64 coreness), max coreness
  coloring   digest(uint32 colours), colour count
  mis        seed 1 (AlgoParams default): digest(uint8 flags), set size
  ldd        beta 0.2, seed 1 (AlgoParams defaults): digests of labels,
             parents, rounds; cluster count, last round
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.bindings import Oracle, Ref, csr_from_pairs, digest, max_degree_source  # noqa: E402

CACHE = os.environ.get("GB_GRAPH_CACHE", "/tmp/gbcache")
UPDATE_SIZES = [10**4, 10**5, 10**6, 10**7]


def sample_ids(n, k=1024):
    """Fixed PageRank sample positions: the first 256 ids plus an even spread."""
    head = np.arange(min(256, n), dtype=np.int64)
    spread = np.linspace(0, n - 1, k - head.size).astype(np.int64)
    return np.unique(np.concatenate([head, spread]))


def graph(ref, S):
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"rmat{S}.npz")
    if os.path.exists(path):
        z = np.load(path)
        return int(z["n"]), z["off"], z["nbr"]
    t = time.time()
    n, pairs = ref.rmat(S, 16 << S, 1)
    print(f"s{S}: generated n={n} m={len(pairs)} in {time.time() - t:.1f}s", flush=True)
    off, nbr = csr_from_pairs(n, pairs)
    del pairs
    np.savez(path, n=n, off=off, nbr=nbr)
    return n, off, nbr


def update_seed(ref, size, rep):
    """hash_combine(hash_combine(seed=2, size), rep), mirroring bench.cpp:161."""
    return ref.hash_combine(ref.hash_combine(2, size), rep)


def updates(ref, n, off, nbr, S, reps=3):
    """Config 5 on the reference dynamic container ("chunked_set",
    registry.cpp:136-137), in run_updates' order (bench.cpp:158-187): per
    size and rep 0..2 sample a batch with seed hash_combine(hash_combine(2,
    size), rep), drop arcs already in the base (bench.cpp:150-169 policy,
    untimed), insert (prepare + apply_insert), BFS from the lowest-id
    max-degree vertex, delete."""
    src_of = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off.astype(np.int64)))
    base_keys = (src_of << np.uint64(32)) | nbr.astype(np.uint64)
    del src_of
    pairs = np.stack([np.repeat(np.arange(n, dtype=np.uint32), np.diff(off.astype(np.int64))), nbr], axis=1)
    t = time.time()
    cont = ref.chunked(n, pairs)
    del pairs
    print(f"s{S}: chunked_set built in {time.time() - t:.1f}s", flush=True)
    out = []
    for size, rep in [(size, rep) for size in UPDATE_SIZES for rep in range(reps)]:
        seed = update_seed(ref, size, rep)
        raw = ref.update_batch(S, size, seed)
        keys = (raw[:, 0].astype(np.uint64) << np.uint64(32)) | raw[:, 1].astype(np.uint64)
        keep = ~np.isin(keys, base_keys)
        fresh = np.ascontiguousarray(raw[keep])
        t = time.time()
        ins = cont.apply(fresh, True)
        m_ins = cont.m
        eo, en = cont.export()
        src = max_degree_source(eo)
        depth = cont.bfs(src)
        dele = cont.apply(fresh, False)
        rec = dict(size=size, rep=rep, seed=seed, raw_digest=digest(raw.reshape(-1)), fresh=int(fresh.shape[0]),
                   fresh_digest=digest(fresh.reshape(-1)), inserted=ins, m_after_insert=m_ins,
                   off_digest_after_insert=digest(eo), nbr_digest_after_insert=digest(en), bfs_source=src,
                   bfs_digest=digest(depth), bfs_reached=int((depth >= 0).sum()), deleted=dele,
                   m_after_delete=cont.m)
        print(f"s{S}: update {size}: {rec} ({time.time() - t:.1f}s)", flush=True)
        out.append(rec)
    return out


def main(scales):
    ref, orc = Ref(), Oracle()
    for S in scales:
        n, off, nbr = graph(ref, S)
        rec = dict(scale=S, seed=1, a=0.57, b=0.19, c=0.19, arcs=16 << S, n=n, m=int(off[n]),
                   off_digest=digest(off), nbr_digest=digest(nbr))
        deg = np.diff(off.astype(np.int64))
        rec["isolated"] = int((deg == 0).sum())
        rec["max_degree"] = int(deg.max())
        src = max_degree_source(off)
        g = ref.csr(n, off, nbr)
        t = time.time()
        depth = g.bfs(src)
        modes, sizes = g.bfs_trace(src)
        rec["bfs"] = dict(source=src, digest=digest(depth), reached=int((depth >= 0).sum()),
                          max_depth=int(depth.max()), modes=modes, frontier_sizes=sizes,
                          graph500_edges=int(deg[depth >= 0].sum() // 2))
        print(f"s{S}: bfs {time.time() - t:.1f}s {rec['bfs']}", flush=True)
        t = time.time()
        pr = g.pagerank(0.85, 20, np.finfo(np.float64).tiny)
        ids = sample_ids(n)
        rec["pagerank"] = dict(damping=0.85, iters=20, sum=float(pr.sum()), sample_ids=ids.tolist(),
                               sample_hex=[float(x).hex() for x in pr[ids]])
        print(f"s{S}: pagerank {time.time() - t:.1f}s sum={pr.sum()!r} p0={pr[0]!r}", flush=True)
        del pr
        t = time.time()
        lab = g.cc()
        rec["cc"] = dict(digest=digest(lab), components=int(np.unique(lab).size))
        print(f"s{S}: cc {time.time() - t:.1f}s {rec['cc']}", flush=True)
        del lab, g
        if S <= 24 and S != 22:
            t = time.time()
            rec["tc"] = dict(triangles=orc.tc(n, off, nbr), source="oracle/gbo.c restatement")
            print(f"s{S}: tc {time.time() - t:.1f}s {rec['tc']}", flush=True)
        if S == 22:
            rec["updates"] = updates(ref, n, off, nbr, S)
        with open(os.path.join(HERE, f"rmat_s{S}.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(f"s{S}: written", flush=True)


def greedy(scales):
    ref = Ref()
    for S in scales:
        n, off, nbr = graph(ref, S)
        path = os.path.join(HERE, f"rmat_s{S}.json")
        with open(path) as f:
            rec = json.load(f)
        g = ref.csr(n, off, nbr)
        t = time.time()
        core = g.kcore()
        rec["kcore"] = dict(digest=digest(core), max_core=int(core.max()))
        print(f"s{S}: kcore {time.time() - t:.1f}s {rec['kcore']}", flush=True)
        t = time.time()
        col = g.coloring()
        rec["coloring"] = dict(digest=digest(col), colors=int(col.max()) + 1)
        print(f"s{S}: coloring {time.time() - t:.1f}s {rec['coloring']}", flush=True)
        t = time.time()
        flags = g.mis(1)
        rec["mis"] = dict(seed=1, digest=digest(flags), size=int(flags.sum()))
        print(f"s{S}: mis {time.time() - t:.1f}s {rec['mis']}", flush=True)
        t = time.time()
        lab, par, rnd = g.ldd(0.2, 1)
        rec["ldd"] = dict(beta=0.2, seed=1, labels_digest=digest(lab), parents_digest=digest(par),
                          rounds_digest=digest(rnd), clusters=int((lab == np.arange(n)).sum()),
                          last_round=int(rnd.max()))
        print(f"s{S}: ldd {time.time() - t:.1f}s {rec['ldd']}", flush=True)
        with open(path, "w") as f:
            json.dump(rec, f, indent=1)


def refresh_updates(S=22):
    """Recompute only the config-5 update sequence of rmat_s{S}.json."""
    ref = Ref()
    n, off, nbr = graph(ref, S)
    path = os.path.join(HERE, f"rmat_s{S}.json")
    with open(path) as f:
        rec = json.load(f)
    assert rec["m"] == int(off[n])
    rec["updates"] = updates(ref, n, off, nbr, S)
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--updates"]:
        refresh_updates(int(sys.argv[2]) if len(sys.argv) > 2 else 22)
    elif sys.argv[1:2] == ["--greedy"]:
        greedy([int(x) for x in sys.argv[2:]])
    else:
        main([int(x) for x in sys.argv[1:]] or [16, 20])

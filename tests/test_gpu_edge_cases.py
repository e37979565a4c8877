"""GPU edge cases the reference tests or its contract imply: empty and
singleton graphs, very deep BFS (more levels than the stats window), hub
rows far above every load-balancing threshold, disconnected pieces, and
degenerate update batches.  Everything is compared with the C oracle."""
import numpy as np
import pytest

from tests.helpers import PR_PATHS, csr, pagerank_on, undirected

pytestmark = pytest.mark.gpu
TINY = np.finfo(np.float64).tiny


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / max(np.abs(b).sum(), 1e-300))


@pytest.mark.parametrize("path", PR_PATHS)
@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_empty_and_singleton_graphs(gbg, kind, path):
    mk = gbg.CsrGraph.build if kind == "csr" else gbg.BlockedGraph.build
    g0 = mk(0, [])
    assert g0.num_vertices() == 0 and g0.num_edges() == 0
    assert pagerank_on(gbg, g0, path).size == 0 and gbg.cc(g0).size == 0
    with pytest.raises(IndexError):
        gbg.bfs(g0, 0)
    g1 = mk(1, [])
    assert gbg.bfs(g1, 0).depth.tolist() == [0]
    assert gbg.cc(g1).tolist() == [0]
    assert np.allclose(pagerank_on(gbg, g1, path, 0.85, 20, TINY), [1.0])
    assert gbg.triangle_count(g1) == 0


@pytest.mark.parametrize("path", PR_PATHS)
@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_deep_path_bfs(gbg, orc, kind, path):
    """A 3000-vertex path: 2999 levels, far beyond GBG_MAX_LEVELS."""
    n = 3000
    nn, pairs = undirected(n, [(i, i + 1) for i in range(n - 1)], orc)
    off, nbr = csr(nn, pairs)
    g = gbg.CsrGraph.build(nn, pairs) if kind == "csr" else gbg.BlockedGraph.build(nn, pairs)
    for src in (0, 1234, n - 1):
        r = gbg.bfs(g, src)
        want, modes, sizes = orc.bfs(nn, off, nbr, src)
        assert np.array_equal(r.depth, want)
        assert r.reached == n
        k = min(len(modes), 64)
        assert r.modes[:k] == modes[:k] and r.frontier_sizes[:k] == sizes[:k]
    assert gbg.cc(g).tolist() == [0] * n
    assert rel_l1(pagerank_on(gbg, g, path, 0.85, 20, TINY), orc.pagerank(nn, off, nbr, 0.85, 20, TINY)) <= 1e-9


@pytest.mark.parametrize("path", PR_PATHS)
def test_huge_star_and_disconnected_pieces(gbg, orc, path):
    """One hub of 200k leaves (far above every split threshold) plus a
    triangle and isolated vertices."""
    leaves = 200_000
    edges = [(0, v) for v in range(1, leaves + 1)] + [(leaves + 1, leaves + 2), (leaves + 2, leaves + 3),
                                                        (leaves + 1, leaves + 3)]
    n = leaves + 10
    nn, pairs = undirected(n, edges, orc)
    off, nbr = csr(nn, pairs)
    g = gbg.CsrGraph.build(nn, pairs)
    for src in (0, 5, leaves + 2, leaves + 7):
        assert np.array_equal(gbg.bfs(g, src).depth, orc.bfs(nn, off, nbr, src)[0])
    assert np.array_equal(gbg.cc(g), orc.cc(nn, off, nbr))
    assert gbg.triangle_count(g) == 1
    assert rel_l1(pagerank_on(gbg, g, path, 0.85, 20, TINY), orc.pagerank(nn, off, nbr, 0.85, 20, TINY)) <= 1e-9
    # early convergence: the tolerance break (algorithms.cpp:552)
    for tol in (1e-3, 1e-6):
        assert rel_l1(pagerank_on(gbg, g, path, 0.85, 100, tol), orc.pagerank(nn, off, nbr, 0.85, 100, tol)) <= 1e-9


@pytest.mark.parametrize("path", PR_PATHS)
def test_complete_graph(gbg, orc, path):
    k = 300
    nn, pairs = undirected(k, [(i, j) for i in range(k) for j in range(i + 1, k)], orc)
    g = gbg.CsrGraph.build(nn, pairs)
    d = gbg.bfs(g, 7).depth
    assert d[7] == 0 and set(d.tolist()) == {0, 1}
    assert np.allclose(pagerank_on(gbg, g, path, 0.85, 20, TINY), 1.0 / k, rtol=1e-12, atol=0)
    assert gbg.triangle_count(g) == k * (k - 1) * (k - 2) // 6


def test_degenerate_batches(gbg, orc):
    edges = [(i, (i * 7 + 3) % 64) for i in range(64)]
    n, pairs = undirected(64, edges, orc)
    g = gbg.BlockedGraph.build(n, pairs)
    off, nbr = csr(n, pairs)

    def expect(batch, insert):
        nonlocal off, nbr
        k, off, nbr = orc.set_apply(n, off, nbr, orc.prepare_global(batch), insert)
        return k

    assert g.insert_batch(np.zeros((0, 2), np.uint32)) == 0
    assert g.insert_batch([[5, 5], [9, 9]]) == 0  # only self-loops (batch.cpp:36)
    assert g.insert_batch(pairs) == 0              # all present
    b = [[1, 2], [1, 2], [1, 2]]                  # duplicates of one arc
    assert g.delete_batch(b) == expect(b, False)
    dup = np.array([[10, 20]] * 1000 + [[20, 10]] * 1000, np.uint32)
    ins = g.insert_batch(dup)
    assert ins == expect(dup, True) and g.num_edges() == int(off[n])
    assert g.delete_batch(dup) == expect(dup, False) == ins
    with pytest.raises(IndexError):
        g.insert_batch([[0, 64]])
    assert g.num_edges() == int(off[n])
    # delete everything, then insert everything back
    off, nbr = g.to_csr()
    allp = np.stack([np.repeat(np.arange(n, dtype=np.uint32), np.diff(off.astype(np.int64))), nbr], axis=1)
    assert g.delete_batch(allp) == allp.shape[0] and g.num_edges() == 0
    assert g.insert_batch(allp) == allp.shape[0]
    o2, n2 = g.to_csr()
    assert np.array_equal(o2, off) and np.array_equal(n2, nbr)


def test_pool_growth_and_relayout(gbg, orc):
    """Insert far more arcs than the initial pool holds (forces grown lists
    and a relayout into a larger pool), then delete them again."""
    n = 5000
    g = gbg.BlockedGraph.build(n, [])
    rng = np.random.default_rng(3)
    off, nbr = csr(n, np.zeros((0, 2), np.uint32))
    for step in range(6):
        raw = rng.integers(0, n, size=(200_000, 2)).astype(np.uint32)
        raw[: 50_000, 0] = step  # a few fast-growing hubs
        want, off, nbr = orc.set_apply(n, off, nbr, orc.prepare_global(raw), True)
        assert g.insert_batch(raw) == want
    go, gn = g.to_csr()
    assert np.array_equal(go, off) and np.array_equal(gn, nbr)
    assert np.array_equal(gbg.bfs(g, 0).depth, orc.bfs(n, off, nbr, 0)[0])
    assert g.memory_bytes() > 0


def test_pipelined_create_with_pagerank_layout(gbg, ref, orc):
    """gbg_csr_create_ex: chunked upload + validation, optional PageRank
    layout built during the upload — same ranks, same rejections."""
    n, pairs = ref.rmat(14, 16 << 14, 1)
    off, nbr = csr(n, pairs)
    a = gbg.CsrGraph.from_csr(off, nbr, prepare_pagerank=True)
    b = gbg.CsrGraph.from_csr(off, nbr)
    pa = gbg.pagerank(a, 0.85, 20, 1e-300)
    pb = gbg.pagerank(b, 0.85, 20, 1e-300)
    assert np.array_equal(pa, pb)
    want = orc.pagerank(n, off, nbr, 0.85, 20, 1e-300)
    assert np.abs(pa - want).sum() / np.abs(want).sum() <= 1e-9
    bad = nbr.copy()
    bad[5] = n + 3  # out of range: rejected, no crash in the layout relabel
    with pytest.raises(gbg.FormatError):
        gbg.CsrGraph.from_csr(off, bad, prepare_pagerank=True)
    bad = nbr.copy()
    bad[[10, 11]] = bad[[11, 10]]  # unsorted segment
    with pytest.raises(gbg.FormatError):
        gbg.CsrGraph.from_csr(off, bad, prepare_pagerank=True)
    boff = off.copy()
    boff[3] = boff[4] + 1
    with pytest.raises(gbg.FormatError):
        gbg.CsrGraph.from_csr(boff, nbr, prepare_pagerank=True)


def test_launch_per_step_paths_match_oracle(gbg, orc, tmp_path):
    """The launch-per-step host loops (used when cooperative launch is
    unavailable; forced here with GBG_COOP=0 in a fresh process) of BFS,
    k-core and coloring give the oracle's outputs and BFS direction trace."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, json; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2405_11671_b200.graph as gbg\n"
        "from oracle.bindings import RMAT_A, RMAT_B, RMAT_C\n"
        "g = gbg.generate_rmat(13, 16 << 13, 1, RMAT_A, RMAT_B, RMAT_C)\n"
        "b = gbg.BlockedGraph.from_csr_graph(g)\n"
        "out = {}\n"
        "for name, h in (('csr', g), ('blocked', b)):\n"
        "    r = gbg.bfs(h, 0)\n"
        "    out[name] = [r.depth.tolist(), r.modes, gbg.kcore(h).tolist(), gbg.coloring(h).tolist()]\n"
        "print(json.dumps(out))\n" % root)
    env = dict(os.environ, GBG_COOP="0")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    n, pairs = orc.rmat(13, 16 << 13, 1)
    off, nbr = csr(n, pairs)
    d, modes, _ = orc.bfs(n, off, nbr, 0)
    core, col = orc.kcore(n, off, nbr), orc.coloring(n, off, nbr)
    for name in ("csr", "blocked"):
        assert np.array_equal(np.array(got[name][0], dtype=np.int32), d), name
        assert got[name][1] == modes, name
        assert np.array_equal(np.array(got[name][2], dtype=np.uint64), core), name
        assert np.array_equal(np.array(got[name][3], dtype=np.uint32), col), name


def test_bfs_list_built_transitions_match_oracle(gbg, orc):
    """GBG_BFS_BITMAP_PUSH=0 (fresh process): the persistent BFS builds the id
    list at every dense -> sparse transition instead of pushing from the
    bitmap; depths, direction trace and examined arcs still match the
    oracle (R-MAT scale 16 and the bitmap-push transition graph)."""
    import json
    import os
    import subprocess
    import sys

    from tests.test_gpu_parity import transition_graph

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n0, edges = transition_graph(1000)
    tn, tpairs = undirected(n0, edges, orc)
    code = (
        "import sys, json; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2405_11671_b200.graph as gbg\n"
        "from oracle.bindings import RMAT_A, RMAT_B, RMAT_C\n"
        "g = gbg.generate_rmat(16, 16 << 16, 1, RMAT_A, RMAT_B, RMAT_C)\n"
        "t = gbg.CsrGraph.build(%d, np.array(json.loads(sys.stdin.read()), dtype=np.uint32))\n"
        "out = {}\n"
        "for name, h in (('rmat', g), ('transition', t)):\n"
        "    r = gbg.bfs(h, 0)\n"
        "    out[name] = [r.depth.tolist(), r.modes, r.examined]\n"
        "print(json.dumps(out))\n" % (root, tn))
    env = dict(os.environ, GBG_BFS_BITMAP_PUSH="0")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                         input=json.dumps(np.asarray(tpairs).tolist()))
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    n, pairs = orc.rmat(16, 16 << 16, 1)
    for name, (nn, pp) in (("rmat", (n, pairs)), ("transition", (tn, tpairs))):
        off, nbr = csr(nn, pp)
        d, modes, _ = orc.bfs(nn, off, nbr, 0)
        assert np.array_equal(np.array(got[name][0], dtype=np.int32), d), name
        assert got[name][1] == modes, name
        assert got[name][2] == orc.bfs_examined(nn, off, nbr, 0), name


def test_concurrent_reads_from_threads(gbg, orc):
    """graph_container.hpp:33-35: read operations are safe from many threads.
    Several host threads run BFS / CC / degree queries on one handle (calls
    are serialised per handle) and on their own handles at once."""
    import threading

    n, pairs = orc.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    want_d = orc.bfs(n, off, nbr, 0)[0]
    want_cc = orc.cc(n, off, nbr)
    shared = gbg.CsrGraph.build(n, pairs)
    errors = []

    def worker(k):
        try:
            own = gbg.BlockedGraph.build(n, pairs)
            for _ in range(5):
                for g in (shared, own):
                    assert np.array_equal(gbg.bfs(g, 0).depth, want_d)
                    assert np.array_equal(gbg.cc(g), want_cc)
                    assert g.degree(k) == int(off[k + 1] - off[k])
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]


def _directed_with_sinks(n, p, sink_frac, seed):
    """Random directed arcs, then every out-arc of a `sink_frac` share of the
    vertices removed: those vertices keep in-arcs but have degree 0."""
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    a[rng.random(n) < sink_frac, :] = False
    s, d = np.nonzero(a)
    return np.stack([s, d], axis=1).astype(np.uint32)


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_directed_bfs_reaches_vertices_without_out_arcs(gbg, ref, kind):
    """A vertex with in-arcs but no out-arcs is reached by a sparse push
    (traversal.cpp:16-46 walks the frontier member's list); it must not be
    pre-marked visited as a zero-degree vertex of a symmetric graph would
    be.  First the advisor's case (arc 0->1 plus a 30-clique: bfs(0) gives
    depth[1] = 1), then seeded directed graphs with sinks and BC on them."""
    mk = gbg.CsrGraph.build if kind == "csr" else gbg.BlockedGraph.build
    arcs = [(0, 1)] + [(i, j) for i in range(2, 32) for j in range(2, 32) if i != j]
    pairs = np.array(sorted(arcs), dtype=np.uint32)
    off, nbr = csr(32, pairs)
    g = mk(32, pairs)
    r = gbg.bfs(g, 0)
    assert np.array_equal(r.depth, ref.csr(32, off, nbr).bfs(0))
    assert r.depth[1] == 1
    for seed, (n, p) in enumerate([(300, 0.02), (2000, 0.004), (2000, 0.03)]):
        pairs = _directed_with_sinks(n, p, 0.3, seed)
        off, nbr = csr(n, pairs)
        rg = ref.csr(n, off, nbr)
        g = mk(n, pairs)
        for src in (0, 1, n // 2, n - 1):
            assert np.array_equal(gbg.bfs(g, src).depth, rg.bfs(src)), (seed, src)
        for src in (0, n // 3):
            want = rg.bc(src)
            assert np.allclose(gbg.bc(g, src), want, rtol=1e-12, atol=1e-12, equal_nan=True), (seed, src)


def test_symmetric_batches_keep_the_premark(gbg, ref, orc):
    """Insert/delete of a reverse-closed batch keeps the blocked container
    symmetric; a one-directional arc makes it asymmetric, and BFS then
    still reaches the new sink (checked against the reference)."""
    n = 64
    nn, pairs = undirected(n, [(i, (i * 7 + 3) % n) for i in range(n)], orc)
    g = gbg.BlockedGraph.build(nn, pairs)
    g.insert_batch(np.array([[1, 40], [40, 1], [5, 6], [6, 5]], dtype=np.uint32))
    g.delete_batch(np.array([[1, 40], [40, 1]], dtype=np.uint32))
    g.insert_batch(np.array([[2, 63]], dtype=np.uint32))  # one direction only
    off, nbr = g.to_csr()
    rg = ref.csr(nn, off, nbr)
    for src in range(0, n, 7):
        assert np.array_equal(gbg.bfs(g, src).depth, rg.bfs(src))
    # equal s < d / s > d counts but not reverse-closed: (2, n) and (n+1, 3)
    # reach the two isolated vertices n, n+1 one way each; the symmetry
    # check must see it (hash sums), or the zero-out-degree pre-mark would
    # hide vertex n from a BFS from 2
    nn2, pairs2 = undirected(n, [(i, (i * 7 + 3) % n) for i in range(n)], orc)
    g2 = gbg.BlockedGraph.build(n + 2, pairs2)
    assert gbg.bfs(g2, 2).depth[n] == -1
    g2.insert_batch(np.array([[2, n], [n + 1, 3]], dtype=np.uint32))
    off, nbr = g2.to_csr()
    rg2 = ref.csr(n + 2, off, nbr)
    for src in (2, 3, n + 1, n):
        assert np.array_equal(gbg.bfs(g2, src).depth, rg2.bfs(src)), src
    assert gbg.bfs(g2, 2).depth[n] == 1


def test_batch_self_loop_with_out_of_range_id_is_dropped(gbg, ref):
    """prepare(GlobalSort) drops self-loops before any id check
    (batch.cpp:34-42), so (n+5, n+5) is ignored, not an out-of-range error;
    a non-loop out-of-range arc still fails."""
    g = gbg.BlockedGraph.build(4, np.array([[0, 1], [1, 0]], dtype=np.uint32))
    assert g.insert_batch(np.array([[9, 9], [2, 3], [3, 2]], dtype=np.uint32)) == 2
    assert g.num_edges() == 4
    with pytest.raises(IndexError):
        g.insert_batch(np.array([[2, 9]], dtype=np.uint32))


def test_pagerank_index_bytes_and_invalidation(gbg, orc):
    """The cached PageRank indexes report their device bytes, and an update
    drops both (derived data of one graph version)."""
    n, pairs = orc.rmat(12, 16 << 12, 3)
    g = gbg.BlockedGraph.build(n, pairs)
    assert gbg.pagerank_index_bytes(g) == (0, 0)
    gbg.pagerank(g, 0.85, 3, 1e-300)  # one-shot call: row layout
    tiled, rows = gbg.pagerank_index_bytes(g)
    assert tiled == 0 and rows >= 4 * g.num_edges()
    gbg.pagerank_prepare(g)
    tiled, rows = gbg.pagerank_index_bytes(g)
    assert tiled >= 2 * g.num_edges()
    g.insert_batch(np.array([[0, n - 1], [n - 1, 0]], dtype=np.uint32))
    assert gbg.pagerank_index_bytes(g) == (0, 0)

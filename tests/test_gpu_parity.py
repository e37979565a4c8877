"""GPU parity tests: the CUDA library (through its C ABI, via the Python
mirror) against the CPU oracle / reference library on identical seeded
inputs, plus the golden fixtures at the BASELINE sizes.

Bars: bit-exact for depths, labels, counts, arc sets; PageRank relative L1
<= 1e-9 in fp64 (north_star), with the reference's own 1e-7 check
(bench.cpp:225-233) implied.
"""
import numpy as np
import pytest

from oracle.bindings import RMAT_A, RMAT_B, RMAT_C, digest, max_degree_source
from tests.conftest import golden
from tests.helpers import PR_PATHS, pagerank_on, T4_PAIRS, complete, csr, members, star, undirected

pytestmark = pytest.mark.gpu
TINY = np.finfo(np.float64).tiny
PR_TOL = 1e-9  # relative L1, BASELINE.json north_star


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


# ---------------------------------------------------------------- subsets
def test_subset_known_answers(gbg):
    assert gbg.subset_to_dense(4, [1, 3]).tolist() == [0b1010]
    assert gbg.subset_to_dense(4, []).tolist() == [0]
    assert gbg.subset_to_dense(1000, [999]).size == 16
    assert gbg.subset_to_sparse(4, np.array([0b0101], np.uint64)).tolist() == [0, 2]
    assert gbg.subset_to_sparse(6, gbg.subset_to_dense(6, [5, 1, 5, 3, 1])).tolist() == [1, 3, 5]
    with pytest.raises(IndexError):
        gbg.subset_to_dense(4, [4])


def test_subset_round_trips(gbg, orc):
    rng = np.random.default_rng(42)
    for _ in range(200):
        n = int(rng.integers(1, 5000))
        ids = rng.integers(0, n, size=int(rng.integers(0, n + 1))).astype(np.uint32)
        dense = gbg.subset_to_dense(n, ids)
        assert np.array_equal(dense, orc.to_dense(n, ids))
        assert np.array_equal(gbg.subset_to_sparse(n, dense), orc.to_sparse(n, dense))


def test_vertex_filter_reference_cases(gbg):
    # test_traversal.cpp:239-261
    evens = [1, 0, 1, 0, 1, 0]
    assert gbg.vertex_filter_sparse(6, [0, 1, 2, 3], evens).tolist() == [0, 2]
    assert gbg.vertex_filter_sparse(6, [0, 1, 2, 3], [1] * 6).tolist() == [0, 1, 2, 3]
    dense = gbg.subset_to_dense(6, [0, 1, 2, 3])
    out = gbg.vertex_filter_dense(6, dense, [1, 1, 0, 0, 0, 0])
    assert gbg.subset_to_sparse(6, out).tolist() == [0, 1]
    assert gbg.vertex_filter_sparse(6, [], evens).size == 0
    assert gbg.vertex_filter_sparse(6, [5, 2, 2, 0], evens).tolist() == [0, 2]  # constructor sorts + dedups
    with pytest.raises(IndexError):
        gbg.vertex_filter_sparse(4, [4], [1] * 4)


def test_vertex_filter_matches_reference(gbg, ref):
    rng = np.random.default_rng(7)
    for trial in range(120):
        n = int(rng.integers(1, 70000 if trial % 10 == 0 else 3000))
        keep = (rng.random(n) < rng.random()).astype(np.uint8)
        ids = rng.integers(0, n, size=int(rng.integers(0, n + 1))).astype(np.uint32)
        if trial % 2:
            ids = np.unique(ids)
        assert np.array_equal(gbg.vertex_filter_sparse(n, ids, keep), ref.vertex_filter_sparse(n, ids, keep))
        words = gbg.subset_to_dense(n, ids)
        assert np.array_equal(gbg.vertex_filter_dense(n, words, keep), ref.vertex_filter_dense(n, words, keep))


# ---------------------------------------------------------------- containers
def test_csr_build_and_read_api(gbg):
    g = gbg.CsrGraph.build(4, T4_PAIRS)
    off, nbr = g.to_csr()
    assert off.tolist() == [0, 2, 4, 7, 8] and nbr.tolist() == [1, 2, 0, 2, 0, 1, 3, 2]
    assert g.num_vertices() == 4 and g.num_edges() == 8 and g.degree(2) == 3
    assert g.map_neighbors(2).tolist() == [0, 1, 3]
    assert g.degrees().tolist() == [2, 2, 3, 1]
    caps = g.capabilities()
    assert caps["has_degree"] and caps["has_map_early_exit"] and not caps["has_batch_updates"]
    e = gbg.CsrGraph.build(3, [])
    assert e.to_csr()[0].tolist() == [0, 0, 0, 0] and e.num_edges() == 0
    for bad, n in (([[1, 0], [0, 1]], 2), ([[0, 1], [0, 1]], 2), ([[0, 5]], 2)):
        with pytest.raises(gbg.FormatError):
            gbg.CsrGraph.build(n, bad)
    with pytest.raises(gbg.FormatError):
        gbg.CsrGraph.from_csr([0, 2, 1], [1, 0])
    with pytest.raises(IndexError):
        g.degree(4)


def test_static_csr_rejects_updates(gbg):
    g = gbg.CsrGraph.build(4, T4_PAIRS)
    for f in (lambda: g.insert_edge(0, 3), lambda: g.delete_edge(0, 1), lambda: g.insert_batch([]),
              lambda: g.delete_batch([[0, 1]])):
        with pytest.raises(gbg.UnsupportedOperation):
            f()


def test_gbcsr1_files_interchange_with_reference(gbg, ref, tmp_path):
    """GBCSR1 (io.cpp:75-114): files written by the reference load on the
    device, and files written from the device are byte-identical to the
    reference's and load back in it."""
    n, pairs = ref.rmat(14, 16 << 14, 3)
    off, nbr = csr(n, pairs)
    ref_file = tmp_path / "ref.gbcsr"
    ref.csr(n, off, nbr).save_binary(str(ref_file))
    for kind in (gbg.KIND_CSR, gbg.KIND_BLOCKED):
        g = gbg.load_binary(str(ref_file), kind)
        go, gn = g.to_csr()
        assert np.array_equal(go, off) and np.array_equal(gn, nbr)
        ours = tmp_path / f"ours{kind}.gbcsr"
        gbg.save_binary(g, str(ours))
        assert ours.read_bytes() == ref_file.read_bytes()
        rn, ro, rb = ref.load_binary(str(ours))
        assert rn == n and np.array_equal(ro, off) and np.array_equal(rb, nbr)
    bad = tmp_path / "bad.gbcsr"
    bad.write_bytes(b"NOTCSR00" + ref_file.read_bytes()[8:])
    with pytest.raises(gbg.FormatError):
        gbg.load_binary(str(bad))
    bad.write_bytes(ref_file.read_bytes()[:100])
    with pytest.raises(gbg.FormatError):
        gbg.load_binary(str(bad))
    raw = bytearray(ref_file.read_bytes())
    hdr = 8 + 16 + 8 * (n + 1)
    raw[hdr:hdr + 8] = raw[hdr + 4:hdr + 8] + raw[hdr:hdr + 4]  # swap two ids of vertex 0's list
    bad.write_bytes(bytes(raw))
    with pytest.raises(gbg.FormatError):
        gbg.load_binary(str(bad))


# ---------------------------------------------------------------- edge_map
def test_edge_map_known_answers(gbg):
    g = gbg.CsrGraph.build(4, T4_PAIRS)
    cond = np.array([0, 1, 1, 1], np.uint8)
    for mode in (gbg.MODE_SPARSE, gbg.MODE_DENSE, gbg.MODE_AUTO):
        out, _, _ = gbg.edge_map(g, [0], cond, mode)
        assert members(out) == {1, 2}
    assert members(gbg.edge_map(g, [], np.ones(4, np.uint8))[0]) == set()
    assert members(gbg.edge_map(g, [0, 1, 2, 3], np.zeros(4, np.uint8))[0]) == set()
    out, _, mode = gbg.edge_map(g, [1, 2], np.array([0, 0, 0, 1], np.uint8), gbg.MODE_DENSE)
    assert members(out) == {3} and mode == gbg.MODE_DENSE
    with pytest.raises(IndexError):
        gbg.edge_map(g, [7], np.ones(4, np.uint8))


def test_edge_map_dense_early_exit_counts(gbg, orc):
    n, pairs = undirected(64, star(63), orc)
    g = gbg.CsrGraph.build(n, pairs)
    cond = np.zeros(64, np.uint8)
    cond[0] = 1
    ids = np.arange(1, 64)
    assert gbg.edge_map(g, ids, cond, gbg.MODE_DENSE, True)[1] == 1
    assert gbg.edge_map(g, ids, cond, gbg.MODE_DENSE, False)[1] == 63


def test_edge_map_sparse_once_per_destination_and_hubs(gbg, orc):
    n, pairs = undirected(32, star(31), orc)
    g = gbg.CsrGraph.build(n, pairs)
    out, upd, _ = gbg.edge_map(g, np.arange(1, 32), np.ones(32, np.uint8), gbg.MODE_SPARSE)
    assert upd == 1 and members(out) == {0}
    edges = [(0, v) for v in range(2, 1502)] + [(1, v) for v in range(1502, 3002)]
    n, pairs = undirected(3002, edges, orc)
    g = gbg.CsrGraph.build(n, pairs)
    cond = np.ones(n, np.uint8)
    cond[:2] = 0
    out, upd, _ = gbg.edge_map(g, [0, 1], cond, gbg.MODE_SPARSE)
    m = sorted(members(out))
    assert len(m) == 3000 and m[0] == 2 and m[-1] == 3001 and upd == 3000


def test_edge_map_threshold_switch(gbg):
    g = gbg.CsrGraph.build(4, T4_PAIRS)
    # |F| + sum deg = 2 <= m/20 = 0.4? no -> dense; reference switch rule
    _, _, mode = gbg.edge_map(g, [3], np.ones(4, np.uint8), gbg.MODE_AUTO)
    assert mode == gbg.MODE_DENSE


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_edge_map_modes_match_oracle(gbg, ref, orc, kind):
    rng = np.random.default_rng(7)
    for trial in range(60):
        nv = 40 + int(rng.integers(0, 200))
        n, pairs = ref.er(nv, 0.08, 1000 + trial)
        off, nbr = csr(n, pairs)
        g = gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)
        ids = np.nonzero(rng.integers(0, 3, size=n) == 0)[0].astype(np.uint32)
        cond = (rng.integers(0, 4, size=n) != 0).astype(np.uint8)
        for mode in (0, 1):
            for ee in (True, False):
                want, wupd = orc.edge_map(n, off, nbr, ids, cond, mode, ee)
                got, upd, _ = gbg.edge_map(g, ids, cond, mode, ee)
                assert np.array_equal(got, want), (trial, mode, ee)
                assert upd == wupd, (trial, mode, ee)


# ---------------------------------------------------------------- BFS
def test_bfs_known_answers(gbg, orc):
    g = gbg.CsrGraph.build(4, T4_PAIRS)
    r = gbg.bfs(g, 0)
    assert r.depth.tolist() == [0, 1, 1, 2] and r.reached == 4
    n, pairs = undirected(4, [(0, 1)], orc)
    r = gbg.bfs(gbg.CsrGraph.build(n, pairs), 3)
    assert r.depth.tolist() == [-1, -1, -1, 0]
    with pytest.raises(IndexError):
        gbg.bfs(g, 9)


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_bfs_unreached_depths(gbg, orc, kind):
    """Unreached vertices read -1 whatever the level pattern and whatever
    the device buffer held before: an isolated source on a tiny graph
    (level 1 dense: 1 > m / 20), a path (never dense), a star (level 1
    dense), with isolated and unreachable vertices in every case."""
    import torch
    cases = []
    n, pairs = undirected(40, [(1, 2), (2, 3), (5, 6)], orc)            # source 0 isolated, m = 6
    cases.append((n, pairs, 0))
    n, pairs = undirected(300, [(i, i + 1) for i in range(200)] + [(250, 251)], orc)  # path + far component
    cases.append((n, pairs, 0))
    n, pairs = undirected(600, [(0, i) for i in range(1, 400)] + [(450, 451)], orc)   # star
    cases.append((n, pairs, 0))
    cases.append((n, pairs, 450))
    cases.append((n, pairs, 599))                                          # isolated source, larger graph
    for n, pairs, src in cases:
        off, nbr = csr(n, pairs)
        g = gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)
        d, modes, sizes = orc.bfs(n, off, nbr, src)
        r = gbg.bfs(g, src)
        assert np.array_equal(r.depth, d) and r.modes == modes and r.frontier_sizes == sizes
        dd = torch.full((n,), 123456, dtype=torch.int32, device="cuda")
        gbg.bfs_device(g, src, dd.data_ptr(), stats=False)
        g.synchronize()
        assert np.array_equal(dd.cpu().numpy(), d)


def test_bfs_large_sparse_push_matches_oracle(gbg, orc):
    """A sparse level of >= 64 K edges (emissions aggregated per CTA): a hub
    with 80,000 leaves inside enough filler edges that m / 20 stays above
    the hub's degree, so level 1 is a push of 80,000 edges that emits all
    of them; levels, sizes and depths against the oracle."""
    hub = 80000
    fill = 800000
    e = np.empty((hub + fill, 2), dtype=np.uint32)
    e[:hub, 0] = 0
    e[:hub, 1] = np.arange(1, hub + 1, dtype=np.uint32)
    base = hub + 1
    e[hub:, 0] = base + 2 * np.arange(fill, dtype=np.uint32)
    e[hub:, 1] = e[hub:, 0] + 1
    n, pairs = orc.normalize(e, base + 2 * fill)
    off, nbr = csr(n, pairs)
    d, modes, sizes = orc.bfs(n, off, nbr, 0)
    assert modes[0] == 0 and sizes[1] == hub  # level 1 really is the large sparse push
    r = gbg.bfs(gbg.CsrGraph.build(n, pairs), 0)
    assert np.array_equal(r.depth, d) and r.modes == modes and r.frontier_sizes == sizes
    assert r.degree_sums[1] == hub  # every leaf emitted once, with its degree


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_bfs_matches_oracle_seeded(gbg, ref, orc, kind):
    for trial in range(20):
        n, pairs = ref.er(150 + 37 * trial, 0.03, 100 + trial)
        off, nbr = csr(n, pairs)
        g = gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)
        d, modes, sizes = orc.bfs(n, off, nbr, trial % n)
        r = gbg.bfs(g, trial % n)
        assert np.array_equal(r.depth, d)
        assert r.modes == modes and r.frontier_sizes == sizes


def transition_graph(hub_degree):
    """A BFS from 0 whose level 2 is dense and whose level 3 is a sparse push
    from that level's bitmap holding one vertex of degree `hub_degree`:
    0 - {1..1200}, 1 - H, H - (hub_degree - 1) leaves, and disjoint filler
    edges that bring m to 40,000 arcs (threshold m/20 = 2000)."""
    edges = [(0, a) for a in range(1, 1201)]
    h = 1201
    edges.append((1, h))
    leaves = range(h + 1, h + hub_degree)
    edges += [(h, x) for x in leaves]
    nxt = h + hub_degree
    fill = 20000 - len(edges)
    edges += [(nxt + 2 * i, nxt + 2 * i + 1) for i in range(fill)]
    return nxt + 2 * fill, edges


@pytest.mark.parametrize("kind", ["csr", "blocked"])
@pytest.mark.parametrize("hub_degree", [40, 1000, 1024, 1025, 1500])
def test_bfs_dense_to_sparse_transition(gbg, orc, kind, hub_degree):
    """The dense -> sparse transition pushes straight from the frontier
    bitmap when every member's degree is <= 1024 (lists above kPullSerial
    finish warp-cooperatively) and builds the id list first otherwise; both
    give the oracle's depths and direction trace."""
    n0, edges = transition_graph(hub_degree)
    n, pairs = undirected(n0, edges, orc)
    off, nbr = csr(n, pairs)
    g = gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)
    d, modes, sizes = orc.bfs(n, off, nbr, 0)
    assert modes[:3] == [0, 1, 0] and sizes[2] == 1
    r = gbg.bfs(g, 0)
    assert np.array_equal(r.depth, d)
    assert r.modes == modes and r.frontier_sizes == sizes
    assert r.examined == orc.bfs_examined(n, off, nbr, 0)


@pytest.mark.parametrize("S", [16, 20])
def test_rmat_generator_and_bfs_cc_match_golden(gbg, S):
    gd = golden(S)
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    off, nbr = g.to_csr()
    assert (g.num_vertices(), g.num_edges()) == (gd["n"], gd["m"])
    assert digest(off) == gd["off_digest"] and digest(nbr) == gd["nbr_digest"]
    src = max_degree_source(off)
    assert src == gd["bfs"]["source"]
    r = gbg.bfs(g, src)
    assert digest(r.depth) == gd["bfs"]["digest"]
    assert r.modes == gd["bfs"]["modes"] and r.frontier_sizes == gd["bfs"]["frontier_sizes"]
    assert r.reached == gd["bfs"]["reached"]
    # NULL statistics: asynchronous on the handle's stream, queued twice
    # back to back into one device buffer; same depths after a synchronise
    import torch
    dd = torch.full((g.num_vertices(),), 7, dtype=torch.int32, device="cuda")
    assert gbg.bfs_device(g, src, dd.data_ptr(), stats=False) is None
    assert gbg.bfs_device(g, src, dd.data_ptr(), stats=False) is None
    g.synchronize()
    assert digest(dd.cpu().numpy()) == gd["bfs"]["digest"]
    assert digest(gbg.cc(g)) == gd["cc"]["digest"]
    assert gbg.triangle_count(g) == gd["tc"]["triangles"]


def test_scale24_bfs_cc_match_golden(gbg):
    gd = golden(24)
    g = gbg.generate_rmat(24, 16 << 24, 1, RMAT_A, RMAT_B, RMAT_C)
    assert (g.num_vertices(), g.num_edges()) == (gd["n"], gd["m"])
    off, nbr = g.to_csr()
    assert digest(off) == gd["off_digest"] and digest(nbr) == gd["nbr_digest"]
    del off, nbr
    r = gbg.bfs(g, gd["bfs"]["source"])
    assert digest(r.depth) == gd["bfs"]["digest"]
    assert r.modes == gd["bfs"]["modes"] and r.frontier_sizes == gd["bfs"]["frontier_sizes"]
    assert digest(gbg.cc(g)) == gd["cc"]["digest"]
    assert gbg.triangle_count(g) == gd["tc"]["triangles"]
    p = gbg.pagerank(g, 0.85, 20, TINY)
    ids = np.array(gd["pagerank"]["sample_ids"])
    want = np.array([float.fromhex(h) for h in gd["pagerank"]["sample_hex"]])
    assert rel_l1(p[ids], want) <= PR_TOL
    assert abs(p.sum() - gd["pagerank"]["sum"]) <= PR_TOL


@pytest.mark.parametrize("path", PR_PATHS)
def test_scale24_pagerank_full_vector_matches_reference(gbg, ref, path):
    """The headline config at the BASELINE bar: all 16.8M ranks of the
    device PageRank against the reference library's own
    gb::pagerank(view, 0.85, 20, DBL_MIN) (algorithms.cpp:508-555) on the
    same graph, relative L1 <= 1e-9 (the reference's own check is absolute
    L1 <= 1e-7, bench.cpp:225-233); also the largest per-vertex error."""
    import os

    g = gbg.generate_rmat(24, 16 << 24, 1, RMAT_A, RMAT_B, RMAT_C)
    n = g.num_vertices()
    off, nbr = g.to_csr()
    ref.set_threads(os.cpu_count() or 1)
    want = ref.csr(n, off, nbr).pagerank(0.85, 20, TINY)
    del off, nbr
    got = pagerank_on(gbg, g, path, 0.85, 20, TINY)
    assert got.shape == want.shape == (n,)
    err = rel_l1(got, want)
    assert err <= PR_TOL, err
    assert np.max(np.abs(got - want) / want) <= 1e-9
    assert abs(got.sum() - want.sum()) <= 1e-10


# ---------------------------------------------------------------- PageRank
def test_pagerank_known_answers(gbg, orc):
    n, pairs = undirected(4, [(0, 1), (1, 2), (2, 3), (3, 0)], orc)
    p = gbg.pagerank(gbg.CsrGraph.build(n, pairs), 0.85, 20, 1e-4)
    assert np.allclose(p, 0.25, rtol=1e-12, atol=0)
    g = gbg.CsrGraph.build(4, T4_PAIRS)
    q = gbg.pagerank(g, 0.85, 20, 1e-4)
    assert q[2] > q[0] and q[2] > q[1] and q[2] > q[3] and abs(q.sum() - 1) < 1e-6
    with pytest.raises(ValueError):
        gbg.pagerank(g, 1.5, 20, 1e-4)
    with pytest.raises(ValueError):
        gbg.pagerank(g, 0.85, 20, 0.0)


@pytest.mark.parametrize("path", PR_PATHS)
@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_pagerank_matches_oracle_seeded(gbg, ref, orc, kind, path):
    for trial in range(15):
        n, pairs = ref.er(150 + 101 * trial, 0.04, 2300 + trial)
        off, nbr = csr(n, pairs)
        g = gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)
        for tol in (1e-4, TINY):
            want = orc.pagerank(n, off, nbr, 0.85, 20, tol)
            got = pagerank_on(gbg, g, path, 0.85, 20, tol)
            assert rel_l1(got, want) <= PR_TOL, (trial, tol)


@pytest.mark.parametrize("path", PR_PATHS)
@pytest.mark.parametrize("S", [16, 20])
def test_pagerank_rmat_matches_reference(gbg, ref, S, path):
    gd = golden(S)
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    off, nbr = g.to_csr()
    want = ref.csr(gd["n"], off, nbr).pagerank(0.85, 20, TINY)
    got = pagerank_on(gbg, g, path, 0.85, 20, TINY)
    assert rel_l1(got, want) <= PR_TOL
    ids = np.array(gd["pagerank"]["sample_ids"])
    gold = np.array([float.fromhex(h) for h in gd["pagerank"]["sample_hex"]])
    assert rel_l1(got[ids], gold) <= PR_TOL


@pytest.mark.parametrize("path", PR_PATHS)
def test_pagerank_hub_rows(gbg, orc, path):
    # rows far above the heavy-row split (kHeavy) and many straddling tiles
    edges = [(0, v) for v in range(1, 20000)] + [(1, v) for v in range(2, 9000, 3)] + complete(60)
    n, pairs = undirected(20001, edges, orc)
    off, nbr = csr(n, pairs)
    got = pagerank_on(gbg, gbg.CsrGraph.build(n, pairs), path, 0.85, 20, TINY)
    want = orc.pagerank(n, off, nbr, 0.85, 20, TINY)
    assert rel_l1(got, want) <= PR_TOL


@pytest.mark.parametrize("path", PR_PATHS)
def test_pagerank_asymmetric_arcs(gbg, orc, path):
    """Directed arc sets: vertices with in-arcs but no out-arcs are dangling
    (contrib 0, mass redistributed) yet gathered by their in-neighbours, on
    both containers, with early stopping and with 20 fixed iterations."""
    rng = np.random.default_rng(5)
    for trial in range(8):
        n = 200 + 150 * trial
        raw = rng.integers(0, n, size=(3 * n, 2)).astype(np.uint32)
        raw = raw[raw[:, 0] % 3 != 0]  # a third of the vertices keep no out-arcs
        pairs = orc.prepare_global(raw)
        off, nbr = csr(n, pairs)
        for g in (gbg.CsrGraph.build(n, pairs), gbg.BlockedGraph.build(n, pairs)):
            for tol in (1e-4, TINY):
                want = orc.pagerank(n, off, nbr, 0.85, 20, tol)
                assert rel_l1(pagerank_on(gbg, g, path, 0.85, 20, tol), want) <= PR_TOL, (trial, tol)


# ---------------------------------------------------------------- CC / TC
@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_cc_matches_oracle(gbg, ref, orc, kind):
    mk = (lambda n, p: gbg.CsrGraph.build(n, p)) if kind == "csr" else (lambda n, p: gbg.BlockedGraph.build(n, p))
    assert gbg.cc(mk(4, T4_PAIRS)).tolist() == [0, 0, 0, 0]
    assert gbg.cc(mk(5, [])).tolist() == [0, 1, 2, 3, 4]
    for trial in range(25):
        n, pairs = ref.er(200 + 53 * trial, 0.008, 900 + trial)
        off, nbr = csr(n, pairs)
        assert np.array_equal(gbg.cc(mk(n, pairs)), orc.cc(n, off, nbr))


def test_cc_asymmetric_arcs(gbg, orc):
    """Directed arc sets (no reverse arcs): the full-hooking path, labels
    still the minimum id of each weakly connected component."""
    rng = np.random.default_rng(11)
    for trial in range(10):
        n = 300 + 100 * trial
        raw = rng.integers(0, n, size=(n // 2, 2)).astype(np.uint32)
        pairs = orc.prepare_global(raw)
        off, nbr = csr(n, pairs)
        for g in (gbg.CsrGraph.build(n, pairs), gbg.BlockedGraph.build(n, pairs)):
            assert np.array_equal(gbg.cc(g), orc.cc(n, off, nbr)), trial


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_bc_matches_oracle(gbg, ref, orc, kind):
    """gb::bc; the reference's own differential check is |Δ| <= 1e-9 per
    vertex (bench.cpp:234-241); large dependencies are compared relatively."""
    mk = (lambda n, p: gbg.CsrGraph.build(n, p)) if kind == "csr" else (lambda n, p: gbg.BlockedGraph.build(n, p))
    assert gbg.bc(mk(4, T4_PAIRS), 3).tolist() == [0.0, 0.0, 2.0, 3.0]
    with pytest.raises(IndexError):
        gbg.bc(mk(4, T4_PAIRS), 9)
    for trial in range(12):
        n, pairs = ref.er(150 + 50 * trial, 0.04, 300 + trial)
        off, nbr = csr(n, pairs)
        want = orc.bc(n, off, nbr, trial)
        got = gbg.bc(mk(n, pairs), trial)
        assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
    for S in (12, 16):
        n, pairs = ref.rmat(S, 16 << S, 1)
        off, nbr = csr(n, pairs)
        want = orc.bc(n, off, nbr, 0)
        got = gbg.bc(mk(n, pairs), 0)
        assert np.abs(got - want).max() <= 1e-9 * np.abs(want).max()


def test_tc_known_answers(gbg, ref, orc):
    assert gbg.triangle_count(gbg.CsrGraph.build(4, T4_PAIRS)) == 1
    for k in (3, 5, 8, 12, 40):
        n, pairs = undirected(k, complete(k), orc)
        assert gbg.triangle_count(gbg.CsrGraph.build(n, pairs)) == k * (k - 1) * (k - 2) // 6
    n, pairs = undirected(50, star(49), orc)
    assert gbg.triangle_count(gbg.CsrGraph.build(n, pairs)) == 0
    for trial in range(10):
        n, pairs = ref.er(300, 0.05, 77 + trial)
        off, nbr = csr(n, pairs)
        assert gbg.triangle_count(gbg.BlockedGraph.build(n, pairs)) == orc.tc(n, off, nbr)


# ---------------------------------------------------------------- updates
def test_update_batch_generator_bit_exact(gbg, orc):
    import torch

    for S, size, seed in ((14, 1000, 42), (22, 100000, 7)):
        buf = torch.empty(4 * size, dtype=torch.int32, device="cuda")
        gbg.generate_update_batch_device(S, size, seed, buf.data_ptr(), RMAT_A, RMAT_B, RMAT_C)
        got = buf.cpu().numpy().view(np.uint32).reshape(-1, 2)
        assert np.array_equal(got, orc.update_batch(S, size, seed))


def test_blocked_t4_apply_counts(gbg):
    g = gbg.BlockedGraph.build(4, T4_PAIRS)
    assert g.capabilities()["has_batch_updates"]
    assert gbg.apply_insert(g, [[0, 3], [3, 0]]) == 2
    assert g.num_edges() == 10 and g.degree(3) == 2
    assert gbg.apply_insert(g, T4_PAIRS) == 0 and g.num_edges() == 10
    assert gbg.apply_delete(g, [[0, 3], [3, 0]]) == 2 and g.num_edges() == 8
    off, nbr = g.to_csr()
    assert off.tolist() == [0, 2, 4, 7, 8] and nbr.tolist() == [1, 2, 0, 2, 0, 1, 3, 2]
    assert gbg.apply_delete(g, [[1, 3], [3, 1]]) == 0
    assert gbg.apply_delete(g, [[2, 3], [3, 2]]) == 2 and g.num_edges() == 6
    gbg.apply_delete(g, T4_PAIRS)
    assert g.num_vertices() == 4 and g.num_edges() == 0
    with pytest.raises(IndexError):
        g.insert_batch([[0, 9]])
    with pytest.raises(ValueError):
        g.insert_edge(1, 1)
    assert g.insert_edge(0, 1) and not g.insert_edge(0, 1) and g.delete_edge(0, 1)


@pytest.mark.parametrize("path", PR_PATHS)
def test_pagerank_after_batches_on_blocked_container(gbg, ref, path):
    """PageRank on the dynamic container after insert and delete batches:
    both derived PageRank layouts are dropped by an update and rebuilt on
    the next call, so every call matches gb::pagerank on the container's
    current arcs (asymmetric batches included)."""
    n, base = ref.rmat(14, 16 << 14, 5, RMAT_A, RMAT_B, RMAT_C)
    g = gbg.BlockedGraph.build(n, base)
    rng = np.random.default_rng(3)
    for step in range(4):
        pagerank_on(gbg, g, path, 0.85, 20, TINY)  # layouts exist before the update
        raw = ref.update_batch(14, 3000, 77 + step, RMAT_A, RMAT_B, RMAT_C)
        if step == 2:
            raw = rng.integers(0, n, size=(500, 2)).astype(np.uint32)  # one-directional arcs
        if step == 3:
            g.delete_batch(raw)
        else:
            g.insert_batch(raw)
        off, nbr = g.to_csr()
        want = ref.csr(n, off, nbr).pagerank(0.85, 20, TINY)
        assert rel_l1(pagerank_on(gbg, g, path, 0.85, 20, TINY), want) <= PR_TOL, step


def test_blocked_churn_matches_oracle(gbg, ref, orc):
    """Random insert/delete batches (with duplicates and self-loops) against
    the restated set semantics; exercises in-place merges, grown lists and
    pool compaction."""
    rng = np.random.default_rng(5)
    n, base = ref.rmat(12, 1 << 14, 3, 0.5, 0.1, 0.1)
    off, nbr = csr(n, base)
    g = gbg.BlockedGraph.build(n, base)
    for step in range(40):
        k = int(rng.integers(1, 20000))
        raw = rng.integers(0, n, size=(k, 2)).astype(np.uint32)
        if step % 3 == 0:
            raw[: k // 3, 0] = int(rng.integers(0, 4))  # hub-heavy batch
        insert = bool(rng.integers(0, 2)) or step < 5
        want, off, nbr = orc.set_apply(n, off, nbr, orc.prepare_global(raw), insert)
        got = g.insert_batch(raw) if insert else g.delete_batch(raw)
        assert got == want, step
        assert g.num_edges() == int(off[n])
        if step % 8 == 7:
            go, gn = g.to_csr()
            assert np.array_equal(go, off) and np.array_equal(gn, nbr), step
    go, gn = g.to_csr()
    assert np.array_equal(go, off) and np.array_equal(gn, nbr)
    assert np.array_equal(gbg.bfs(g, 0).depth, orc.bfs(n, off, nbr, 0)[0])


def test_blocked_round_trip_matches_chunked_set(gbg, ref):
    n, base = ref.rmat(14, 1 << 16, 11, 0.5, 0.1, 0.1)
    raw = ref.update_batch(14, 20000, 777, 0.5, 0.1, 0.1)
    keys = set(map(tuple, base.tolist()))
    batch = np.array([e for e in raw.tolist() if tuple(e) not in keys], dtype=np.uint32)
    batch = np.concatenate([batch, batch[: len(batch) // 2]])
    c = ref.chunked(n, base)
    g = gbg.BlockedGraph.build(n, base)
    ins = g.insert_batch(batch)
    assert ins == c.apply(batch, True) > 0
    eo, en = c.export()
    go, gn = g.to_csr()
    assert np.array_equal(go, eo) and np.array_equal(gn, en)
    assert g.delete_batch(batch) == c.apply(batch, False) == ins
    go, gn = g.to_csr()
    bo, bn = csr(n, base)
    assert np.array_equal(go, bo) and np.array_equal(gn, bn)


def test_scale22_update_sequence_matches_golden(gbg):
    """Config 5: s22 base, batches 1e4..1e7 x reps 0..2 (seeds
    hash_combine(hash_combine(2,size),rep), bench.cpp:159-161; base-disjoint),
    BFS after each insert, each batch deleted again — all against the
    chunked_set replay recorded in tests/golden/rmat_s22.json."""
    import torch

    gd = golden(22)
    g = gbg.generate_rmat(22, 16 << 22, 1, RMAT_A, RMAT_B, RMAT_C, kind=gbg.KIND_BLOCKED)
    assert g.num_edges() == gd["m"]
    assert sorted({(r["size"], r.get("rep", 0)) for r in gd["updates"]}) == [
        (s, r) for s in (10**4, 10**5, 10**6, 10**7) for r in range(3)]
    for rec in gd["updates"]:
        size = rec["size"]
        buf = torch.empty(4 * size, dtype=torch.int32, device="cuda")
        gbg.generate_update_batch_device(22, size, rec["seed"], buf.data_ptr(), RMAT_A, RMAT_B, RMAT_C)
        raw = buf.cpu().numpy().view(np.uint32).reshape(-1, 2)
        assert digest(raw.reshape(-1)) == rec["raw_digest"]
        # base-disjoint filter (bench.cpp:150-169) with the device membership query
        present = torch.empty(2 * size, dtype=torch.uint8, device="cuda")
        g.contains_device(buf.data_ptr(), 2 * size, present.data_ptr())
        fresh = np.ascontiguousarray(raw[present.cpu().numpy() == 0])
        assert digest(fresh.reshape(-1)) == rec["fresh_digest"]
        assert g.insert_batch(fresh) == rec["inserted"]
        assert g.num_edges() == rec["m_after_insert"]
        off, nbr = g.to_csr()
        assert digest(off) == rec["off_digest_after_insert"] and digest(nbr) == rec["nbr_digest_after_insert"]
        src = max_degree_source(off)
        del off, nbr
        assert src == rec["bfs_source"]
        r = gbg.bfs(g, src)
        assert digest(r.depth) == rec["bfs_digest"] and r.reached == rec["bfs_reached"]
        assert g.delete_batch(fresh) == rec["deleted"]
        assert g.num_edges() == rec["m_after_delete"]


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_bfs_examined_arcs(gbg, orc, kind):
    """gbg_bfs_stats.examined equals the arcs the reference inspects per level
    (SURVEY App. A3 / oracle gbo_bfs_examined): sum deg(F) for pushes, list
    prefixes up to the first frontier hit for early-exit pulls."""
    for S, want in ((16, [9709, 38520, 1569, 1735, 6]), (20, [64840, 624964, 39715, 46114, 139])):
        g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C,
                              kind=gbg.KIND_CSR if kind == "csr" else gbg.KIND_BLOCKED)
        assert gbg.bfs(g, 0).examined == want, S
    n, pairs = orc.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    g = gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)
    for src in (0, 5, 77):
        assert gbg.bfs(g, src).examined == orc.bfs_examined(n, off, nbr, src), src


def test_scale24_bfs_examined_arcs(gbg):
    """SURVEY App. A3 at scale 24: 11,810,112 arcs inspected over six levels."""
    g = gbg.generate_rmat(24, 16 << 24, 1, RMAT_A, RMAT_B, RMAT_C)
    r = gbg.bfs(g, 0)
    assert r.examined == [406360, 9510944, 851503, 1038253, 3041, 11]

"""CPU tests: pin the C restatement oracle (oracle/gbo.c) against the
reference library itself (oracle/_ref/libgbref.so, built from
/root/reference) and against the reference test suite's known answers and
the golden fixtures.  No GPU needed."""
import numpy as np
import pytest

from oracle.bindings import RefError, digest, max_degree_source
from tests.conftest import golden
from tests.helpers import T4_PAIRS, complete, csr, members, star, undirected

TINY = np.finfo(np.float64).tiny


# ---------------------------------------------------------------- generators
@pytest.mark.parametrize("a,b,c", [(0.5, 0.1, 0.1), (0.57, 0.19, 0.19)])
@pytest.mark.parametrize("seed", [1, 42, 12345])
def test_update_batch_matches_reference(ref, orc, a, b, c, seed):
    for log2_n in (4, 14, 22):
        x = ref.update_batch(log2_n, 1000, seed, a, b, c)
        y = orc.update_batch(log2_n, 1000, seed, a, b, c)
        assert np.array_equal(x, y)


def test_update_batch_shape_and_pairs(orc):
    # test_batch.cpp:162-182
    one = orc.update_batch(14, 10, 42, 0.5, 0.1, 0.1)
    assert one.shape == (20, 2)
    assert np.array_equal(one[0::2, 0], one[1::2, 1]) and np.array_equal(one[0::2, 1], one[1::2, 0])
    assert np.array_equal(one, orc.update_batch(14, 10, 42, 0.5, 0.1, 0.1))
    assert not np.array_equal(one, orc.update_batch(14, 10, 43, 0.5, 0.1, 0.1))


def test_rng_and_hash_match_reference(ref, orc):
    for a, b in [(0, 0), (1, 2), (2**63, 7), (123456789, 987654321)]:
        assert ref.L.gbref_hash_combine(a, b) == orc.L.gbo_hash_combine(a, b)
    for s, st, cn in [(1, 0, 0), (1, 5, 3), (99, 2**40, 17)]:
        assert ref.L.gbref_rng_double(s, st, cn) == orc.L.gbo_rng_double(s, st, cn)


@pytest.mark.parametrize("S", [10, 14])
def test_rmat_graph_matches_reference(ref, orc, S):
    n1, p1 = ref.rmat(S, 16 << S, 1)
    n2, p2 = orc.rmat(S, 16 << S, 1)
    assert n1 == n2 == 1 << S
    assert np.array_equal(p1, p2)


def test_rmat_s16_matches_golden(orc):
    gd = golden(16)
    n, pairs = orc.rmat(16, 16 << 16, 1)
    off, nbr = csr(n, pairs)
    assert (n, int(off[n])) == (gd["n"], gd["m"])
    assert digest(off) == gd["off_digest"] and digest(nbr) == gd["nbr_digest"]


@pytest.mark.parametrize("S,seed,abc", [(1, 1, (0.57, 0.19, 0.19)), (10, 1, (0.57, 0.19, 0.19)),
                                         (14, 1, (0.57, 0.19, 0.19)), (12, 42, (0.5, 0.1, 0.1)),
                                         (13, 7, (0.45, 0.15, 0.25))])
def test_parallel_rmat_csr_matches_reference(ref, orc, S, seed, abc):
    """oracle/gbo_omp.c (the bench's host-side generator for the CPU
    reference arm) against gb::generate_rmat + CsrGraph::build."""
    n, pairs = ref.rmat(S, 16 << S, seed, *abc)
    want_off, want_nbr = csr(n, pairs)
    off, nbr = orc.rmat_csr(S, 16 << S, seed, *abc)
    assert np.array_equal(off, want_off) and np.array_equal(nbr, want_nbr)


def test_parallel_rmat_s16_golden_and_gbcsr1_bytes(ref, orc, tmp_path):
    """Scale 16 against the golden digests, and the GBCSR1 writer against
    gb::save_binary byte for byte; gb::load_binary_csr reads it back."""
    gd = golden(16)
    off, nbr = orc.rmat_csr(16, 16 << 16, 1)
    assert digest(off) == gd["off_digest"] and digest(nbr) == gd["nbr_digest"]
    n = off.size - 1
    ours, theirs = tmp_path / "ours.gbcsr1", tmp_path / "ref.gbcsr1"
    orc.save_gbcsr1(str(ours), n, off, nbr)
    ref.csr(n, off, nbr).save_binary(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    g = ref.load_binary_graph(str(ours))
    assert g.n == n
    assert np.array_equal(g.bfs(0), ref.csr(n, off, nbr).bfs(0))


def test_normalize_and_fixture(ref, orc):
    n, p = ref.t4()
    assert n == 4 and np.array_equal(p, T4_PAIRS)
    n2, p2 = orc.normalize([[0, 1], [1, 2], [0, 2], [2, 3]], 4)
    assert n2 == 4 and np.array_equal(p2, T4_PAIRS)
    # n = max(min_n, 1 + max id), loops counted for n but dropped
    n3, p3 = orc.normalize([[5, 5], [0, 1]], 0)
    assert n3 == 6 and p3.tolist() == [[0, 1], [1, 0]]


def test_csr_build_known_answers(orc):
    # test_containers.cpp:17-39
    off, nbr = orc.csr(4, T4_PAIRS)
    assert off.tolist() == [0, 2, 4, 7, 8] and nbr.tolist() == [1, 2, 0, 2, 0, 1, 3, 2]
    off, nbr = orc.csr(3, np.zeros((0, 2), np.uint32))
    assert off.tolist() == [0, 0, 0, 0]
    for bad, n in (([[1, 0], [0, 1]], 2), ([[0, 1], [0, 1]], 2), ([[0, 5]], 2)):
        with pytest.raises(ValueError):
            orc.csr(n, bad)


# ---------------------------------------------------------------- subsets
def test_subset_known_answers(orc):
    # test_vertex_subset.cpp:22-57
    assert orc.to_dense(4, [1, 3]).tolist() == [0b1010]
    assert orc.to_dense(1000, [999]).size == (1000 + 63) // 64
    assert orc.to_sparse(4, np.array([0b0101], np.uint64)).tolist() == [0, 2]
    assert orc.to_sparse(6, orc.to_dense(6, [5, 1, 5, 3, 1])).tolist() == [1, 3, 5]
    assert orc.to_sparse(4, np.array([0b1111], np.uint64)).tolist() == [0, 1, 2, 3]


def test_subset_round_trips(orc):
    # test_vertex_subset.cpp:69-92
    rng = np.random.default_rng(42)
    for _ in range(300):
        n = int(rng.integers(1, 301))
        ids = rng.integers(0, n, size=int(rng.integers(0, n + 1))).astype(np.uint32)
        dense = orc.to_dense(n, ids)
        back = orc.to_sparse(n, dense)
        assert back.tolist() == sorted(set(ids.tolist()))
        assert np.array_equal(orc.to_dense(n, back), dense)


# ---------------------------------------------------------------- edge_map
def test_ref_vertex_filter_known_answers(ref):
    # test_traversal.cpp:239-261 through the compiled reference
    evens = [1, 0, 1, 0, 1, 0]
    assert ref.vertex_filter_sparse(6, [0, 1, 2, 3], evens).tolist() == [0, 2]
    assert ref.vertex_filter_sparse(6, [0, 1, 2, 3], [1] * 6).tolist() == [0, 1, 2, 3]
    out = ref.vertex_filter_dense(6, np.array([0b1111], np.uint64), [1, 1, 0, 0, 0, 0])
    assert out.tolist() == [0b11]
    assert ref.vertex_filter_sparse(6, [5, 2, 2, 0], evens).tolist() == [0, 2]


def test_edge_map_known_answers(ref, orc):
    off, nbr = csr(4, T4_PAIRS)
    g = ref.csr(4, off, nbr)
    allc = np.ones(4, np.uint8)
    # T4 bfs step {0} -> {1,2} (test_traversal.cpp:25-44)
    cond = np.array([0, 1, 1, 1], np.uint8)
    for mode in (0, 1):
        out, upd = orc.edge_map(4, off, nbr, [0], cond, mode)
        assert members(out) == {1, 2}
        rout, rupd, _ = g.edge_map([0], cond, mode)
        assert members(rout) == {1, 2} and rupd == upd
    # empty frontier, always-false cond (46-61)
    assert members(orc.edge_map(4, off, nbr, [], allc, 0)[0]) == set()
    assert members(orc.edge_map(4, off, nbr, [0, 1, 2, 3], np.zeros(4, np.uint8), 1)[0]) == set()
    # pull step with cond v == 3 (63-75)
    assert members(orc.edge_map(4, off, nbr, [1, 2], np.array([0, 0, 0, 1], np.uint8), 1)[0]) == {3}


def test_dense_early_exit_counts(ref, orc):
    # test_traversal.cpp:77-114: star 0-(1..63), frontier 1..63, cond v == 0
    n, pairs = undirected(64, star(63), orc)
    off, nbr = csr(n, pairs)
    cond = np.zeros(64, np.uint8)
    cond[0] = 1
    ids = np.arange(1, 64, dtype=np.uint32)
    assert orc.edge_map(n, off, nbr, ids, cond, 1, True)[1] == 1
    assert orc.edge_map(n, off, nbr, ids, cond, 1, False)[1] == 63
    g = ref.csr(n, off, nbr)
    assert g.edge_map(ids, cond, 1, True)[1] == 1
    assert g.edge_map(ids, cond, 1, False)[1] == 63


def test_sparse_once_per_destination(orc):
    # test_traversal.cpp:138-161
    n, pairs = undirected(32, star(31), orc)
    off, nbr = csr(n, pairs)
    out, upd = orc.edge_map(n, off, nbr, np.arange(1, 32), np.ones(32, np.uint8), 0)
    assert upd == 1 and members(out) == {0}


def test_modes_agree_on_seeded_graphs(ref, orc):
    # test_traversal.cpp:163-185 / acceptance.cpp:238-268 (same construction)
    rng = np.random.default_rng(7)
    for trial in range(60):
        nv = 40 + int(rng.integers(0, 40))
        n, pairs = ref.er(nv, 0.08, 1000 + trial)
        off, nbr = csr(n, pairs)
        ids = np.nonzero(rng.integers(0, 3, size=n) == 0)[0].astype(np.uint32)
        cond = (rng.integers(0, 4, size=n) != 0).astype(np.uint8)
        a, _ = orc.edge_map(n, off, nbr, ids, cond, 0)
        b, _ = orc.edge_map(n, off, nbr, ids, cond, 1)
        assert members(a) == members(b)
        r, _, _ = ref.csr(n, off, nbr).edge_map(ids, cond, 0)
        assert members(r) == members(a)


def test_two_hubs(orc):
    # test_traversal.cpp:220-237
    edges = [(0, v) for v in range(2, 1502)] + [(1, v) for v in range(1502, 3002)]
    n, pairs = undirected(3002, edges, orc)
    off, nbr = csr(n, pairs)
    cond = np.ones(n, np.uint8)
    cond[:2] = 0
    out, _ = orc.edge_map(n, off, nbr, [0, 1], cond, 0)
    m = sorted(members(out))
    assert len(m) == 3000 and m[0] == 2 and m[-1] == 3001


# ---------------------------------------------------------------- algorithms
def test_bfs_known_answers(orc):
    off, nbr = csr(4, T4_PAIRS)
    assert orc.bfs(4, off, nbr, 0)[0].tolist() == [0, 1, 1, 2]
    n, pairs = undirected(4, [(0, 1)], orc)
    off, nbr = csr(n, pairs)
    assert orc.bfs(n, off, nbr, 3)[0].tolist() == [-1, -1, -1, 0]
    with pytest.raises(IndexError):
        orc.bfs(4, *csr(4, T4_PAIRS), 9)


def test_bfs_matches_reference_on_seeded_graphs(ref, orc):
    for trial in range(20):
        n, pairs = ref.er(150, 0.03, 100 + trial)
        off, nbr = csr(n, pairs)
        g = ref.csr(n, off, nbr)
        d, modes, sizes = orc.bfs(n, off, nbr, trial % 150)
        assert np.array_equal(d, g.bfs(trial % 150))
        assert (modes, sizes) == g.bfs_trace(trial % 150)


def test_cc_known_answers_and_seeded(ref, orc):
    off, nbr = csr(4, T4_PAIRS)
    assert orc.cc(4, off, nbr).tolist() == [0, 0, 0, 0]
    off, nbr = csr(5, np.zeros((0, 2), np.uint32))
    assert orc.cc(5, off, nbr).tolist() == [0, 1, 2, 3, 4]
    for trial in range(25):
        n, pairs = ref.er(200, 0.008, 900 + trial)
        off, nbr = csr(n, pairs)
        assert np.array_equal(orc.cc(n, off, nbr), ref.csr(n, off, nbr).cc())


def test_pagerank_known_answers(ref, orc):
    # test_algorithms.cpp:294-313
    n, pairs = undirected(4, [(0, 1), (1, 2), (2, 3), (3, 0)], orc)
    p = orc.pagerank(n, *csr(n, pairs), 0.85, 20, 1e-4)
    assert np.allclose(p, 0.25, rtol=1e-12, atol=0)
    q = orc.pagerank(4, *csr(4, T4_PAIRS), 0.85, 20, 1e-4)
    assert q[2] > q[0] and q[2] > q[1] and q[2] > q[3] and abs(q.sum() - 1) < 1e-6
    with pytest.raises(ValueError):
        orc.pagerank(4, *csr(4, T4_PAIRS), 1.5, 20, 1e-4)
    with pytest.raises(ValueError):
        orc.pagerank(4, *csr(4, T4_PAIRS), 0.85, 20, 0.0)


def test_pagerank_matches_reference(ref, orc):
    for trial in range(15):
        n, pairs = ref.er(150, 0.04, 2300 + trial)
        off, nbr = csr(n, pairs)
        g = ref.csr(n, off, nbr)
        for tol in (1e-4, TINY):
            a = orc.pagerank(n, off, nbr, 0.85, 20, tol)
            b = g.pagerank(0.85, 20, tol)
            assert np.abs(a - b).sum() <= 1e-12


def test_bc_matches_reference(ref, orc):
    # test_algorithms.cpp:57-66: from the pendant of T4
    off, nbr = csr(4, T4_PAIRS)
    assert orc.bc(4, off, nbr, 3).tolist() == ref.csr(4, off, nbr).bc(3).tolist() == [0.0, 0.0, 2.0, 3.0]
    for trial in range(10):
        n, pairs = ref.er(150, 0.04, 300 + trial)
        off, nbr = csr(n, pairs)
        assert np.array_equal(orc.bc(n, off, nbr, trial), ref.csr(n, off, nbr).bc(trial))
    n, pairs = ref.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    assert np.array_equal(orc.bc(n, off, nbr, 0), ref.csr(n, off, nbr).bc(0))


def test_tc_known_answers(orc):
    off, nbr = csr(4, T4_PAIRS)
    assert orc.tc(4, off, nbr) == 1
    for k in (3, 5, 8, 12):
        n, pairs = undirected(k, complete(k), orc)
        assert orc.tc(n, *csr(n, pairs)) == k * (k - 1) * (k - 2) // 6
    n, pairs = undirected(50, star(49), orc)
    assert orc.tc(n, *csr(n, pairs)) == 0
    n, pairs = undirected(7, [(0, 1), (1, 2), (1, 3), (3, 4), (3, 5), (5, 6)], orc)  # tree
    assert orc.tc(n, *csr(n, pairs)) == 0


def test_tc_brute_force_small(ref, orc):
    for trial in range(10):
        n, pairs = ref.er(40, 0.2, 77 + trial)
        adj = np.zeros((n, n), dtype=np.int64)
        adj[pairs[:, 0], pairs[:, 1]] = 1
        brute = int(np.trace(adj @ adj @ adj)) // 6
        assert orc.tc(n, *csr(n, pairs)) == brute


def test_s16_outputs_match_golden(orc):
    gd = golden(16)
    n, pairs = orc.rmat(16, 16 << 16, 1)
    off, nbr = csr(n, pairs)
    src = max_degree_source(off)
    assert src == gd["bfs"]["source"]
    d, modes, sizes = orc.bfs(n, off, nbr, src)
    assert digest(d) == gd["bfs"]["digest"]
    assert modes == gd["bfs"]["modes"] and sizes == gd["bfs"]["frontier_sizes"]
    assert digest(orc.cc(n, off, nbr)) == gd["cc"]["digest"]
    p = orc.pagerank(n, off, nbr, 0.85, 20, TINY)
    ids = np.array(gd["pagerank"]["sample_ids"])
    want = np.array([float.fromhex(h) for h in gd["pagerank"]["sample_hex"]])
    assert np.abs(p[ids] - want).max() <= 1e-15
    assert orc.tc(n, off, nbr) == gd["tc"]["triangles"]


# ---------------------------------------------------------------- batches
def test_prepare_global_known_answers(ref, orc):
    # test_batch.cpp:25-30, 50-62
    raw = [[2, 3], [0, 1], [2, 1], [0, 1]]
    assert orc.prepare_global(raw).tolist() == [[0, 1], [2, 1], [2, 3]]
    assert ref.prepare_global(raw).tolist() == [[0, 1], [2, 1], [2, 3]]
    loops = [[1, 1], [2, 2], [1, 2], [1, 2], [2, 1]]
    assert orc.prepare_global(loops).tolist() == [[1, 2], [2, 1]]
    assert orc.prepare_global(np.zeros((0, 2), np.uint32)).shape[0] == 0


def test_set_apply_t4_counts(orc):
    # test_batch.cpp:85-125
    off, nbr = csr(4, T4_PAIRS)
    add = orc.prepare_global([[0, 3], [3, 0]])
    k, off, nbr = orc.set_apply(4, off, nbr, add, True)
    assert k == 2 and int(off[4]) == 10 and int(off[4] - off[3]) == 2
    k, off, nbr = orc.set_apply(4, off, nbr, orc.prepare_global(T4_PAIRS), True)
    assert k == 0 and int(off[4]) == 10
    k, off, nbr = orc.set_apply(4, off, nbr, add, False)
    assert k == 2 and int(off[4]) == 8
    t_off, t_nbr = csr(4, T4_PAIRS)
    assert np.array_equal(off, t_off) and np.array_equal(nbr, t_nbr)
    k, off, nbr = orc.set_apply(4, off, nbr, orc.prepare_global([[1, 3], [3, 1]]), False)
    assert k == 0
    k, off, nbr = orc.set_apply(4, off, nbr, orc.prepare_global([[2, 3], [3, 2]]), False)
    assert k == 2 and int(off[4]) == 6
    k, off, nbr = orc.set_apply(4, off, nbr, orc.prepare_global(T4_PAIRS), False)
    assert int(off[4]) == 0 and off.size == 5


def test_set_apply_matches_chunked_set(ref, orc):
    # acceptance.cpp:272-320 shape: base-disjoint batch with duplicates
    n, base = ref.rmat(14, 1 << 16, 11, 0.5, 0.1, 0.1)
    off, nbr = csr(n, base)
    raw = ref.update_batch(14, 20000, 777, 0.5, 0.1, 0.1)
    keys = set(map(tuple, base.tolist()))
    batch = np.array([e for e in raw.tolist() if tuple(e) not in keys], dtype=np.uint32)
    batch = np.concatenate([batch, batch[: len(batch) // 2]])
    c = ref.chunked(n, base)
    ins = c.apply(batch, True)
    k, o2, n2 = orc.set_apply(n, off, nbr, orc.prepare_global(batch), True)
    assert k == ins > 0
    eo, en = c.export()
    assert np.array_equal(eo, o2) and np.array_equal(en, n2)
    dele = c.apply(batch, False)
    k2, o3, n3 = orc.set_apply(n, o2, n2, orc.prepare_global(batch), False)
    assert k2 == dele == ins
    assert np.array_equal(o3, off) and np.array_equal(n3, nbr)


# ------------------------------------------- priority-order consumers (§8f)
def _directed(n, p, seed):
    """Sorted unique arcs without self-loops, no reverse pairing."""
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    s, d = np.nonzero(a)
    return np.stack([s, d], axis=1).astype(np.uint32)


def _check_coloring(n, pairs, colors):
    """checks.cpp:42-58"""
    deg = np.bincount(pairs[:, 0], minlength=n) if len(pairs) else np.zeros(n, np.int64)
    assert not np.any(colors[pairs[:, 0]] == colors[pairs[:, 1]])
    assert colors.max(initial=0) <= deg.max(initial=0)


def _check_mis(n, off, nbr, flags):
    """checks.cpp:60-81"""
    src = np.repeat(np.arange(n), np.diff(off.astype(np.int64)))
    assert not np.any(flags[src] & flags[nbr])
    covered = flags.astype(bool).copy()
    covered[src[flags[nbr] == 1]] = True
    assert covered.all()


def test_kcore_known_answers(ref, orc):
    # test_algorithms.cpp:228-241
    off, nbr = csr(4, T4_PAIRS)
    assert orc.kcore(4, off, nbr).tolist() == ref.csr(4, off, nbr).kcore().tolist() == [2, 2, 2, 1]
    n, pairs = undirected(7, [(0, 1), (0, 2), (1, 3), (1, 4), (2, 5), (2, 6)], orc)
    assert orc.kcore(n, *csr(n, pairs)).tolist() == [1] * 7
    for k in (4, 9):
        n, pairs = undirected(k, complete(k), orc)
        assert orc.kcore(n, *csr(n, pairs)).tolist() == [k - 1] * k
    off, nbr = csr(5, np.zeros((0, 2), np.uint32))
    assert orc.kcore(5, off, nbr).tolist() == [0] * 5


def test_kcore_matches_reference(ref, orc):
    # test_algorithms.cpp:243-250 (seeded graphs) plus directed inputs: the
    # out-degree peel is order-independent there too
    for trial in range(15):
        n, pairs = ref.er(200, 0.03, 1700 + trial)
        off, nbr = csr(n, pairs)
        assert np.array_equal(orc.kcore(n, off, nbr), ref.csr(n, off, nbr).kcore())
    for trial in range(5):
        pairs = _directed(120, 0.05, trial)
        off, nbr = csr(120, pairs)
        assert np.array_equal(orc.kcore(120, off, nbr), ref.csr(120, off, nbr).kcore())
    n, pairs = ref.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    assert np.array_equal(orc.kcore(n, off, nbr), ref.csr(n, off, nbr).kcore())


def test_coloring_matches_reference(ref, orc):
    # test_algorithms.cpp:252-264
    off, nbr = csr(5, np.zeros((0, 2), np.uint32))
    assert orc.coloring(5, off, nbr).tolist() == ref.csr(5, off, nbr).coloring().tolist() == [0] * 5
    for trial in range(20):
        n, pairs = ref.er(120, 0.06, 1900 + trial)
        off, nbr = csr(n, pairs)
        c = orc.coloring(n, off, nbr)
        assert np.array_equal(c, ref.csr(n, off, nbr).coloring())
        _check_coloring(n, pairs, c)
    n, pairs = ref.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    c = orc.coloring(n, off, nbr)
    assert np.array_equal(c, ref.csr(n, off, nbr).coloring())
    _check_coloring(n, pairs, c)


def test_mis_matches_reference(ref, orc):
    # test_algorithms.cpp:266-292
    off, nbr = csr(4, T4_PAIRS)
    f = orc.mis(4, off, nbr, 3)
    assert np.array_equal(f, ref.csr(4, off, nbr).mis(3))
    assert (f.sum() == 1 and f[2]) or (f.sum() == 2 and f[3])
    off, nbr = csr(4, np.zeros((0, 2), np.uint32))
    assert orc.mis(4, off, nbr, 1).tolist() == [1, 1, 1, 1]
    for trial in range(50):
        n, pairs = ref.er(150, 0.05, 2100 + trial)
        off, nbr = csr(n, pairs)
        f = orc.mis(n, off, nbr, trial)
        assert np.array_equal(f, ref.csr(n, off, nbr).mis(trial))
        _check_mis(n, off, nbr, f)
    n, pairs = ref.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    f = orc.mis(n, off, nbr, 1)
    assert np.array_equal(f, ref.csr(n, off, nbr).mis(1))
    _check_mis(n, off, nbr, f)


def test_mis_is_lexicographically_first(orc):
    """The rounds give the sequential greedy MIS in (rank, id) order."""
    for trial in range(10):
        n, pairs = undirected(60, [tuple(e) for e in _directed(60, 0.1, 50 + trial)], orc)
        off, nbr = csr(n, pairs)
        f = orc.mis(n, off, nbr, trial)
        rank = [orc.rng_u64(trial, 7, v) for v in range(n)]
        chosen = np.zeros(n, np.uint8)
        blocked = np.zeros(n, bool)
        for v in sorted(range(n), key=lambda v: (rank[v], v)):
            if not blocked[v]:
                chosen[v] = 1
                blocked[nbr[off[v]:off[v + 1]]] = True
        assert np.array_equal(f, chosen)


def _check_ldd(n, off, nbr, labels):
    """checks.cpp:83-117: every vertex labelled, centres in their own
    cluster, clusters connected through same-cluster arcs."""
    assert (labels < n).all()
    assert (labels[labels] == labels).all()
    reached = labels == np.arange(n)
    stack = list(np.nonzero(reached)[0])
    while stack:
        u = stack.pop()
        for v in nbr[off[u]:off[u + 1]]:
            if not reached[v] and labels[v] == labels[u]:
                reached[v] = True
                stack.append(v)
    assert reached.all()


def test_ldd_matches_reference(ref, orc):
    # test_algorithms.cpp:90-104 (partition per trial, beta range) + exact outputs
    off, nbr = csr(4, T4_PAIRS)
    for bad in (0.0, 1.5, -1.0):
        with pytest.raises(ValueError):
            orc.ldd(4, off, nbr, bad, 1)
        with pytest.raises(RefError, match="reference error 2"):  # std::invalid_argument
            ref.csr(4, off, nbr).ldd(bad, 1)
    for trial in range(20):
        n, pairs = ref.er(150, 0.03, 700 + trial)
        off, nbr = csr(n, pairs)
        beta = (0.05, 0.2, 0.5, 1.0)[trial % 4]
        got = orc.ldd(n, off, nbr, beta, trial)
        want = ref.csr(n, off, nbr).ldd(beta, trial)
        for a, b in zip(got, want):
            assert np.array_equal(a, b), trial
        _check_ldd(n, off, nbr, got[0])
    pairs = _directed(100, 0.04, 3)  # directed: parents may be missing, still exact
    off, nbr = csr(100, pairs)
    for a, b in zip(orc.ldd(100, off, nbr, 0.3, 5), ref.csr(100, off, nbr).ldd(0.3, 5)):
        assert np.array_equal(a, b)
    n, pairs = ref.rmat(12, 16 << 12, 1)
    off, nbr = csr(n, pairs)
    for a, b in zip(orc.ldd(n, off, nbr, 0.2, 1), ref.csr(n, off, nbr).ldd(0.2, 1)):
        assert np.array_equal(a, b)


def test_bytecode_known_answers_and_reference(ref, orc):
    # test_containers.cpp:54-65: pinned wire examples
    off, nbr = csr(11, [(6, 5), (6, 7), (6, 10)])
    bo, b = orc.bytecode_encode(11, off, nbr)
    assert b[bo[6]:bo[7]].tolist() == [0x01, 0x02, 0x03] and bo[7] - bo[6] == 3 and bo[11] == 3
    off, nbr = csr(201, [(0, 200)])
    bo, b = orc.bytecode_encode(201, off, nbr)
    assert b.tolist() == [0x90, 0x03]
    off, nbr = csr(3, np.zeros((0, 2), np.uint32))
    bo, b = orc.bytecode_encode(3, off, nbr)
    assert b.size == 0 and bo.tolist() == [0, 0, 0, 0]
    for n, pairs in [ref.er(300, 0.05, 41), ref.rmat(12, 16 << 12, 1), (120, _directed(120, 0.1, 2))]:
        off, nbr = csr(n, pairs)
        want = ref.csr(n, off, nbr).compressed()
        got = orc.bytecode_encode(n, off, nbr)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_greedy_consumers_with_self_loops(ref, orc):
    """Self-loops are legal CsrGraph input (csr.cpp:9-25); kcore counts them
    in the degree, coloring / mis never let a vertex beat itself."""
    rng = np.random.default_rng(11)
    for trial in range(4):
        n, pairs = ref.er(80, 0.08, 50 + trial)
        loops = np.repeat(rng.choice(n, 10, replace=False).astype(np.uint32), 2).reshape(-1, 2)
        allp = np.unique(np.concatenate([pairs, loops]), axis=0)
        off, nbr = csr(n, allp)
        g = ref.csr(n, off, nbr)
        assert np.array_equal(orc.kcore(n, off, nbr), g.kcore())
        assert np.array_equal(orc.coloring(n, off, nbr), g.coloring())
        assert np.array_equal(orc.mis(n, off, nbr, trial), g.mis(trial))
        for a, b in zip(orc.ldd(n, off, nbr, 0.3, trial), g.ldd(0.3, trial)):
            assert np.array_equal(a, b)


def test_bfs_examined_arcs_match_survey(orc):
    """Per-level arcs inspected (measured with the reference
    library: sorted-order early exit in dense levels)."""
    n, pairs = orc.rmat(16, 16 << 16, 1)
    off, nbr = csr(n, pairs)
    assert orc.bfs_examined(n, off, nbr, 0) == [9709, 38520, 1569, 1735, 6]
    gd = golden(20)
    n, pairs = orc.rmat(20, 16 << 20, 1)
    off, nbr = csr(n, pairs)
    assert orc.bfs_examined(n, off, nbr, gd["bfs"]["source"]) == [64840, 624964, 39715, 46114, 139]

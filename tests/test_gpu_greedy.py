"""GPU parity for the §8(f) row-3 consumers on the frontier primitives:
k-core (gb::kcore, algorithms.cpp:330-374), coloring (gb::coloring,
algorithms.cpp:376-432) and MIS (gb::mis, algorithms.cpp:434-504), through
the C ABI against the C restatement (itself pinned to the reference in
tests/test_oracle.py) and the reference-generated golden digests.  All
three outputs are integers and unique for the input, so the bar is
bit-exact."""
import numpy as np
import pytest

from oracle.bindings import RMAT_A, RMAT_B, RMAT_C, digest
from tests.conftest import golden
from tests.helpers import T4_PAIRS, complete, csr, star, undirected

pytestmark = pytest.mark.gpu
KINDS = ["csr", "blocked"]


def build(gbg, kind, n, pairs):
    pairs = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
    return gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)


def directed(n, p, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    s, d = np.nonzero(a)
    return np.stack([s, d], axis=1).astype(np.uint32)


@pytest.mark.parametrize("kind", KINDS)
def test_known_answers(gbg, orc, kind):
    g = build(gbg, kind, 4, T4_PAIRS)
    assert gbg.kcore(g).tolist() == [2, 2, 2, 1]  # test_algorithms.cpp:228-232
    f = gbg.mis(g, 3)
    assert (f.sum() == 1 and f[2]) or (f.sum() == 2 and f[3])  # test_algorithms.cpp:266-281
    c = gbg.coloring(g)
    assert c[0] != c[1] != c[2] != c[0] and c[3] != c[2]
    e = build(gbg, kind, 5, [])
    assert gbg.kcore(e).tolist() == [0] * 5
    assert gbg.coloring(e).tolist() == [0] * 5  # test_algorithms.cpp:253-256
    assert gbg.mis(e, 1).tolist() == [1] * 5  # test_algorithms.cpp:282-284
    n, pairs = undirected(7, [(0, 1), (0, 2), (1, 3), (1, 4), (2, 5), (2, 6)], orc)
    assert gbg.kcore(build(gbg, kind, n, pairs)).tolist() == [1] * 7  # tree
    for k in (5, 40, 70):  # cliques: heavy colour path once k >= 64
        n, pairs = undirected(k, complete(k), orc)
        g = build(gbg, kind, n, pairs)
        assert gbg.kcore(g).tolist() == [k - 1] * k
        assert sorted(gbg.coloring(g).tolist()) == list(range(k))
        assert gbg.mis(g, 9).sum() == 1


@pytest.mark.parametrize("kind", KINDS)
def test_seeded_graphs_match_oracle(gbg, ref, orc, kind):
    for trial in range(15):
        n, pairs = ref.er(150 + 40 * trial, 0.04, 1700 + trial)
        off, nbr = csr(n, pairs)
        g = build(gbg, kind, n, pairs)
        assert np.array_equal(gbg.kcore(g), orc.kcore(n, off, nbr)), trial
        assert np.array_equal(gbg.coloring(g), orc.coloring(n, off, nbr)), trial
        for seed in (trial, 12345):
            assert np.array_equal(gbg.mis(g, seed), orc.mis(n, off, nbr, seed)), (trial, seed)


@pytest.mark.parametrize("kind", KINDS)
def test_hubs_and_stars(gbg, orc, kind):
    """Hub rows span many push tiles; a star's centre is the heavy path."""
    n, pairs = undirected(3001, star(3000), orc)
    off, nbr = csr(n, pairs)
    g = build(gbg, kind, n, pairs)
    assert gbg.kcore(g).tolist() == [1] * n
    assert np.array_equal(gbg.coloring(g), orc.coloring(n, off, nbr))
    assert np.array_equal(gbg.mis(g, 4), orc.mis(n, off, nbr, 4))
    # two dense communities bridged by hubs
    rng = np.random.default_rng(5)
    e = [(int(a), int(b)) for a, b in rng.integers(0, 400, size=(6000, 2)) if a != b]
    e += [(0, v) for v in range(1, 2000)] + [(1, v) for v in range(2, 2000, 3)]
    n, pairs = undirected(2000, e, orc)
    off, nbr = csr(n, pairs)
    g = build(gbg, kind, n, pairs)
    assert np.array_equal(gbg.kcore(g), orc.kcore(n, off, nbr))
    assert np.array_equal(gbg.coloring(g), orc.coloring(n, off, nbr))
    assert np.array_equal(gbg.mis(g, 2), orc.mis(n, off, nbr, 2))


def test_kcore_directed_and_asymmetric_rejects(gbg, ref, orc):
    """kcore's out-degree peel is order-independent on directed input too;
    coloring / mis refuse asymmetric graphs (the reference's own result is
    schedule-dependent there)."""
    for trial in range(6):
        pairs = directed(300, 0.03, trial)
        off, nbr = csr(300, pairs)
        g = gbg.CsrGraph.build(300, pairs)
        assert np.array_equal(gbg.kcore(g), orc.kcore(300, off, nbr))
        assert np.array_equal(gbg.kcore(g), ref.csr(300, off, nbr).kcore())
        with pytest.raises(ValueError):
            gbg.coloring(g)
        with pytest.raises(ValueError):
            gbg.mis(g, 1)


def test_blocked_after_updates(gbg, ref, orc):
    """The blocked container after insert/delete batches (non-contiguous
    segments) still matches the oracle on the resulting arc set."""
    n, pairs = ref.rmat(12, 16 << 12, 1)
    g = gbg.BlockedGraph.build(n, pairs)
    batch = orc.update_batch(12, 20000, 99)
    gbg.apply_insert(g, batch)
    gbg.apply_delete(g, batch[: (len(batch) // 3) & ~1])  # whole (u,v),(v,u) pairs
    off, nbr = g.to_csr()
    assert np.array_equal(gbg.kcore(g), orc.kcore(n, off, nbr))
    assert np.array_equal(gbg.coloring(g), orc.coloring(n, off, nbr))
    assert np.array_equal(gbg.mis(g, 1), orc.mis(n, off, nbr, 1))


@pytest.mark.parametrize("S", [16, 20])
def test_rmat_match_golden(gbg, S):
    gd = golden(S)
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    core = gbg.kcore(g)
    assert digest(core) == gd["kcore"]["digest"] and int(core.max()) == gd["kcore"]["max_core"]
    col = gbg.coloring(g)
    assert digest(col) == gd["coloring"]["digest"] and int(col.max()) + 1 == gd["coloring"]["colors"]
    f = gbg.mis(g, gd["mis"]["seed"])
    assert digest(f) == gd["mis"]["digest"] and int(f.sum()) == gd["mis"]["size"]


def test_scale24_match_golden(gbg):
    gd = golden(24)
    if "kcore" not in gd:
        pytest.skip("s24 greedy digests not generated")
    g = gbg.generate_rmat(24, 16 << 24, 1, RMAT_A, RMAT_B, RMAT_C)
    assert digest(gbg.kcore(g)) == gd["kcore"]["digest"]
    assert digest(gbg.coloring(g)) == gd["coloring"]["digest"]
    assert digest(gbg.mis(g, gd["mis"]["seed"])) == gd["mis"]["digest"]


@pytest.mark.parametrize("kind", KINDS)
def test_empty_single_and_self_loops(gbg, ref, orc, kind):
    """n = 0 and n = 1 handles; self-loops (CsrGraph::build accepts them,
    csr.cpp:9-25) take the reference's paths: a self-loop never beats its
    own vertex and is released like any other arc."""
    z = build(gbg, kind, 0, [])
    assert gbg.kcore(z).size == 0 and gbg.coloring(z).size == 0 and gbg.mis(z, 1).size == 0
    assert gbg.ldd(z, 0.2, 1)[0].size == 0
    one = build(gbg, kind, 1, [])
    assert gbg.kcore(one).tolist() == [0] and gbg.coloring(one).tolist() == [0] and gbg.mis(one, 1).tolist() == [1]
    rng = np.random.default_rng(11)
    for trial in range(4):
        n, pairs = ref.er(80, 0.08, 50 + trial)
        loops = np.repeat(rng.choice(n, 10, replace=False).astype(np.uint32), 2).reshape(-1, 2)
        allp = np.unique(np.concatenate([pairs, loops]), axis=0)
        off, nbr = csr(n, allp)
        g = build(gbg, kind, n, allp)
        want_ref = ref.csr(n, off, nbr)
        assert np.array_equal(gbg.kcore(g), want_ref.kcore())
        assert np.array_equal(gbg.kcore(g), orc.kcore(n, off, nbr))
        assert np.array_equal(gbg.coloring(g), orc.coloring(n, off, nbr))
        assert np.array_equal(gbg.mis(g, trial), orc.mis(n, off, nbr, trial))
        for a, b in zip(gbg.ldd(g, 0.3, trial), want_ref.ldd(0.3, trial)):
            assert np.array_equal(a, b)

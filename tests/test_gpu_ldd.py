"""GPU parity for gb::ldd (algorithms.cpp:114-188): labels, parents and
rounds bit-exact against the C restatement (pinned to the reference in
tests/test_oracle.py) and the reference-generated golden digests.  The
device Exponential shifts must equal the host C library's, so the device
log1p is first checked bit for bit against the reference's own libm call."""
import numpy as np
import pytest

from oracle.bindings import RMAT_A, RMAT_B, RMAT_C, digest
from tests.conftest import golden
from tests.helpers import T4_PAIRS, csr, undirected

pytestmark = pytest.mark.gpu


def build(gbg, kind, n, pairs):
    pairs = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
    return gbg.CsrGraph.build(n, pairs) if kind == "csr" else gbg.BlockedGraph.build(n, pairs)


def test_device_log1p_matches_host_libm(gbg, ref):
    rng = np.random.default_rng(0)
    u = rng.random(1 << 22)  # k * 2^-53, the form of rng_double
    xs = [-u,  # the ldd arguments: -rng_double
          rng.uniform(-1.0, 1.0, 1 << 20),
          -np.ldexp(rng.random(1 << 18), -rng.integers(0, 60, 1 << 18)),
          np.ldexp(rng.random(1 << 18), -rng.integers(0, 60, 1 << 18)),
          np.array([0.0, -0.0, -1.0, -0.5, 0.41422, -0.2929, 1e-300, 2.0 ** -29, 1e3, 1e300])]
    for x in xs:
        got, want = gbg.selftest_log1p(x), ref.log1p(x)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("kind", ["csr", "blocked"])
def test_ldd_matches_oracle(gbg, ref, orc, kind):
    g = build(gbg, kind, 4, T4_PAIRS)
    for bad in (0.0, 1.5):
        with pytest.raises(ValueError):
            gbg.ldd(g, bad, 1)
    e = build(gbg, kind, 6, [])
    lab, par, rnd = gbg.ldd(e, 0.2, 1)
    assert lab.tolist() == list(range(6)) and par.tolist() == list(range(6))
    for trial in range(16):
        n, pairs = ref.er(120 + 60 * trial, 0.03, 700 + trial)
        off, nbr = csr(n, pairs)
        beta = (0.05, 0.2, 0.5, 1.0)[trial % 4]
        got = gbg.ldd(build(gbg, kind, n, pairs), beta, trial)
        want = orc.ldd(n, off, nbr, beta, trial)
        for a, b in zip(got, want):
            assert np.array_equal(a, b), trial


def test_ldd_directed_and_hubs(gbg, orc):
    rng = np.random.default_rng(9)
    a = rng.random((300, 300)) < 0.02
    np.fill_diagonal(a, False)
    s, d = np.nonzero(a)
    pairs = np.stack([s, d], axis=1).astype(np.uint32)
    off, nbr = csr(300, pairs)
    for x, y in zip(gbg.ldd(gbg.CsrGraph.build(300, pairs), 0.3, 4), orc.ldd(300, off, nbr, 0.3, 4)):
        assert np.array_equal(x, y)
    e = [(0, v) for v in range(1, 5000)] + [(v, v + 1) for v in range(1, 4999, 2)]
    n, pairs = undirected(5000, e, orc)
    off, nbr = csr(n, pairs)
    for x, y in zip(gbg.ldd(gbg.CsrGraph.build(n, pairs), 0.2, 2), orc.ldd(n, off, nbr, 0.2, 2)):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("S", [16, 20, 24])
def test_ldd_rmat_golden(gbg, S):
    gd = golden(S)
    if "ldd" not in gd:
        pytest.skip("ldd digests not generated")
    g = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C)
    lab, par, rnd = gbg.ldd(g, gd["ldd"]["beta"], gd["ldd"]["seed"])
    assert digest(lab) == gd["ldd"]["labels_digest"]
    assert digest(par) == gd["ldd"]["parents_digest"]
    assert digest(rnd) == gd["ldd"]["rounds_digest"]
    assert int((lab == np.arange(lab.size)).sum()) == gd["ldd"]["clusters"]

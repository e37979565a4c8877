"""GPU parity for the compressed CSR container (§8f row 4):
gb::CompressedCsrGraph (compressed_csr.hpp:12-46) with the byte code of
bytecode.hpp:11-62, encoded and decoded on the device.  The device encoding
must be byte-identical to the reference's (and the C restatement's), the
warp-parallel decode must give back the lists, and every algorithm on a
compressed handle must equal the CSR result."""
import numpy as np
import pytest

from oracle.bindings import RMAT_A, RMAT_B, RMAT_C, digest
from tests.conftest import golden
from tests.helpers import T4_PAIRS, csr

pytestmark = pytest.mark.gpu
TINY = np.finfo(np.float64).tiny


def test_wire_examples(gbg):
    # test_containers.cpp:54-65
    z = gbg.CompressedGraph.build(11, [(6, 5), (6, 7), (6, 10)])
    bo, b = z.encoding()
    assert b[bo[6]:bo[7]].tolist() == [0x01, 0x02, 0x03] and bo[11] == 3
    assert z.map_neighbors(6).tolist() == [5, 7, 10] and z.degree(6) == 3 and z.degree(5) == 0
    z = gbg.CompressedGraph.build(201, [(0, 200)])
    assert z.encoding()[1].tolist() == [0x90, 0x03]
    z = gbg.CompressedGraph.build(3, np.zeros((0, 2), np.uint32))
    assert z.encoding()[1].size == 0 and z.num_edges() == 0


def test_static_container_contract(gbg):
    """test_containers.cpp:26-52: static, rejects updates; capabilities
    {1,1,1,0,0,0} (compressed_csr.hpp:27-29)."""
    z = gbg.CompressedGraph.build(4, T4_PAIRS)
    caps = z.capabilities()
    assert [caps[k] for k in ("has_num_edges", "has_degree", "has_map_early_exit", "has_parallel_map",
                              "has_parallel_map_early_exit", "has_batch_updates")] == [1, 1, 1, 0, 0, 0]
    with pytest.raises(NotImplementedError):
        z.insert_batch(np.array([[0, 3]], np.uint32))
    with pytest.raises(NotImplementedError):
        z.delete_edge(0, 1)
    with pytest.raises(IndexError):
        z.degree(9)
    assert z.memory_bytes() > 0
    with pytest.raises(Exception):
        gbg.CompressedGraph.from_csr(np.array([0, 2, 1], np.uint64), np.array([1, 0], np.uint32))


def test_encoding_matches_reference(gbg, ref, orc):
    cases = [ref.er(400, 0.05, 41), ref.rmat(14, 16 << 14, 1)]
    for nn, pairs in cases:
        off, nbr = csr(nn, pairs)
        want = ref.csr(nn, off, nbr).compressed()
        for src in (gbg.CsrGraph.build(nn, pairs), gbg.BlockedGraph.build(nn, pairs)):
            z = gbg.CompressedGraph.from_graph(src)
            got = z.encoding()
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
            o2, n2 = z.to_csr()
            assert np.array_equal(o2, off) and np.array_equal(n2, nbr)
    # 4- and 5-byte varints: a 2^28 gap and a first neighbour 2^28 below its source
    nn = (1 << 28) + 1
    lists = {5: [1, 1 << 20, 1 << 28], 1 << 28: [0, 7]}
    pairs = np.array([(v, u) for v in sorted(lists) for u in lists[v]], np.uint32)
    z = gbg.CompressedGraph.build(nn, pairs)
    for v, lst in lists.items():
        assert z.map_neighbors(v).tolist() == lst
    bo, b = z.encoding()
    assert b.tolist() == _encode(5, lists[5]) + _encode(1 << 28, lists[1 << 28])
    assert bo[6] == len(_encode(5, lists[5])) and bo[nn] == b.size


def _encode(v, lst):
    """bytecode_encode (bytecode.hpp:11-27), restated for the test."""
    out = []
    for i, x in enumerate(lst):
        d = x - v if i == 0 else x - lst[i - 1]
        z = d if i > 0 else (2 * d if d >= 0 else -2 * d - 1)  # gaps plain, first zig-zag
        while True:
            byte, z = z & 0x7F, z >> 7
            out.append(byte | (0x80 if z else 0))
            if not z:
                break
    return out


@pytest.mark.parametrize("S", [16, 20])
def test_rmat_compressed_algorithms_match_golden(gbg, S):
    gd = golden(S)
    z = gbg.generate_rmat(S, 16 << S, 1, RMAT_A, RMAT_B, RMAT_C, kind=gbg.KIND_COMPRESSED)
    assert (z.num_vertices(), z.num_edges()) == (gd["n"], gd["m"])
    off, nbr = z.to_csr()
    assert digest(off) == gd["off_digest"] and digest(nbr) == gd["nbr_digest"]
    r = gbg.bfs(z, gd["bfs"]["source"])
    assert digest(r.depth) == gd["bfs"]["digest"] and r.modes == gd["bfs"]["modes"]
    assert digest(gbg.cc(z)) == gd["cc"]["digest"]
    assert gbg.triangle_count(z) == gd["tc"]["triangles"]
    assert digest(gbg.kcore(z)) == gd["kcore"]["digest"]
    assert digest(gbg.coloring(z)) == gd["coloring"]["digest"]
    assert digest(gbg.mis(z, 1)) == gd["mis"]["digest"]
    assert digest(gbg.ldd(z, 0.2, 1)[0]) == gd["ldd"]["labels_digest"]
    p = gbg.pagerank(z, 0.85, 20, TINY)
    ids = np.array(gd["pagerank"]["sample_ids"])
    want = np.array([float.fromhex(h) for h in gd["pagerank"]["sample_hex"]])
    assert float(np.abs(p[ids] - want).sum() / np.abs(want).sum()) <= 1e-9
    gbg.pagerank_prepare(z)  # the tiled index path on the compressed container
    p = gbg.pagerank(z, 0.85, 20, TINY)
    assert float(np.abs(p[ids] - want).sum() / np.abs(want).sum()) <= 1e-9
    with gbg.CsrGraph.from_csr(off, nbr) as c:
        assert np.array_equal(gbg.bc(z, 0), gbg.bc(c, 0))


def test_gbcsr1_into_compressed(gbg, tmp_path):
    g = gbg.generate_rmat(12, 16 << 12, 1, RMAT_A, RMAT_B, RMAT_C)
    path = str(tmp_path / "g.gbcsr1")
    gbg.save_binary(g, path)
    z = gbg.load_binary(path, gbg.KIND_COMPRESSED)
    assert isinstance(z, gbg.CompressedGraph)
    o1, n1 = g.to_csr()
    o2, n2 = z.to_csr()
    assert np.array_equal(o1, o2) and np.array_equal(n1, n2)
    path2 = str(tmp_path / "z.gbcsr1")
    gbg.save_binary(z, path2)
    assert open(path, "rb").read() == open(path2, "rb").read()

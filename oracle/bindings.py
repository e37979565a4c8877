"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Ref``: the UNMODIFIED reference library (``/root/reference/proj/src``
  compiled in place by ``oracle/Makefile`` into ``oracle/_ref/libgbref.so``,
  entry points in ``oracle/ref_shim.cpp``).
* ``Oracle``: our plain-C restatement (``oracle/gbo.c`` -> ``oracle/liboracle.so``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product library never does.  ``digest`` is the
array fingerprint shared by the golden fixtures and the GPU parity tests.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgbref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

# BASELINE.json R-MAT parameters (Graph500): a=.57, b=c=.19 (d=.05 implied).
RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------- digest
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(x: np.ndarray) -> np.ndarray:
    x = x + _G
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def digest(a: np.ndarray, chunk: int = 1 << 24) -> int:
    """Order-sensitive 64-bit fingerprint: sum_i mix(v_i + mix(i)) mod 2^64,
    values taken as their integer bit patterns widened to uint64."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        a = a.view(np.uint64)
    elif a.dtype == np.int32:
        a = a.view(np.uint32)
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for s in range(0, a.size, chunk):
            v = a[s : s + chunk].astype(np.uint64)
            i = np.arange(s, s + v.size, dtype=np.uint64)
            total = total + np.sum(_mix(v + _mix(i)), dtype=np.uint64)
    return int(total)


def csr_from_pairs(n: int, pairs: np.ndarray):
    """Sorted, deduplicated (src,dst) pairs -> (offsets u64[n+1], nbrs u32[m])."""
    pairs = pairs.reshape(-1, 2)
    counts = np.bincount(pairs[:, 0].astype(np.int64), minlength=n).astype(np.uint64)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(counts, out=off[1:])
    return off, np.ascontiguousarray(pairs[:, 1], dtype=np.uint32)


def max_degree_source(off: np.ndarray) -> int:
    """Lowest-id vertex of maximum degree (BASELINE configs' BFS source)."""
    deg = np.diff(off.astype(np.int64))
    return int(np.argmax(deg))


# ---------------------------------------------------------------- reference
class RefError(RuntimeError):
    pass


class Ref:
    """The reference library itself (oracle/_ref/libgbref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.L = C.CDLL(path)
        L.gbref_last_error.restype = C.c_char_p
        L.gbref_rmat.restype = C.c_void_p
        L.gbref_rmat.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64]
        L.gbref_er.restype = C.c_void_p
        L.gbref_er.argtypes = [C.c_uint64, C.c_double, C.c_uint64]
        L.gbref_t4.restype = C.c_void_p
        L.gbref_normalize.restype = C.c_void_p
        L.gbref_normalize.argtypes = [_u32p, C.c_uint64, C.c_uint64]
        for f in ("gbref_graph_n", "gbref_graph_m"):
            getattr(L, f).restype = C.c_uint64
            getattr(L, f).argtypes = [C.c_void_p]
        L.gbref_graph_arcs.argtypes = [C.c_void_p, _u32p]
        L.gbref_graph_free.argtypes = [C.c_void_p]
        L.gbref_csr_create.restype = C.c_void_p
        L.gbref_csr_create.argtypes = [C.c_uint64, _u64p, _u32p]
        L.gbref_csr_from_pairs.restype = C.c_void_p
        L.gbref_csr_from_pairs.argtypes = [C.c_uint64, _u32p, C.c_uint64]
        L.gbref_csr_free.argtypes = [C.c_void_p]
        L.gbref_bfs.argtypes = [C.c_void_p, C.c_uint32, _i32p]
        L.gbref_bfs_trace.argtypes = [C.c_void_p, C.c_uint32, _i32p, _u64p, C.c_uint64, _u64p]
        L.gbref_pagerank.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_double, _f64p]
        L.gbref_cc.argtypes = [C.c_void_p, _u32p]
        L.gbref_edge_map.argtypes = [C.c_void_p, _u32p, C.c_uint64, _u8p, C.c_int, C.c_int, _u8p, _u64p,
                                     C.POINTER(C.c_int)]
        L.gbref_update_batch.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                         C.c_uint64, _u32p]
        L.gbref_prepare_global.argtypes = [_u32p, C.c_uint64, _u32p, _u64p]
        L.gbref_chunked_build.restype = C.c_void_p
        L.gbref_chunked_build.argtypes = [C.c_uint64, _u32p, C.c_uint64]
        L.gbref_container_free.argtypes = [C.c_void_p]
        L.gbref_chunked_apply.argtypes = [C.c_void_p, _u32p, C.c_uint64, C.c_int, _u64p]
        for f in ("gbref_container_m", "gbref_container_n"):
            getattr(L, f).restype = C.c_uint64
            getattr(L, f).argtypes = [C.c_void_p]
        L.gbref_container_degree.restype = C.c_uint64
        L.gbref_container_degree.argtypes = [C.c_void_p, C.c_uint32]
        L.gbref_container_export.argtypes = [C.c_void_p, _u64p, _u32p]
        L.gbref_container_bfs.argtypes = [C.c_void_p, C.c_uint32, _i32p]
        L.gbref_hash_combine.restype = C.c_uint64
        L.gbref_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
        L.gbref_mix64.restype = C.c_uint64
        L.gbref_mix64.argtypes = [C.c_uint64]
        L.gbref_rng_double.restype = C.c_double
        L.gbref_rng_double.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.gbref_set_threads.argtypes = [C.c_int]
        L.gbref_num_threads.restype = C.c_int

    def _check(self, rc: int):
        if rc != 0:
            raise RefError(f"reference error {rc}: {self.L.gbref_last_error().decode()}")

    def set_threads(self, t: int):
        self.L.gbref_set_threads(t)

    def num_threads(self) -> int:
        return self.L.gbref_num_threads()

    def hash_combine(self, a: int, b: int) -> int:
        return self.L.gbref_hash_combine(a, b)

    def vertex_filter_sparse(self, n, ids, keep):
        """vertex_filter (traversal.cpp:117-131) on a sparse VertexSubset."""
        self._bind_vertex_filter()
        return _ref_vertex_filter(self, n, ids, None, keep)

    def vertex_filter_dense(self, n, words, keep):
        """vertex_filter on a dense VertexSubset; the result stays dense."""
        self._bind_vertex_filter()
        return _ref_vertex_filter(self, n, None, words, keep)

    def _bind_vertex_filter(self):
        f = self.L.gbref_vertex_filter
        f.argtypes = [C.c_uint64, _u32p, C.c_uint64, _u64p, _u8p, _u32p, _u64p, C.POINTER(C.c_uint64),
                      C.POINTER(C.c_int)]
        f.restype = C.c_int

    def log1p(self, x):
        """std::log1p as the reference's C library computes it (rng.hpp:33)."""
        self.L.gbref_log1p.argtypes = [_f64p, C.c_uint64, _f64p]
        self.L.gbref_log1p.restype = None
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self.L.gbref_log1p(ptr(x, _f64p), x.size, ptr(out, _f64p))
        return out

    # graphs -> (n, pairs[m,2] u32)
    def _take_graph(self, h):
        if not h:
            raise RefError(self.L.gbref_last_error().decode())
        n = self.L.gbref_graph_n(h)
        m = self.L.gbref_graph_m(h)
        pairs = np.empty((m, 2), dtype=np.uint32)
        if m:
            self.L.gbref_graph_arcs(h, ptr(pairs, _u32p))
        self.L.gbref_graph_free(h)
        return n, pairs

    def rmat(self, log2_n, arcs, seed, a=RMAT_A, b=RMAT_B, c=RMAT_C):
        return self._take_graph(self.L.gbref_rmat(log2_n, arcs, a, b, c, seed))

    def er(self, n, p, seed):
        return self._take_graph(self.L.gbref_er(n, p, seed))

    def t4(self):
        return self._take_graph(self.L.gbref_t4())

    def normalize(self, undirected_pairs, min_n):
        up = np.ascontiguousarray(np.asarray(undirected_pairs, dtype=np.uint32).reshape(-1, 2))
        return self._take_graph(self.L.gbref_normalize(ptr(up, _u32p), up.shape[0], min_n))

    # CSR handle
    def csr(self, n, off, nbr):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        h = self.L.gbref_csr_create(n, ptr(off, _u64p), ptr(nbr, _u32p))
        if not h:
            raise RefError(self.L.gbref_last_error().decode())
        return RefCsr(self, h, n)

    def update_batch(self, log2_n, size, seed, a=RMAT_A, b=RMAT_B, c=RMAT_C):
        out = np.empty((2 * size, 2), dtype=np.uint32)
        self._check(self.L.gbref_update_batch(log2_n, a, b, c, size, seed, ptr(out, _u32p)))
        return out

    def load_binary(self, path):
        """gb::load_binary_csr (io.cpp:87-110) -> (n, offsets, neighbors)."""
        L = self.L
        L.gbref_load_binary.restype = C.c_void_p
        L.gbref_load_binary.argtypes = [C.c_char_p]
        for f in ("gbref_csr_n", "gbref_csr_m"):
            getattr(L, f).restype = C.c_uint64
            getattr(L, f).argtypes = [C.c_void_p]
        L.gbref_csr_arrays.argtypes = [C.c_void_p, _u64p, _u32p]
        h = L.gbref_load_binary(os.fsencode(path))
        if not h:
            raise RefError(L.gbref_last_error().decode())
        n, m = L.gbref_csr_n(h), L.gbref_csr_m(h)
        off = np.empty(n + 1, dtype=np.uint64)
        nbr = np.empty(max(m, 1), dtype=np.uint32)
        L.gbref_csr_arrays(h, ptr(off, _u64p), ptr(nbr, _u32p))
        L.gbref_csr_free(h)
        return n, off, nbr[:m]

    def load_binary_graph(self, path):
        """gb::load_binary_csr (io.cpp:87-110), kept as a reference CsrGraph
        (the input path bench.cpp uses for cached graphs)."""
        L = self.L
        L.gbref_load_binary.restype = C.c_void_p
        L.gbref_load_binary.argtypes = [C.c_char_p]
        L.gbref_csr_n.restype = C.c_uint64
        L.gbref_csr_n.argtypes = [C.c_void_p]
        h = L.gbref_load_binary(os.fsencode(path))
        if not h:
            raise RefError(L.gbref_last_error().decode())
        return RefCsr(self, h, int(L.gbref_csr_n(h)))

    def prepare_global(self, pairs):
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
        out = np.empty_like(pairs)
        cnt = C.c_uint64(0)
        self._check(self.L.gbref_prepare_global(ptr(pairs, _u32p), pairs.shape[0], ptr(out, _u32p),
                                                C.byref(cnt)))
        return out[: cnt.value]

    def chunked(self, n, pairs):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        h = self.L.gbref_chunked_build(n, ptr(pairs, _u32p), pairs.shape[0])
        if not h:
            raise RefError(self.L.gbref_last_error().decode())
        return RefChunked(self, h)


class RefCsr:
    def __init__(self, ref: Ref, h, n):
        self.ref, self.h, self.n = ref, h, n

    def __del__(self):
        try:
            self.ref.L.gbref_csr_free(self.h)
        except Exception:
            pass

    @property
    def m(self):
        L = self.ref.L
        L.gbref_csr_m.restype = C.c_uint64
        L.gbref_csr_m.argtypes = [C.c_void_p]
        return int(L.gbref_csr_m(self.h))

    def bfs(self, src):
        out = np.empty(self.n, dtype=np.int32)
        self.ref._check(self.ref.L.gbref_bfs(self.h, src, ptr(out, _i32p)))
        return out

    def save_binary(self, path):
        """gb::save_binary (io.cpp:75-85)."""
        L = self.ref.L
        L.gbref_save_binary.argtypes = [C.c_void_p, C.c_char_p]
        self.ref._check(L.gbref_save_binary(self.h, os.fsencode(path)))

    def bfs_trace(self, src, cap=64):
        modes = np.zeros(cap, dtype=np.int32)
        sizes = np.zeros(cap, dtype=np.uint64)
        lv = C.c_uint64(0)
        self.ref._check(self.ref.L.gbref_bfs_trace(self.h, src, ptr(modes, _i32p), ptr(sizes, _u64p), cap,
                                                   C.byref(lv)))
        k = min(lv.value, cap)
        return [int(x) for x in modes[:k]], [int(x) for x in sizes[:k]]

    def pagerank(self, damping=0.85, iters=20, tol=np.finfo(np.float64).tiny):
        out = np.empty(self.n, dtype=np.float64)
        self.ref._check(self.ref.L.gbref_pagerank(self.h, damping, iters, tol, ptr(out, _f64p)))
        return out

    def time_pagerank(self, damping=0.85, iters=20, tol=np.finfo(np.float64).tiny):
        """Seconds of one gb::pagerank call (steady_clock inside the shim) and
        the rank sum."""
        L = self.ref.L
        L.gbref_time_pagerank.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_double, _f64p, _f64p]
        sec, tot = C.c_double(), C.c_double()
        self.ref._check(L.gbref_time_pagerank(self.h, damping, iters, tol, C.byref(sec), C.byref(tot)))
        return sec.value, tot.value

    def time_bfs(self, src):
        L = self.ref.L
        L.gbref_time_bfs.argtypes = [C.c_void_p, C.c_uint32, _f64p, _u64p]
        sec, k = C.c_double(), C.c_uint64()
        self.ref._check(L.gbref_time_bfs(self.h, src, C.byref(sec), C.byref(k)))
        return sec.value, k.value

    def time_cc(self):
        L = self.ref.L
        L.gbref_time_cc.argtypes = [C.c_void_p, _f64p, _u64p]
        sec, k = C.c_double(), C.c_uint64()
        self.ref._check(L.gbref_time_cc(self.h, C.byref(sec), C.byref(k)))
        return sec.value, k.value

    def cc(self):
        out = np.empty(self.n, dtype=np.uint32)
        self.ref._check(self.ref.L.gbref_cc(self.h, ptr(out, _u32p)))
        return out

    def bc(self, src):
        """gb::bc (algorithms.cpp:60-103)."""
        L = self.ref.L
        L.gbref_bc.argtypes = [C.c_void_p, C.c_uint32, _f64p]
        out = np.empty(self.n, dtype=np.float64)
        self.ref._check(L.gbref_bc(self.h, src, ptr(out, _f64p)))
        return out

    def kcore(self):
        """gb::kcore (algorithms.cpp:330-374)."""
        L = self.ref.L
        L.gbref_kcore.argtypes = [C.c_void_p, _u64p]
        out = np.empty(self.n, dtype=np.uint64)
        self.ref._check(L.gbref_kcore(self.h, ptr(out, _u64p)))
        return out

    def coloring(self):
        """gb::coloring (algorithms.cpp:376-432)."""
        L = self.ref.L
        L.gbref_coloring.argtypes = [C.c_void_p, _u32p]
        out = np.empty(self.n, dtype=np.uint32)
        self.ref._check(L.gbref_coloring(self.h, ptr(out, _u32p)))
        return out

    def mis(self, seed=1):
        """gb::mis (algorithms.cpp:434-504)."""
        L = self.ref.L
        L.gbref_mis.argtypes = [C.c_void_p, C.c_uint64, _u8p]
        out = np.empty(self.n, dtype=np.uint8)
        self.ref._check(L.gbref_mis(self.h, seed, ptr(out, _u8p)))
        return out

    def compressed(self):
        """CompressedCsrGraph::build (compressed_csr.cpp:5-17) -> (byte_offsets, bytes)."""
        L = self.ref.L
        L.gbref_compressed.argtypes = [C.c_void_p, _u64p, _u8p, _u64p]
        nb = C.c_uint64()
        self.ref._check(L.gbref_compressed(self.h, None, None, C.byref(nb)))
        off = np.empty(self.n + 1, dtype=np.uint64)
        b = np.empty(max(nb.value, 1), dtype=np.uint8)
        self.ref._check(L.gbref_compressed(self.h, ptr(off, _u64p), ptr(b, _u8p), C.byref(nb)))
        return off, b[: nb.value]

    def ldd(self, beta=0.2, seed=1):
        """gb::ldd (algorithms.cpp:114-188) -> (labels, parents, rounds)."""
        L = self.ref.L
        L.gbref_ldd.argtypes = [C.c_void_p, C.c_double, C.c_uint64, _u32p, _u32p, _u64p]
        lab = np.empty(self.n, dtype=np.uint32)
        par = np.empty(self.n, dtype=np.uint32)
        rnd = np.empty(self.n, dtype=np.uint64)
        self.ref._check(L.gbref_ldd(self.h, beta, seed, ptr(lab, _u32p), ptr(par, _u32p), ptr(rnd, _u64p)))
        return lab, par, rnd

    def edge_map(self, ids, cond_mask, mode, early_exit=True):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        cond = np.ascontiguousarray(cond_mask, dtype=np.uint8)
        out = np.zeros(self.n, dtype=np.uint8)
        upd = C.c_uint64(0)
        chosen = C.c_int(0)
        self.ref._check(self.ref.L.gbref_edge_map(self.h, ptr(ids, _u32p), ids.size, ptr(cond, _u8p), mode,
                                                  int(early_exit), ptr(out, _u8p), C.byref(upd),
                                                  C.byref(chosen)))
        return out.astype(bool), upd.value, chosen.value


def _ref_vertex_filter(ref, n, ids, words, keep):
    keep = np.ascontiguousarray(keep, dtype=np.uint8)
    k = C.c_uint64(0)
    dense = C.c_int(0)
    nw = (n + 63) // 64
    out_words = np.zeros(max(nw, 1), dtype=np.uint64)
    if words is None:
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        out_ids = np.empty(max(ids.size, 1), dtype=np.uint32)
        ref._check(ref.L.gbref_vertex_filter(n, ptr(ids, _u32p), ids.size, None, ptr(keep, _u8p),
                                             ptr(out_ids, _u32p), ptr(out_words, _u64p), C.byref(k),
                                             C.byref(dense)))
        assert not dense.value
        return out_ids[: k.value].copy()
    words = np.ascontiguousarray(words, dtype=np.uint64)
    out_ids = np.empty(1, dtype=np.uint32)
    ref._check(ref.L.gbref_vertex_filter(n, None, 0, ptr(words, _u64p), ptr(keep, _u8p), ptr(out_ids, _u32p),
                                         ptr(out_words, _u64p), C.byref(k), C.byref(dense)))
    assert dense.value
    return out_words[:nw].copy()


class RefChunked:
    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h
        self.n = ref.L.gbref_container_n(h)

    def __del__(self):
        try:
            self.ref.L.gbref_container_free(self.h)
        except Exception:
            pass

    @property
    def m(self):
        return self.ref.L.gbref_container_m(self.h)

    def apply(self, pairs, insert: bool) -> int:
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        applied = C.c_uint64(0)
        self.ref._check(self.ref.L.gbref_chunked_apply(self.h, ptr(pairs, _u32p), pairs.shape[0], int(insert),
                                                       C.byref(applied)))
        return applied.value

    def apply_timed(self, pairs, insert: bool):
        """(applied, seconds of prepare + apply) as bench.cpp:171-186 times them."""
        L = self.ref.L
        L.gbref_chunked_apply_timed.argtypes = [C.c_void_p, _u32p, C.c_uint64, C.c_int, _u64p, _f64p]
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        applied, sec = C.c_uint64(0), C.c_double()
        self.ref._check(L.gbref_chunked_apply_timed(self.h, ptr(pairs, _u32p), pairs.shape[0], int(insert),
                                                    C.byref(applied), C.byref(sec)))
        return applied.value, sec.value

    def time_bfs(self, src):
        L = self.ref.L
        L.gbref_container_bfs_timed.argtypes = [C.c_void_p, C.c_uint32, _f64p, _u64p]
        sec, k = C.c_double(), C.c_uint64()
        self.ref._check(L.gbref_container_bfs_timed(self.h, src, C.byref(sec), C.byref(k)))
        return sec.value, k.value

    def export(self):
        off = np.empty(self.n + 1, dtype=np.uint64)
        nbr = np.empty(self.m, dtype=np.uint32)
        self.ref._check(self.ref.L.gbref_container_export(self.h, ptr(off, _u64p), ptr(nbr, _u32p)))
        return off, nbr

    def bfs(self, src):
        out = np.empty(self.n, dtype=np.int32)
        self.ref._check(self.ref.L.gbref_container_bfs(self.h, src, ptr(out, _i32p)))
        return out


# ---------------------------------------------------------------- restatement
class Oracle:
    """Plain-C restatement (oracle/gbo.c), pinned against ``Ref`` and goldens."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle restatement`")
        L = self.L = C.CDLL(path)
        L.gbo_mix64.restype = C.c_uint64
        L.gbo_mix64.argtypes = [C.c_uint64]
        L.gbo_hash_combine.restype = C.c_uint64
        L.gbo_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
        L.gbo_rng_double.restype = C.c_double
        L.gbo_rng_double.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.gbo_rng_u64.restype = C.c_uint64
        L.gbo_rng_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.gbo_update_batch.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                       C.c_uint64, _u32p]
        L.gbo_normalize.restype = C.c_uint64
        L.gbo_normalize.argtypes = [_u32p, C.c_uint64, C.c_uint64, _u32p, _u64p]
        L.gbo_prepare_global.restype = C.c_uint64
        L.gbo_prepare_global.argtypes = [_u32p, C.c_uint64, _u32p]
        L.gbo_csr_build.argtypes = [C.c_uint64, _u32p, C.c_uint64, _u64p, _u32p]
        L.gbo_bfs.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint32, _i32p, _i32p, _u64p, C.c_uint64, _u64p]
        L.gbo_pagerank.argtypes = [C.c_uint64, _u64p, _u32p, C.c_double, C.c_uint64, C.c_double, _f64p]
        L.gbo_cc.argtypes = [C.c_uint64, _u64p, _u32p, _u32p]
        L.gbo_tc.restype = C.c_uint64
        L.gbo_tc.argtypes = [C.c_uint64, _u64p, _u32p]
        L.gbo_subset_to_dense.argtypes = [C.c_uint64, _u32p, C.c_uint64, _u64p]
        L.gbo_subset_to_sparse.restype = C.c_uint64
        L.gbo_subset_to_sparse.argtypes = [C.c_uint64, _u64p, _u32p]
        L.gbo_edge_map.argtypes = [C.c_uint64, _u64p, _u32p, _u32p, C.c_uint64, _u8p, C.c_int, C.c_int, _u8p,
                                   _u64p]
        L.gbo_set_apply.restype = C.c_uint64
        L.gbo_set_apply.argtypes = [C.c_uint64, _u64p, _u32p, _u32p, C.c_uint64, C.c_int, _u64p, _u32p]

    def rmat_csr(self, log2_n, draws, seed, a=RMAT_A, b=RMAT_B, c=RMAT_C):
        """generate_rmat (generators.cpp:67-72) as (offsets, neighbours),
        OpenMP on every host core (oracle/gbo_omp.c)."""
        L = self.L
        L.gbo_rmat_csr_omp.restype = C.c_uint64
        L.gbo_rmat_csr_omp.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                       _u64p, C.POINTER(_u32p)]
        L.gbo_free.argtypes = [C.c_void_p]
        n = 1 << log2_n
        off = np.empty(n + 1, dtype=np.uint64)
        p = _u32p()
        m = L.gbo_rmat_csr_omp(log2_n, a, b, c, draws, seed, ptr(off, _u64p), C.byref(p))
        if m == (1 << 64) - 1:
            raise MemoryError("gbo_rmat_csr_omp: out of host memory")
        nbr = np.ctypeslib.as_array(p, shape=(max(m, 1),))[:m].copy()
        L.gbo_free(C.cast(p, C.c_void_p))
        return off, nbr

    def save_gbcsr1(self, path, n, off, nbr):
        """GBCSR1 file as gb::save_binary writes it (io.cpp:75-85)."""
        L = self.L
        L.gbo_save_gbcsr1.argtypes = [C.c_char_p, C.c_uint64, _u64p, _u32p]
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        if L.gbo_save_gbcsr1(os.fsencode(path), n, ptr(off, _u64p), ptr(nbr if nbr.size else np.zeros(1, np.uint32), _u32p)):
            raise OSError(f"cannot write {path}")

    def update_batch(self, log2_n, size, seed, a=RMAT_A, b=RMAT_B, c=RMAT_C):
        out = np.empty((2 * size, 2), dtype=np.uint32)
        self.L.gbo_update_batch(log2_n, a, b, c, size, seed, ptr(out, _u32p))
        return out

    def normalize(self, raw_pairs, min_n):
        raw = np.ascontiguousarray(np.asarray(raw_pairs, dtype=np.uint32).reshape(-1, 2))
        out = np.empty((2 * raw.shape[0] + 1, 2), dtype=np.uint32)
        n = C.c_uint64(0)
        m = self.L.gbo_normalize(ptr(raw, _u32p), raw.shape[0], min_n, ptr(out, _u32p), C.byref(n))
        return n.value, out[:m].copy()

    def rmat(self, log2_n, arcs, seed, a=RMAT_A, b=RMAT_B, c=RMAT_C):
        """generators.cpp:67-72 = update batch + normalize with n = 2^log2_n."""
        return self.normalize(self.update_batch(log2_n, arcs, seed, a, b, c), 1 << log2_n)

    def prepare_global(self, pairs):
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
        out = np.empty_like(p)
        k = self.L.gbo_prepare_global(ptr(p, _u32p), p.shape[0], ptr(out, _u32p))
        return out[:k].copy()

    def csr(self, n, pairs):
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
        off = np.empty(n + 1, dtype=np.uint64)
        nbr = np.empty(max(p.shape[0], 1), dtype=np.uint32)
        rc = self.L.gbo_csr_build(n, ptr(p, _u32p), p.shape[0], ptr(off, _u64p), ptr(nbr, _u32p))
        if rc:
            raise ValueError("csr_build: format error")
        return off, nbr[: p.shape[0]]

    def bfs_examined(self, n, off, nbr, src, cap=64):
        """Arcs inspected per level in the reference's order (sum deg(F) for a
        push level, list prefixes up to the first hit for a dense one)."""
        self.L.gbo_bfs_examined.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint32, _u64p, C.c_uint64]
        self.L.gbo_bfs_examined.restype = C.c_uint64
        ex = np.zeros(cap, dtype=np.uint64)
        k = self.L.gbo_bfs_examined(n, *self._csr_args(off, nbr), src, ptr(ex, _u64p), cap)
        return [int(x) for x in ex[:min(k, cap)]]

    def bfs(self, n, off, nbr, src, cap=64):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        depth = np.empty(n, dtype=np.int32)
        modes = np.zeros(cap, dtype=np.int32)
        sizes = np.zeros(cap, dtype=np.uint64)
        lv = C.c_uint64(0)
        rc = self.L.gbo_bfs(n, ptr(off, _u64p), ptr(nbr, _u32p), src, ptr(depth, _i32p), ptr(modes, _i32p),
                            ptr(sizes, _u64p), cap, C.byref(lv))
        if rc:
            raise IndexError("bfs: source out of range")
        k = min(lv.value, cap)
        return depth, [int(x) for x in modes[:k]], [int(x) for x in sizes[:k]]

    def pagerank(self, n, off, nbr, damping=0.85, iters=20, tol=np.finfo(np.float64).tiny):
        out = np.empty(n, dtype=np.float64)
        rc = self.L.gbo_pagerank(n, ptr(np.ascontiguousarray(off, dtype=np.uint64), _u64p),
                                 ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p), damping, iters, tol,
                                 ptr(out, _f64p))
        if rc:
            raise ValueError("pagerank: invalid argument")
        return out

    def cc(self, n, off, nbr):
        out = np.empty(n, dtype=np.uint32)
        self.L.gbo_cc(n, ptr(np.ascontiguousarray(off, dtype=np.uint64), _u64p),
                      ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p), ptr(out, _u32p))
        return out

    def bc(self, n, off, nbr, src):
        L = self.L
        L.gbo_bc.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint32, _f64p]
        out = np.empty(max(n, 1), dtype=np.float64)
        rc = L.gbo_bc(n, ptr(np.ascontiguousarray(off, dtype=np.uint64), _u64p),
                      ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p), src, ptr(out, _f64p))
        if rc:
            raise IndexError("bc: source out of range")
        return out[:n]

    def rng_u64(self, seed, stream, counter) -> int:
        return int(self.L.gbo_rng_u64(seed, stream, counter))

    def _csr_args(self, off, nbr):
        return (ptr(np.ascontiguousarray(off, dtype=np.uint64), _u64p),
                ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p))

    def bytecode_encode(self, n, off, nbr):
        """-> (byte_offsets u64[n+1], bytes u8[...])"""
        self.L.gbo_bytecode_encode.argtypes = [C.c_uint64, _u64p, _u32p, _u64p, _u8p]
        self.L.gbo_bytecode_encode.restype = C.c_uint64
        total = self.L.gbo_bytecode_encode(n, *self._csr_args(off, nbr), None, None)
        bo = np.empty(n + 1, dtype=np.uint64)
        b = np.empty(max(total, 1), dtype=np.uint8)
        self.L.gbo_bytecode_encode(n, *self._csr_args(off, nbr), ptr(bo, _u64p), ptr(b, _u8p))
        return bo, b[:total]

    def ldd(self, n, off, nbr, beta=0.2, seed=1):
        self.L.gbo_ldd.argtypes = [C.c_uint64, _u64p, _u32p, C.c_double, C.c_uint64, _u32p, _u32p, _u64p]
        lab = np.empty(max(n, 1), dtype=np.uint32)
        par = np.empty(max(n, 1), dtype=np.uint32)
        rnd = np.empty(max(n, 1), dtype=np.uint64)
        if self.L.gbo_ldd(n, *self._csr_args(off, nbr), beta, seed, ptr(lab, _u32p), ptr(par, _u32p), ptr(rnd, _u64p)):
            raise ValueError("ldd: beta must be in (0, 1]")
        return lab[:n], par[:n], rnd[:n]

    def kcore(self, n, off, nbr):
        self.L.gbo_kcore.argtypes = [C.c_uint64, _u64p, _u32p, _u64p]
        out = np.empty(max(n, 1), dtype=np.uint64)
        self.L.gbo_kcore(n, *self._csr_args(off, nbr), ptr(out, _u64p))
        return out[:n]

    def coloring(self, n, off, nbr):
        self.L.gbo_coloring.argtypes = [C.c_uint64, _u64p, _u32p, _u32p]
        out = np.empty(max(n, 1), dtype=np.uint32)
        self.L.gbo_coloring(n, *self._csr_args(off, nbr), ptr(out, _u32p))
        return out[:n]

    def mis(self, n, off, nbr, seed=1):
        self.L.gbo_mis.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint64, _u8p]
        out = np.empty(max(n, 1), dtype=np.uint8)
        self.L.gbo_mis(n, *self._csr_args(off, nbr), seed, ptr(out, _u8p))
        return out[:n]

    def tc(self, n, off, nbr) -> int:
        return int(self.L.gbo_tc(n, ptr(np.ascontiguousarray(off, dtype=np.uint64), _u64p),
                                 ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p)))

    def to_dense(self, n, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        w = np.zeros(max((n + 63) // 64, 1), dtype=np.uint64)
        self.L.gbo_subset_to_dense(n, ptr(ids, _u32p), ids.size, ptr(w, _u64p))
        return w[: (n + 63) // 64]

    def to_sparse(self, n, words):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        ids = np.empty(max(n, 1), dtype=np.uint32)
        k = self.L.gbo_subset_to_sparse(n, ptr(words, _u64p), ptr(ids, _u32p))
        return ids[:k].copy()

    def edge_map(self, n, off, nbr, ids, cond_mask, mode, early_exit=True):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        cond = np.ascontiguousarray(cond_mask, dtype=np.uint8)
        out = np.zeros(max(n, 1), dtype=np.uint8)
        upd = C.c_uint64(0)
        rc = self.L.gbo_edge_map(n, ptr(np.ascontiguousarray(off, dtype=np.uint64), _u64p),
                                 ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p), ptr(ids, _u32p),
                                 ids.size, ptr(cond, _u8p), mode, int(early_exit), ptr(out, _u8p),
                                 C.byref(upd))
        if rc:
            raise IndexError("edge_map: id out of range")
        return out[:n].astype(bool), upd.value

    def set_apply(self, n, off, nbr, prepared_pairs, insert: bool):
        b = np.ascontiguousarray(np.asarray(prepared_pairs, dtype=np.uint32).reshape(-1, 2))
        off = np.ascontiguousarray(off, dtype=np.uint64)
        off_out = np.empty(n + 1, dtype=np.uint64)
        nbr_out = np.empty(int(off[n]) + b.shape[0] + 1, dtype=np.uint32)
        applied = self.L.gbo_set_apply(n, ptr(off, _u64p), ptr(np.ascontiguousarray(nbr, dtype=np.uint32), _u32p),
                                       ptr(b, _u32p), b.shape[0], int(insert), ptr(off_out, _u64p),
                                       ptr(nbr_out, _u32p))
        return int(applied), off_out, nbr_out[: int(off_out[n])].copy()

"""Python host mirror of the reference's container / algorithm surface over
the C ABI (include/gbg_c.h, libgbg.so).

Names follow the reference (``/root/reference/proj/include/gb``):
``CsrGraph`` (csr.hpp:12-53), ``BlockedGraph`` (the dynamic container in the
role of ``SetGraph<ChunkedSortedSet>``, set_graph.hpp:26-249), ``bfs`` /
``pagerank`` / ``cc`` (algorithms.hpp:28-76), ``edge_map`` (traversal.hpp:37-56),
``subset_to_dense`` / ``subset_to_sparse`` (vertex_subset.hpp:85-91),
``generate_rmat`` / ``generate_update_batch`` (generators.hpp:19-20,
batch.hpp:52-56), ``apply_insert`` / ``apply_delete`` (batch.hpp:47-48).
Errors raise the Python analogue of the reference exception type.

There is no CPU fallback: importing this module without the built
``libgbg.so`` raises, and every call runs the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgbg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_2405_11671_b200.build` "
                      "(the CUDA library is the only implementation; there is no CPU fallback)")

_L = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- errors
GBG_OK, GBG_ERR_CUDA, GBG_ERR_OOM, GBG_ERR_OUT_OF_RANGE, GBG_ERR_INVALID_ARGUMENT = 0, 1, 2, 3, 4
GBG_ERR_UNSUPPORTED, GBG_ERR_CONFIG, GBG_ERR_FORMAT, GBG_ERR_LOGIC = 5, 6, 7, 8
KIND_CSR, KIND_BLOCKED, KIND_COMPRESSED = 0, 1, 2
GBG_CREATE_PAGERANK_LAYOUT = 1
MODE_SPARSE, MODE_DENSE, MODE_AUTO = 0, 1, 2
MAX_LEVELS = 64


class GbgError(RuntimeError):
    status = -1


class CudaError(GbgError):
    status = GBG_ERR_CUDA


class OutOfMemory(GbgError, MemoryError):
    status = GBG_ERR_OOM


class OutOfRange(GbgError, IndexError):
    """std::out_of_range"""
    status = GBG_ERR_OUT_OF_RANGE


class InvalidArgument(GbgError, ValueError):
    """std::invalid_argument"""
    status = GBG_ERR_INVALID_ARGUMENT


class UnsupportedOperation(GbgError, NotImplementedError):
    """gb::unsupported_operation (types.hpp:45-49)"""
    status = GBG_ERR_UNSUPPORTED


class ConfigError(GbgError):
    """gb::config_error (types.hpp:53-56)"""
    status = GBG_ERR_CONFIG


class FormatError(GbgError):
    """gb::format_error (types.hpp:59-62)"""
    status = GBG_ERR_FORMAT


class LogicError(GbgError):
    """std::logic_error"""
    status = GBG_ERR_LOGIC


_ERRORS = {c.status: c for c in (CudaError, OutOfMemory, OutOfRange, InvalidArgument, UnsupportedOperation,
                                 ConfigError, FormatError, LogicError)}

_L.gbg_last_error.restype = C.c_char_p


def _check(st: int):
    if st != GBG_OK:
        msg = _L.gbg_last_error().decode(errors="replace")
        raise _ERRORS.get(st, GbgError)(msg)


# ---------------------------------------------------------------- ABI
_vp = C.c_void_p
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_gpp = C.POINTER(C.c_void_p)


class BfsStats(C.Structure):
    _fields_ = [("levels", C.c_uint64), ("mode", C.c_int32 * MAX_LEVELS), ("frontier", C.c_uint64 * MAX_LEVELS),
                ("degree_sum", C.c_uint64 * MAX_LEVELS), ("reached", C.c_uint64), ("level_ms", C.c_float * MAX_LEVELS),
                ("examined", C.c_uint64 * MAX_LEVELS)]


class Caps(C.Structure):
    _fields_ = [("has_num_edges", C.c_int), ("has_degree", C.c_int), ("has_map_early_exit", C.c_int),
                ("has_parallel_map", C.c_int), ("has_parallel_map_early_exit", C.c_int),
                ("has_batch_updates", C.c_int)]


_SIGS = {
    "gbg_set_device": [C.c_int],
    "gbg_synchronize": [_vp],
    "gbg_csr_create": [C.c_uint64, C.c_uint64, _u64p, _u32p, _gpp],
    "gbg_csr_from_arcs": [C.c_uint64, _u32p, C.c_uint64, _gpp],
    "gbg_csr_create_ex": [C.c_uint64, C.c_uint64, _u64p, _u32p, C.c_uint32, _gpp],
    "gbg_blocked_create": [C.c_uint64, _u32p, C.c_uint64, _gpp],
    "gbg_blocked_from_csr": [_vp, _gpp],
    "gbg_rmat_create": [C.c_uint32, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int, _gpp],
    "gbg_graph_destroy": [_vp],
    "gbg_kind": [_vp, C.POINTER(C.c_int)],
    "gbg_num_vertices": [_vp, _u64p],
    "gbg_num_edges": [_vp, _u64p],
    "gbg_degree": [_vp, C.c_uint32, _u64p],
    "gbg_degrees": [_vp, _u64p],
    "gbg_neighbors": [_vp, C.c_uint32, _u32p, C.c_uint64, _u64p],
    "gbg_export_csr": [_vp, _u64p, _u32p],
    "gbg_capabilities": [_vp, C.POINTER(Caps)],
    "gbg_memory_bytes": [_vp, _u64p],
    "gbg_subset_to_dense": [C.c_uint64, _u32p, C.c_uint64, _u64p],
    "gbg_subset_to_sparse": [C.c_uint64, _u64p, _u32p, _u64p],
    "gbg_vertex_filter_sparse": [C.c_uint64, _u32p, C.c_uint64, _u8p, _u32p, _u64p],
    "gbg_vertex_filter_dense": [C.c_uint64, _u64p, _u8p, _u64p],
    "gbg_edge_map": [_vp, _u32p, C.c_uint64, _u8p, C.c_int, C.c_int, _u8p, _u64p, C.POINTER(C.c_int)],
    "gbg_bfs": [_vp, C.c_uint32, _i32p, C.POINTER(BfsStats)],
    "gbg_bfs_device": [_vp, C.c_uint32, _vp, C.POINTER(BfsStats)],
    "gbg_pagerank": [_vp, C.c_double, C.c_uint64, C.c_double, _f64p, _u64p],
    "gbg_pagerank_device": [_vp, C.c_double, C.c_uint64, C.c_double, _vp, _u64p],
    "gbg_cc": [_vp, _u32p],
    "gbg_cc_device": [_vp, _vp],
    "gbg_tc": [_vp, _u64p],
    "gbg_insert_batch": [_vp, _u32p, C.c_uint64, _u64p],
    "gbg_delete_batch": [_vp, _u32p, C.c_uint64, _u64p],
    "gbg_insert_batch_device": [_vp, _vp, C.c_uint64, _u64p],
    "gbg_delete_batch_device": [_vp, _vp, C.c_uint64, _u64p],
    "gbg_insert_edge": [_vp, C.c_uint32, C.c_uint32, C.POINTER(C.c_int)],
    "gbg_delete_edge": [_vp, C.c_uint32, C.c_uint32, C.POINTER(C.c_int)],
    "gbg_update_batch_device": [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_uint64, _vp],
    "gbg_contains_device": [_vp, _vp, C.c_uint64, _vp],
    "gbg_pagerank_prepare": [_vp, _f64p],
    "gbg_pagerank_index_bytes": [_vp, _u64p, _u64p],
    "gbg_bc": [_vp, C.c_uint32, _f64p],
    "gbg_bc_device": [_vp, C.c_uint32, _vp],
    "gbg_kcore": [_vp, _u64p],
    "gbg_coloring": [_vp, _u32p],
    "gbg_mis": [_vp, C.c_uint64, _u8p],
    "gbg_compressed_from": [_vp, _gpp],
    "gbg_compressed_create": [C.c_uint64, C.c_uint64, _u64p, _u32p, _gpp],
    "gbg_compressed_bytes": [_vp, _u64p, _u8p, _u64p],
    "gbg_ldd": [_vp, C.c_double, C.c_uint64, _u32p, _u32p, _u64p],
    "gbg_selftest_log1p": [_f64p, C.c_uint64, _f64p],
    "gbg_load_gbcsr1": [C.c_char_p, C.c_int, _gpp],
    "gbg_save_gbcsr1": [_vp, C.c_char_p],
}
for _name, _args in _SIGS.items():
    _f = getattr(_L, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_L.gbg_launch_count.argtypes = [_vp]
_L.gbg_launch_count.restype = C.c_uint64
_L.gbg_stream.argtypes = [_vp]
_L.gbg_stream.restype = C.c_void_p

EXPORTED = sorted(list(_SIGS) + ["gbg_last_error", "gbg_launch_count", "gbg_stream"])


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _pairs(arcs) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(arcs, dtype=np.uint32))
    if a.size == 0:
        return np.zeros((0, 2), dtype=np.uint32)
    return a.reshape(-1, 2)


def set_device(device: int):
    _check(_L.gbg_set_device(device))


# ---------------------------------------------------------------- containers
class _Graph:
    """Owner of one gbg_graph handle (GraphContainerPtr, graph_container.hpp:89)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        self.close()

    def close(self):
        h = getattr(self, "_h", None)
        if h and _L is not None:  # module globals may be gone at interpreter exit
            _L.gbg_graph_destroy(h)
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    # ---- read API (graph_container.hpp:39-60)
    def num_vertices(self) -> int:
        n = C.c_uint64()
        _check(_L.gbg_num_vertices(self._h, C.byref(n)))
        return n.value

    def num_edges(self) -> int:
        m = C.c_uint64()
        _check(_L.gbg_num_edges(self._h, C.byref(m)))
        return m.value

    def degree(self, v: int) -> int:
        d = C.c_uint64()
        _check(_L.gbg_degree(self._h, v, C.byref(d)))
        return d.value

    def degrees(self) -> np.ndarray:
        out = np.empty(self.num_vertices(), dtype=np.uint64)
        _check(_L.gbg_degrees(self._h, _p(out, _u64p)))
        return out

    def map_neighbors(self, v: int) -> np.ndarray:
        """Neighbours of v in ascending order (materialised map_neighbors)."""
        d = C.c_uint64()
        _check(_L.gbg_neighbors(self._h, v, None, 0, C.byref(d)))
        out = np.empty(d.value, dtype=np.uint32)
        if d.value:
            _check(_L.gbg_neighbors(self._h, v, _p(out, _u32p), d.value, C.byref(d)))
        return out

    def to_csr(self):
        n, m = self.num_vertices(), self.num_edges()
        off = np.empty(n + 1, dtype=np.uint64)
        nbr = np.empty(max(m, 1), dtype=np.uint32)
        _check(_L.gbg_export_csr(self._h, _p(off, _u64p), _p(nbr, _u32p)))
        return off, nbr[:m]

    def capabilities(self) -> dict:
        c = Caps()
        _check(_L.gbg_capabilities(self._h, C.byref(c)))
        return {k: bool(getattr(c, k)) for k, _ in Caps._fields_}

    def memory_bytes(self) -> int:
        b = C.c_uint64()
        _check(_L.gbg_memory_bytes(self._h, C.byref(b)))
        return b.value

    def kind(self) -> int:
        k = C.c_int()
        _check(_L.gbg_kind(self._h, C.byref(k)))
        return k.value

    # ---- updates (graph_container.hpp:64-78)
    def insert_edge(self, src: int, dst: int) -> bool:
        ch = C.c_int()
        _check(_L.gbg_insert_edge(self._h, src, dst, C.byref(ch)))
        return bool(ch.value)

    def delete_edge(self, src: int, dst: int) -> bool:
        ch = C.c_int()
        _check(_L.gbg_delete_edge(self._h, src, dst, C.byref(ch)))
        return bool(ch.value)

    def insert_batch(self, arcs) -> int:
        a = _pairs(arcs)
        applied = C.c_uint64()
        _check(_L.gbg_insert_batch(self._h, _p(a, _u32p), a.shape[0], C.byref(applied)))
        return applied.value

    def delete_batch(self, arcs) -> int:
        a = _pairs(arcs)
        applied = C.c_uint64()
        _check(_L.gbg_delete_batch(self._h, _p(a, _u32p), a.shape[0], C.byref(applied)))
        return applied.value

    def insert_batch_device(self, arcs_ptr: int, count: int) -> int:
        applied = C.c_uint64()
        _check(_L.gbg_insert_batch_device(self._h, arcs_ptr, count, C.byref(applied)))
        return applied.value

    def delete_batch_device(self, arcs_ptr: int, count: int) -> int:
        applied = C.c_uint64()
        _check(_L.gbg_delete_batch_device(self._h, arcs_ptr, count, C.byref(applied)))
        return applied.value

    def contains_device(self, arcs_ptr: int, count: int, out_ptr: int):
        """out[i] = 1 iff arc i (device uint32 pairs) is present."""
        _check(_L.gbg_contains_device(self._h, arcs_ptr, count, out_ptr))

    # ---- runtime
    def stream(self) -> int:
        return _L.gbg_stream(self._h) or 0

    def launch_count(self) -> int:
        return _L.gbg_launch_count(self._h)

    def synchronize(self):
        _check(_L.gbg_synchronize(self._h))


class CsrGraph(_Graph):
    """Device-resident static CSR (csr.hpp:12-53): uint64 offsets, uint32 ids."""

    @classmethod
    def build(cls, n: int, arcs) -> "CsrGraph":
        """CsrGraph::build(n, arcs): arcs sorted by (src,dst), deduplicated."""
        a = _pairs(arcs)
        h = C.c_void_p()
        _check(_L.gbg_csr_from_arcs(n, _p(a, _u32p), a.shape[0], C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_csr(cls, offsets, neighbors, prepare_pagerank: bool = False) -> "CsrGraph":
        """CsrGraph::build from CSR arrays (validated like csr.cpp:14-18).
        The upload is chunked and overlapped with validation; with
        prepare_pagerank the PageRank layout is built during the upload."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        h = C.c_void_p()
        flags = GBG_CREATE_PAGERANK_LAYOUT if prepare_pagerank else 0
        _check(_L.gbg_csr_create_ex(off.size - 1, nbr.size, _p(off, _u64p), _p(nbr, _u32p), flags, C.byref(h)))
        return cls(h.value)


class BlockedGraph(_Graph):
    """Dynamic blocked sorted adjacency: the chunked_set role
    (registry.cpp:136-137) with device batch insert/delete."""

    @classmethod
    def build(cls, n: int, arcs) -> "BlockedGraph":
        a = _pairs(arcs)
        h = C.c_void_p()
        _check(_L.gbg_blocked_create(n, _p(a, _u32p), a.shape[0], C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_csr_graph(cls, g: CsrGraph) -> "BlockedGraph":
        h = C.c_void_p()
        _check(_L.gbg_blocked_from_csr(g.handle, C.byref(h)))
        return cls(h.value)


class CompressedGraph(_Graph):
    """gb::CompressedCsrGraph (compressed_csr.hpp:12-46) on the device: the
    byte code of bytecode.hpp, static, no parallel maps."""

    @classmethod
    def build(cls, n: int, arcs) -> "CompressedGraph":
        with CsrGraph.build(n, arcs) as csr:
            return cls.from_graph(csr)

    @classmethod
    def from_csr(cls, offsets, neighbors) -> "CompressedGraph":
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        h = C.c_void_p()
        _check(_L.gbg_compressed_create(off.size - 1, nbr.size, _p(off, _u64p), _p(nbr, _u32p), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_graph(cls, g: _Graph) -> "CompressedGraph":
        """CompressedCsrGraph::build (compressed_csr.cpp:5-17) from any handle."""
        h = C.c_void_p()
        _check(_L.gbg_compressed_from(g.handle, C.byref(h)))
        return cls(h.value)

    def encoding(self):
        """(byte_offsets u64[n+1], bytes u8[...]): the raw byte code."""
        nb = C.c_uint64()
        _check(_L.gbg_compressed_bytes(self.handle, None, None, C.byref(nb)))
        off = np.empty(self.num_vertices() + 1, dtype=np.uint64)
        b = np.empty(max(nb.value, 1), dtype=np.uint8)
        _check(_L.gbg_compressed_bytes(self.handle, _p(off, _u64p), _p(b, _u8p), C.byref(nb)))
        return off, b[: nb.value]


def _cls_of(kind: int):
    return {KIND_CSR: CsrGraph, KIND_BLOCKED: BlockedGraph, KIND_COMPRESSED: CompressedGraph}[kind]


def generate_rmat(log2_n: int, arcs: int, seed: int, a=0.5, b=0.1, c=0.1, kind: int = KIND_CSR):
    """gb::generate_rmat (generators.cpp:67-72) on the device, bit-exact.
    Defaults are RmatParams' (batch.hpp:44-50)."""
    h = C.c_void_p()
    _check(_L.gbg_rmat_create(log2_n, arcs, a, b, c, seed, kind, C.byref(h)))
    return _cls_of(kind)(h.value)


def load_binary(path: str, kind: int = KIND_CSR):
    """gb::load_binary_csr (io.cpp:87-110): a GBCSR1 file into a device container."""
    h = C.c_void_p()
    _check(_L.gbg_load_gbcsr1(os.fsencode(path), kind, C.byref(h)))
    return _cls_of(kind)(h.value)


def save_binary(g: _Graph, path: str):
    """gb::save_binary (io.cpp:75-85) from a device container."""
    _check(_L.gbg_save_gbcsr1(g.handle, os.fsencode(path)))


def generate_update_batch_device(log2_n: int, size: int, seed: int, out_ptr: int, a=0.5, b=0.1, c=0.1):
    """gb::generate_update_batch (batch.cpp:128-154) into device memory at
    out_ptr (2*size uint32 pairs)."""
    _check(_L.gbg_update_batch_device(log2_n, a, b, c, size, seed, out_ptr))


def apply_insert(g: _Graph, raw_arcs) -> int:
    """prepare(GlobalSort) + apply_insert (batch.cpp:34-42, 120-122)."""
    return g.insert_batch(raw_arcs)


def apply_delete(g: _Graph, raw_arcs) -> int:
    """prepare(GlobalSort) + apply_delete (batch.cpp:34-42, 124-126)."""
    return g.delete_batch(raw_arcs)


# ---------------------------------------------------------------- algorithms
@dataclass
class BfsResult:
    depth: np.ndarray  # int32, -1 = unreached (kInfiniteDistance)
    modes: List[int] = field(default_factory=list)
    frontier_sizes: List[int] = field(default_factory=list)
    degree_sums: List[int] = field(default_factory=list)
    reached: int = 0
    level_ms: List[float] = field(default_factory=list)
    examined: List[int] = field(default_factory=list)


def _stats(st: BfsStats) -> dict:
    k = min(st.levels, MAX_LEVELS)
    return dict(modes=[st.mode[i] for i in range(k)], frontier_sizes=[st.frontier[i] for i in range(k)],
                degree_sums=[st.degree_sum[i] for i in range(k)], reached=st.reached,
                level_ms=[round(st.level_ms[i], 4) for i in range(k)], examined=[st.examined[i] for i in range(k)])


def bfs(g: _Graph, source: int) -> BfsResult:
    """gb::bfs (algorithms.cpp:29-58): depths with the reference switch."""
    depth = np.empty(g.num_vertices(), dtype=np.int32)
    st = BfsStats()
    _check(_L.gbg_bfs(g.handle, source, _p(depth, _i32p), C.byref(st)))
    return BfsResult(depth=depth, **_stats(st))


def bfs_device(g: _Graph, source: int, depth_ptr: int, stats: bool = True):
    """gbg_bfs_device: depths stay on the device.  stats=False passes NULL
    statistics: the call is then asynchronous on the handle's stream
    (nothing returns to the host) and the result is None."""
    if not stats:
        _check(_L.gbg_bfs_device(g.handle, source, depth_ptr, None))
        return None
    st = BfsStats()
    _check(_L.gbg_bfs_device(g.handle, source, depth_ptr, C.byref(st)))
    return _stats(st)


def pagerank(g: _Graph, damping: float = 0.85, max_iters: int = 20, tolerance: float = 1e-4, out=None):
    """gb::pagerank (algorithms.cpp:508-555), fp64.  AlgoParams defaults
    (algorithms.hpp:16-18).  `out`: optional host float64 array (pinned
    memory makes the device->host copy run at link speed)."""
    if out is None:
        out = np.empty(g.num_vertices(), dtype=np.float64)
    elif out.dtype != np.float64 or out.size != g.num_vertices() or not out.flags.c_contiguous:
        raise InvalidArgument("out must be a contiguous float64 array of num_vertices() entries")
    it = C.c_uint64()
    _check(_L.gbg_pagerank(g.handle, damping, max_iters, tolerance, _p(out, _f64p), C.byref(it)))
    return out


def pagerank_kernel_name() -> str:
    """Name of the per-iteration PageRank kernel (for ncu lookups)."""
    return "pr_tile_k"


def pagerank_prepare(g: _Graph) -> float:
    """Build the cached degree-ordered PageRank layout; returns its build ms."""
    ms = C.c_double()
    _check(_L.gbg_pagerank_prepare(g.handle, C.byref(ms)))
    return ms.value


def pagerank_index_bytes(g: _Graph) -> tuple:
    """(tiled index bytes, row layout bytes) currently cached on the handle."""
    a, b = C.c_uint64(), C.c_uint64()
    _check(_L.gbg_pagerank_index_bytes(g.handle, C.byref(a), C.byref(b)))
    return a.value, b.value


def pagerank_device(g: _Graph, out_ptr: int, damping=0.85, max_iters=20, tolerance=1e-4) -> int:
    it = C.c_uint64()
    _check(_L.gbg_pagerank_device(g.handle, damping, max_iters, tolerance, out_ptr, C.byref(it)))
    return it.value


def bc(g: _Graph, source: int) -> np.ndarray:
    """gb::bc (algorithms.cpp:60-103): single-source Brandes dependencies."""
    out = np.empty(g.num_vertices(), dtype=np.float64)
    _check(_L.gbg_bc(g.handle, source, _p(out, _f64p)))
    return out


def bc_device(g: _Graph, source: int, out_ptr: int):
    _check(_L.gbg_bc_device(g.handle, source, out_ptr))


def cc(g: _Graph) -> np.ndarray:
    """gb::cc (algorithms.cpp:194-234): min-id component labels."""
    out = np.empty(g.num_vertices(), dtype=np.uint32)
    _check(_L.gbg_cc(g.handle, _p(out, _u32p)))
    return out


def cc_device(g: _Graph, out_ptr: int):
    _check(_L.gbg_cc_device(g.handle, out_ptr))


def kcore(g: _Graph) -> np.ndarray:
    """gb::kcore (algorithms.cpp:330-374): coreness per vertex (uint64)."""
    out = np.empty(g.num_vertices(), dtype=np.uint64)
    _check(_L.gbg_kcore(g.handle, _p(out, _u64p)))
    return out


def coloring(g: _Graph) -> np.ndarray:
    """gb::coloring (algorithms.cpp:376-432): first-fit colours in
    largest-log-degree-first order (uint32).  Symmetric graphs only."""
    out = np.empty(g.num_vertices(), dtype=np.uint32)
    _check(_L.gbg_coloring(g.handle, _p(out, _u32p)))
    return out


def mis(g: _Graph, seed: int = 1) -> np.ndarray:
    """gb::mis (algorithms.cpp:434-504): 0/1 membership (uint8) of the
    lexicographically-first MIS under (rng_u64(seed, 7, v), v).  Symmetric
    graphs only."""
    out = np.empty(g.num_vertices(), dtype=np.uint8)
    _check(_L.gbg_mis(g.handle, seed, _p(out, _u8p)))
    return out


def ldd(g: _Graph, beta: float = 0.2, seed: int = 1):
    """gb::ldd (algorithms.cpp:114-188) -> (labels u32, parents u32,
    rounds u64); UINT32_MAX marks no parent."""
    n = g.num_vertices()
    labels = np.empty(n, dtype=np.uint32)
    parents = np.empty(n, dtype=np.uint32)
    rounds = np.empty(n, dtype=np.uint64)
    _check(_L.gbg_ldd(g.handle, beta, seed, _p(labels, _u32p), _p(parents, _u32p), _p(rounds, _u64p)))
    return labels, parents, rounds


def selftest_log1p(x) -> np.ndarray:
    """The device log1p used for ldd's shifts, on host values (test hook)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _check(_L.gbg_selftest_log1p(_p(x, _f64p), x.size, _p(out, _f64p)))
    return out


def triangle_count(g: _Graph) -> int:
    t = C.c_uint64()
    _check(_L.gbg_tc(g.handle, C.byref(t)))
    return t.value


def vertex_filter_sparse(n: int, ids, keep) -> np.ndarray:
    """vertex_filter (traversal.cpp:117-131) on a sparse subset: the members
    with keep[v] != 0, ascending and unique as VertexSubset holds them."""
    a = np.ascontiguousarray(ids, dtype=np.uint32)
    k = np.ascontiguousarray(keep, dtype=np.uint8)
    out = np.empty(max(a.size, 1), dtype=np.uint32)
    cnt = C.c_uint64()
    _check(_L.gbg_vertex_filter_sparse(n, _p(a, _u32p), a.size, _p(k, _u8p), _p(out, _u32p), C.byref(cnt)))
    return out[: cnt.value]


def vertex_filter_dense(n: int, words, keep) -> np.ndarray:
    """vertex_filter on a dense subset (uint64 words, LSB first): stays dense."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    k = np.ascontiguousarray(keep, dtype=np.uint8)
    out = np.zeros(max(w.size, 1), dtype=np.uint64)
    _check(_L.gbg_vertex_filter_dense(n, _p(w, _u64p), _p(k, _u8p), _p(out, _u64p)))
    return out[: w.size]


def edge_map(g: _Graph, frontier_ids, cond_mask, mode: int = MODE_AUTO, early_exit: bool = True):
    """One gb::edge_map (traversal.cpp:16-111) with cond(v) = cond_mask[v]
    and an always-true update.  Returns (member bool[n], updates, mode)."""
    ids = np.ascontiguousarray(frontier_ids, dtype=np.uint32)
    cond = np.ascontiguousarray(cond_mask, dtype=np.uint8)
    n = g.num_vertices()
    if cond.size != n:
        raise InvalidArgument("cond_mask must have num_vertices() entries")
    out = np.zeros(max(n, 1), dtype=np.uint8)
    upd = C.c_uint64()
    chosen = C.c_int()
    _check(_L.gbg_edge_map(g.handle, _p(ids, _u32p), ids.size, _p(cond, _u8p), mode, int(early_exit),
                           _p(out, _u8p), C.byref(upd), C.byref(chosen)))
    return out[:n].astype(bool), upd.value, chosen.value


def subset_to_dense(n: int, ids) -> np.ndarray:
    """VertexSubset::to_dense (vertex_subset.cpp:32-37): uint64 words, LSB first."""
    a = np.ascontiguousarray(ids, dtype=np.uint32)
    words = np.zeros(max((n + 63) // 64, 1), dtype=np.uint64)
    _check(_L.gbg_subset_to_dense(n, _p(a, _u32p), a.size, _p(words, _u64p)))
    return words[: (n + 63) // 64]


def subset_to_sparse(n: int, words) -> np.ndarray:
    """VertexSubset::to_sparse (vertex_subset.cpp:39-45): ascending ids."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    ids = np.empty(max(n, 1), dtype=np.uint32)
    k = C.c_uint64()
    _check(_L.gbg_subset_to_sparse(n, _p(w, _u64p), _p(ids, _u32p), C.byref(k)))
    return ids[: k.value].copy()

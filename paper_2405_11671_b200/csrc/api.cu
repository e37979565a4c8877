// Container handles and the read API of the C ABI (include/gbg_c.h).
//
// Reference surface replaced: gb::GraphContainer (graph_container.hpp:36-87),
// gb::CsrGraph (csr.hpp:12-53, csr.cpp:9-25), VertexSubset conversions
// (vertex_subset.cpp:8-45).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "edges.cuh"
#include "traverse.cuh"

namespace gbg {

namespace {
thread_local std::string t_err;
thread_local int t_device = -1;
}  // namespace

void set_last_error(const std::string& m) { t_err = m; }

void read_scalars(gbg_graph* g, const void* dev, size_t bytes, void* host) {
  if (bytes > kHostScalarBytes) fail(GBG_ERR_LOGIC, "read_scalars: too large");
  GBG_CUDA(cudaMemcpyAsync(g->hscalar, dev, bytes, cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  std::memcpy(host, g->hscalar, bytes);
}

gbg_graph* new_handle(int kind, uint64_t n) {
  if (n > (uint64_t{1} << 32) - 1)
    fail(GBG_ERR_INVALID_ARGUMENT, "vertex count must fit uint32 ids (types.hpp:11)");
  auto* g = new gbg_graph();
  try {
    if (t_device >= 0) GBG_CUDA(cudaSetDevice(t_device));
    GBG_CUDA(cudaGetDevice(&g->device));
    GBG_CUDA(cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, g->device));
    GBG_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    GBG_CUDA(cudaDeviceGetDefaultMemPool(&pool, g->device));
    uint64_t keep = UINT64_MAX;  // keep freed blocks in the pool for reuse
    GBG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    GBG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&g->hscalar), kHostScalarBytes));
  } catch (...) {
    delete g;
    throw;
  }
  g->kind = kind;
  g->n = n;
  return g;
}

// ---------------------------------------------------------------- kernels
__global__ void list_to_bitmap_k(const uint32_t* ids, uint64_t k, uint32_t* bm) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = ids[i];
    atomicOr(bm + (v >> 5), 1u << (v & 31));
  }
}

// vertex_filter (traversal.cpp:117-131): members with keep[v] != 0, in the
// input's representation (sparse: order kept; dense: word-wise AND)
struct KeepIn {
  const uint32_t* ids;
  const uint8_t* keep;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return keep[ids[i]] != 0; }
};
struct KeepOut {
  const uint32_t* ids;
  const uint8_t* keep;
  uint32_t* out;
  __device__ __forceinline__ void operator()(uint64_t i, uint32_t pre) const {
    if (keep[ids[i]]) out[pre] = ids[i];
  }
};
__global__ void filter_dense_k(uint64_t n, const uint32_t* in, const uint8_t* keep, uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~uint64_t{31}; base < n; base += stride) {
    const uint64_t v = base + (threadIdx.x & 31);
    const uint32_t m = __ballot_sync(0xffffffffu, v < n && keep[v] != 0);
    if ((threadIdx.x & 31) == 0) out[base >> 5] = in[base >> 5] & m;
  }
}

// csr.cpp:14-18 split in two passes: the offsets are monotone from 0 to m
// (vertex-parallel), then every id is in range and strictly above its
// predecessor within the segment (edge-parallel, balanced).
__global__ void csr_validate_offsets_k(uint64_t n, uint64_t m, const uint64_t* off, int* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    uint64_t b = off[v], e = off[v + 1];
    if (e < b || e > m) *bad = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m)) *bad = 1;
}

struct SegmentOrderOp {
  const uint64_t* off;
  const uint32_t* nbr;
  uint64_t n;
  int* bad;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t e) const {
    if (v >= n || (e > off[u] && nbr[e - 1] >= v)) *bad = 1;
  }
};

// arcs sorted strictly increasing by (src,dst), ids < n.  src/dst split out.
__global__ void arcs_validate_split_k(uint64_t n, uint64_t m, const uint32_t* pairs, uint32_t* src,
                                      uint32_t* dst, int* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
    uint32_t s = pairs[2 * i], d = pairs[2 * i + 1];
    if (s >= n || d >= n) *bad = 1;
    if (i > 0) {
      uint64_t prev = ((uint64_t)pairs[2 * i - 2] << 32) | pairs[2 * i - 1];
      uint64_t cur = ((uint64_t)s << 32) | d;
      if (!(prev < cur)) *bad = 1;
    }
    src[i] = s;
    dst[i] = d;
  }
}

// offsets from a sorted source array: off[x] = first i with src[i] >= x.
__global__ void offsets_from_sorted_k(const uint32_t* src, uint64_t m, uint64_t n, uint64_t* off) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= m; i += stride) {
    uint64_t lo = i == 0 ? 0 : (uint64_t)src[i - 1] + 1;
    uint64_t hi = i == m ? n : (uint64_t)src[i];
    for (uint64_t x = lo; x <= hi; ++x) off[x] = i;
  }
}

void build_csr_offsets_from_sorted_src(gbg_graph* g, const uint32_t* src, uint64_t m, uint64_t* off) {
  GBG_LAUNCH(g, offsets_from_sorted_k, grid_for(m + 1, 256), 256, 0, src, m, g->n, off);
}

__global__ void widen_k(const uint32_t* in, uint64_t n, uint64_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) out[v] = in[v];
}

template <class G>
__global__ void degrees_k(G gv, uint64_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < gv.n; v += stride)
    out[v] = gv.degree(static_cast<uint32_t>(v));
}

template <class G>
__global__ void gather_csr_k(G gv, const uint64_t* voff, uint32_t* out) {
  // one warp per vertex
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t v = w0; v < gv.n; v += nw) {
    uint64_t b;
    uint32_t d;
    gv.seg(static_cast<uint32_t>(v), b, d);
    uint64_t o = voff[v];
    for (uint32_t j = lane; j < d; j += 32) out[o + j] = gv.at(b + j);
  }
}

}  // namespace gbg

using namespace gbg;

gbg_graph::~gbg_graph() {
  DeviceScope ds(device);
  AllocStream as(stream);
  ws.clear();
  dfree(off);
  dfree(nbr);
  dfree(bstart);
  dfree(bdeg);
  dfree(bcap);
  dfree(pool);
  dfree(voff);
  dfree(first);
  dfree(coff);
  dfree(cbytes);
  dfree(cdeg);
  invalidate_derived();
  if (hscalar) cudaFreeHost(hscalar);
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

extern "C" {

const char* gbg_last_error(void) { return t_err.c_str(); }

gbg_status gbg_set_device(int device) {
  return guard([&] {
    int count = 0;
    GBG_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(GBG_ERR_OUT_OF_RANGE, "gbg_set_device: no such device");
    GBG_CUDA(cudaSetDevice(device));
    t_device = device;
  });
}

uint64_t gbg_launch_count(const gbg_graph* g) { return g ? g->launches : 0; }
void* gbg_stream(const gbg_graph* g) { return g ? static_cast<void*>(g->stream) : nullptr; }

gbg_status gbg_synchronize(gbg_graph* g) {
  return guard([&] {
    GBG_HANDLE(g);
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

// The upload is pipelined: offsets first, then the neighbour ids in chunks
// on a copy stream, each chunk validated (and, with
// GBG_CREATE_PAGERANK_LAYOUT, relabelled into the PageRank layout) on the
// handle's stream as soon as it lands, so host->device transfer hides the
// checks and the layout build.  Pinned host buffers make the copies
// asynchronous; pageable ones still work (the driver stages them).
gbg_status gbg_csr_create_ex(uint64_t n, uint64_t m, const uint64_t* offsets, const uint32_t* neighbors,
                             uint32_t flags, gbg_graph** out) {
  return guard([&] {
    if (!out || !offsets || (m && !neighbors)) fail(GBG_ERR_INVALID_ARGUMENT, "gbg_csr_create: null argument");
    if (flags & ~uint32_t{GBG_CREATE_PAGERANK_LAYOUT}) fail(GBG_ERR_INVALID_ARGUMENT, "gbg_csr_create: unknown flags");
    *out = nullptr;
    gbg_graph* g = new_handle(GBG_KIND_CSR, n);
    std::unique_ptr<gbg_graph> hold(g);
    AllocStream as(g->stream);
    g->m = m;
    g->off = dalloc<uint64_t>(n + 1);
    g->nbr = dalloc<uint32_t>(m);
    GBG_CUDA(cudaStreamSynchronize(g->stream));  // allocations visible to the copy stream
    constexpr uint64_t kChunkIds = uint64_t{1} << 26;  // 256 MB of ids per chunk
    const uint64_t nchunks = (m + kChunkIds - 1) / kChunkIds;
    struct Copier {  // copy stream + per-chunk events; drained before the handle can be freed
      cudaStream_t cs = nullptr;
      std::vector<cudaEvent_t> ev;
      ~Copier() {
        if (cs) {
          cudaStreamSynchronize(cs);
          cudaStreamDestroy(cs);
        }
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
      }
    } cp;
    GBG_CUDA(cudaStreamCreateWithFlags(&cp.cs, cudaStreamNonBlocking));
    cp.ev.resize(nchunks + 1);
    for (auto& e : cp.ev) GBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    GBG_CUDA(cudaMemcpyAsync(g->off, offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, cp.cs));
    GBG_CUDA(cudaEventRecord(cp.ev[0], cp.cs));
    for (uint64_t c = 0; c < nchunks; ++c) {
      const uint64_t e0 = c * kChunkIds, e1 = std::min(m, e0 + kChunkIds);
      GBG_CUDA(cudaMemcpyAsync(g->nbr + e0, neighbors + e0, (e1 - e0) * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               cp.cs));
      GBG_CUDA(cudaEventRecord(cp.ev[c + 1], cp.cs));
    }
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    GBG_CUDA(cudaEventCreate(&t0));
    GBG_CUDA(cudaEventCreate(&t1));
    GBG_CUDA(cudaStreamWaitEvent(g->stream, cp.ev[0], 0));
    GBG_CUDA(cudaEventRecord(t0, g->stream));
    int* bad = g->ws.get<int>("bad", 1);
    GBG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), g->stream));
    GBG_LAUNCH(g, csr_validate_offsets_k, grid_for(n + 1, 256), 256, 0, n, m, g->off, bad);
    int hb = 0;
    read_scalars(g, bad, sizeof(int), &hb);
    if (hb) fail(GBG_ERR_FORMAT, "csr_build: offsets must rise monotonically from 0 to m");
    prrows::PrRows* L = nullptr;
    struct LayoutHold {
      prrows::PrRows*& L;
      ~LayoutHold() {
        if (L) prrows::pr_layout_free(L);
      }
    } lh{L};
    if ((flags & GBG_CREATE_PAGERANK_LAYOUT) && n) L = prrows::pr_layout_rows_csr(g);  // offsets only
    for (uint64_t c = 0; c < nchunks; ++c) {
      const uint64_t e0 = c * kChunkIds, e1 = std::min(m, e0 + kChunkIds);
      GBG_CUDA(cudaStreamWaitEvent(g->stream, cp.ev[c + 1], 0));
      for_each_edge_range(g, g->csr_view(), g->off, e0, e1, SegmentOrderOp{g->off, g->nbr, n, bad});
      if (L) prrows::pr_layout_relabel_csr(g, L, e0, e1);
    }
    GBG_CUDA(cudaEventRecord(t1, g->stream));
    read_scalars(g, bad, sizeof(int), &hb);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (hb) fail(GBG_ERR_FORMAT, "csr_build: arcs must be sorted, deduplicated and in range");
    if (L) {
      prrows::pr_layout_attach(g, L, ms);
      L = nullptr;
    }
    *out = hold.release();
  });
}

gbg_status gbg_csr_create(uint64_t n, uint64_t m, const uint64_t* offsets, const uint32_t* neighbors,
                          gbg_graph** out) {
  return gbg_csr_create_ex(n, m, offsets, neighbors, 0, out);
}

gbg_status gbg_csr_from_arcs(uint64_t n, const uint32_t* arcs, uint64_t m, gbg_graph** out) {
  return guard([&] {
    if (!out || (m && !arcs)) fail(GBG_ERR_INVALID_ARGUMENT, "gbg_csr_from_arcs: null argument");
    *out = nullptr;
    gbg_graph* g = new_handle(GBG_KIND_CSR, n);
    std::unique_ptr<gbg_graph> hold(g);
    AllocStream as(g->stream);
    g->m = m;
    g->off = dalloc<uint64_t>(n + 1);
    g->nbr = dalloc<uint32_t>(m);
    uint32_t* pairs = g->ws.get<uint32_t>("pairs", 2 * m);
    uint32_t* src = g->ws.get<uint32_t>("src", m);
    if (m) GBG_CUDA(cudaMemcpyAsync(pairs, arcs, 2 * m * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
    int* bad = g->ws.get<int>("bad", 1);
    GBG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), g->stream));
    if (m) GBG_LAUNCH(g, arcs_validate_split_k, grid_for(m, 256), 256, 0, n, m, pairs, src, g->nbr, bad);
    int hb = 0;
    read_scalars(g, bad, sizeof(int), &hb);
    if (hb) fail(GBG_ERR_FORMAT, "csr_build: arcs must be sorted, deduplicated and in range");
    build_csr_offsets_from_sorted_src(g, src, m, g->off);
    g->ws.release("pairs");
    g->ws.release("src");
    GBG_CUDA(cudaStreamSynchronize(g->stream));
    *out = hold.release();
  });
}

gbg_status gbg_graph_destroy(gbg_graph* g) {
  return guard([&] { delete g; });
}

// ---- GBCSR1 files (io.cpp:75-114) ---------------------------------------
static const char kGbcsrMagic[8] = {'G', 'B', 'C', 'S', 'R', '1', '\0', '\0'};

gbg_status gbg_load_gbcsr1(const char* path, int kind, gbg_graph** out) {
  return guard([&] {
    if (!path || !out) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (kind != GBG_KIND_CSR && kind != GBG_KIND_BLOCKED && kind != GBG_KIND_COMPRESSED)
      fail(GBG_ERR_CONFIG, "unknown container kind");
    *out = nullptr;
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), &std::fclose);
    if (!f) fail(GBG_ERR_FORMAT, std::string("cannot open binary graph: ") + path);
    char magic[8];
    uint64_t nm[2];
    if (std::fread(magic, 1, 8, f.get()) != 8 || std::memcmp(magic, kGbcsrMagic, 8) != 0)
      fail(GBG_ERR_FORMAT, std::string("binary graph: bad magic: ") + path);
    if (std::fread(nm, sizeof(uint64_t), 2, f.get()) != 2) fail(GBG_ERR_FORMAT, "binary graph: truncated header");
    const uint64_t n = nm[0], m = nm[1];
    uint64_t* off = nullptr;
    uint32_t* nbr = nullptr;
    GBG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&off), (n + 1) * sizeof(uint64_t)));
    std::unique_ptr<uint64_t, cudaError_t (*)(void*)> hold_off(off, &cudaFreeHost);
    GBG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&nbr), (m ? m : 1) * sizeof(uint32_t)));
    std::unique_ptr<uint32_t, cudaError_t (*)(void*)> hold_nbr(nbr, &cudaFreeHost);
    if (std::fread(off, sizeof(uint64_t), n + 1, f.get()) != n + 1) fail(GBG_ERR_FORMAT, "binary graph: truncated offsets");
    if (m && std::fread(nbr, sizeof(uint32_t), m, f.get()) != m) fail(GBG_ERR_FORMAT, "binary graph: truncated neighbors");
    gbg_graph* csr = nullptr;
    gbg_status st = gbg_csr_create(n, m, off, nbr, &csr);  // validates on the device
    if (st != GBG_OK) fail(st, gbg_last_error());
    if (kind == GBG_KIND_CSR) {
      *out = csr;
      return;
    }
    std::unique_ptr<gbg_graph> hold_csr(csr);
    gbg_graph* b = nullptr;
    st = kind == GBG_KIND_BLOCKED ? gbg_blocked_from_csr(csr, &b) : gbg_compressed_from(csr, &b);
    if (st != GBG_OK) fail(st, gbg_last_error());
    *out = b;
  });
}

gbg_status gbg_save_gbcsr1(gbg_graph* g, const char* path) {
  return guard([&] {
    if (!g || !path) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    const uint64_t n = g->n, m = g->m;
    std::vector<uint64_t> off(n + 1);
    std::vector<uint32_t> nbr(m ? m : 1);
    gbg_status st = gbg_export_csr(g, off.data(), nbr.data());
    if (st != GBG_OK) fail(st, gbg_last_error());
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), &std::fclose);
    if (!f) fail(GBG_ERR_FORMAT, std::string("cannot write binary graph: ") + path);
    const uint64_t nm[2] = {n, m};
    bool ok = std::fwrite(kGbcsrMagic, 1, 8, f.get()) == 8 && std::fwrite(nm, sizeof(uint64_t), 2, f.get()) == 2 &&
              std::fwrite(off.data(), sizeof(uint64_t), n + 1, f.get()) == n + 1 &&
              (m == 0 || std::fwrite(nbr.data(), sizeof(uint32_t), m, f.get()) == m);
    if (!ok) fail(GBG_ERR_FORMAT, std::string("write failed: ") + path);
  });
}

gbg_status gbg_kind(const gbg_graph* g, int* kind) {
  return guard([&] {
    if (!g || !kind) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    *kind = g->kind;
  });
}

gbg_status gbg_num_vertices(const gbg_graph* g, uint64_t* n) {
  return guard([&] {
    if (!g || !n) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    *n = g->n;
  });
}

gbg_status gbg_num_edges(const gbg_graph* g, uint64_t* m) {
  return guard([&] {
    if (!g || !m) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    *m = g->m;
  });
}

gbg_status gbg_degree(gbg_graph* g, uint32_t v, uint64_t* deg) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!deg) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (v >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "degree: vertex out of range");
    if (g->kind == GBG_KIND_CSR) {
      uint64_t o[2];
      read_scalars(g, g->off + v, sizeof(o), o);
      *deg = o[1] - o[0];
    } else {
      uint32_t d = 0;
      read_scalars(g, (g->kind == GBG_KIND_BLOCKED ? g->bdeg : g->cdeg) + v, sizeof(d), &d);
      *deg = d;
    }
  });
}

gbg_status gbg_degrees(gbg_graph* g, uint64_t* out) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!out) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    uint64_t* d = g->ws.get<uint64_t>("degrees", g->n);
    if (g->kind == GBG_KIND_COMPRESSED) {
      GBG_LAUNCH(g, widen_k, grid_for(g->n, 256), 256, 0, g->cdeg, g->n, d);
    } else {
      with_view(g, [&](auto view) {
        GBG_LAUNCH(g, degrees_k<decltype(view)>, grid_for(g->n, 256), 256, 0, view, d);
      });
    }
    GBG_CUDA(cudaMemcpyAsync(out, d, g->n * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_neighbors(gbg_graph* g, uint32_t v, uint32_t* out, uint64_t cap, uint64_t* deg) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!deg || (cap && !out)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (v >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "neighbors: vertex out of range");
    uint64_t begin = 0, d = 0;
    const uint32_t* base;
    if (g->kind == GBG_KIND_COMPRESSED) {
      uint32_t dd = 0;
      read_scalars(g, g->cdeg + v, sizeof(dd), &dd);
      uint32_t* tmp = g->ws.get<uint32_t>("nbrs", dd);
      if (dd) compressed_neighbors(g, v, tmp);
      d = dd;
      base = tmp;
    } else if (g->kind == GBG_KIND_CSR) {
      uint64_t o[2];
      read_scalars(g, g->off + v, sizeof(o), o);
      begin = o[0];
      d = o[1] - o[0];
      base = g->nbr;
    } else {
      uint64_t b = 0;
      uint32_t dd = 0;
      read_scalars(g, g->bstart + v, sizeof(b), &b);
      read_scalars(g, g->bdeg + v, sizeof(dd), &dd);
      begin = b;
      d = dd;
      base = g->pool;
    }
    *deg = d;
    uint64_t k = std::min(d, cap);
    if (k) {
      GBG_CUDA(cudaMemcpyAsync(out, base + begin, k * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
      GBG_CUDA(cudaStreamSynchronize(g->stream));
    }
  });
}

gbg_status gbg_export_csr(gbg_graph* g, uint64_t* offsets, uint32_t* neighbors) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!offsets || (g->m && !neighbors)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (g->kind == GBG_KIND_CSR || g->kind == GBG_KIND_COMPRESSED) {
      const CsrView v = g->kind == GBG_KIND_CSR ? g->csr_view() : compressed_decoded(g);
      GBG_CUDA(cudaMemcpyAsync(offsets, v.off, (g->n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
      if (g->m)
        GBG_CUDA(cudaMemcpyAsync(neighbors, v.nbr, g->m * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    } else {
      const uint64_t* voff = virtual_offsets(g);
      uint32_t* tmp = g->ws.get<uint32_t>("export", g->m);
      GBG_LAUNCH(g, gather_csr_k<BlockedView>, grid_for(g->n * 32, 256, 148 * 32), 256, 0, g->blocked_view(), voff,
                 tmp);
      GBG_CUDA(cudaMemcpyAsync(offsets, voff, (g->n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
      if (g->m)
        GBG_CUDA(cudaMemcpyAsync(neighbors, tmp, g->m * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
      GBG_CUDA(cudaStreamSynchronize(g->stream));
      g->ws.release("export");
    }
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_capabilities(const gbg_graph* g, gbg_caps* caps) {
  return guard([&] {
    if (!g || !caps) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    // CSR pattern (csr.hpp:31-33); the blocked container adds batch updates
    // (set_graph.hpp:95-98).
    // The compressed container decodes sequentially: no parallel maps
    // (compressed_csr.hpp:27-29).
    if (g->kind == GBG_KIND_COMPRESSED)
      *caps = gbg_caps{1, 1, 1, 0, 0, 0};
    else
      *caps = gbg_caps{1, 1, 1, 1, 1, g->kind == GBG_KIND_BLOCKED ? 1 : 0};
  });
}

gbg_status gbg_memory_bytes(const gbg_graph* g, uint64_t* bytes) {
  return guard([&] {
    if (!g || !bytes) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (g->kind == GBG_KIND_CSR)
      *bytes = (g->n + 1) * sizeof(uint64_t) + g->m * sizeof(uint32_t);
    else if (g->kind == GBG_KIND_COMPRESSED)  // compressed_csr.hpp:31-33 plus the degree array
      *bytes = (g->n + 1) * sizeof(uint64_t) + g->cbytes_len + g->n * sizeof(uint32_t);
    else
      *bytes = g->n * (sizeof(uint64_t) + 2 * sizeof(uint32_t)) + g->pool_cap * sizeof(uint32_t);
  });
}

// ---- vertex_subset conversions (vertex_subset.cpp:8-45) ----------------
gbg_status gbg_subset_to_dense(uint64_t n, const uint32_t* ids, uint64_t k, uint64_t* words) {
  return guard([&] {
    if ((k && !ids) || (n && !words)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    for (uint64_t i = 0; i < k; ++i)
      if (ids[i] >= n) fail(GBG_ERR_OUT_OF_RANGE, "VertexSubset: id out of range");
    std::unique_ptr<gbg_graph> g(new_handle(GBG_KIND_CSR, n));
    AllocStream as(g->stream);
    uint64_t nw32 = (n + 31) / 32, nw64 = (n + 63) / 64;
    uint32_t* bm = g->ws.get<uint32_t>("bm", 2 * nw64);
    uint32_t* dids = g->ws.get<uint32_t>("ids", k);
    GBG_CUDA(cudaMemsetAsync(bm, 0, 2 * nw64 * sizeof(uint32_t), g->stream));
    if (k) {
      GBG_CUDA(cudaMemcpyAsync(dids, ids, k * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
      GBG_LAUNCH(g.get(), list_to_bitmap_k, grid_for(k, 256), 256, 0, dids, k, bm);
    }
    (void)nw32;
    if (nw64)
      GBG_CUDA(cudaMemcpyAsync(words, bm, nw64 * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_vertex_filter_sparse(uint64_t n, const uint32_t* ids, uint64_t k, const uint8_t* keep, uint32_t* out,
                                    uint64_t* out_k) {
  return guard([&] {
    if (!out_k || (k && (!ids || !out)) || (n && !keep)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (k > 0xffffffffull) fail(GBG_ERR_INVALID_ARGUMENT, "subset too large");
    bool canonical = true;  // strictly increasing, as VertexSubset stores ids
    for (uint64_t i = 0; i < k; ++i) {
      if (ids[i] >= n) fail(GBG_ERR_OUT_OF_RANGE, "VertexSubset: id out of range");
      if (i && ids[i] <= ids[i - 1]) canonical = false;
    }
    *out_k = 0;
    if (!k) return;
    std::unique_ptr<gbg_graph> g(new_handle(GBG_KIND_CSR, n));
    AllocStream as(g->stream);
    uint32_t* dids = g->ws.get<uint32_t>("ids", k);
    uint32_t* dout = g->ws.get<uint32_t>("out", k);
    uint8_t* dkeep = g->ws.get<uint8_t>("keep", n);
    uint32_t* cnt = g->ws.get<uint32_t>("cnt", 1);
    GBG_CUDA(cudaMemcpyAsync(dids, ids, k * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
    GBG_CUDA(cudaMemcpyAsync(dkeep, keep, n, cudaMemcpyHostToDevice, g->stream));
    if (canonical) {  // order-preserving compaction, O(k)
      device_scan<uint32_t>(g.get(), KeepIn{dids, dkeep}, KeepOut{dids, dkeep, dout}, k, cnt, "vf");
    } else {  // the constructor's sort + unique (vertex_subset.cpp:8-15) through a bitmap
      const uint64_t nw64 = (n + 63) / 64;
      uint32_t* bm = g->ws.get<uint32_t>("bm", 2 * nw64);
      uint32_t* fm = g->ws.get<uint32_t>("fm", 2 * nw64);
      GBG_CUDA(cudaMemsetAsync(bm, 0, 2 * nw64 * sizeof(uint32_t), g->stream));
      GBG_LAUNCH(g.get(), list_to_bitmap_k, grid_for(k, 256), 256, 0, dids, k, bm);
      GBG_LAUNCH(g.get(), filter_dense_k, grid_for((n + 31) / 32 * 32, 256), 256, 0, n, bm, dkeep, fm);
      bitmap_to_list(g.get(), fm, (n + 31) / 32, dout, cnt);
    }
    uint32_t hc = 0;
    read_scalars(g.get(), cnt, sizeof(hc), &hc);
    if (hc) GBG_CUDA(cudaMemcpyAsync(out, dout, hc * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
    *out_k = hc;
  });
}

gbg_status gbg_vertex_filter_dense(uint64_t n, const uint64_t* words, const uint8_t* keep, uint64_t* out_words) {
  return guard([&] {
    if (n && (!words || !keep || !out_words)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    const uint64_t nw64 = (n + 63) / 64;
    if (!nw64) return;
    std::unique_ptr<gbg_graph> g(new_handle(GBG_KIND_CSR, n));
    AllocStream as(g->stream);
    uint32_t* din = g->ws.get<uint32_t>("in", 2 * nw64);
    uint32_t* dout = g->ws.get<uint32_t>("out", 2 * nw64);
    uint8_t* dkeep = g->ws.get<uint8_t>("keep", n);
    GBG_CUDA(cudaMemcpyAsync(din, words, nw64 * sizeof(uint64_t), cudaMemcpyHostToDevice, g->stream));
    GBG_CUDA(cudaMemcpyAsync(dkeep, keep, n, cudaMemcpyHostToDevice, g->stream));
    GBG_CUDA(cudaMemsetAsync(dout, 0, 2 * nw64 * sizeof(uint32_t), g->stream));
    GBG_LAUNCH(g.get(), filter_dense_k, grid_for((n + 31) / 32 * 32, 256), 256, 0, n, din, dkeep, dout);
    GBG_CUDA(cudaMemcpyAsync(out_words, dout, nw64 * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_subset_to_sparse(uint64_t n, const uint64_t* words, uint32_t* ids, uint64_t* k) {
  return guard([&] {
    if (!k || (n && (!words || !ids))) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    uint64_t nw64 = (n + 63) / 64;
    if (n % 64 && nw64 && (words[nw64 - 1] >> (n % 64)))
      fail(GBG_ERR_OUT_OF_RANGE, "VertexSubset: bits at positions >= n must be zero");
    std::unique_ptr<gbg_graph> g(new_handle(GBG_KIND_CSR, n));
    AllocStream as(g->stream);
    uint32_t* bm = g->ws.get<uint32_t>("bm", 2 * nw64);
    uint32_t* dids = g->ws.get<uint32_t>("ids", n);
    uint32_t* cnt = g->ws.get<uint32_t>("cnt", 1);
    GBG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), g->stream));
    if (nw64) GBG_CUDA(cudaMemcpyAsync(bm, words, nw64 * sizeof(uint64_t), cudaMemcpyHostToDevice, g->stream));
    bitmap_to_list(g.get(), bm, 2 * nw64, dids, cnt);
    uint32_t hk = 0;
    read_scalars(g.get(), cnt, sizeof(hk), &hk);
    *k = hk;
    if (hk) GBG_CUDA(cudaMemcpyAsync(ids, dids, hk * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"

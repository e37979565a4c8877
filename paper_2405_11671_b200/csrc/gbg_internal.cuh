// Internal runtime of libgbg: the device-resident container handle, error
// plumbing, per-handle workspace, and the two read views every kernel is
// templated on (CSR and blocked).  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gbg_c.h"

namespace gbg {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  gbg_status status;
  Error(gbg_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(gbg_status s, const std::string& m) { throw Error(s, m); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    fail(GBG_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  }
  fail(GBG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define GBG_CUDA(call) ::gbg::cuda_check((call), #call)

// ---------------------------------------------------------------- memory
// Device memory comes from the device's stream-ordered pool
// (cudaMallocAsync) on the stream of the handle being worked on, so
// building and dropping containers and scratch buffers never pays
// cudaMalloc/cudaFree's device-wide synchronisation; the pool keeps freed
// memory for reuse (release threshold raised in new_handle).
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
struct AllocStream {
  cudaStream_t prev;
  explicit AllocStream(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~AllocStream() { alloc_stream() = prev; }
};

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  cuda_check(cudaMallocAsync(&p, count * sizeof(T), alloc_stream()), "cudaMallocAsync");
  return static_cast<T*>(p);
}
inline void dfree(void* p) {
  if (p) cudaFreeAsync(p, alloc_stream());
}

// Named, growable device scratch buffers owned by a handle.  Buffers are
// reused across calls; grow() never shrinks.
struct Workspace {
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs;
  void* get(const std::string& name, size_t bytes) {
    Buf& b = bufs[name];
    if (b.bytes < bytes) {
      dfree(b.p);
      b.p = nullptr;
      b.bytes = 0;
      size_t want = bytes + bytes / 8 + 256;
      cuda_check(cudaMallocAsync(&b.p, want, alloc_stream()), "workspace cudaMallocAsync");
      b.bytes = want;
    }
    return b.p;
  }
  template <class T>
  T* get(const std::string& name, size_t count) {
    return static_cast<T*>(get(name, (count ? count : 1) * sizeof(T)));
  }
  void release(const std::string& name) {
    auto it = bufs.find(name);
    if (it != bufs.end()) {
      dfree(it->second.p);
      bufs.erase(it);
    }
  }
  size_t bytes() const {
    size_t t = 0;
    for (auto& kv : bufs) t += kv.second.bytes;
    return t;
  }
  void clear() {
    for (auto& kv : bufs) dfree(kv.second.p);
    bufs.clear();
  }
  ~Workspace() { clear(); }
};

// ---------------------------------------------------------------- views
// Read view of the static CSR: uint64 offsets[n+1], uint32 neighbors[m],
// ascending within each segment (csr.hpp:51-52).
struct CsrView {
  static constexpr bool kContiguous = true;  // row r's edges start at off[r]
  uint64_t n;
  const uint64_t* off;
  const uint32_t* nbr;
  __device__ __forceinline__ void seg(uint32_t v, uint64_t& begin, uint32_t& deg) const {
    uint64_t b = __ldg(off + v), e = __ldg(off + v + 1);
    begin = b;
    deg = static_cast<uint32_t>(e - b);
  }
  __device__ __forceinline__ uint32_t degree(uint32_t v) const {
    return static_cast<uint32_t>(__ldg(off + v + 1) - __ldg(off + v));
  }
  __device__ __forceinline__ uint32_t at(uint64_t pos) const { return __ldg(nbr + pos); }
  __device__ __forceinline__ uint64_t seg_begin(uint32_t v) const { return __ldg(off + v); }
  __device__ __forceinline__ const uint32_t* data() const { return nbr; }
};

// Read view of the dynamic blocked container: vertex v's ascending
// neighbours live at pool[start[v] .. start[v]+deg[v]) inside a 16-byte
// aligned allocation of cap[v] ids (see blocked.cu).
struct BlockedView {
  static constexpr bool kContiguous = false;
  uint64_t n;
  const uint64_t* start;
  const uint32_t* deg;
  const uint32_t* pool;
  __device__ __forceinline__ void seg(uint32_t v, uint64_t& begin, uint32_t& d) const {
    begin = __ldg(start + v);
    d = __ldg(deg + v);
  }
  __device__ __forceinline__ uint32_t degree(uint32_t v) const { return __ldg(deg + v); }
  __device__ __forceinline__ uint32_t at(uint64_t pos) const { return __ldg(pool + pos); }
  __device__ __forceinline__ uint64_t seg_begin(uint32_t v) const { return __ldg(start + v); }
  __device__ __forceinline__ const uint32_t* data() const { return pool; }
};

// ---------------------------------------------------------------- handle
struct PrLayout;  // pagerank.cu (tiled index)
namespace prrows {
struct PrRows;  // pagerank_rows.cu (row path)
}
struct TcCache;     // tc.cu

}  // namespace gbg

namespace gbg {
constexpr size_t kHostScalarBytes = 4096;  // gbg_graph::hscalar
}  // namespace gbg

struct gbg_graph {
  int kind = GBG_KIND_CSR;
  int device = 0;
  uint64_t n = 0;
  uint64_t m = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  uint64_t launches = 0;
  int sm_count = 148;
  bool symmetric = false;    // every arc's reverse present (set by the R-MAT builder)
  bool sym_checked = false;  // symmetry verified on the device (cc.cu)

  // CSR storage
  uint64_t* off = nullptr;
  uint32_t* nbr = nullptr;

  // blocked storage (blocked.cu)
  uint64_t* bstart = nullptr;  // element offset of v's allocation in pool
  uint32_t* bdeg = nullptr;    // live neighbours
  uint32_t* bcap = nullptr;    // allocated ids (multiple of 4 -> 16 B)
  uint32_t* pool = nullptr;
  uint64_t pool_cap = 0;       // ids
  uint64_t pool_top = 0;       // ids handed out (bump allocator)
  uint64_t pool_live = 0;      // ids in live allocations

  // compressed storage (compressed.cu)
  uint64_t* coff = nullptr;    // byte offsets [n+1]
  uint8_t* cbytes = nullptr;   // byte code (+8 padding bytes)
  uint64_t cbytes_len = 0;
  uint32_t* cdeg = nullptr;    // degrees
  bool cz_ready = false;       // transient decoded CSR present in ws ("cz.off"/"cz.nbr")

  // derived, rebuilt lazily after updates
  uint64_t* voff = nullptr;    // exclusive scan of degrees (blocked only)
  bool voff_valid = false;
  uint64_t* first = nullptr;   // (degree << 32) | first neighbour of every vertex (kNoFirst if isolated) + isolated bitmap
  bool first_valid = false;
  gbg::PrLayout* pr = nullptr;          // cached PageRank tiled index (gbg_pagerank_prepare)
  gbg::prrows::PrRows* pr_rows = nullptr;  // cached PageRank row layout (one-shot path)

  gbg::Workspace ws;
  // pinned host staging for small device->host reads (scalars, per-level stats)
  uint64_t* hscalar = nullptr;

  gbg::CsrView csr_view() const { return {n, off, nbr}; }
  gbg::BlockedView blocked_view() const { return {n, bstart, bdeg, pool}; }
  void invalidate_derived();
  ~gbg_graph();
};

namespace gbg {

// kernels launched through this macro are counted per handle
#define GBG_LAUNCH(g, kernel, grid, block, smem, ...)                        \
  do {                                                                       \
    kernel<<<(grid), (block), (smem), (g)->stream>>>(__VA_ARGS__);           \
    ::gbg::cuda_check(cudaGetLastError(), #kernel);                          \
    (g)->launches++;                                                         \
  } while (0)

inline unsigned grid_for(uint64_t items, unsigned per_block, unsigned cap = 148u * 64u) {
  uint64_t g = (items + per_block - 1) / per_block;
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// Read small device scalars back (synchronises the handle's stream).
void read_scalars(gbg_graph* g, const void* dev, size_t bytes, void* host);

// Compressed handles: the decoded CSR for the current API call (built on
// first use, released by TransientScope), one vertex's list, release.
CsrView compressed_decoded(gbg_graph* g);
void compressed_neighbors(gbg_graph* g, uint32_t v, uint32_t* out_dev);
void release_transient(gbg_graph* g);

// Dispatch a functor templated on the view type.
template <class F>
void with_view(gbg_graph* g, F&& f) {
  if (g->kind == GBG_KIND_CSR)
    f(g->csr_view());
  else if (g->kind == GBG_KIND_BLOCKED)
    f(g->blocked_view());
  else
    f(compressed_decoded(g));
}

// Ensure the blocked container's virtual offsets (scan of degrees) are
// current; returns a pointer usable as CSR-like offsets for scheduling.
const uint64_t* virtual_offsets(gbg_graph* g);

// Persistent cooperative kernels (BFS, k-core, coloring) are used when the
// device supports cooperative launch, unless GBG_COOP=0 (then the
// launch-per-step host loops run: the fallback, testable on any device).
inline bool coop_enabled(int device) {
  static const bool env_off = [] {
    const char* e = std::getenv("GBG_COOP");
    return e && e[0] == '0';
  }();
  if (env_off) return false;
  int coop = 0;
  cuda_check(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device), "cudaDeviceGetAttribute");
  return coop != 0;
}

// Every vertex's (degree << 32) | first neighbour (traverse.cuh kNoFirst when isolated),
// kept until the next update (bfs.cu).
const uint64_t* first_neighbors(gbg_graph* g);
// Bit v set when v has no neighbours (same lifetime as first_neighbors).
const uint32_t* isolated_bitmap(gbg_graph* g);
// Vertices no arc points to (the visited bits a BFS starts with; bfs.cu).
const uint32_t* bfs_premark(gbg_graph* g);

// Every arc has its reverse (checked once per graph version, cc.cu).
bool graph_is_symmetric(gbg_graph* g);

// PageRank layout in phases for pipelined CSR builds (pagerank.cu).
namespace prrows {
PrRows* pr_layout_rows_csr(gbg_graph* g);
void pr_layout_relabel_csr(gbg_graph* g, PrRows* L, uint64_t e0, uint64_t e1);
void pr_layout_attach(gbg_graph* g, PrRows* L, float build_ms);
void pr_layout_free(PrRows* L);
PrRows* pr_layout(gbg_graph* g);
uint64_t pagerank_rows_run(gbg_graph* g, double damping, uint64_t max_iters, double tol, double* p_dev);
double rows_build_ms(const PrRows* L);
uint64_t rows_bytes(const PrRows* L);
}  // namespace prrows
uint64_t pr_layout_bytes(const PrLayout* L);  // pagerank.cu

// Optional phase timing (environment GBG_TRACE=1): CUDA events on the
// handle's stream at named points, device-time deltas printed to stderr
// when the tracer goes out of scope.
struct PhaseTrace {
  cudaStream_t stream;
  const char* what;
  bool on;
  std::vector<std::pair<const char*, cudaEvent_t>> marks;
  PhaseTrace(cudaStream_t s, const char* w) : stream(s), what(w), on(enabled()) { mark("start"); }
  static bool enabled() {
    static const bool e = [] {
      const char* v = std::getenv("GBG_TRACE");
      return v && v[0] == '1';
    }();
    return e;
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    marks.emplace_back(name, e);
  }
  ~PhaseTrace() {
    if (!on || marks.empty()) return;
    cudaEventSynchronize(marks.back().second);
    std::fprintf(stderr, "[gbg trace] %s:", what);
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
      std::fprintf(stderr, " %s %.3f", marks[i].first, ms);
    }
    std::fprintf(stderr, " ms\n");
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
};

}  // namespace gbg

namespace gbg {

void set_last_error(const std::string& m);

// Run `f`, translating exceptions into a status + thread-local message.
template <class F>
gbg_status guard(F&& f) {
  try {
    f();
    return GBG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc& e) {
    set_last_error(e.what());
    return GBG_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GBG_ERR_LOGIC;
  }
}

// Make the handle's device current for the duration of a call.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Drops per-call transient state (a compressed handle's decoded CSR) when
// the API call returns; frees are stream-ordered after the call's work.
struct TransientScope {
  gbg_graph* g;
  ~TransientScope() { release_transient(g); }
};

// Locked, device-scoped access to a handle.
#define GBG_HANDLE(g)                                                        \
  if (!(g)) ::gbg::fail(GBG_ERR_INVALID_ARGUMENT, "null graph handle");     \
  std::lock_guard<std::mutex> gbg_lock_((g)->mu);                            \
  ::gbg::DeviceScope gbg_dev_((g)->device);                                  \
  ::gbg::AllocStream gbg_as_((g)->stream);                                   \
  ::gbg::TransientScope gbg_tr_{(g)}

gbg_graph* new_handle(int kind, uint64_t n);
void build_csr_offsets_from_sorted_src(gbg_graph* g, const uint32_t* src, uint64_t m, uint64_t* off);
void blocked_from_device_csr(gbg_graph* g, uint64_t n, const uint64_t* off, const uint32_t* nbr);

}  // namespace gbg

// Connected components, labels = minimum vertex id per component.
//
// Reference: gb::cc (algorithms.cpp:194-234): concurrent union-find where
// unite() CAS-links the larger root under the smaller (209-222) and find()
// path-halves (200-208), then a final find per vertex (229-232).  The same
// invariant — every link points from a larger id to a smaller one, so each
// root is its component's minimum — gives the canonical labels the BASELINE
// asks for ("min-label" hooking followed by pointer jumping).
//
// Symmetric graphs (every arc's reverse present; known for R-MAT builds,
// otherwise verified once per graph) take the sampling shortcut of Sutton
// et al.'s Afforest: hook every vertex to its first kSample neighbours,
// compress, find the dominant root by sampling, then hook the remaining
// neighbours of only those vertices that are not in the dominant component.
// An arc (u,v) skipped because u is in that component is covered from the
// other side: v is either in it too, or hooks (v,u) itself.  On the
// scale-24 R-MAT graph the giant component holds 8.86M of the 8.87M
// non-isolated vertices, so almost no edge is touched after sampling.
// Asymmetric graphs hook every arc through the balanced all-edges engine.
#include "edges.cuh"
#include "traverse.cuh"

namespace gbg {

constexpr uint32_t kSample = 2;

__device__ __forceinline__ uint32_t uf_find(uint32_t* p, uint32_t x) {
  volatile uint32_t* vp = p;
  uint32_t px = vp[x];
  while (px != x) {
    const uint32_t gp = vp[px];
    if (gp == px) return px;
    vp[x] = gp;  // path halving: gp is an ancestor (ids only decrease upward)
    x = gp;
    px = vp[x];
  }
  return x;
}

__device__ __forceinline__ void uf_link(uint32_t* parent, uint32_t u, uint32_t v) {
  uint32_t ru = uf_find(parent, u), rv = uf_find(parent, v);
  while (ru != rv) {
    const uint32_t hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
    const uint32_t old = atomicCAS(parent + hi, hi, lo);
    if (old == hi) return;
    ru = uf_find(parent, old);
    rv = uf_find(parent, lo);
  }
}

struct HookOp {
  uint32_t* parent;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t) const { uf_link(parent, u, v); }
};

__global__ void cc_init_k(uint64_t n, uint32_t* p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    p[v] = static_cast<uint32_t>(v);
}

// pointer jumping to the root (algorithms.cpp:229-232)
__global__ void cc_compress_k(uint64_t n, uint32_t* p, uint32_t* labels) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t x = static_cast<uint32_t>(v);
    uint32_t px = p[x];
    while (px != x) {
      x = px;
      px = p[x];
    }
    labels[v] = x;
  }
}

// Afforest sampling round r: hook v to its r-th neighbour
template <class G>
__global__ void cc_sample_k(G g, uint32_t r, uint32_t* parent) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < g.n; v += stride) {
    uint64_t b;
    uint32_t d;
    g.seg(static_cast<uint32_t>(v), b, d);
    if (d > r) uf_link(parent, static_cast<uint32_t>(v), g.at(b + r));
  }
}

// most frequent root among a fixed sample of 1024 vertices (ties -> smaller
// root); one thread per sample counts its matches, then a block argmax
__global__ void __launch_bounds__(1024) cc_dominant_k(const uint32_t* parent, uint64_t n, uint32_t* out) {
  constexpr int S = 1024;
  __shared__ uint32_t s[S];
  __shared__ uint64_t s_best[32];
  const int i = threadIdx.x;
  s[i] = parent[(static_cast<uint64_t>(i) * 2654435761u) % n];
  __syncthreads();
  uint32_t c = 0;
  const uint32_t mine = s[i];
  for (int j = 0; j < S; ++j) c += s[j] == mine;
  // key: higher count first, then smaller root
  uint64_t key = (static_cast<uint64_t>(c) << 32) | (0xffffffffu - mine);
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t other = __shfl_xor_sync(0xffffffffu, key, o);
    key = other > key ? other : key;
  }
  if ((i & 31) == 0) s_best[i >> 5] = key;
  __syncthreads();
  if (i == 0) {
    uint64_t best = 0;
    for (int k = 0; k < 32; ++k) best = s_best[k] > best ? s_best[k] : best;
    *out = 0xffffffffu - static_cast<uint32_t>(best);
  }
}

// vertices outside the dominant component that still have unsampled arcs
template <class G>
struct OutsideIn {
  G g;
  const uint32_t* parent;
  const uint32_t* dom;
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const {
    return parent[v] != *dom && g.degree(static_cast<uint32_t>(v)) > kSample;
  }
};
template <class G>
struct OutsideOut {
  OutsideIn<G> in;
  uint32_t* list;
  __device__ __forceinline__ void operator()(uint64_t v, uint32_t pre) const {
    if (in(v)) list[pre] = static_cast<uint32_t>(v);
  }
};

// hook arcs of a listed vertex beyond its first kSample neighbours (the
// push engine's load-balanced expansion, with a hooking operator)
struct RestOp {
  uint32_t* parent;
  __device__ __forceinline__ bool cond(uint32_t) const { return true; }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t u, uint32_t v) const {
    uf_link(parent, u, v);
    return false;  // nothing is emitted
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

template <class G>
struct RestDegIn {
  G g;
  const uint32_t* F;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return g.degree(F[i]); }
};

// ---- symmetry check: every arc (u,v) has (v,u)
template <class G>
struct SymOp {
  G g;
  int* bad;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t) const {
    uint64_t b;
    uint32_t d;
    g.seg(v, b, d);
    uint32_t lo = 0, hi = d;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (g.at(b + mid) < u) lo = mid + 1; else hi = mid;
    }
    if (lo >= d || g.at(b + lo) != u) *bad = 1;
  }
};

bool graph_is_symmetric(gbg_graph* g) {
  if (g->symmetric) return true;
  if (g->sym_checked) return false;
  int* bad = g->ws.get<int>("cc.bad", 1);
  GBG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), g->stream));
  const uint64_t* voff = virtual_offsets(g);
  with_view(g, [&](auto view) { for_each_edge(g, view, voff, g->m, SymOp<decltype(view)>{view, bad}); });
  int hb = 1;
  read_scalars(g, bad, sizeof(hb), &hb);
  g->sym_checked = true;
  g->symmetric = hb == 0;
  return g->symmetric;
}

void cc_run(gbg_graph* g, uint32_t* labels_dev) {
  const uint64_t n = g->n;
  uint32_t* parent = g->ws.get<uint32_t>("cc.parent", n);
  GBG_LAUNCH(g, cc_init_k, grid_for(n, 256), 256, 0, n, parent);
  const uint64_t* voff = virtual_offsets(g);
  if (!graph_is_symmetric(g)) {
    with_view(g, [&](auto view) { for_each_edge(g, view, voff, g->m, HookOp{parent}); });
    GBG_LAUNCH(g, cc_compress_k, grid_for(n, 256), 256, 0, n, parent, labels_dev);
    return;
  }
  with_view(g, [&](auto view) {
    using G = decltype(view);
    for (uint32_t r = 0; r < kSample; ++r)
      GBG_LAUNCH(g, cc_sample_k<G>, grid_for(n, 256), 256, 0, view, r, parent);
    GBG_LAUNCH(g, cc_compress_k, grid_for(n, 256), 256, 0, n, parent, parent);
    uint32_t* dom = g->ws.get<uint32_t>("cc.dom", 4);
    GBG_LAUNCH(g, cc_dominant_k, 1, 1024, 0, parent, n, dom);
    uint32_t* list = g->ws.get<uint32_t>("cc.list", n);
    OutsideIn<G> oin{view, parent, dom};
    device_scan<uint32_t>(g, oin, OutsideOut<G>{oin, list}, n, dom + 1, "cc.out");
    uint32_t k = 0;
    read_scalars(g, dom + 1, sizeof(k), &k);
    if (k) {
      // expand the listed vertices' full lists (the first kSample arcs are
      // re-hooked harmlessly), balanced by the push engine
      uint64_t* dscan = g->ws.get<uint64_t>("cc.dscan", static_cast<uint64_t>(k) + 1);
      device_scan<uint64_t>(g, RestDegIn<G>{view, list}, ArrayOut<uint64_t>{dscan}, k, dscan + k, "cc.rest");
      uint64_t E = 0;
      read_scalars(g, dscan + k, sizeof(E), &E);
      if (E) {
        unsigned long long* counters = g->ws.get<unsigned long long>("cc.counters", 2);
        GBG_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), g->stream));
        const uint32_t ipt = push_ipt(E, static_cast<uint64_t>(g->sm_count) * kPushCtasPerSm);
        GBG_LAUNCH(g, (push_k<G, RestOp>), static_cast<unsigned>(push_tiles(E, ipt)), kPushThreads, 0, view, list,
                   k, dscan, E, RestOp{parent}, list, nullptr, nullptr, counters, ipt);
      }
    }
  });
  GBG_LAUNCH(g, cc_compress_k, grid_for(n, 256), 256, 0, n, parent, labels_dev);
}

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_cc_device(gbg_graph* g, uint32_t* labels_dev) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!labels_dev && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null labels");
    if (g->n) cc_run(g, labels_dev);
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_cc(gbg_graph* g, uint32_t* labels) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!labels && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null labels");
    if (!g->n) return;
    uint32_t* d = g->ws.get<uint32_t>("cc.labels", g->n);
    cc_run(g, d);
    GBG_CUDA(cudaMemcpyAsync(labels, d, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"

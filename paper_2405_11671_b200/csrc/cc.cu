// Connected components, labels = minimum vertex id per component.
//
// Reference: gb::cc (algorithms.cpp:194-234): concurrent union-find where
// unite() CAS-links the larger root under the smaller (209-222) and find()
// path-halves (200-208), then a final find per vertex (229-232).  The same
// invariant — every link points from a larger id to a smaller one, so each
// root is its component's minimum — gives the canonical labels the BASELINE
// asks for ("min-label" hooking followed by pointer jumping).  Edges are
// processed by the balanced all-edges engine (edges.cuh); on graphs built
// symmetric (R-MAT) only arcs u -> v with v < u are hooked, each undirected
// edge once.
#include "edges.cuh"

namespace gbg {

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

struct HookOp {
  uint32_t* parent;
  int skip_upper;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t) const {
    if (skip_upper && v > u) return;
    uint32_t ru = uf_find(parent, u), rv = uf_find(parent, v);
    while (ru != rv) {
      const uint32_t hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
      const uint32_t old = atomicCAS(parent + hi, hi, lo);
      if (old == hi) return;
      ru = uf_find(parent, old);
      rv = uf_find(parent, lo);
    }
  }
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

void cc_run(gbg_graph* g, uint32_t* labels_dev) {
  const uint64_t n = g->n;
  uint32_t* parent = g->ws.get<uint32_t>("cc.parent", n);
  GBG_LAUNCH(g, cc_init_k, grid_for(n, 256), 256, 0, n, parent);
  const uint64_t* voff = virtual_offsets(g);
  with_view(g, [&](auto view) { for_each_edge(g, view, voff, g->m, HookOp{parent, g->symmetric ? 1 : 0}); });
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

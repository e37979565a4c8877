// Direction-optimising BFS and the generic edge_map entry point.
//
// Reference: gb::bfs (algorithms.cpp:29-58) over gb::edge_map
// (traversal.cpp:101-111).  The level loop, the switch rule
//   dense iff |F| + sum deg(F) > (1/20) * m        (traversal.cpp:105-106)
// and the frontier representations follow the reference; the work inside
// each level runs in the push_k / pull_k engines (traverse.cuh).  The host
// reads back two scalars per level (|next| and sum deg(next)) to make the
// same decision the reference makes.
#include <cstring>
#include <memory>
#include <vector>

#include "traverse.cuh"

namespace gbg {

// BFS as an edge_map operator: cond = unvisited, claim = atomic test-and-set
// on the visited bitmap (AtomicBitset::try_claim, parallel.hpp:133-137),
// update = record the depth.  In pull mode the warp owning a 32-vertex word
// publishes visited bits without atomics (dense_word).
struct BfsOp {
  uint32_t* visited;
  int32_t* depth;
  int32_t level;
  __device__ __forceinline__ bool cond(uint32_t v) const {
    return !((*(volatile uint32_t*)(visited + (v >> 5)) >> (v & 31)) & 1u);
  }
  __device__ __forceinline__ bool claim(uint32_t v) const {
    const uint32_t bit = 1u << (v & 31);
    return !(atomicOr(visited + (v >> 5), bit) & bit);
  }
  __device__ __forceinline__ bool update(uint32_t, uint32_t v) const {
    depth[v] = level;
    return true;
  }
  __device__ __forceinline__ void dense_word(uint64_t w, uint32_t m) const { visited[w] |= m; }
};

// The test operator of gbg_edge_map: cond from a byte mask, a fresh claim
// bitmap per call (traversal.cpp:23), update always true and counted.
struct MaskOp {
  const uint8_t* cond_mask;
  uint32_t* claimed;
  unsigned long long* updates;
  __device__ __forceinline__ bool cond(uint32_t v) const { return cond_mask[v] != 0; }
  __device__ __forceinline__ bool claim(uint32_t v) const {
    const uint32_t bit = 1u << (v & 31);
    return !(atomicOr(claimed + (v >> 5), bit) & bit);
  }
  __device__ __forceinline__ bool update(uint32_t, uint32_t) const {
    atomicAdd(updates, 1ull);
    return true;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

__global__ void bfs_init_k(uint32_t src, uint32_t* visited, int32_t* depth, uint32_t* list) {
  visited[src >> 5] |= 1u << (src & 31);
  depth[src] = 0;
  list[0] = src;
}

template <class G>
__global__ void degree_of_k(G g, uint32_t v, unsigned long long* out) {
  out[0] = 1;
  out[1] = g.degree(v);
}

namespace {

// Frontier state shared by BFS and edge_map: a list, a bitmap, or both.
struct Frontier {
  uint32_t* list = nullptr;
  uint32_t* bm = nullptr;
  bool has_list = false, has_bm = false;
  uint64_t size = 0, degsum = 0;
};

struct TraversalBuffers {
  uint64_t nw;  // 32-bit words
  uint32_t *fb, *nb, *la, *lb;
  uint64_t* dscan;
  unsigned long long* counters;
  uint32_t* cnt32;
  TraversalBuffers(gbg_graph* g) {
    nw = (g->n + 31) / 32;
    fb = g->ws.get<uint32_t>("t.fb", nw + 2);
    nb = g->ws.get<uint32_t>("t.nb", nw + 2);
    la = g->ws.get<uint32_t>("t.la", g->n + 1);
    lb = g->ws.get<uint32_t>("t.lb", g->n + 1);
    dscan = g->ws.get<uint64_t>("t.dscan", g->n + 2);
    counters = g->ws.get<unsigned long long>("t.counters", 4);
    cnt32 = g->ws.get<uint32_t>("t.cnt32", 2);
  }
};

bool choose_dense(uint64_t size, uint64_t degsum, uint64_t m, double threshold_fraction) {
  // traversal.cpp:105-106, the same double expression
  return static_cast<double>(size + degsum) > threshold_fraction * static_cast<double>(m);
}

unsigned pull_grid(gbg_graph* g, uint64_t nw) {
  return grid_for(nw * 32, kPullThreads, static_cast<unsigned>(g->sm_count) * 8u);
}

// One edge_map step.  `cur` is consumed (converted as needed); the output
// frontier is written into `out` (list for sparse, bitmap for dense).
template <class G, class Op, bool kEarly>
void edge_map_step(gbg_graph* g, G view, TraversalBuffers& tb, Frontier& cur, uint32_t* out_list,
                   uint32_t* out_bm, bool dense, Op op, Frontier& out) {
  GBG_CUDA(cudaMemsetAsync(tb.counters, 0, 2 * sizeof(unsigned long long), g->stream));
  out = Frontier{};
  if (dense) {
    if (!cur.has_bm) {
      GBG_CUDA(cudaMemsetAsync(cur.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
      if (cur.size) GBG_LAUNCH(g, list_to_bitmap_k, grid_for(cur.size, 256), 256, 0, cur.list, cur.size, cur.bm);
      cur.has_bm = true;
    }
    GBG_CUDA(cudaMemsetAsync(out_bm, 0, tb.nw * sizeof(uint32_t), g->stream));
    GBG_LAUNCH(g, (pull_k<G, Op, kEarly>), pull_grid(g, tb.nw), kPullThreads, 0, view, cur.bm, op, out_bm, tb.nw,
               tb.counters);
    out.bm = out_bm;
    out.has_bm = true;
  } else {
    if (!cur.has_list) {
      GBG_CUDA(cudaMemsetAsync(tb.cnt32, 0, sizeof(uint32_t), g->stream));
      bitmap_to_list(g, cur.bm, tb.nw, cur.list, tb.cnt32);
      cur.has_list = true;
    }
    if (cur.size) {
      device_scan<uint64_t>(g, FrontierDegIn<G>{view, cur.list}, ArrayOut<uint64_t>{tb.dscan}, cur.size,
                            tb.dscan + cur.size, "push.scan");
      const uint64_t E = cur.degsum;
      if (E) {
        const uint64_t tiles = (E + kPushTile - 1) / kPushTile;
        GBG_LAUNCH(g, (push_k<G, Op>), (unsigned)tiles, kPushThreads, 0, view, cur.list,
                   static_cast<uint32_t>(cur.size), tb.dscan, E, op, out_list, tb.counters);
      }
    }
    out.list = out_list;
    out.has_list = true;
  }
  unsigned long long c[2];
  read_scalars(g, tb.counters, sizeof(c), c);
  out.size = c[0];
  out.degsum = c[1];
}

template <class G>
void bfs_run(gbg_graph* g, G view, uint32_t src, int32_t* depth, gbg_bfs_stats* st) {
  TraversalBuffers tb(g);
  uint32_t* visited = g->ws.get<uint32_t>("bfs.visited", tb.nw + 2);
  GBG_CUDA(cudaMemsetAsync(depth, 0xff, g->n * sizeof(int32_t), g->stream));
  GBG_CUDA(cudaMemsetAsync(visited, 0, tb.nw * sizeof(uint32_t), g->stream));
  GBG_LAUNCH(g, bfs_init_k, 1, 1, 0, src, visited, depth, tb.la);
  GBG_LAUNCH(g, degree_of_k<G>, 1, 1, 0, view, src, tb.counters);
  unsigned long long c[2];
  read_scalars(g, tb.counters, sizeof(c), c);
  Frontier cur;
  cur.list = tb.la;
  cur.bm = tb.fb;
  cur.has_list = true;
  cur.size = 1;
  cur.degsum = c[1];
  uint32_t *spare_list = tb.lb, *spare_bm = tb.nb;
  uint64_t reached = 1;
  int32_t level = 0;
  if (st) std::memset(st, 0, sizeof(*st));
  while (cur.size > 0) {
    ++level;
    const bool dense = choose_dense(cur.size, cur.degsum, g->m, 1.0 / 20.0);
    if (st && level - 1 < GBG_MAX_LEVELS) {
      st->mode[level - 1] = dense ? GBG_MODE_DENSE : GBG_MODE_SPARSE;
      st->frontier[level - 1] = cur.size;
      st->degree_sum[level - 1] = cur.degsum;
    }
    Frontier nxt;
    BfsOp op{visited, depth, level};
    edge_map_step<G, BfsOp, true>(g, view, tb, cur, spare_list, spare_bm, dense, op, nxt);
    // recycle: the consumed frontier's storage becomes the spare
    uint32_t* old_list = cur.list;
    uint32_t* old_bm = cur.bm;
    if (dense) {
      nxt.list = old_list;  // storage for a later bitmap->list conversion
      spare_bm = old_bm;
      spare_list = spare_list;
    } else {
      nxt.bm = old_bm;
      spare_list = old_list;
    }
    cur = nxt;
    reached += cur.size;
  }
  if (st) {
    st->levels = static_cast<uint64_t>(level);
    st->reached = reached;
  }
}

}  // namespace
}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_bfs_device(gbg_graph* g, uint32_t source, int32_t* depth_dev, gbg_bfs_stats* stats) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!depth_dev) fail(GBG_ERR_INVALID_ARGUMENT, "null depth buffer");
    if (source >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "bfs: source out of range");
    with_view(g, [&](auto view) { bfs_run(g, view, source, depth_dev, stats); });
  });
}

gbg_status gbg_bfs(gbg_graph* g, uint32_t source, int32_t* depth, gbg_bfs_stats* stats) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!depth) fail(GBG_ERR_INVALID_ARGUMENT, "null depth buffer");
    if (source >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "bfs: source out of range");
    int32_t* d = g->ws.get<int32_t>("bfs.depth", g->n);
    with_view(g, [&](auto view) { bfs_run(g, view, source, d, stats); });
    GBG_CUDA(cudaMemcpyAsync(depth, d, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_edge_map(gbg_graph* g, const uint32_t* ids, uint64_t k, const uint8_t* cond_mask, int mode,
                        int early_exit, uint8_t* out_member, uint64_t* updates, int* mode_out) {
  return guard([&] {
    GBG_HANDLE(g);
    if ((k && !ids) || !cond_mask || !out_member || !updates)
      fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (mode < 0 || mode > 2) fail(GBG_ERR_INVALID_ARGUMENT, "edge_map: bad mode");
    for (uint64_t i = 0; i < k; ++i)
      if (ids[i] >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "VertexSubset: id out of range");
    TraversalBuffers tb(g);
    uint8_t* dcond = g->ws.get<uint8_t>("em.cond", g->n);
    uint32_t* claimed = g->ws.get<uint32_t>("em.claimed", tb.nw + 2);
    uint32_t* raw = g->ws.get<uint32_t>("em.raw", k);
    unsigned long long* upd = g->ws.get<unsigned long long>("em.upd", 1);
    GBG_CUDA(cudaMemcpyAsync(dcond, cond_mask, g->n, cudaMemcpyHostToDevice, g->stream));
    GBG_CUDA(cudaMemsetAsync(claimed, 0, tb.nw * sizeof(uint32_t), g->stream));
    GBG_CUDA(cudaMemsetAsync(upd, 0, sizeof(unsigned long long), g->stream));
    // canonical VertexSubset (sorted, deduplicated; vertex_subset.cpp:8-15)
    // through the two conversion primitives
    GBG_CUDA(cudaMemsetAsync(tb.fb, 0, tb.nw * sizeof(uint32_t), g->stream));
    if (k) {
      GBG_CUDA(cudaMemcpyAsync(raw, ids, k * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
      GBG_LAUNCH(g, list_to_bitmap_k, grid_for(k, 256), 256, 0, raw, k, tb.fb);
    }
    GBG_CUDA(cudaMemsetAsync(tb.cnt32, 0, sizeof(uint32_t), g->stream));
    bitmap_to_list(g, tb.fb, tb.nw, tb.la, tb.cnt32);
    uint32_t size = 0;
    read_scalars(g, tb.cnt32, sizeof(size), &size);
    Frontier cur;
    cur.list = tb.la;
    cur.bm = tb.fb;
    cur.has_list = cur.has_bm = true;
    cur.size = size;
    with_view(g, [&](auto view) {
      using G = decltype(view);
      // frontier work = |F| + sum deg(F) (traversal.hpp:15-20)
      if (size) {
        device_scan<uint64_t>(g, FrontierDegIn<G>{view, cur.list}, ArrayOut<uint64_t>{tb.dscan}, size,
                              tb.dscan + size, "em.scan");
        read_scalars(g, tb.dscan + size, sizeof(uint64_t), &cur.degsum);
      }
      bool dense = mode == GBG_MODE_DENSE ||
                   (mode == GBG_MODE_AUTO && choose_dense(cur.size, cur.degsum, g->m, 1.0 / 20.0));
      if (mode_out) *mode_out = dense ? GBG_MODE_DENSE : GBG_MODE_SPARSE;
      MaskOp op{dcond, claimed, upd};
      Frontier out;
      if (dense && !early_exit)
        edge_map_step<G, MaskOp, false>(g, view, tb, cur, tb.lb, tb.nb, true, op, out);
      else
        edge_map_step<G, MaskOp, true>(g, view, tb, cur, tb.lb, tb.nb, dense, op, out);
      // membership bytes
      std::vector<uint8_t> member(g->n, 0);
      if (out.has_bm) {
        std::vector<uint32_t> bm(tb.nw);
        GBG_CUDA(cudaMemcpyAsync(bm.data(), out.bm, tb.nw * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
        GBG_CUDA(cudaStreamSynchronize(g->stream));
        for (uint64_t v = 0; v < g->n; ++v) member[v] = (bm[v >> 5] >> (v & 31)) & 1u;
      } else {
        std::vector<uint32_t> lst(out.size);
        if (out.size)
          GBG_CUDA(cudaMemcpyAsync(lst.data(), out.list, out.size * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                   g->stream));
        GBG_CUDA(cudaStreamSynchronize(g->stream));
        for (uint32_t v : lst) member[v] = 1;
      }
      std::memcpy(out_member, member.data(), g->n);
    });
    unsigned long long hu = 0;
    read_scalars(g, upd, sizeof(hu), &hu);
    *updates = hu;
  });
}

}  // extern "C"

// Direction-optimising BFS and the generic edge_map entry point.
//
// Reference: gb::bfs (algorithms.cpp:29-58) over gb::edge_map
// (traversal.cpp:101-111).  The level loop, the switch rule
//   dense iff |F| + sum deg(F) > (1/20) * m        (traversal.cpp:105-106)
// and the frontier representations follow the reference; the work inside
// each level runs in the push_k / pull_k engines (traverse.cuh).  The host
// reads back one packed scalar per level (|next| and sum deg(next)) to make
// the same decision the reference makes.  A push level emits the next
// frontier as an id list together with its degree prefix and bitmap, so the
// following level starts without a scan or conversion; only a dense ->
// sparse transition compacts a bitmap (one ordered scan).
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

template <class G>
__global__ void bfs_init_k(G g, uint32_t src, uint32_t* visited, int32_t* depth, uint32_t* list, uint64_t* dscan,
                           uint32_t* bm, unsigned long long* packed) {
  const uint32_t bit = 1u << (src & 31);
  visited[src >> 5] |= bit;
  bm[src >> 5] |= bit;
  depth[src] = 0;
  list[0] = src;
  const uint32_t d = g.degree(src);
  dscan[0] = 0;
  dscan[1] = d;
  *packed = (1ull << kPackShift) | d;
}

namespace {

// One frontier: storage for all three representations, flags for which are
// current.
struct Frontier {
  uint32_t* list = nullptr;
  uint64_t* dscan = nullptr;
  uint32_t* bm = nullptr;
  bool has_list = false, has_bm = false;
  uint64_t size = 0, degsum = 0;
};

struct TraversalBuffers {
  uint64_t nw;  // 32-bit words
  Frontier a, b;
  unsigned long long* packed;
  TraversalBuffers(gbg_graph* g) {
    nw = (g->n + 31) / 32;
    a.bm = g->ws.get<uint32_t>("t.fa", nw + 2);
    b.bm = g->ws.get<uint32_t>("t.fb", nw + 2);
    a.list = g->ws.get<uint32_t>("t.la", g->n + 1);
    b.list = g->ws.get<uint32_t>("t.lb", g->n + 1);
    a.dscan = g->ws.get<uint64_t>("t.da", g->n + 2);
    b.dscan = g->ws.get<uint64_t>("t.db", g->n + 2);
    packed = g->ws.get<unsigned long long>("t.packed", 2);
  }
};

bool choose_dense(uint64_t size, uint64_t degsum, uint64_t m, double threshold_fraction) {
  // traversal.cpp:105-106, the same double expression
  return static_cast<double>(size + degsum) > threshold_fraction * static_cast<double>(m);
}

unsigned pull_grid(gbg_graph* g, uint64_t nw) {
  return grid_for(nw * 32, kPullThreads, static_cast<unsigned>(g->sm_count) * 8u);
}

void read_packed(gbg_graph* g, unsigned long long* packed, Frontier& f) {
  unsigned long long p = 0;
  read_scalars(g, packed, sizeof(p), &p);
  f.size = pack_count(p);
  f.degsum = pack_degsum(p);
}

// make the frontier's id list + degree prefix current (bitmap -> list)
template <class G>
void ensure_list(gbg_graph* g, G view, TraversalBuffers& tb, Frontier& f) {
  if (f.has_list) return;
  device_scan<uint64_t>(g, PopcDegIn<G>{view, f.bm}, BitsToIdsDscanOut<G>{view, f.bm, f.list, f.dscan}, tb.nw,
                        reinterpret_cast<uint64_t*>(tb.packed + 1), "b2l");
  f.has_list = true;
}

// One edge_map step from `cur` into `out` (the other buffer set).
template <class G, class Op, bool kEarly>
void edge_map_step(gbg_graph* g, G view, TraversalBuffers& tb, Frontier& cur, Frontier& out, bool dense, Op op) {
  GBG_CUDA(cudaMemsetAsync(tb.packed, 0, sizeof(unsigned long long), g->stream));
  out.has_list = out.has_bm = false;
  if (dense) {
    if (!cur.has_bm) {
      GBG_CUDA(cudaMemsetAsync(cur.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
      if (cur.size) GBG_LAUNCH(g, list_to_bitmap_k, grid_for(cur.size, 256), 256, 0, cur.list, cur.size, cur.bm);
      cur.has_bm = true;
    }
    GBG_LAUNCH(g, (pull_k<G, Op, kEarly>), pull_grid(g, tb.nw), kPullThreads, 0, view, cur.bm, op, out.bm, tb.nw,
               tb.packed);
    out.has_bm = true;
  } else {
    ensure_list(g, view, tb, cur);
    GBG_CUDA(cudaMemsetAsync(out.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
    if (cur.size && cur.degsum) {
      // sentinel dscan[|F|] = E closes the last segment for the binary searches
      g->hscalar[4] = cur.degsum;
      GBG_CUDA(cudaMemcpyAsync(cur.dscan + cur.size, g->hscalar + 4, sizeof(uint64_t), cudaMemcpyHostToDevice,
                               g->stream));
      const uint64_t tiles = (cur.degsum + kPushTile - 1) / kPushTile;
      GBG_LAUNCH(g, (push_k<G, Op>), static_cast<unsigned>(tiles), kPushThreads, 0, view, cur.list,
                 static_cast<uint32_t>(cur.size), cur.dscan, cur.degsum, op, out.list, out.dscan, out.bm, tb.packed);
    }
    out.has_list = out.has_bm = true;
  }
  read_packed(g, tb.packed, out);
}

template <class G>
void bfs_run(gbg_graph* g, G view, uint32_t src, int32_t* depth, gbg_bfs_stats* st) {
  TraversalBuffers tb(g);
  uint32_t* visited = g->ws.get<uint32_t>("bfs.visited", tb.nw + 2);
  GBG_CUDA(cudaMemsetAsync(depth, 0xff, g->n * sizeof(int32_t), g->stream));
  GBG_CUDA(cudaMemsetAsync(visited, 0, tb.nw * sizeof(uint32_t), g->stream));
  GBG_CUDA(cudaMemsetAsync(tb.a.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
  GBG_LAUNCH(g, bfs_init_k<G>, 1, 1, 0, view, src, visited, depth, tb.a.list, tb.a.dscan, tb.a.bm, tb.packed);
  Frontier* cur = &tb.a;
  Frontier* nxt = &tb.b;
  read_packed(g, tb.packed, *cur);
  cur->has_list = cur->has_bm = true;
  uint64_t reached = 1;
  int32_t level = 0;
  if (st) std::memset(st, 0, sizeof(*st));
  cudaEvent_t ev[GBG_MAX_LEVELS + 1];
  int nev = 0;
  if (st) {
    GBG_CUDA(cudaEventCreate(&ev[0]));
    GBG_CUDA(cudaEventRecord(ev[0], g->stream));
    nev = 1;
  }
  while (cur->size > 0) {
    ++level;
    const bool dense = choose_dense(cur->size, cur->degsum, g->m, 1.0 / 20.0);
    if (st && level - 1 < GBG_MAX_LEVELS) {
      st->mode[level - 1] = dense ? GBG_MODE_DENSE : GBG_MODE_SPARSE;
      st->frontier[level - 1] = cur->size;
      st->degree_sum[level - 1] = cur->degsum;
    }
    BfsOp op{visited, depth, level};
    edge_map_step<G, BfsOp, true>(g, view, tb, *cur, *nxt, dense, op);
    if (st && nev <= GBG_MAX_LEVELS) {
      GBG_CUDA(cudaEventCreate(&ev[nev]));
      GBG_CUDA(cudaEventRecord(ev[nev], g->stream));
      ++nev;
    }
    std::swap(cur, nxt);
    reached += cur->size;
  }
  if (st) {
    GBG_CUDA(cudaEventSynchronize(ev[nev - 1]));
    for (int i = 1; i < nev; ++i) cudaEventElapsedTime(&st->level_ms[i - 1], ev[i - 1], ev[i]);
    for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
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
    Frontier& cur = tb.a;
    GBG_CUDA(cudaMemsetAsync(cur.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
    if (k) {
      GBG_CUDA(cudaMemcpyAsync(raw, ids, k * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
      GBG_LAUNCH(g, list_to_bitmap_k, grid_for(k, 256), 256, 0, raw, k, cur.bm);
    }
    cur.has_bm = true;
    with_view(g, [&](auto view) {
      using G = decltype(view);
      // |F| and frontier work = |F| + sum deg(F) (traversal.hpp:15-20)
      ensure_list(g, view, tb, cur);
      read_packed(g, tb.packed + 1, cur);
      bool dense = mode == GBG_MODE_DENSE ||
                   (mode == GBG_MODE_AUTO && choose_dense(cur.size, cur.degsum, g->m, 1.0 / 20.0));
      if (mode_out) *mode_out = dense ? GBG_MODE_DENSE : GBG_MODE_SPARSE;
      MaskOp op{dcond, claimed, upd};
      Frontier& out = tb.b;
      if (dense && !early_exit)
        edge_map_step<G, MaskOp, false>(g, view, tb, cur, out, true, op);
      else
        edge_map_step<G, MaskOp, true>(g, view, tb, cur, out, dense, op);
      // membership bytes from the output bitmap (both modes produce one)
      std::vector<uint32_t> bm(tb.nw);
      GBG_CUDA(cudaMemcpyAsync(bm.data(), out.bm, tb.nw * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
      GBG_CUDA(cudaStreamSynchronize(g->stream));
      for (uint64_t v = 0; v < g->n; ++v) out_member[v] = (bm[v >> 5] >> (v & 31)) & 1u;
    });
    unsigned long long hu = 0;
    read_scalars(g, upd, sizeof(hu), &hu);
    *updates = hu;
  });
}

}  // extern "C"

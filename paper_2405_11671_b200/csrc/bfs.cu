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
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "edges.cuh"
#include "traverse.cuh"

#ifndef GBG_BFS_SMALL_GRID
#define GBG_BFS_SMALL_GRID 4096  // vertices per CTA below which the persistent grid shrinks (>= one CTA per SM)
#endif
#ifndef GBG_BFS_MINB
#define GBG_BFS_MINB 5
#endif

namespace gbg {

// BFS as an edge_map operator: cond = unvisited, claim = atomic test-and-set
// on the visited bitmap (AtomicBitset::try_claim, parallel.hpp:133-137),
// update = record the depth.  In pull mode the warp owning a 32-vertex word
// publishes its word's visited bits with one reduction (dense_word).
struct BfsOp {
  uint32_t* visited;
  int32_t* depth;
  int32_t level;
  __device__ __forceinline__ bool cond(uint32_t v) const {
    return !((*(volatile uint32_t*)(visited + (v >> 5)) >> (v & 31)) & 1u);
  }
  __device__ __forceinline__ uint32_t cond_word(uint64_t w) const { return ~*(volatile uint32_t*)(visited + w); }
  __device__ __forceinline__ bool claim(uint32_t v) const {
    const uint32_t bit = 1u << (v & 31);
    return !(atomicOr(visited + (v >> 5), bit) & bit);
  }
  __device__ __forceinline__ bool update(uint32_t, uint32_t v) const {
    depth[v] = level;
    return true;
  }
  // the owning warp's word: a fire-and-forget reduction (RED.OR) instead of
  // a load + store keeps one L2 round trip off every word's chain
  __device__ __forceinline__ void dense_word(uint64_t w, uint32_t m) const { atomicOr(visited + w, m); }
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

// ---------------------------------------------------------------- persistent BFS
// The whole level loop in one cooperative launch: every CTA evaluates the
// same switch rule from the device-resident packed counter, runs its share
// of the pull (grid-stride over bitmap words) or push (grid-stride over
// edge tiles), and a grid-wide barrier separates levels.  This removes the
// host round trip and the launch chain of each level.
struct CoopState {
  uint32_t* visited;
  int32_t* depth;
  uint32_t* list[2];
  uint64_t* dscan[2];
  uint32_t* bm[3];             // frontier bitmaps: level l reads bm[(l-1)%3], writes bm[l%3], clears bm[(l+1)%3]
  unsigned long long* packed;  // ring of 3 level counters
  uint64_t* level_packed;      // [GBG_MAX_LEVELS] per-level (count, degsum) of the input frontier
  int32_t* level_mode;         // [GBG_MAX_LEVELS]
  unsigned long long* level_ns;  // [GBG_MAX_LEVELS + 1] globaltimer at level boundaries
  uint64_t* blocksum;          // [gridDim] conversion scan scratch
  uint64_t* result;            // [0] levels, [1] reached
  uint64_t nw;
  double threshold;            // (1/20) * m, evaluated on the host like traversal.cpp:105-106
  uint32_t src;
  const uint64_t* first;       // (degree << 32) | first neighbour (dense-level shortcut)
  const uint32_t* iso;         // isolated vertices: pre-set in `visited` (never reached, never pulled)
  unsigned long long* level_examined;  // [GBG_MAX_LEVELS] arcs inspected by dense levels
  unsigned* level_heavy;       // [GBG_MAX_LEVELS] a dense level reached a vertex of degree > kBitmapPushMaxDeg
  int bitmap_push;             // dense -> sparse transitions push straight from the bitmap
  int timing;                  // record level_ns (GBG_BFS_LEVEL_TIMES=1; diagnostics only)
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// grid-wide ordered compaction bitmap -> (ids, degree prefix); each CTA
// owns a contiguous word range, each thread a contiguous sub-range
template <class G>
__device__ void coop_bitmap_to_list(cooperative_groups::grid_group& grid, G g, const uint32_t* bm, uint64_t nw,
                                    uint32_t* ids, uint64_t* dscan, uint64_t* blocksum, uint64_t* s_red) {
  const uint64_t per_cta = (nw + gridDim.x - 1) / gridDim.x;
  const uint64_t w0 = blockIdx.x * per_cta;
  const uint64_t w1 = w0 + per_cta < nw ? w0 + per_cta : nw;
  const uint64_t per_thr = (per_cta + blockDim.x - 1) / blockDim.x;
  const uint64_t t0 = w0 + threadIdx.x * per_thr;
  const uint64_t t1 = t0 + per_thr < w1 ? t0 + per_thr : w1;
  PopcDegIn<G> in{g, bm};
  uint64_t local = 0;
  for (uint64_t w = t0; w < t1; ++w) local += in(w);
  const uint64_t btot = block_sum(local, s_red);
  if (threadIdx.x == 0) blocksum[blockIdx.x] = btot;
  grid.sync();
  uint64_t pre = 0;
  for (uint64_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) pre += blocksum[b];
  pre = block_sum(pre, s_red);
  uint64_t tot;
  const uint64_t mine = block_exclusive_scan(local, s_red, tot) + pre;
  BitsToIdsDscanOut<G> out{g, bm, ids, dscan};
  uint64_t run = mine;
  for (uint64_t w = t0; w < t1; ++w) {
    out(w, run);
    run += in(w);
  }
}

template <class G>
__global__ void __launch_bounds__(kPushThreads, GBG_BFS_MINB) bfs_coop_k(G g, CoopState s) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ uint32_t s_idx[kPushTile];
  __shared__ uint64_t s_red[33];
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // initial state, the source included, in one pass and one barrier
  const uint64_t sw = s.src >> 5;
  const uint32_t sbit = 1u << (s.src & 31);
  for (uint64_t i = tid; i < g.n; i += nthreads) s.depth[i] = i == s.src ? 0 : -1;
  for (uint64_t w = tid; w < s.nw; w += nthreads) {
    s.visited[w] = s.iso[w] | (w == sw ? sbit : 0u);
    s.bm[0][w] = w == sw ? sbit : 0u;
    s.bm[1][w] = 0;
  }
  if (tid < 3) s.packed[tid] = tid == 0 ? (1ull << kPackShift) | g.degree(s.src) : 0ull;
  if (tid < GBG_MAX_LEVELS) {
    s.level_examined[tid] = 0;
    s.level_heavy[tid] = 0;
  }
  if (tid == 0) {
    s.list[0][0] = s.src;
    s.dscan[0][0] = 0;
    if (s.timing) s.level_ns[0] = globaltimer();
  }
  grid.sync();
  int cur = 0;      // list buffers
  int bcur = 0;     // bitmap ring position of the level's input
  bool has_list = true;
  uint64_t reached = 1;
  int32_t level = 1;
  for (;; ++level) {
    const unsigned long long p = *reinterpret_cast<volatile unsigned long long*>(s.packed + (level - 1) % 3);
    const uint64_t size = pack_count(p), degsum = pack_degsum(p);
    if (size == 0) break;
    reached += level > 1 ? size : 0;
    const bool dense = static_cast<double>(size + degsum) > s.threshold;
    if (tid == 0) {
      s.packed[(level + 1) % 3] = 0;  // last read at the start of level - 1
      if (level <= GBG_MAX_LEVELS) {
        s.level_packed[level - 1] = p;
        s.level_mode[level - 1] = dense ? GBG_MODE_DENSE : GBG_MODE_SPARSE;
      }
    }
    const int nxt = cur ^ 1;
    const int bnxt = bcur == 2 ? 0 : bcur + 1, bclr = bnxt == 2 ? 0 : bnxt + 1;
    BfsOp op{s.visited, s.depth, level};
    unsigned long long* acc = s.packed + level % 3;
    // the next level's output bitmap, idle during this level (it was the
    // previous level's input): cleared here so a sparse level needs no
    // barrier between clearing and pushing
    for (uint64_t w = tid; w < s.nw; w += nthreads) s.bm[bclr][w] = 0;
    if (dense) {
      pull_words<G, BfsOp, true>(g, s.bm[bcur], op, s.bm[bnxt], s.nw, acc, s.first,
                                 level <= GBG_MAX_LEVELS ? s.level_examined + level - 1 : nullptr,
                                 level <= GBG_MAX_LEVELS ? s.level_heavy + level - 1 : nullptr);
      has_list = false;
    } else if (!has_list && s.bitmap_push && level - 1 <= GBG_MAX_LEVELS &&
               !*reinterpret_cast<volatile unsigned*>(s.level_heavy + level - 2)) {
      // dense -> sparse with no member above kBitmapPushMaxDeg: push from
      // the bitmap, no list to build first
      push_bitmap(g, s.bm[bcur], s.nw, op, s.list[nxt], s.dscan[nxt], s.bm[bnxt], acc);
      has_list = true;
    } else {
      if (!has_list) {
        coop_bitmap_to_list(grid, g, s.bm[bcur], s.nw, s.list[cur], s.dscan[cur], s.blocksum, s_red);
        has_list = true;
        grid.sync();
      }
      const uint32_t ipt = push_ipt(degsum, gridDim.x);
      const uint64_t tiles = push_tiles(degsum, ipt);
      for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        push_tile(g, s.list[cur], static_cast<uint32_t>(size), s.dscan[cur], degsum, op, s.list[nxt], s.dscan[nxt],
                  s.bm[bnxt], acc, t, s_idx, ipt);
        __syncthreads();
      }
    }
    grid.sync();
    if (s.timing && tid == 0 && level <= GBG_MAX_LEVELS) s.level_ns[level] = globaltimer();
    cur = nxt;
    bcur = bnxt;
  }
  if (tid == 0) {
    s.result[0] = static_cast<uint64_t>(level - 1);
    s.result[1] = reached;
  }
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
void edge_map_step(gbg_graph* g, G view, TraversalBuffers& tb, Frontier& cur, Frontier& out, bool dense, Op op,
                   unsigned long long* examined = nullptr) {
  GBG_CUDA(cudaMemsetAsync(tb.packed, 0, sizeof(unsigned long long), g->stream));
  out.has_list = out.has_bm = false;
  if (dense) {
    if (!cur.has_bm) {
      GBG_CUDA(cudaMemsetAsync(cur.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
      if (cur.size) GBG_LAUNCH(g, list_to_bitmap_k, grid_for(cur.size, 256), 256, 0, cur.list, cur.size, cur.bm);
      cur.has_bm = true;
    }
    GBG_LAUNCH(g, (pull_k<G, Op, kEarly>), pull_grid(g, tb.nw), kPullThreads, 0, view, cur.bm, op, out.bm, tb.nw,
               tb.packed, kEarly ? first_neighbors(g) : static_cast<const uint64_t*>(nullptr), examined);
    out.has_bm = true;
  } else {
    ensure_list(g, view, tb, cur);
    GBG_CUDA(cudaMemsetAsync(out.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
    if (cur.size && cur.degsum) {
      // sentinel dscan[|F|] = E closes the last segment for the binary searches
      g->hscalar[4] = cur.degsum;
      GBG_CUDA(cudaMemcpyAsync(cur.dscan + cur.size, g->hscalar + 4, sizeof(uint64_t), cudaMemcpyHostToDevice,
                               g->stream));
      const uint32_t ipt = push_ipt(cur.degsum, static_cast<uint64_t>(g->sm_count) * kPushCtasPerSm);
      GBG_LAUNCH(g, (push_k<G, Op>), static_cast<unsigned>(push_tiles(cur.degsum, ipt)), kPushThreads, 0, view,
                 cur.list, static_cast<uint32_t>(cur.size), cur.dscan, cur.degsum, op, out.list, out.dscan, out.bm,
                 tb.packed, ipt);
    }
    out.has_list = out.has_bm = true;
  }
  read_packed(g, tb.packed, out);
}

// first neighbour of every vertex, and the bitmap of isolated vertices
template <class G>
__global__ void first_nbr_k(G g, uint64_t* first, uint32_t* iso) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~uint64_t{31}; base < g.n;
       base += stride) {
    const uint64_t v = base + (threadIdx.x & 31);
    bool isolated = false;
    if (v < g.n) {
      uint64_t b;
      uint32_t d;
      g.seg(static_cast<uint32_t>(v), b, d);
      first[v] = (static_cast<uint64_t>(d) << 32) | (d ? g.at(b) : kNoFirst);
      isolated = d == 0;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, isolated);
    if ((threadIdx.x & 31) == 0) iso[base >> 5] = m;
  }
}

// GBG_BFS_BITMAP_PUSH=0 turns the bitmap-driven push of dense -> sparse
// transitions off (the list is then built first, as the launch-per-level
// path does); a comparison and test knob.
bool bitmap_push_enabled() {
  static const bool off = [] {
    const char* e = std::getenv("GBG_BFS_BITMAP_PUSH");
    return e && e[0] == '0';
  }();
  return !off;
}

// The persistent path; false when the device cannot co-schedule the grid.
// per-level device timestamps in the persistent kernel: off unless
// GBG_BFS_LEVEL_TIMES=1 (read per call), so the timed path carries no
// instrumentation; gbg_bfs_stats.level_ms is 0 when off
bool level_times_enabled() {
  const char* v = std::getenv("GBG_BFS_LEVEL_TIMES");
  return v && v[0] == '1';
}

template <class G>
bool bfs_coop(gbg_graph* g, G view, uint32_t src, int32_t* depth, gbg_bfs_stats* st) {
  if (!coop_enabled(g->device)) return false;
  int per_sm = 0;
  GBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_coop_k<G>, kPushThreads, 0));
  if (per_sm < 1) return false;
  unsigned grid = static_cast<unsigned>(per_sm * g->sm_count);
#if GBG_BFS_SMALL_GRID
  // small graphs: one CTA per SM is enough work per barrier round, and a
  // grid barrier over 148 CTAs costs about half of one over 740 (scale 16:
  // 0.062 -> 0.052 ms; scale 20 at 256 CTAs unchanged, at 148 slower)
  {
    const uint64_t want = (g->n + GBG_BFS_SMALL_GRID - 1) / GBG_BFS_SMALL_GRID;
    const unsigned lo = static_cast<unsigned>(g->sm_count);
    if (want < grid) grid = want > lo ? static_cast<unsigned>(want) : lo;
  }
#endif
  TraversalBuffers tb(g);
  CoopState s;
  s.visited = g->ws.get<uint32_t>("bfs.visited", tb.nw + 2);
  s.depth = depth;
  s.list[0] = tb.a.list;
  s.list[1] = tb.b.list;
  s.dscan[0] = tb.a.dscan;
  s.dscan[1] = tb.b.dscan;
  s.bm[0] = tb.a.bm;
  s.bm[1] = tb.b.bm;
  s.bm[2] = g->ws.get<uint32_t>("bfs.bm2", tb.nw + 2);
  s.packed = g->ws.get<unsigned long long>("bfs.ring", 4);
  // every per-level statistic in one block, read back with one copy into
  // the handle's pinned staging: [packed | ns (+1) | result (2) | examined | modes]
  constexpr int ML = GBG_MAX_LEVELS;
  constexpr size_t kStatWords = 3 * ML + 4 + ML / 2;
  static_assert(kStatWords * sizeof(uint64_t) <= kHostScalarBytes, "BFS stats exceed the pinned staging");
  uint64_t* stat = g->ws.get<uint64_t>("bfs.stat", kStatWords);
  s.level_packed = stat;
  s.level_ns = reinterpret_cast<unsigned long long*>(stat + ML);
  s.result = stat + 2 * ML + 2;
  s.level_examined = reinterpret_cast<unsigned long long*>(stat + 2 * ML + 4);
  s.level_mode = reinterpret_cast<int32_t*>(stat + 3 * ML + 4);
  s.level_heavy = g->ws.get<unsigned>("bfs.heavy", ML);
  s.bitmap_push = bitmap_push_enabled();
  s.timing = level_times_enabled();
  s.blocksum = g->ws.get<uint64_t>("bfs.blocksum", grid);
  s.nw = tb.nw;
  s.threshold = (1.0 / 20.0) * static_cast<double>(g->m);
  s.src = src;
  s.first = first_neighbors(g);
  s.iso = bfs_premark(g);
  void* args[] = {&view, &s};
  GBG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bfs_coop_k<G>), grid, kPushThreads, args, 0,
                                       g->stream));
  g->launches++;
  // no statistics wanted: nothing comes back to the host, so the call is
  // asynchronous on the handle's stream (one launch, no readback or sync)
  if (!st) return true;
  GBG_CUDA(cudaMemcpyAsync(g->hscalar, stat, kStatWords * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  const uint64_t* hs = g->hscalar;
  const unsigned long long* hx = reinterpret_cast<const unsigned long long*>(hs + 2 * ML + 4);
  const int32_t* hm = reinterpret_cast<const int32_t*>(hs + 3 * ML + 4);
  {
    std::memset(st, 0, sizeof(*st));
    const uint64_t levels = hs[2 * GBG_MAX_LEVELS + 2];
    st->levels = levels;
    st->reached = hs[2 * GBG_MAX_LEVELS + 3];
    for (uint64_t i = 0; i < levels && i < GBG_MAX_LEVELS; ++i) {
      st->mode[i] = hm[i];
      st->frontier[i] = pack_count(hs[i]);
      st->degree_sum[i] = pack_degsum(hs[i]);
      st->level_ms[i] =
          s.timing ? static_cast<float>((hs[GBG_MAX_LEVELS + i + 1] - hs[GBG_MAX_LEVELS + i]) * 1e-6) : 0.0f;
      st->examined[i] = hm[i] == GBG_MODE_DENSE ? hx[i] : st->degree_sum[i];
    }
  }
  return true;
}

template <class G>
void bfs_run(gbg_graph* g, G view, uint32_t src, int32_t* depth, gbg_bfs_stats* st) {
  if (bfs_coop(g, view, src, depth, st)) return;
  TraversalBuffers tb(g);
  uint32_t* visited = g->ws.get<uint32_t>("bfs.visited", tb.nw + 2);
  GBG_CUDA(cudaMemsetAsync(depth, 0xff, g->n * sizeof(int32_t), g->stream));
  GBG_CUDA(cudaMemcpyAsync(visited, bfs_premark(g), tb.nw * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                           g->stream));
  GBG_CUDA(cudaMemsetAsync(tb.a.bm, 0, tb.nw * sizeof(uint32_t), g->stream));
  GBG_LAUNCH(g, bfs_init_k<G>, 1, 1, 0, view, src, visited, depth, tb.a.list, tb.a.dscan, tb.a.bm, tb.packed);
  Frontier* cur = &tb.a;
  Frontier* nxt = &tb.b;
  read_packed(g, tb.packed, *cur);
  cur->has_list = cur->has_bm = true;
  uint64_t reached = 1;
  int32_t level = 0;
  if (st) std::memset(st, 0, sizeof(*st));
  unsigned long long* xcnt = g->ws.get<unsigned long long>("bfs.examined", GBG_MAX_LEVELS);
  GBG_CUDA(cudaMemsetAsync(xcnt, 0, GBG_MAX_LEVELS * sizeof(unsigned long long), g->stream));
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
    edge_map_step<G, BfsOp, true>(g, view, tb, *cur, *nxt, dense, op,
                                  st && level <= GBG_MAX_LEVELS ? xcnt + level - 1 : nullptr);
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
    unsigned long long hx[GBG_MAX_LEVELS];
    GBG_CUDA(cudaMemcpyAsync(hx, xcnt, sizeof(hx), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
    for (int32_t i = 0; i < level && i < GBG_MAX_LEVELS; ++i)
      st->examined[i] = st->mode[i] == GBG_MODE_DENSE ? hx[i] : st->degree_sum[i];
  }
}

// ---------------------------------------------------------------- betweenness
// gb::bc (algorithms.cpp:60-103): BFS depths, vertices bucketed by depth,
// then path counts pulled level by level from the previous layer and
// dependencies pulled from the next layer in reverse level order.  One warp
// per vertex of the level; each sum is a fixed shuffle tree.
__global__ void level_count_k(const int32_t* depth, uint64_t n, uint32_t* cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    if (depth[v] >= 0) atomicAdd(cnt + depth[v], 1u);
}
__global__ void level_scatter_k(const int32_t* depth, uint64_t n, uint32_t* cursor, uint32_t* list) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    if (depth[v] >= 0) list[atomicAdd(cursor + depth[v], 1u)] = static_cast<uint32_t>(v);
}

template <class G, bool kSigma>
__global__ void bc_level_k(G g, const uint32_t* list, uint32_t count, const int32_t* depth, int32_t d,
                           double* sigma, double* delta) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w0; i < count; i += nw) {
    const uint32_t v = list[i];
    uint64_t b;
    uint32_t deg;
    g.seg(v, b, deg);
    double acc = 0.0;
    const double sv = kSigma ? 0.0 : sigma[v];
    for (uint32_t j = lane; j < deg; j += 32) {
      const uint32_t u = g.at(b + j);
      if (kSigma) {
        if (depth[u] == d - 1) acc += sigma[u];
      } else if (depth[u] == d + 1) {
        acc += (sv / sigma[u]) * (1.0 + delta[u]);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) (kSigma ? sigma : delta)[v] = acc;
  }
}

template <class G>
void bc_run(gbg_graph* g, G view, uint32_t src, double* delta) {
  const uint64_t n = g->n;
  int32_t* depth = g->ws.get<int32_t>("bc.depth", n);
  gbg_bfs_stats st;
  bfs_run(g, view, src, depth, &st);
  const uint64_t nlev = st.levels;  // depths 0 .. nlev-1
  uint32_t* cnt = g->ws.get<uint32_t>("bc.cnt", nlev + 1);
  uint32_t* list = g->ws.get<uint32_t>("bc.list", n);
  double* sigma = g->ws.get<double>("bc.sigma", n);
  GBG_CUDA(cudaMemsetAsync(cnt, 0, (nlev + 1) * sizeof(uint32_t), g->stream));
  GBG_LAUNCH(g, level_count_k, grid_for(n, 256), 256, 0, depth, n, cnt);
  std::vector<uint32_t> hc(nlev + 1), start(nlev + 1);
  GBG_CUDA(cudaMemcpyAsync(hc.data(), cnt, (nlev + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  uint32_t run = 0;
  for (uint64_t d = 0; d <= nlev; ++d) {
    start[d] = run;
    run += hc[d];
  }
  GBG_CUDA(cudaMemcpyAsync(cnt, start.data(), (nlev + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
  GBG_LAUNCH(g, level_scatter_k, grid_for(n, 256), 256, 0, depth, n, cnt, list);
  GBG_CUDA(cudaMemsetAsync(sigma, 0, n * sizeof(double), g->stream));
  GBG_CUDA(cudaMemsetAsync(delta, 0, n * sizeof(double), g->stream));
  const double one = 1.0;
  GBG_CUDA(cudaMemcpyAsync(sigma + src, &one, sizeof(double), cudaMemcpyHostToDevice, g->stream));
  auto grid = [&](uint32_t c) { return grid_for(static_cast<uint64_t>(c) * 32, 256, g->sm_count * 16); };
  for (uint64_t d = 1; d < nlev; ++d)
    if (hc[d])
      GBG_LAUNCH(g, (bc_level_k<G, true>), grid(hc[d]), 256, 0, view, list + start[d], hc[d], depth,
                 static_cast<int32_t>(d), sigma, delta);
  for (uint64_t d = nlev; d-- > 0;)
    if (hc[d] && d + 1 < nlev)
      GBG_LAUNCH(g, (bc_level_k<G, false>), grid(hc[d]), 256, 0, view, list + start[d], hc[d], depth,
                 static_cast<int32_t>(d), sigma, delta);
}

}  // namespace
}  // namespace gbg

namespace gbg {
const uint64_t* first_neighbors(gbg_graph* g) {
  const uint64_t nw = (g->n + 31) / 32;
  // (degree, first) words, then the isolated bitmap
  if (!g->first) g->first = dalloc<uint64_t>(g->n + nw / 2 + 1);
  if (!g->first_valid) {
    with_view(g, [&](auto view) {
      GBG_LAUNCH(g, first_nbr_k<decltype(view)>, grid_for(nw * 32, 256), 256, 0, view, g->first,
                 reinterpret_cast<uint32_t*>(g->first + g->n));
    });
    g->first_valid = true;
  }
  return g->first;
}
const uint32_t* isolated_bitmap(gbg_graph* g) { return reinterpret_cast<const uint32_t*>(first_neighbors(g) + g->n); }

namespace {
struct ClearTargetOp {
  uint32_t* bm;
  __device__ __forceinline__ void operator()(uint32_t, uint32_t v, uint64_t) const {
    atomicAnd(bm + (v >> 5), ~(1u << (v & 31)));
  }
};
}  // namespace

// The visited bits a BFS may set before it starts: vertices no level can
// reach.  A sparse level reaches v through an arc u -> v (traversal.cpp:
// 16-46 walks u's list); a dense level through v's own list (traversal.cpp:
// 48-95 scans N(v) for a frontier member).  So only vertices with neither
// in-arcs nor out-arcs are unreachable.  On a symmetric graph those are the
// zero-degree vertices (the cached isolated bitmap); on a directed graph
// the isolated bitmap minus every arc target, built per call.
const uint32_t* bfs_premark(gbg_graph* g) {
  if (graph_is_symmetric(g)) return isolated_bitmap(g);
  const uint64_t nw = (g->n + 31) / 32;
  uint32_t* bm = g->ws.get<uint32_t>("bfs.premark", nw + 1);
  GBG_CUDA(cudaMemcpyAsync(bm, isolated_bitmap(g), nw * sizeof(uint32_t), cudaMemcpyDeviceToDevice, g->stream));
  const uint64_t* voff = virtual_offsets(g);
  with_view(g, [&](auto view) { for_each_edge(g, view, voff, g->m, ClearTargetOp{bm}); });
  return bm;
}
}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_bc_device(gbg_graph* g, uint32_t source, double* delta_dev) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!delta_dev) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    if (source >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "bc: source out of range");  // algorithms.cpp:62
    with_view(g, [&](auto view) { bc_run(g, view, source, delta_dev); });
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_bc(gbg_graph* g, uint32_t source, double* delta) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!delta) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    if (source >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "bc: source out of range");
    double* d = g->ws.get<double>("bc.delta", g->n);
    with_view(g, [&](auto view) { bc_run(g, view, source, d); });
    GBG_CUDA(cudaMemcpyAsync(delta, d, g->n * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

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

// PageRank: one persistent pull kernel per power iteration over a tiled,
// source-sorted index of the graph (a container-side index built once per
// graph version and cached in the handle).
//
// Reference: gb::pagerank (algorithms.cpp:508-555).  Per iteration the
// reference runs a serial contrib/dangling loop (528-532), the dense pull
// next[v] += contrib[u] over every v (535-542: edge_map on "everyone" with
// early exit off, i.e. map_neighbors of every vertex), then a serial
// finalize + L1 loop (544-551) and an early break when err < tolerance
// (552).  Here all three are one launch:
//
//   X_i[r] = p_i[r]/deg(r)  if deg(r) > 0   (the contrib the gather reads)
//          = -p_i[r]        if deg(r) = 0   (dangling mass; fmax(X,0) = 0)
//
// so a gather of fmax(X_i[u], 0) yields contrib[u], and the finalize of
// row r emits X_{i+1}[r] directly.  The dangling mass of the zero-degree
// rows and the L1 error are folded deterministically (per-block partials,
// last-CTA fold in block order) and published for the next launch, which
// forms the same base term (1-d)/n + d*dangling/n as algorithms.cpp:544-545.
//
// Why a tiled index.  A row-by-row pull gathers one fp64 per arc from a
// vector that is mostly L2-resident, and the kernel ends up bound by the
// L1 -> L2 request rate (~1 request per SM per cycle): 520 M gathers per
// iteration at scale 24, one 32-byte sector each (r01: 1.85 ms, 0.2 of the
// HBM roofline).  The index instead
//   * renumbers vertices by (degree desc, id asc), so the gathered vector's
//     hot part is contiguous and rows of similar degree are adjacent;
//   * cuts the rows with edges into blocks of kRows = 8192 consecutive
//     rows, and sorts each block's arcs by SOURCE (the gathered vertex):
//     one warp load then reads 32 consecutive arcs whose sources share a
//     few 128-byte lines (scale 24: ~0.1 line requests per arc instead of
//     ~1.03 sectors), and an arc of a hub source becomes part of a "run" of
//     equal sources (~0.25 runs per arc);
//   * stores per arc only its row inside the block (13 bits) and a run-start
//     bit, in 16 bits, plus one uint32 source id per run: ~3 B per arc
//     against 4 B of neighbour id in the CSR;
//   * accumulates each block's row sums in shared memory (64 KiB per CTA)
//     as 64-bit fixed point (2^-F units, F from the arc count, see
//     fix_bits_for): integer atomics are order-independent, so the result
//     is deterministic whatever the schedule, and the rounding stays ~6e-11
//     in relative L1 after 20 iterations, inside the 1e-9 bar.  sm_100
//     has no native 64-bit shared-memory add (it compiles to a CAS loop),
//     so each sum is two 32-bit words: the low word takes the term's low
//     half with a native atomic add that returns the old value, and the
//     carry out of it goes to the high word with the term's high half --
//     the pair is the exact 64-bit sum.
// Blocks with many arcs (the hub rows) are cut into tiles of about kTileArcs
// arcs along their source order; a tile of such a block flushes its
// partial sums into a global fixed-point vector (red.add) and the block's
// last tile finalizes the rows.  CTAs take tiles from an atomic queue.
#include "radix.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "cache.cuh"
#include "edges.cuh"

namespace gbg {

#ifndef GBG_PR_ROW_BITS
#define GBG_PR_ROW_BITS 13
#endif
constexpr int kRowBits = GBG_PR_ROW_BITS;
constexpr uint32_t kRows = 1u << kRowBits;  // rows per block: 8 B of fixed-point sum each in shared memory
constexpr uint16_t kRunStart = 0x8000;      // arc word: run-start bit | row in block
constexpr uint32_t kGroup = 256;            // arcs per warp work item (8 rounds of 32)
constexpr int kConsumers = 31;              // consumer warps; warp 31 issues the bulk copies
#ifndef GBG_PR_WARP_GROUPS
#define GBG_PR_WARP_GROUPS 1
#endif
constexpr uint32_t kWarpGroups = GBG_PR_WARP_GROUPS;            // groups per consumer warp per chunk
constexpr uint32_t kChunkGroups = kConsumers * kWarpGroups;     // groups per staged chunk at most
constexpr uint32_t kChunk = kChunkGroups * kGroup;
#ifndef GBG_PR_RUN_BUF
#define GBG_PR_RUN_BUF 4096
#endif
#ifndef GBG_PR_STAGES
#define GBG_PR_STAGES 3
#endif
constexpr uint32_t kRunBuf = GBG_PR_RUN_BUF + 8;  // staged runs per chunk at most (u32)
constexpr uint32_t kArcBuf = kChunk + 16;   // staged arc words (u16, + 16-byte alignment slack)
constexpr uint32_t kGrpBuf = (kChunkGroups + 8 + 3) & ~3u;  // staged group run bases (u32)
constexpr int kStages = GBG_PR_STAGES;
      // shared-memory ring depth
#ifndef GBG_PR_TILE_ARCS
#define GBG_PR_TILE_ARCS (1u << 19)
#endif
constexpr uint32_t kTileArcs = GBG_PR_TILE_ARCS;
#ifndef GBG_PR_MIN_TILES_PER_SM
#define GBG_PR_MIN_TILES_PER_SM 4
#endif
constexpr uint32_t kMinTilesPerSm = GBG_PR_MIN_TILES_PER_SM;
#ifndef GBG_PR_THREADS
#define GBG_PR_THREADS 1024
#endif
constexpr int kPrThreads = GBG_PR_THREADS;
// Fixed-point scale of the row sums: 2^F, F = ceil(log2(m)) + kFixMargin
// (at most 62; 62 up to 2^22 arcs).  A contrib is about 1/m of the rank
// mass (PageRank of an undirected graph is close to degree / 2m), so its
// rounding error relative to its size is ~2^-kFixMargin at every scale:
// measured 5.8e-11 / 6.1e-11 relative L1 after 20 iterations at scales 22 /
// 24 (F = 55 / 57) against the reference, inside the 1e-9 bar (each bit of
// margin halves it).  The same choice keeps a term below 2^32 units, so the
// high word of a row sum only takes the carries out of the low word (a few
// percent of the adds), and the high-word add is skipped when there is
// none.  Row sums stay below 2^(64-F) >= 4.
#ifndef GBG_PR_FIN_PREFETCH
#define GBG_PR_FIN_PREFETCH 1
#endif
#ifndef GBG_PR_FIX_MARGIN
#define GBG_PR_FIX_MARGIN 28
#endif
constexpr int kFixMargin = GBG_PR_FIX_MARGIN;
#ifndef GBG_PR_FIX_FLOOR_LG
#define GBG_PR_FIX_FLOOR_LG 22
#endif
inline int fix_bits_for(uint64_t m) {
  int lg = 0;  // ceil(log2(m))
  while ((uint64_t{1} << lg) < m) ++lg;
  // up to 2^22 arcs the finest scale: small graphs keep ~1e-13 sums
  // (equal-contrib graphs such as K_n round every term the same way)
  return lg <= GBG_PR_FIX_FLOOR_LG ? 62 : std::min(62, lg + kFixMargin);
}

// One staged chunk of a tile: arcs [e0, e0 + len), work groups [g0, g0 +
// ng), the runs they touch [rlo, rhi) (both widened to 16-byte bounds for
// the bulk copies), the block, and whether it is its tile's first / last
// chunk and its block has several tiles.
struct PrChunk {
  uint64_t e0;
  uint32_t len, g0, rlo, rhi, block, flags;  // flags: ng | first << 8 | last << 9 | multi << 10
};
static_assert(sizeof(PrChunk) == 32, "chunk record");

struct PrLayout {
  uint64_t n = 0, m = 0;
  uint32_t nz = 0;      // rows with edges: new ids [0, nz)
  int idb = 1;          // id bits
  uint32_t* ord = nullptr;  // new -> old id
  uint32_t* pos = nullptr;  // old -> new id
  uint32_t* deg = nullptr;  // degree of new row r (r < n)
  uint64_t* keys = nullptr;  // build only: (block, source, row-in-block) per arc
  // the index
  uint16_t* arc = nullptr;      // [m] row in block | run-start bit, block by block, sources ascending
  uint32_t* run_src = nullptr;  // [nruns] source (new id) of each run
  uint64_t nruns = 0;
  uint32_t nblocks = 0, ntiles = 0, ngroups = 0;
  uint64_t* tile_arc = nullptr;    // [ntiles + 1] first arc of each tile
  uint32_t* tile_grp = nullptr;    // [ntiles + 1] first work group of each tile
  uint32_t* tile_block = nullptr;  // [ntiles]
  uint32_t* first_tile = nullptr;  // [nblocks + 1]
  uint32_t* grp_rbase = nullptr;   // [ngroups + 1] run index before the group's first arc
  uint32_t nchunks = 0;
  uint32_t* tile_chunk = nullptr;  // [ntiles + 1] first chunk of each tile
  PrChunk* chunk = nullptr;        // [nchunks]
  // iteration state
  unsigned long long* gsum = nullptr;  // [nz] fixed-point partials of multi-tile blocks
  unsigned* bcount = nullptr;          // [nblocks] tiles done per block
  double* blk_err = nullptr;           // [nblocks]
  unsigned* work = nullptr;            // tile queue
  unsigned* done_counter = nullptr;
  uint32_t grid = 0;
  double build_ms = 0;
  uint64_t bytes() const {
    return m * 2 + nruns * 4 + (ntiles + 1) * 20ull + ntiles * 4ull + (nblocks + 1) * 4ull + ngroups * 4ull +
           nchunks * 32ull + n * 12ull + nz * 8ull + nblocks * 12ull;
  }
  ~PrLayout() {
    for (void* p : {(void*)ord, (void*)pos, (void*)deg, (void*)keys, (void*)arc, (void*)run_src, (void*)tile_arc,
                    (void*)tile_grp, (void*)tile_block, (void*)first_tile, (void*)grp_rbase, (void*)gsum,
                    (void*)bcount, (void*)blk_err, (void*)work, (void*)done_counter, (void*)tile_chunk,
                    (void*)chunk})
      dfree(p);
  }
};

// ---------------------------------------------------------------- index build
// (degree desc, id asc) as one key: inverted degree above the L id bits
template <class G>
__global__ void degree_keys_k(G g, int L, uint64_t* keys) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < g.n; v += stride)
    keys[v] = (static_cast<uint64_t>(0xffffffffu - g.degree(static_cast<uint32_t>(v))) << L) | v;
}

__global__ void order_from_keys_k(const uint64_t* sorted, uint64_t n, int L, uint32_t* ord, uint32_t* pos,
                                  uint32_t* deg, uint32_t* nz) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint64_t k = sorted[r];
    const uint32_t v = static_cast<uint32_t>(k & ((uint64_t{1} << L) - 1));
    const uint32_t d = 0xffffffffu - static_cast<uint32_t>(k >> L);
    ord[r] = v;
    pos[v] = static_cast<uint32_t>(r);
    deg[r] = d;
    // first zero-degree row (degrees descend)
    if (d == 0 && (r == 0 || (0xffffffffu - static_cast<uint32_t>(sorted[r - 1] >> L)) != 0))
      *nz = static_cast<uint32_t>(r);
  }
}

// Phase 1 (degrees only): the degree order and the per-arc key buffer.
// Phase 2 (layout_keys) fills the keys for any range of edges, so a
// pipelined container build can key each chunk of neighbour ids as it
// lands (gbg_csr_create_ex, api.cu).  Phase 3 (layout_finish) sorts the
// keys and builds the index.
template <class G>
PrLayout* layout_rows(gbg_graph* g, G view) {
  const uint64_t n = g->n, m = g->m;
  if (m > 0xffffffffull) fail(GBG_ERR_INVALID_ARGUMENT, "pagerank: more than 2^32-1 arcs");
  auto L = std::make_unique<PrLayout>();
  L->n = n;
  L->m = m;
  uint64_t* keys = g->ws.get<uint64_t>("prl.keys", n);
  uint64_t* scratch = g->ws.get<uint64_t>("prl.sorted", n);
  int idb = 1;
  while ((uint64_t{1} << idb) < n) ++idb;
  L->idb = idb;
  GBG_LAUNCH(g, degree_keys_k<G>, grid_for(n, 256), 256, 0, view, idb, keys);
  const uint64_t* sorted = radix_sort_u64(g, keys, scratch, n, 32 + idb, "prl.sort");
  L->ord = dalloc<uint32_t>(n);
  L->pos = dalloc<uint32_t>(n);
  L->deg = dalloc<uint32_t>(n);
  uint32_t* nz = g->ws.get<uint32_t>("prl.nz", 1);
  const uint32_t all = static_cast<uint32_t>(n);
  GBG_CUDA(cudaMemcpyAsync(nz, &all, sizeof(all), cudaMemcpyHostToDevice, g->stream));
  GBG_LAUNCH(g, order_from_keys_k, grid_for(n, 256), 256, 0, sorted, n, idb, L->ord, L->pos, L->deg, nz);
  read_scalars(g, nz, sizeof(uint32_t), &L->nz);
  L->keys = dalloc<uint64_t>(m ? m : 1);
  g->ws.release("prl.keys");
  g->ws.release("prl.sorted");
  g->ws.release("prl.sort.hist");
  g->ws.release("prl.sort.lb");
  return L.release();
}

// key of arc u -> v (u's list holds v): block of row pos[u], source pos[v],
// row in block; out-of-range ids (not yet validated input, which the
// caller then rejects) get source 0
struct ArcKeyOp {
  const uint32_t* pos;
  uint64_t* keys;
  uint64_t n;
  int idb;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t e) const {
    const uint32_t r = pos[u];
    const uint32_t s = v < n ? pos[v] : 0u;
    keys[e] = (static_cast<uint64_t>(r >> kRowBits) << (idb + kRowBits)) |
              (static_cast<uint64_t>(s) << kRowBits) | (r & (kRows - 1));
  }
};

template <class G>
void layout_keys(gbg_graph* g, G view, const uint64_t* voff, PrLayout* L, uint64_t e0, uint64_t e1) {
  for_each_edge_range(g, view, voff, e0, e1, ArcKeyOp{L->pos, L->keys, g->n, L->idb});
}

// run start: first arc, or (block, source) differs from the previous arc's
__device__ __forceinline__ bool run_start(const uint64_t* k, uint64_t e) {
  return e == 0 || (k[e] >> kRowBits) != (k[e - 1] >> kRowBits);
}

__global__ void arc_words_k(const uint64_t* k, uint64_t m, uint16_t* arc) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += stride)
    arc[e] = static_cast<uint16_t>((k[e] & (kRows - 1)) | (run_start(k, e) ? kRunStart : 0));
}

struct RunIn {
  const uint64_t* k;
  __device__ __forceinline__ uint32_t operator()(uint64_t e) const { return run_start(k, e) ? 1u : 0u; }
};
struct RunOut {
  const uint64_t* k;
  uint64_t idmask;
  uint32_t* run_src;
  uint64_t* run_off;
  __device__ __forceinline__ void operator()(uint64_t e, uint32_t r) const {
    if (run_start(k, e)) {
      run_src[r] = static_cast<uint32_t>((k[e] >> kRowBits) & idmask);
      run_off[r] = e;
    }
  }
};

__device__ __forceinline__ uint32_t run_block(const uint64_t* k, const uint64_t* run_off, uint64_t r, int shift) {
  return static_cast<uint32_t>(k[run_off[r]] >> shift);
}

// block starts (every block has arcs: its rows have degree > 0)
__global__ void block_starts_k(const uint64_t* k, const uint64_t* run_off, uint64_t nruns, int shift,
                               uint64_t* block_arc) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nruns; r += stride) {
    const uint32_t b = run_block(k, run_off, r, shift);
    if (r == 0 || run_block(k, run_off, r - 1, shift) != b) block_arc[b] = run_off[r];
  }
}

// tile start: the block's first run, or a run whose arc offset in the block
// crosses a multiple of the tile size (2^tile_bits arcs)
struct TileIn {
  const uint64_t* k;
  const uint64_t* run_off;
  const uint64_t* block_arc;
  int shift;
  int tile_bits;
  __device__ __forceinline__ bool start(uint64_t r) const {
    const uint32_t b = run_block(k, run_off, r, shift);
    if (r == 0 || run_block(k, run_off, r - 1, shift) != b) return true;
    const uint64_t base = block_arc[b];
    return (run_off[r] - base) >> tile_bits != (run_off[r - 1] - base) >> tile_bits;
  }
  __device__ __forceinline__ uint32_t operator()(uint64_t r) const { return start(r) ? 1u : 0u; }
};
struct TileOut {
  TileIn in;
  uint64_t* tile_arc;
  uint32_t* tile_block;
  __device__ __forceinline__ void operator()(uint64_t r, uint32_t t) const {
    if (in.start(r)) {
      tile_arc[t] = in.run_off[r];
      tile_block[t] = run_block(in.k, in.run_off, r, in.shift);
    }
  }
};

struct GroupsIn {
  const uint64_t* tile_arc;
  __device__ __forceinline__ uint32_t operator()(uint64_t t) const {
    // groups are 256-arc windows aligned to the tile's first arc rounded
    // down to 8 (16-byte shared-memory loads), clipped to the tile
    return static_cast<uint32_t>((tile_arc[t + 1] - (tile_arc[t] & ~uint64_t{7}) + kGroup - 1) / kGroup);
  }
};

__global__ void first_tiles_k(const uint32_t* tile_block, uint32_t ntiles, uint32_t nblocks, uint32_t* first) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles; t += stride) {
    if (t == ntiles) {
      first[nblocks] = ntiles;
    } else if (t == 0 || tile_block[t] != tile_block[t - 1]) {
      first[tile_block[t]] = t;
    }
  }
}

__global__ void block_tiles_k(const uint32_t* first, uint32_t nblocks, unsigned* bcount) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += stride)
    bcount[2 * b + 1] = first[b + 1] - first[b];
}

// run index just before the group's first arc: (runs starting before it) - 1
struct GroupBaseOp {
  const uint64_t* tile_arc;
  const uint64_t* run_off;
  uint64_t nruns;
  uint32_t* grp_rbase;
  __device__ __forceinline__ void operator()(uint32_t t, uint32_t rank, uint64_t flat) const {
    const uint64_t e0 = max(tile_arc[t], (tile_arc[t] & ~uint64_t{7}) + static_cast<uint64_t>(rank) * kGroup);
    uint64_t lo = 0, hi = nruns;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (run_off[mid] < e0) lo = mid + 1; else hi = mid;
    }
    grp_rbase[flat] = static_cast<uint32_t>(lo) - 1u;
  }
};

// Chunks: consecutive work groups of one tile, at most kChunkGroups and at
// most kRunBuf staged runs (run range widened to 16-byte bounds), cut
// greedily by one thread per tile (a tile has at most ~520 groups).
__device__ __forceinline__ uint32_t run_lo(uint32_t rb) { return (rb == ~0u ? 0u : rb) & ~3u; }
__device__ __forceinline__ uint32_t run_hi(uint32_t rb_end) { return (rb_end + 1u + 3u) & ~3u; }

template <bool kFill>
__global__ void chunk_cut_k(const uint64_t* tile_arc, const uint32_t* tile_grp, const uint32_t* tile_block,
                            const uint32_t* first_tile, const uint32_t* grp_rbase, uint32_t ntiles,
                            uint32_t* tile_chunk, PrChunk* chunk) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += stride) {
    const uint32_t ga = tile_grp[t], gb = tile_grp[t + 1];
    const uint64_t tb = tile_arc[t], te = tile_arc[t + 1];
    const uint32_t b = tile_block[t];
    const bool multi = first_tile[b + 1] - first_tile[b] > 1;
    uint32_t c = kFill ? tile_chunk[t] : 0u, k = 0;
    for (uint32_t g0 = ga; g0 < gb; ++k) {
      const uint32_t rlo = run_lo(grp_rbase[g0]);
      uint32_t g1 = g0 + 1;
      while (g1 < gb && g1 - g0 < kChunkGroups && run_hi(grp_rbase[g1 + 1]) - rlo <= kRunBuf) ++g1;
      if (kFill) {
        PrChunk ch;
        const uint64_t ta = tb & ~uint64_t{7};
        ch.e0 = max(tb, ta + static_cast<uint64_t>(g0 - ga) * kGroup);
        const uint64_t e1 = g1 == gb ? te : ta + static_cast<uint64_t>(g1 - ga) * kGroup;
        ch.len = static_cast<uint32_t>(e1 - ch.e0);
        ch.g0 = g0;
        ch.rlo = rlo;
        ch.rhi = run_hi(grp_rbase[g1]);
        ch.block = b;
        ch.flags = (g1 - g0) | (g0 == ga ? 1u << 8 : 0u) | (g1 == gb ? 1u << 9 : 0u) | (multi ? 1u << 10 : 0u);
        chunk[c + k] = ch;
      }
      g0 = g1;
    }
    if (!kFill) tile_chunk[t] = k;
  }
}

void layout_finish(gbg_graph* g, PrLayout* L) {
  const uint64_t m = L->m;
  const uint32_t nz = L->nz;
  L->nblocks = (nz + kRows - 1) / kRows;
  int bb = 1;
  while ((1u << bb) < std::max(L->nblocks, 2u)) ++bb;
  const int shift = L->idb + kRowBits;  // key >> shift = block
  L->arc = dalloc<uint16_t>(m + 16);  // bulk copies read up to 16 bytes past the end
  L->first_tile = dalloc<uint32_t>(L->nblocks + 1);
  L->gsum = dalloc<unsigned long long>(nz ? nz : 1);
  L->bcount = dalloc<unsigned>(2 * (L->nblocks ? L->nblocks : 1));
  L->blk_err = dalloc<double>(L->nblocks ? L->nblocks : 1);
  L->work = dalloc<unsigned>(1);
  L->done_counter = dalloc<unsigned>(1);
  GBG_CUDA(cudaMemsetAsync(L->gsum, 0, (nz ? nz : 1) * sizeof(unsigned long long), g->stream));
  GBG_CUDA(cudaMemsetAsync(L->bcount, 0, 2 * (L->nblocks ? L->nblocks : 1) * sizeof(unsigned), g->stream));
  GBG_CUDA(cudaMemsetAsync(L->work, 0, sizeof(unsigned), g->stream));
  GBG_CUDA(cudaMemsetAsync(L->done_counter, 0, sizeof(unsigned), g->stream));
  if (m == 0) {
    L->tile_arc = dalloc<uint64_t>(1);
    L->tile_grp = dalloc<uint32_t>(1);
    L->tile_block = dalloc<uint32_t>(1);
    L->grp_rbase = dalloc<uint32_t>(1);
    L->run_src = dalloc<uint32_t>(1);
    L->tile_chunk = dalloc<uint32_t>(1);
    L->chunk = dalloc<PrChunk>(1);
    dfree(L->keys);
    L->keys = nullptr;
    return;
  }
  PhaseTrace tr(g->stream, "pagerank index");
  // 1. sort the arcs by (block, source, row)
  uint64_t* scratch = g->ws.get<uint64_t>("prl.ksort", m);
  tr.mark("alloc");
  uint64_t* k = radix_sort_u64(g, L->keys, scratch, m, bb + L->idb + kRowBits, "prl.asort");
  tr.mark("sort");
  // 2. arc words, runs
  GBG_LAUNCH(g, arc_words_k, grid_for(m, 256), 256, 0, k, m, L->arc);
  uint32_t* cnt = g->ws.get<uint32_t>("prl.cnt", 4);
  device_scan<uint32_t>(g, RunIn{k}, NullOut{}, m, cnt, "prl.runs");
  uint32_t nruns = 0;
  read_scalars(g, cnt, sizeof(nruns), &nruns);
  L->nruns = nruns;
  tr.mark("runs-count");
  L->run_src = dalloc<uint32_t>(nruns + 8);
  uint64_t* run_off = g->ws.get<uint64_t>("prl.runoff", nruns + 1);
  device_scan<uint32_t>(g, RunIn{k}, RunOut{k, (uint64_t{1} << L->idb) - 1, L->run_src, run_off}, m, cnt,
                        "prl.runs");
  tr.mark("runs");
  // 3. blocks and tiles
  uint64_t* block_arc = g->ws.get<uint64_t>("prl.blockarc", L->nblocks);
  GBG_LAUNCH(g, block_starts_k, grid_for(nruns, 256), 256, 0, k, run_off, nruns, shift, block_arc);
  // tiles of up to kTileArcs arcs, smaller on smaller graphs so that there
  // are at least kMinTilesPerSm tiles per SM to balance over, but not below
  // 2^17 arcs (measured: s24 best at 2^19, s22 and s20 at 2^17 -- s20 1.99
  // -> 1.79 ms against 2^16)
  int tile_bits = 0;
  while ((2ull << tile_bits) <= kTileArcs) ++tile_bits;
  while (tile_bits > 17 && (m >> tile_bits) < uint64_t{kMinTilesPerSm} * g->sm_count) --tile_bits;
#ifdef GBG_PR_TILE_BITS_FORCE
  tile_bits = GBG_PR_TILE_BITS_FORCE;
#endif
  TileIn tin{k, run_off, block_arc, shift, tile_bits};
  device_scan<uint32_t>(g, tin, NullOut{}, nruns, cnt + 1, "prl.tiles");
  read_scalars(g, cnt + 1, sizeof(uint32_t), &L->ntiles);
  L->tile_arc = dalloc<uint64_t>(L->ntiles + 1);
  L->tile_grp = dalloc<uint32_t>(L->ntiles + 1);
  L->tile_block = dalloc<uint32_t>(L->ntiles);
  device_scan<uint32_t>(g, tin, TileOut{tin, L->tile_arc, L->tile_block}, nruns, cnt + 1, "prl.tiles");
  GBG_CUDA(cudaMemcpyAsync(L->tile_arc + L->ntiles, &L->m, sizeof(uint64_t), cudaMemcpyHostToDevice, g->stream));
  GBG_LAUNCH(g, first_tiles_k, grid_for(L->ntiles + 1, 256), 256, 0, L->tile_block, L->ntiles, L->nblocks,
             L->first_tile);
  GBG_LAUNCH(g, block_tiles_k, grid_for(L->nblocks, 256), 256, 0, L->first_tile, L->nblocks, L->bcount);
  tr.mark("tiles");
  // 4. work groups of kGroup arcs per tile, and each one's run base
  device_scan<uint32_t>(g, GroupsIn{L->tile_arc}, ArrayOut<uint32_t>{L->tile_grp}, L->ntiles,
                        L->tile_grp + L->ntiles, "prl.grp");
  read_scalars(g, L->tile_grp + L->ntiles, sizeof(uint32_t), &L->ngroups);
  L->grp_rbase = dalloc<uint32_t>(L->ngroups + 8);
  expand(g, L->tile_grp, L->ntiles, L->ngroups, GroupBaseOp{L->tile_arc, run_off, nruns, L->grp_rbase});
  {  // sentinel: the run of the last arc
    const uint32_t last = nruns - 1;
    GBG_CUDA(cudaMemcpyAsync(L->grp_rbase + L->ngroups, &last, sizeof(last), cudaMemcpyHostToDevice, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  }
  tr.mark("groups");
  // 5. staged chunks per tile
  L->tile_chunk = dalloc<uint32_t>(L->ntiles + 1);
  uint32_t* cnts = g->ws.get<uint32_t>("prl.chkcnt", L->ntiles + 1);
  GBG_LAUNCH(g, chunk_cut_k<false>, grid_for(L->ntiles, 128), 128, 0, L->tile_arc, L->tile_grp, L->tile_block,
             L->first_tile, L->grp_rbase, L->ntiles, cnts, nullptr);
  device_scan<uint32_t>(g, ArrayIn<uint32_t>{cnts}, ArrayOut<uint32_t>{L->tile_chunk}, L->ntiles,
                        L->tile_chunk + L->ntiles, "prl.chk");
  read_scalars(g, L->tile_chunk + L->ntiles, sizeof(uint32_t), &L->nchunks);
  L->chunk = dalloc<PrChunk>(L->nchunks);
  GBG_LAUNCH(g, chunk_cut_k<true>, grid_for(L->ntiles, 128), 128, 0, L->tile_arc, L->tile_grp, L->tile_block,
             L->first_tile, L->grp_rbase, L->ntiles, L->tile_chunk, L->chunk);
  tr.mark("chunks");
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  dfree(L->keys);
  L->keys = nullptr;
  for (const char* b : {"prl.ksort", "prl.asort.hist", "prl.asort.lb", "prl.asort.ctr", "prl.runoff",
                        "prl.blockarc", "prl.runs.sums", "prl.tiles.sums", "prl.grp.sums", "prl.chk.sums", "prl.chkcnt"})
    g->ws.release(b);
}

template <class G>
PrLayout* build_layout(gbg_graph* g, G view, const uint64_t* voff) {
  cudaEvent_t e0, e1;
  GBG_CUDA(cudaEventCreate(&e0));
  GBG_CUDA(cudaEventCreate(&e1));
  GBG_CUDA(cudaEventRecord(e0, g->stream));
  std::unique_ptr<PrLayout> L(layout_rows(g, view));
  layout_keys(g, view, voff, L.get(), 0, g->m);
  layout_finish(g, L.get());
  GBG_CUDA(cudaEventRecord(e1, g->stream));
  GBG_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  L->build_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return L.release();
}

// ---------------------------------------------------------------- iteration
struct PrScalars {
  double dangling[2];  // ping-pong: iteration i reads [i&1], writes [(i+1)&1]
  double p_zero;       // rank of every zero-degree row after the last executed iteration
  double err;          // L1 step difference of the last executed iteration
  int done;            // set once err < tolerance (algorithms.cpp:552)
  int iterations;      // iterations executed
};

struct PrArgs {
  const uint16_t* arc;
  const uint32_t* run_src;
  const uint32_t* grp_rbase;
  const PrChunk* chunk;
  const uint32_t* tile_chunk;
  const uint32_t* deg;
  const double* x_old;
  double* x_new;
  const unsigned long long* t_old;  // fixed-point contribs the gathers read
  unsigned long long* t_new;
  unsigned long long* gsum;
  unsigned* bcount;  // per block: finished tiles, tile count
  double* blk_err;
  unsigned* work;
  unsigned* done_counter;
  PrScalars* sc;
  uint32_t ntiles, nblocks, nz;
  double damping, nd, tol;
  double fix, unfix;  // fixed-point scale of the contribs and row sums
  double n_zero;  // zero-degree rows
  int iter;
};

// ---- shared-memory staging: 1-D bulk copies (TMA) into a two-stage ring,
// completion signalled on an mbarrier per stage
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ unsigned long long ld_fix(const unsigned long long* a, uint64_t pol) {
  unsigned long long v;
  asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

// predicated gather (0 when !p) in one asm block, so the compiler cannot
// fold the later register select into the load's destination (which would
// chain the loads one after the other)
__device__ __forceinline__ unsigned long long ld_fix_if(const unsigned long long* a, uint64_t pol, uint32_t p) {
  unsigned long long v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n mov.b64 %0, 0;\n"
      " @q ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;\n}"
      : "=l"(v)
      : "l"(a), "l"(pol), "r"(p));
  return v;
}

// contrib in fixed point (gathered by the next iteration)
__device__ __forceinline__ unsigned long long to_fix(double contrib, double fix) {
  return __double2ull_rn(fmax(contrib, 0.0) * fix);
}

// L2 residency: the fixed-point contribs of the kHot highest-degree rows
// take ~98% of the gathers (scale 24); they are written and gathered with
// evict_last, everything else streams with evict_first, so the hot part of
// both contrib buffers (2 x 32 MiB) stays in the 126 MB L2 while the arcs,
// the fp64 ranks and the cold contribs pass through.
#ifndef GBG_PR_HOT_BITS
#define GBG_PR_HOT_BITS 22
#endif
constexpr uint32_t kHot = 1u << GBG_PR_HOT_BITS;
__device__ __forceinline__ void st_hint_u64(unsigned long long* a, unsigned long long v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint_f64(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_first_f64(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}

// Finalize row r (d > 0; algorithms.cpp:544-550 for one vertex) from its
// fixed-point sum and emit the next iteration's contrib forms.
__device__ __forceinline__ void pr_finalize(const PrArgs& a, double base, uint32_t r, unsigned long long fsum,
                                            double& err, uint64_t pf, uint64_t pl) {
  const double d = static_cast<double>(ld_stream_u32(a.deg + r, pf));
  const double next = base + a.damping * (static_cast<double>(fsum) * a.unfix);
  const double xo = ld_first_f64(a.x_old + r, pf);
  err += fabs(next - xo * d);
  const double c = next / d;
  st_hint_f64(a.x_new + r, c, pf);
  st_hint_u64(a.t_new + r, to_fix(c, a.fix), r < kHot ? pl : pf);
}

// exact 64-bit fixed-point add into a (lo, hi) pair of shared words
__device__ __forceinline__ void acc_add(uint32_t* lo, uint32_t* hi, uint32_t i, unsigned long long t) {
  const uint32_t l = static_cast<uint32_t>(t), h = static_cast<uint32_t>(t >> 32);
  const uint32_t old = atomicAdd(lo + i, l);
  const uint32_t c = h + (old + l < old ? 1u : 0u);
  if (c) atomicAdd(hi + i, c);
}
__device__ __forceinline__ unsigned long long acc_get(const uint32_t* lo, const uint32_t* hi, uint32_t i) {
  return (static_cast<unsigned long long>(hi[i]) << 32) | lo[i];
}

// Shared-memory layout of pr_tile_k (dynamic): the block's sums, then
// kStages stages of {arc words, run sources, group run bases}.
constexpr size_t kSmemAcc = 2ull * kRows * sizeof(uint32_t);
constexpr size_t kSmemStage = kArcBuf * 2 + kRunBuf * 4 + kGrpBuf * 4;
constexpr size_t kSmemBytes = kSmemAcc + kStages * kSmemStage;
static_assert(kSmemStage % 16 == 0, "stage alignment");

#ifdef GBG_PR_TRACE
// timing trace (analysis builds only): per CTA up to 64 tiles of
// {block, arcs, t_first_chunk, t_groups_done, t_finalized, smid}
__device__ unsigned long long g_pr_trace[148 * 64 * 6];
__device__ unsigned g_pr_trace_n[148];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
struct StageInfo {
  PrChunk ch;
  uint64_t abase;  // arc index of the stage's first staged word
  uint32_t qbase;  // group index of the stage's first staged run base
  uint32_t valid;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier among the consumer warps only (the producer warp never joins)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
}
__device__ __forceinline__ double consumer_sum(double v, double* red) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  consumer_sync();
  if (warp == 0) {
    double w = lane < kConsumers ? red[lane] : 0.0;
    w = warp_sum(w);
    if (lane == 0) red[32] = w;
  }
  consumer_sync();
  const double r = red[32];
  consumer_sync();
  return r;
}

// high word += high half of the term + carry out of the low word's add
// (old = the low word before the add)
__device__ __forceinline__ uint32_t carry_hi(uint32_t old, uint32_t l, uint32_t h) {
  uint32_t c;
  asm("{\n .reg .u32 t;\n add.cc.u32 t, %1, %2;\n addc.u32 %0, %3, 0;\n}" : "=r"(c) : "r"(old), "r"(l), "r"(h));
  return c;
}

// One work group: a 256-arc window of the staged chunk, arcs [vlo, vhi) of
// it valid (kFull: all), as 8 rounds of 32 consecutive arcs.  A round's
// run starts are ballot-ranked onto the run index carried from the group's
// base, so every lane finds its arc's source in the staged runs; lanes of
// one run gather the same contrib (one request), and consecutive runs have
// consecutive sources.  All 8 gathers are in flight before the first add;
// then the 8 low-word adds (with return), then the 8 high-word adds (high
// half + carry; no return).
template <bool kFull>
__device__ __forceinline__ void pr_group(const PrArgs& a, uint32_t* lo, uint32_t* hi, const uint16_t* win,
                                         const uint32_t* srun, uint32_t vlo, uint32_t vhi, uint32_t rbase,
                                         uint32_t lane, uint64_t pf, uint64_t pl) {
  constexpr int R = kGroup / 32;
  uint32_t row[R];
  bool on[R];
  uint32_t flags[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t i = j * 32 + lane;
    on[j] = kFull || (i >= vlo && i < vhi);
    const uint32_t w = on[j] ? win[i] : 0u;
    row[j] = w & (kRows - 1);
    flags[j] = __ballot_sync(0xffffffffu, (w & kRunStart) != 0);
  }
  const uint32_t le = (2u << lane) - 1u;  // lanes <= this one
  // one L2 policy for the whole group: sources ascend inside a block, so
  // the group's last run decides (evict_last when it is hot; a group that
  // straddles kHot is rare)
  uint32_t rend = rbase;
#pragma unroll
  for (int j = 0; j < R; ++j) rend += __popc(flags[j]);
  const uint64_t pol = srun[rend] < kHot ? pl : pf;
  unsigned long long x[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t run = rbase + __popc(flags[j] & le);
    rbase += __popc(flags[j]);
    const uint32_t u = srun[run];
    x[j] = on[j] ? ld_fix(a.t_old + u, pol) : 0ull;
  }
  uint32_t old[R];
#pragma unroll
  for (int j = 0; j < R; ++j) old[j] = on[j] ? atomicAdd(lo + row[j], static_cast<uint32_t>(x[j])) : 0u;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t c = carry_hi(old[j], static_cast<uint32_t>(x[j]), static_cast<uint32_t>(x[j] >> 32));
    if ((kFull || on[j]) && c) atomicAdd(hi + row[j], c);  // result unused: RED
  }
}

// Persistent, warp-specialised: warp 31 is the producer -- it takes tiles
// from an atomic queue and streams each tile's chunks into a kStages-deep
// shared-memory ring with 1-D bulk copies (TMA), one "full" mbarrier per
// stage carrying the byte count, and reuses a stage once every consumer
// warp has arrived on its "empty" mbarrier.  Warps 0..30 are consumers:
// warp w takes group w of each chunk (a chunk has at most 31 groups), so
// no barrier ties them together inside a tile -- gathers of some warps
// overlap the shared-memory adds of others.  Consumers synchronise (named
// barrier 1) only at tile boundaries: clearing the sums before a tile,
// finalizing or flushing them after it.  Per-block error partials are
// folded in block order by the last CTA (deterministic whatever the
// schedule).
__global__ void __launch_bounds__(kPrThreads, 1) pr_tile_k(PrArgs a) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  __shared__ __align__(8) uint64_t s_full[kStages];
  __shared__ __align__(8) uint64_t s_empty[kStages];
  __shared__ StageInfo s_stage[kStages];
  __shared__ double s_red[33];
  __shared__ int s_flag;
  if (a.sc->done) return;
  uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_dyn);
  uint32_t* s_hi = s_lo + kRows;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto stage_ptrs = [&](int s, uint16_t*& arcb, uint32_t*& runb, uint32_t*& grpb) {
    unsigned char* p = s_dyn + kSmemAcc + s * kSmemStage;
    arcb = reinterpret_cast<uint16_t*>(p);
    runb = reinterpret_cast<uint32_t*>(p + kArcBuf * 2);
    grpb = reinterpret_cast<uint32_t*>(p + kArcBuf * 2 + kRunBuf * 4);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      // everything fetched one step ahead: the record of the next chunk
      // (nx) and the chunk range of the tile after the current one (qc, qe)
      uint32_t pc = 0, pe = 0, qc = 0, qe = 0;
      auto take_tile = [&](uint32_t& b, uint32_t& e) {
        const uint32_t t = atomicAdd(a.work, 1u);
        b = e = 0;
        if (t < a.ntiles) {
          b = __ldg(a.tile_chunk + t);
          e = __ldg(a.tile_chunk + t + 1);
        }
      };
      PrChunk nx{};
      take_tile(pc, pe);
      if (pc < pe) {
        take_tile(qc, qe);
        nx = a.chunk[pc];
      }
      for (uint32_t c = 0;; ++c) {
        const int s = c % kStages;
        if (c >= kStages) mbar_wait(&s_empty[s], ((c / kStages) - 1) & 1);
        if (pc == pe) {
          s_stage[s].valid = 0;
          mbar_arrive(&s_full[s]);
          break;
        }
        const PrChunk ch = nx;
#if GBG_PR_FIN_PREFETCH
        if ((ch.flags & (1u << 8)) && !(ch.flags & (1u << 10))) {
          // the first chunk of a single-tile block: pull the block's degrees
          // and previous contribs (read by its finalize) into L2
          const uint32_t row0 = ch.block * kRows;
          const uint32_t nrows = min(kRows, a.nz - row0);
          const uint32_t bd = (nrows * 4u) & ~15u, bx = (nrows * 8u) & ~15u;
          if (bd) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.deg + row0), "r"(bd) : "memory");
          if (bx) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.x_old + row0), "r"(bx) : "memory");
        }
#endif
        uint16_t* arcb;
        uint32_t* runb;
        uint32_t* grpb;
        stage_ptrs(s, arcb, runb, grpb);
        const uint64_t alo = ch.e0 & ~uint64_t{7}, ahi = (ch.e0 + ch.len + 7) & ~uint64_t{7};
        const uint32_t ng = ch.flags & 0xff;
        const uint32_t qlo = ch.g0 & ~3u, qhi = (ch.g0 + ng + 3) & ~3u;
        const uint32_t ba = static_cast<uint32_t>(ahi - alo) * 2, br = (ch.rhi - ch.rlo) * 4,
                       bq = (qhi - qlo) * 4;
        s_stage[s].ch = ch;
        s_stage[s].abase = alo;
        s_stage[s].qbase = qlo;
        s_stage[s].valid = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&s_full[s], ba + br + bq);
        bulk_g2s(arcb, a.arc + alo, ba, &s_full[s], pf);
        bulk_g2s(runb, a.run_src + ch.rlo, br, &s_full[s], pf);
        bulk_g2s(grpb, a.grp_rbase + qlo, bq, &s_full[s], pf);
        // advance: the next chunk of this tile, or the prefetched tile (and
        // take the one after it)
        if (++pc == pe) {
          pc = qc;
          pe = qe;
          if (pc < pe) take_tile(qc, qe);
        }
        if (pc < pe) nx = a.chunk[pc];
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------- consumers
    const double dcur = a.sc->dangling[a.iter & 1];
    const double base = (1.0 - a.damping) / a.nd + a.damping * dcur / a.nd;
    const uint32_t ctid = threadIdx.x;  // < kConsumers * 32
    constexpr uint32_t kCT = kConsumers * 32;
    uint32_t rot = 0;
    for (uint32_t c = 0;; ++c) {
      const int s = c % kStages;
      mbar_wait(&s_full[s], (c / kStages) & 1);
      if (!s_stage[s].valid) break;
      const PrChunk ch = s_stage[s].ch;
      const uint64_t abase = s_stage[s].abase;
      const uint32_t qbase = s_stage[s].qbase;
      const uint32_t row0 = ch.block * kRows;
      const uint32_t nrows = min(kRows, a.nz - row0);
#ifdef GBG_PR_TRACE
      if (ctid == 0 && (ch.flags & (1u << 8))) {
        const unsigned k = g_pr_trace_n[blockIdx.x]++;
        if (k < 64) {
          unsigned long long* r = g_pr_trace + (blockIdx.x * 64 + k) * 6;
          r[0] = ch.block;
          r[1] = 0;
          r[2] = gtime();
          unsigned smid;
          asm("mov.u32 %0, %smid;" : "=r"(smid));
          r[5] = smid;
        }
      }
      if (ctid == 0) {
        const unsigned k = g_pr_trace_n[blockIdx.x] - 1;
        if (k < 64) g_pr_trace[(blockIdx.x * 64 + k) * 6 + 1] += ch.len;
      }
#endif
      if (ch.flags & (1u << 8)) {  // the tile's first chunk: clear the sums
        for (uint32_t i = ctid; i < nrows; i += kCT) s_lo[i] = s_hi[i] = 0u;
        consumer_sync();
      }
      {
        uint16_t* arcb;
        uint32_t* runb;
        uint32_t* grpb;
        stage_ptrs(s, arcb, runb, grpb);
        const uint32_t ng = ch.flags & 0xff;
        // group gi goes to warp (rot + gi) mod 31: the assignment rotates
        // from chunk to chunk, so no warp takes the extra group of every
        // chunk (a chunk's group count is rarely a multiple of 31)
        // group gi = the 256-arc window at staged arc gi * 256 (the stage
        // starts at ch.e0 rounded down to 8), valid arcs [v0, v1) of it
        const uint32_t v0 = static_cast<uint32_t>(ch.e0 - abase), v1 = v0 + ch.len;
        for (uint32_t gi = (warp + kConsumers - rot) % kConsumers; gi < ng; gi += kConsumers) {
          const uint32_t off = gi * kGroup;
          const uint32_t vlo = gi == 0 ? v0 : 0u, vhi = min(kGroup, v1 - off);
          const uint32_t rb = grpb[ch.g0 + gi - qbase];
          // staged run index = global run index - rlo (rb may be ~0u: wraps consistently)
          const uint32_t rs = rb - ch.rlo;
          if (vlo == 0 && vhi == kGroup)
            pr_group<true>(a, s_lo, s_hi, arcb + off, runb, 0, kGroup, rs, lane, pf, pl);
          else
            pr_group<false>(a, s_lo, s_hi, arcb + off, runb, vlo, vhi, rs, lane, pf, pl);
        }
        rot = (rot + ng) % kConsumers;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[s]);
      if (ch.flags & (1u << 9)) {  // the tile's last chunk: finalize or flush
        consumer_sync();
#ifdef GBG_PR_TRACE
        if (ctid == 0 && g_pr_trace_n[blockIdx.x] - 1 < 64)
          g_pr_trace[(blockIdx.x * 64 + g_pr_trace_n[blockIdx.x] - 1) * 6 + 3] = gtime();
#endif
        double err = 0.0;
        bool fin = false;
        const uint32_t b = ch.block;
        if (!(ch.flags & (1u << 10))) {
          // the whole block in this tile: finalize from shared memory
          for (uint32_t i = ctid; i < nrows; i += kCT)
            pr_finalize(a, base, row0 + i, acc_get(s_lo, s_hi, i), err, pf, pl);
          fin = true;
        } else {
          for (uint32_t i = ctid; i < nrows; i += kCT) {
            const unsigned long long v = acc_get(s_lo, s_hi, i);
            if (v) atomicAdd(a.gsum + row0 + i, v);
          }
          __threadfence();
          consumer_sync();
          // bcount[2b] counts the block's finished tiles, bcount[2b + 1] is
          // its tile count (set at build time)
          if (ctid == 0) s_flag = atomicAdd(a.bcount + 2 * b, 1u) + 1 == __ldg(a.bcount + 2 * b + 1);
          consumer_sync();
          if (s_flag) {
            __threadfence();
            for (uint32_t i = ctid; i < nrows; i += kCT) {
              unsigned long long* p = a.gsum + row0 + i;
              pr_finalize(a, base, row0 + i, __ldcg(p), err, pf, pl);
              *p = 0ull;
            }
            if (ctid == 0) a.bcount[2 * b] = 0;
            fin = true;
          }
        }
        if (fin) {  // uniform across the consumers
          const double be = consumer_sum(err, s_red);
          if (ctid == 0) a.blk_err[b] = be;
        }
        consumer_sync();
#ifdef GBG_PR_TRACE
        if (ctid == 0 && g_pr_trace_n[blockIdx.x] - 1 < 64)
          g_pr_trace[(blockIdx.x * 64 + g_pr_trace_n[blockIdx.x] - 1) * 6 + 4] = gtime();
#endif
      }
    }
  }

  // ---- last CTA: fold the block partials in block order
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_flag = atomicAdd(a.done_counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_flag) {
    __threadfence();
    double e = 0.0;
    for (uint32_t k = threadIdx.x; k < a.nblocks; k += kPrThreads) e += __ldcg(a.blk_err + k);
    e = block_sum(e, s_red);
    if (threadIdx.x == 0) {
      const double dcur = a.sc->dangling[a.iter & 1];
      const double base = (1.0 - a.damping) / a.nd + a.damping * dcur / a.nd;
      // zero-degree rows (not in any block): rank exactly `base`, dangling
      // mass n_zero * base, L1 step n_zero * |base - previous base|
      e += a.n_zero * fabs(base - a.sc->p_zero);
      a.sc->dangling[(a.iter + 1) & 1] = a.n_zero * base;
      a.sc->p_zero = base;
      a.sc->err = e;
      a.sc->iterations = a.iter + 1;
      if (e < a.tol) a.sc->done = 1;
      *a.done_counter = 0;
      *a.work = 0;
    }
  }
}

// X0 = contrib form of p0; zero-degree rows (never written by the
// iterations) hold a non-positive value in both buffers, so a gather of
// one (an arc into a vertex without out-arcs on a directed graph)
// contributes fmax(x, 0) = 0 as the reference's contrib[u] = 0 does
// (the fixed-point forms the gathers read are 0 for those rows)
__global__ void pr_init_k(const uint32_t* deg, uint64_t n, double* x, double* x1, unsigned long long* t,
                          unsigned long long* t1, double fix) {
  const double p0 = 1.0 / static_cast<double>(n);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint32_t d = deg[r];
    x[r] = d ? p0 / static_cast<double>(d) : -p0;
    t[r] = d ? to_fix(p0 / static_cast<double>(d), fix) : 0ull;
    if (!d) {
      x1[r] = -p0;
      t1[r] = 0ull;
    }
  }
}

// p[old id] from the contrib form of the renumbered vector (zero-degree
// rows: the rank of the last executed iteration, sc->p_zero)
__global__ void pr_to_p_k(const uint32_t* deg, const uint32_t* pos, uint64_t n, const double* x,
                          const PrScalars* sc, double* p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const double pz = sc->p_zero;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    const uint32_t r = pos[v];
    const uint32_t d = deg[r];
    p[v] = d ? x[r] * static_cast<double>(d) : pz;
  }
}

__global__ void pr_scalars_init_k(PrScalars* sc, double dangling0, double p0) {
  sc->dangling[0] = dangling0;
  sc->dangling[1] = 0.0;
  sc->p_zero = p0;
  sc->err = 0.0;
  sc->done = 0;
  sc->iterations = 0;
}

size_t pr_smem_bytes() { return kSmemBytes; }

PrLayout* pr_layout(gbg_graph* g) {
  if (!g->pr) {
    const uint64_t* voff = virtual_offsets(g);
    with_view(g, [&](auto view) { g->pr = build_layout(g, view, voff); });
  }
  if (!g->pr->grid) {
    GBG_CUDA(cudaFuncSetAttribute(pr_tile_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(pr_smem_bytes())));
    int per_sm = 1;
    GBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pr_tile_k, kPrThreads, pr_smem_bytes()));
    g->pr->grid = static_cast<uint32_t>(std::max(per_sm, 1) * g->sm_count);
  }
  return g->pr;
}

uint64_t pr_layout_bytes(const PrLayout* L) { return L ? L->bytes() : 0; }

uint64_t pagerank_run(gbg_graph* g, double damping, uint64_t max_iters, double tol, double* p_dev) {
  const uint64_t n = g->n;
  PrLayout* L = pr_layout(g);
  double* X0 = g->ws.get<double>("pr.x0", n);
  double* X1 = g->ws.get<double>("pr.x1", n);
  PrScalars* sc = g->ws.get<PrScalars>("pr.sc", 1);
  const double p0 = 1.0 / static_cast<double>(n);
  unsigned long long* T0 = g->ws.get<unsigned long long>("pr.t0", n);
  unsigned long long* T1 = g->ws.get<unsigned long long>("pr.t1", n);
  const double fix = std::ldexp(1.0, fix_bits_for(L->m));
  GBG_LAUNCH(g, pr_init_k, grid_for(n, 256), 256, 0, L->deg, n, X0, X1, T0, T1, fix);
  // initial dangling mass: every zero-degree row holds p0
  const double n_zero = static_cast<double>(n - L->nz);
  GBG_LAUNCH(g, pr_scalars_init_k, 1, 1, 0, sc, n_zero * p0, p0);
  double* X[2] = {X0, X1};
  unsigned long long* T[2] = {T0, T1};
  PrArgs a;
  a.arc = L->arc;
  a.run_src = L->run_src;
  a.grp_rbase = L->grp_rbase;
  a.chunk = L->chunk;
  a.tile_chunk = L->tile_chunk;
  a.deg = L->deg;
  a.gsum = L->gsum;
  a.bcount = L->bcount;
  a.blk_err = L->blk_err;
  a.work = L->work;
  a.done_counter = L->done_counter;
  a.sc = sc;
  a.ntiles = L->ntiles;
  a.nblocks = L->nblocks;
  a.nz = L->nz;
  a.damping = damping;
  a.fix = fix;
  a.unfix = 1.0 / fix;
  a.nd = static_cast<double>(n);
  a.tol = tol;
  a.n_zero = n_zero;
  for (uint64_t it = 0; it < max_iters; ++it) {
    a.x_old = X[it & 1];
    a.x_new = X[(it + 1) & 1];
    a.t_old = T[it & 1];
    a.t_new = T[(it + 1) & 1];
    a.iter = static_cast<int>(it);
    GBG_LAUNCH(g, pr_tile_k, L->grid, kPrThreads, pr_smem_bytes(), a);
  }
  PrScalars hs;
  GBG_CUDA(cudaMemcpyAsync(g->hscalar, sc, sizeof(PrScalars), cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  std::memcpy(&hs, g->hscalar, sizeof(PrScalars));
  const uint64_t done = static_cast<uint64_t>(hs.iterations);
  // p lives in the X buffer written by the last executed iteration
  GBG_LAUNCH(g, pr_to_p_k, grid_for(n, 256), 256, 0, L->deg, L->pos, n, X[done & 1], sc, p_dev);
  return done;
}

}  // namespace gbg

void gbg_graph::invalidate_derived() {
  delete pr;
  pr = nullptr;
  if (pr_rows) gbg::prrows::pr_layout_free(pr_rows);
  pr_rows = nullptr;
  voff_valid = false;
  first_valid = false;
}

using namespace gbg;

namespace {
gbg_status pagerank_entry(gbg_graph* g, double damping, uint64_t max_iters, double tol, double* out, bool host,
                          uint64_t* iterations) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!out && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    // algorithms.cpp:510-513
    if (!(damping > 0.0 && damping < 1.0)) fail(GBG_ERR_INVALID_ARGUMENT, "pagerank: damping must be in (0, 1)");
    if (!(tol > 0.0)) fail(GBG_ERR_INVALID_ARGUMENT, "pagerank: tolerance must be > 0");
    uint64_t done = 0;
    if (g->n == 0) {
      if (iterations) *iterations = 0;
      return;
    }
    double* p = host ? g->ws.get<double>("pr.out", g->n) : out;
    if (max_iters == 0) {
      // no iteration: p = 1/n (algorithms.cpp:520)
      std::vector<double> init(g->n, 1.0 / static_cast<double>(g->n));
      GBG_CUDA(cudaMemcpyAsync(p, init.data(), g->n * sizeof(double), cudaMemcpyHostToDevice, g->stream));
    } else if (g->pr) {
      done = pagerank_run(g, damping, max_iters, tol, p);  // tiled index (prepared)
    } else {
      done = prrows::pagerank_rows_run(g, damping, max_iters, tol, p);  // one-shot row path
    }
    if (host) GBG_CUDA(cudaMemcpyAsync(out, p, g->n * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
    if (iterations) *iterations = done;
  });
}
}  // namespace

extern "C" {
gbg_status gbg_pagerank(gbg_graph* g, double damping, uint64_t max_iters, double tolerance, double* ranks,
                        uint64_t* iterations) {
  return pagerank_entry(g, damping, max_iters, tolerance, ranks, true, iterations);
}
gbg_status gbg_pagerank_device(gbg_graph* g, double damping, uint64_t max_iters, double tolerance, double* ranks_dev,
                               uint64_t* iterations) {
  return pagerank_entry(g, damping, max_iters, tolerance, ranks_dev, false, iterations);
}
#ifdef GBG_PR_TRACE
// analysis builds only: copy out and reset the per-CTA tile trace of the
// last pr_tile_k launch ([148][64][6] u64 + [148] counts)
gbg_status gbg_debug_pr_trace(unsigned long long* out, unsigned* counts) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_pr_trace, sizeof(g_pr_trace));
  cudaMemcpyFromSymbol(counts, g_pr_trace_n, sizeof(g_pr_trace_n));
  static unsigned zero[148] = {};
  cudaMemcpyToSymbol(g_pr_trace_n, zero, sizeof(zero));
  static unsigned long long z2[148 * 64 * 6] = {};
  cudaMemcpyToSymbol(g_pr_trace, z2, sizeof(z2));
  return GBG_OK;
}
#endif
gbg_status gbg_pagerank_index_bytes(const gbg_graph* g, uint64_t* tiled, uint64_t* rows) {
  return guard([&] {
    if (!g) fail(GBG_ERR_INVALID_ARGUMENT, "null handle");
    if (tiled) *tiled = pr_layout_bytes(g->pr);
    if (rows) *rows = prrows::rows_bytes(g->pr_rows);
  });
}
gbg_status gbg_pagerank_prepare(gbg_graph* g, double* build_ms) {
  return guard([&] {
    GBG_HANDLE(g);
    if (g->n) {
      PrLayout* L = pr_layout(g);
      if (build_ms) *build_ms = L->build_ms;
    } else if (build_ms) {
      *build_ms = 0;
    }
  });
}
}

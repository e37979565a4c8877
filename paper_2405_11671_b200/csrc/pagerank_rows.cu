// PageRank, row path: one fused pull kernel per power iteration over a
// degree-ordered copy of the graph, one row (or row chunk) per thread group.
// This is the index-free path: its layout (degree sort + relabel, ~19 ms at
// scale 24, overlapped with the upload in gbg_csr_create_ex) is cheap, so
// it serves one-shot calls; the tiled index of pagerank.cu (faster
// iterations, ~5x costlier to build) is used once gbg_pagerank_prepare has
// built it.  Semantics are identical (see pagerank.cu).
//
// Reference: gb::pagerank (algorithms.cpp:508-555).  Per iteration the
// reference runs a serial contrib/dangling loop (528-532), the dense pull
// next[v] += contrib[u] over every v (535-542, edge_map on "everyone" with
// early exit off), then a serial finalize + L1 loop (544-551) and an early
// break when err < tolerance (552).  Here all three are one launch:
//
//   X_i[r] = p_i[r]/deg(r)  if deg(r) > 0   (the contrib the gather reads)
//          = -p_i[r]        if deg(r) = 0   (dangling mass; fmax(X,0) = 0)
//
// so a gather of fmax(X_i[u], 0) yields contrib[u], and the finalize of
// row r emits X_{i+1}[r] directly.  The dangling sum and the L1 error are
// reduced deterministically (per-CTA partials, last-CTA fold in a fixed
// order) and published for the next launch.
//
// Layout (PrRows, built once per graph and cached; rebuilt after updates):
// vertices are renumbered by (degree desc, id asc); the 2^22
// highest-degree vertices (32 MiB of X) receive 98% of all gathers at scale
// 24; streamed arrays load evict_first, gathers evict_last.  Rows of equal
// degree are adjacent, so rows are processed in degree classes, each with a
// fixed thread group per row and a fixed, unrolled number of edges per
// thread.  Results are mapped back to original ids at the end.
#include "radix.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "cache.cuh"
#include "edges.cuh"

namespace gbg {
namespace prrows {

constexpr int kPrThreads = 256;
// edges per heavy-row chunk (32 per thread, issued 8 at a time); 8192 beat
// 2048 / 4096 / 16384 / 32768 at scales 20 and 24 (r01_pr_class_table.md)
constexpr uint32_t kChunk = 8192;
// Gathers of the kL1Hot highest-degree vertices (128 KiB of contribs, ~28%
// of all gathers at scale 24) may stay in L1; the rest bypass it.
#ifndef GBG_PR_MINB
#define GBG_PR_MINB 8  // CTAs of 256 per SM: the 32-register budget
#endif
#ifndef GBG_PR_L1HOT
#define GBG_PR_L1HOT 16384
#endif
constexpr uint32_t kL1Hot = GBG_PR_L1HOT;
// Degree classes over the degree-descending rows: class c gives each row
// T threads and each thread up to K edges, for degrees in (T*K/2, T*K], so
// at most half of the unrolled, predicated slots are idle.  Class 0 (deg >
// 4096) splits rows into kChunk-edge chunks across CTAs (the class-0 K
// entry is unused: a chunk gives each of the 256 threads kChunk/256 edges);
// class 1 (2049 to 4096) takes a CTA per row, class 2 (1025 to 2048) half a
// CTA (4 warps x 16 edges per lane; s20 2.17 -> 2.11 ms, s24 unchanged);
// class 3 (513 to 1024) a warp per row in two
// 512-edge passes (no block barrier: better at scale 24, while the CTA form
// stays better for the longer rows, which dominate at scale 20); below 513
// edges a row gets 16 / 8 / 4 / 2 / 1 lanes walking 16-32 edges each in
// batches of 8 (fewer lanes per row, more rows per warp: scale 24 42.3 ->
// 38.8 ms against the former 32 / 16 lanes x 4-16 edges, see
// profiles/r01_pr_class_table.md); the last class is the isolated rows
// (resolved analytically, not visited).
constexpr int kClasses = 15;
__host__ __device__ constexpr uint32_t class_threads(int c) {
  constexpr uint32_t t[kClasses] = {256, 256, 128, 32, 16, 8, 8, 4, 2, 1, 1, 1, 1, 1, 1};
  return t[c];
}
__host__ __device__ constexpr uint32_t class_k(int c) {
  constexpr uint32_t k[kClasses] = {16, 16, 16, 32, 32, 32, 16, 16, 16, 16, 8, 4, 2, 1, 0};
  return k[c];
}
__host__ __device__ constexpr uint32_t class_max_deg(int c) { return c == 0 ? 0xffffffffu : class_threads(c) * class_k(c); }

struct PrRows {
  uint64_t n = 0, m = 0;
  uint64_t* off = nullptr;   // [n+1] relabelled CSR
  uint32_t* nbr = nullptr;   // [m]
  uint32_t* ord = nullptr;   // new -> old id
  uint32_t* pos = nullptr;   // old -> new id
  uint32_t row_begin[kClasses + 1] = {};
  uint64_t unit_begin[kClasses + 1] = {};  // work units, class by class
  uint64_t* hchunk = nullptr;  // heavy rows: exclusive scan of chunk counts [nheavy+1]
  uint32_t* hrow = nullptr;    // heavy chunk -> row
  unsigned* heavy_counter = nullptr;
  double* heavy_partial = nullptr;
  double* blk = nullptr;
  unsigned* done_counter = nullptr;
  uint32_t grid = 0;
  double build_ms = 0;
  ~PrRows() {
    dfree(off);
    dfree(nbr);
    dfree(ord);
    dfree(pos);
    dfree(hchunk);
    dfree(hrow);
    dfree(heavy_counter);
    dfree(heavy_partial);
    dfree(blk);
    dfree(done_counter);
  }
};

// ---------------------------------------------------------------- layout build
// (degree desc, id asc) as one key: inverted degree above the L id bits
template <class G>
__global__ void degree_keys_k(G g, int L, uint64_t* keys) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < g.n; v += stride)
    keys[v] = (static_cast<uint64_t>(0xffffffffu - g.degree(static_cast<uint32_t>(v))) << L) | v;
}

__global__ void order_from_keys_k(const uint64_t* sorted, uint64_t n, int L, uint32_t* ord, uint32_t* pos) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint32_t v = static_cast<uint32_t>(sorted[r] & ((uint64_t{1} << L) - 1));
    ord[r] = v;
    pos[v] = static_cast<uint32_t>(r);
  }
}

struct SortedDegIn {
  const uint64_t* sorted;
  int L;
  __device__ __forceinline__ uint64_t operator()(uint64_t r) const {
    return 0xffffffffu - static_cast<uint32_t>(sorted[r] >> L);
  }
};

struct RelabelOp {
  const uint64_t* voff;  // source graph prefix (CSR offsets / blocked virtual offsets)
  const uint32_t* pos;
  const uint64_t* new_off;
  uint32_t* new_nbr;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t e) const {
    new_nbr[new_off[pos[u]] + (e - voff[u])] = pos[v];
  }
};

// first row (degree-descending order) whose degree is <= class_max_deg(c+1)
__global__ void class_bounds_k(const uint64_t* off, uint64_t n, uint32_t* out) {
  const int c = threadIdx.x;
  if (c >= kClasses - 1) return;
  const uint32_t bound = class_max_deg(c + 1);
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (off[mid + 1] - off[mid] <= bound) hi = mid; else lo = mid + 1;
  }
  out[c] = static_cast<uint32_t>(lo);
}

struct HeavyChunksIn {
  const uint64_t* off;
  __device__ __forceinline__ uint64_t operator()(uint64_t r) const {
    return (off[r + 1] - off[r] + kChunk - 1) / kChunk;
  }
};
struct HeavyChunksOut {
  const uint64_t* off;
  uint64_t* hchunk;
  uint32_t* hrow;
  __device__ __forceinline__ void operator()(uint64_t r, uint64_t pre) const {
    hchunk[r] = pre;
    const uint64_t c = HeavyChunksIn{off}(r);
    for (uint64_t k = 0; k < c; ++k) hrow[pre + k] = static_cast<uint32_t>(r);
  }
};

// Phase 1 (offsets only): the degree order, the relabelled offsets, the
// degree classes and the heavy-row chunk map; L->nbr is allocated but not
// filled.  Phase 2 (layout_relabel) fills it for any range of edges, so a
// pipelined container build can relabel each chunk of neighbour ids as it
// lands (gbg_csr_create_ex, api.cu).
template <class G>
PrRows* layout_rows(gbg_graph* g, G view) {
  const uint64_t n = g->n, m = g->m;
  auto L = std::make_unique<PrRows>();
  L->n = n;
  L->m = m;
  uint64_t* keys = g->ws.get<uint64_t>("prl.keys", n);
  uint64_t* scratch = g->ws.get<uint64_t>("prl.sorted", n);
  int idb = 1;  // id bits
  while ((uint64_t{1} << idb) < n) ++idb;
  GBG_LAUNCH(g, degree_keys_k<G>, grid_for(n, 256), 256, 0, view, idb, keys);
  const uint64_t* sorted = radix_sort_u64(g, keys, scratch, n, 32 + idb, "prl.sort");
  L->ord = dalloc<uint32_t>(n);
  L->pos = dalloc<uint32_t>(n);
  L->off = dalloc<uint64_t>(n + 1);
  L->nbr = dalloc<uint32_t>(m);
  GBG_LAUNCH(g, order_from_keys_k, grid_for(n, 256), 256, 0, sorted, n, idb, L->ord, L->pos);
  device_scan<uint64_t>(g, SortedDegIn{sorted, idb}, ArrayOut<uint64_t>{L->off}, n, L->off + n, "prl.scan");
  uint32_t* bnd = g->ws.get<uint32_t>("prl.bnd", kClasses);
  GBG_LAUNCH(g, class_bounds_k, 1, 32, 0, L->off, n, bnd);
  uint32_t hb[kClasses];
  GBG_CUDA(cudaMemcpyAsync(hb, bnd, sizeof(hb), cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  L->row_begin[0] = 0;
  for (int c = 0; c < kClasses - 1; ++c) L->row_begin[c + 1] = hb[c];
  L->row_begin[kClasses] = static_cast<uint32_t>(n);
  const uint32_t nheavy = L->row_begin[1];
  L->hchunk = dalloc<uint64_t>(nheavy + 1);
  uint64_t nchunks = 0;
  device_scan<uint64_t>(g, HeavyChunksIn{L->off}, NullOut{}, nheavy, L->hchunk + nheavy, "prl.heavy");
  read_scalars(g, L->hchunk + nheavy, sizeof(nchunks), &nchunks);
  L->hrow = dalloc<uint32_t>(nchunks + 1);
  device_scan<uint64_t>(g, HeavyChunksIn{L->off}, HeavyChunksOut{L->off, L->hchunk, L->hrow}, nheavy,
                        L->hchunk + nheavy, "prl.heavy");
  L->unit_begin[0] = 0;
  L->unit_begin[1] = nchunks;
  for (int c = 1; c < kClasses; ++c) {
    const uint64_t rows = L->row_begin[c + 1] - L->row_begin[c];
    const uint64_t per_unit = kPrThreads / class_threads(c);
    L->unit_begin[c + 1] = L->unit_begin[c] + (rows + per_unit - 1) / per_unit;
  }
  L->heavy_counter = dalloc<unsigned>(nheavy + 1);
  L->heavy_partial = dalloc<double>(nchunks + 1);
  L->done_counter = dalloc<unsigned>(1);
  GBG_CUDA(cudaMemsetAsync(L->heavy_counter, 0, (nheavy + 1) * sizeof(unsigned), g->stream));
  GBG_CUDA(cudaMemsetAsync(L->done_counter, 0, sizeof(unsigned), g->stream));
  g->ws.release("prl.keys");
  g->ws.release("prl.sorted");
  g->ws.release("prl.sort.hist");
  g->ws.release("prl.sort.lb");
  return L.release();
}

// relabel op for not-yet-validated input: out-of-range ids are skipped (the
// caller's validation rejects the graph)
struct RelabelCheckedOp {
  RelabelOp op;
  uint64_t n;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t e) const {
    if (v < n) op(u, v, e);
  }
};

template <class G>
void layout_relabel(gbg_graph* g, G view, const uint64_t* voff, PrRows* L, uint64_t e0, uint64_t e1) {
  for_each_edge_range(g, view, voff, e0, e1, RelabelCheckedOp{RelabelOp{voff, L->pos, L->off, L->nbr}, g->n});
}

// Heavy rows (> 4096 edges: the hubs, first in the degree order) get their
// relabelled lists sorted ascending.  A warp of the chunked heavy-row path
// reads 32 consecutive entries per gather, and in a sorted hub list the
// many neighbours inside the dense hot region share 128-byte lines, so the
// gather instruction needs fewer L1 wavefronts (scale 24: 48.2 -> 46.4 ms
// for 20 iterations; sorting the other rows as well gains nothing more,
// sorting only within 4096-entry chunks half as much).  One stable radix
// sort of (row, id) keys over the heavy rows' arcs: +10.8 ms of layout
// build at scale 24, paid once per graph version by gbg_pagerank_prepare /
// the first PageRank call.  The pipelined create (gbg_csr_create_ex with
// GBG_CREATE_PAGERANK_LAYOUT) skips it: hub rows complete only when their
// last chunk lands, anywhere in the upload, so the sort would be exposed
// (+10-18 ms) for a 1.8 ms saving on a 20-iteration call.
struct HeavyKeyOp {
  uint64_t* keys;
  int idb;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t v, uint64_t e) const {
    keys[e] = (static_cast<uint64_t>(u) << idb) | v;
  }
};
__global__ void heavy_unkey_k(const uint64_t* keys, uint64_t count, int idb, uint32_t* nbr) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count; e += stride)
    nbr[e] = static_cast<uint32_t>(keys[e] & ((uint64_t{1} << idb) - 1));
}
void layout_sort_heavy(gbg_graph* g, PrRows* L) {
  const uint32_t nheavy = L->row_begin[1];
  if (!nheavy) return;
  uint64_t H = 0;
  read_scalars(g, L->off + nheavy, sizeof(H), &H);
  if (!H) return;
  int idb = 1, rb = 1;
  while ((uint64_t{1} << idb) < L->n) ++idb;
  while ((uint64_t{1} << rb) < nheavy) ++rb;
  uint64_t* keys = g->ws.get<uint64_t>("prl.hkeys", H);
  uint64_t* scr = g->ws.get<uint64_t>("prl.hscr", H);
  CsrView lv{L->n, L->off, L->nbr};
  for_each_edge_range(g, lv, L->off, 0, H, HeavyKeyOp{keys, idb});
  const uint64_t* sorted = radix_sort_u64(g, keys, scr, H, rb + idb, "prl.hsort");
  GBG_LAUNCH(g, heavy_unkey_k, grid_for(H, 256), 256, 0, sorted, H, idb, L->nbr);
  g->ws.release("prl.hkeys");
  g->ws.release("prl.hscr");
  g->ws.release("prl.hsort.hist");
  g->ws.release("prl.hsort.lb");
}

template <class G>
PrRows* build_layout(gbg_graph* g, G view, const uint64_t* voff) {
  cudaEvent_t e0, e1;
  GBG_CUDA(cudaEventCreate(&e0));
  GBG_CUDA(cudaEventCreate(&e1));
  GBG_CUDA(cudaEventRecord(e0, g->stream));
  PrRows* L = layout_rows(g, view);
  layout_relabel(g, view, voff, L, 0, g->m);
  layout_sort_heavy(g, L);
  GBG_CUDA(cudaEventRecord(e1, g->stream));
  GBG_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  L->build_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return L;
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
  const uint64_t* off;
  const uint32_t* nbr;
  const double* x_old;
  double* x_new;
  const uint64_t* hchunk;
  const uint32_t* hrow;
  double* heavy_partial;
  unsigned* heavy_counter;
  double* blk;
  unsigned* done_counter;
  PrScalars* sc;
  uint32_t row_begin[kClasses + 1];
  uint64_t unit_begin[kClasses + 1];
  double damping, nd, tol;
  double n_zero;  // zero-degree rows (the last class)
  int iter;
};

// Finalize row r (d > 0; algorithms.cpp:544-550 for one vertex) and emit
// the next iteration's contrib form.
__device__ __forceinline__ void pr_finalize(const PrArgs& a, double base, uint32_t r, uint64_t d, double sum,
                                            double& err) {
  const double next = base + a.damping * sum;
  const double xo = __ldcs(a.x_old + r);
  err += fabs(next - xo * static_cast<double>(d));
  a.x_new[r] = next / static_cast<double>(d);
}

// Sum of fmax(X[nbr[e]], 0) over e = b + t, b + t + T, ... (< b + d), with
// all K id loads issued before the K gathers.
// At most 8 id loads, then 8 gathers, in flight per thread: longer unrolls
// (K = 16 / 32 in the class table) run as sequential batches of 8.  The
// 16-wide form spilled the ids to local memory at the 32-register budget,
// and every spilled line is an L1->L2 request on the path that limits this
// kernel (l1tex2xbar request cycles ~70% of peak): s24 46.4 -> 44.8 ms.
#ifndef GBG_PR_KMAX
#define GBG_PR_KMAX 8
#endif
template <int K>
__device__ __forceinline__ double gather_sum(const PrArgs& a, uint64_t b, uint32_t d, uint32_t t, uint32_t T,
                                             uint64_t pf, uint64_t pl) {
  if constexpr (K > GBG_PR_KMAX) {
    const double lo = gather_sum<GBG_PR_KMAX>(a, b, d, t, T, pf, pl);
    return lo + gather_sum<K - GBG_PR_KMAX>(a, b, d, t + GBG_PR_KMAX * T, T, pf, pl);
  }
  const uint32_t* nb = a.nbr + b;
  uint32_t ids[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const uint32_t k = t + j * T;
    ids[j] = k < d ? ld_stream_u32(nb + k, pf) : 0u;
  }
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const uint32_t k = t + j * T;
    double x = 0.0;
    if (k < d) x = ids[j] < kL1Hot ? ld_hot_f64(a.x_old + ids[j], pl) : ld_cold_f64(a.x_old + ids[j], pl);
    acc += fmax(x, 0.0);
  }
  return acc;
}

// Persistent: CTA b owns work units b, b + grid, ... (static assignment, so
// the err / dangling fold is deterministic).
__global__ void __launch_bounds__(kPrThreads, GBG_PR_MINB) pr_iter_k(PrArgs a) {
  __shared__ double s_red[33];
  __shared__ int s_flag;
  if (a.sc->done) return;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const double dcur = a.sc->dangling[a.iter & 1];
  const double base = (1.0 - a.damping) / a.nd + a.damping * dcur / a.nd;
  double err = 0.0;
  // Zero-degree rows (the last class; 7.9M of 16.8M at scale 24) are not
  // visited: they gather nothing (an arc into one on a directed graph reads
  // the non-positive contrib form pr_init_k leaves in both buffers, i.e.
  // contributes 0, as the reference's contrib[u] = 0), and each one's next rank is exactly
  // `base` (base + damping * 0), so their dangling mass is n_zero * base and
  // their L1 step is n_zero * |base - previous base|, folded in below, and
  // the output maps them to the last base (pr_to_p_k).
  const uint32_t total = static_cast<uint32_t>(a.unit_begin[kClasses - 1]);

  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    int c = 0;
#pragma unroll
    for (int k = 1; k < kClasses; ++k)
      if (w >= a.unit_begin[k]) c = k;
    if (c == 0) {
      // ---- heavy row chunk: deterministic two-level sum
      const uint32_t r = __ldg(a.hrow + w);
      const uint64_t c0 = __ldg(a.hchunk + r);
      const uint64_t rb = __ldg(a.off + r), re = __ldg(a.off + r + 1);
      const uint32_t nch = static_cast<uint32_t>((re - rb + kChunk - 1) / kChunk);
      const uint64_t eb = rb + (w - c0) * kChunk;
      const uint32_t len = static_cast<uint32_t>(eb + kChunk < re ? kChunk : re - eb);
      const double s = block_sum(gather_sum<kChunk / kPrThreads>(a, eb, len, threadIdx.x, kPrThreads, pf, pl), s_red);
      if (threadIdx.x == 0) {
        a.heavy_partial[w] = s;
        __threadfence();
        s_flag = atomicAdd(a.heavy_counter + r, 1u) == nch - 1;
      }
      __syncthreads();
      if (s_flag && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (uint32_t k = 0; k < nch; ++k) tot += __ldcg(a.heavy_partial + c0 + k);
        pr_finalize(a, base, r, re - rb, tot, err);
        a.heavy_counter[r] = 0;
      }
      __syncthreads();
    } else if (class_threads(c) == kPrThreads / 2) {
      // ---- half a CTA (4 warps) per row, two rows per unit
      const uint32_t half = threadIdx.x >> 7, t = threadIdx.x & 127;
      const uint64_t r64 = a.row_begin[c] + static_cast<uint64_t>(w - a.unit_begin[c]) * 2 + half;
      const bool valid = r64 < a.row_begin[c + 1];
      const uint32_t r = static_cast<uint32_t>(r64);
      double p = 0.0;
      uint32_t d = 0;
      if (valid) {
        const uint64_t rb = __ldg(a.off + r);
        d = static_cast<uint32_t>(__ldg(a.off + r + 1) - rb);
        if (class_k(c) == 32) p = gather_sum<32>(a, rb, d, t, 128, pf, pl);
        else p = gather_sum<16>(a, rb, d, t, 128, pf, pl);
      }
      for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = p;
      __syncthreads();
      if (t == 0 && valid) {
        const double s = (s_red[4 * half] + s_red[4 * half + 1]) + (s_red[4 * half + 2] + s_red[4 * half + 3]);
        pr_finalize(a, base, r, d, s, err);
      }
      __syncthreads();
    } else if (class_threads(c) == kPrThreads) {
      // ---- one CTA per row
      const uint32_t r = a.row_begin[c] + static_cast<uint32_t>(w - a.unit_begin[c]);
      const uint64_t rb = __ldg(a.off + r);
      const uint32_t d = static_cast<uint32_t>(__ldg(a.off + r + 1) - rb);
      double p;
      if (class_k(c) == 16) p = gather_sum<16>(a, rb, d, threadIdx.x, kPrThreads, pf, pl);
      else if (class_k(c) == 8) p = gather_sum<8>(a, rb, d, threadIdx.x, kPrThreads, pf, pl);
      else p = gather_sum<4>(a, rb, d, threadIdx.x, kPrThreads, pf, pl);
      const double s = block_sum(p, s_red);
      if (threadIdx.x == 0) pr_finalize(a, base, r, d, s, err);
    } else {
      // ---- a fixed group of lanes per row, rows of the unit consecutive
      const uint32_t lanes = class_threads(c);
      const uint32_t rows_per_unit = kPrThreads / lanes;
      const uint64_t r64 = a.row_begin[c] + (w - a.unit_begin[c]) * rows_per_unit + threadIdx.x / lanes;
      const bool valid = r64 < a.row_begin[c + 1];
      const uint32_t r = static_cast<uint32_t>(r64);
      const uint32_t l = threadIdx.x & (lanes - 1);
      double acc = 0.0;
      uint32_t d = 0;
      if (valid) {
        const uint64_t rb = ld_stream_u64(a.off + r, pf);
        d = static_cast<uint32_t>(ld_stream_u64(a.off + r + 1, pf) - rb);
        switch (class_k(c)) {
          case 32:
            if (lanes == 32) {  // warp per row, 512 edges per pass (no block barrier)
              for (uint32_t o = 0; o < d; o += 16 * 32) acc += gather_sum<16>(a, rb + o, d - o, l, 32, pf, pl);
            } else {  // (the table has K = 32 only, below a full warp)
              acc = gather_sum<32>(a, rb, d, l, lanes, pf, pl);
            }
            break;
          case 16: acc = gather_sum<16>(a, rb, d, l, lanes, pf, pl); break;
          case 8: acc = gather_sum<8>(a, rb, d, l, lanes, pf, pl); break;
          case 4: acc = gather_sum<4>(a, rb, d, l, lanes, pf, pl); break;
          case 2: acc = gather_sum<2>(a, rb, d, l, lanes, pf, pl); break;
          case 1: acc = gather_sum<1>(a, rb, d, l, lanes, pf, pl); break;
          default: break;
        }
      }
      for (uint32_t o = lanes >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, lanes);
      if (valid && l == 0) pr_finalize(a, base, r, d, acc, err);
    }
  }

  // ---- per-CTA partials, last CTA folds them in order
  const double be = block_sum(err, s_red);
  if (threadIdx.x == 0) {
    a.blk[blockIdx.x] = be;
    __threadfence();
    s_flag = atomicAdd(a.done_counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_flag) {
    __threadfence();
    double e = 0.0;
    for (uint64_t k = threadIdx.x; k < gridDim.x; k += kPrThreads) e += __ldcg(a.blk + k);
    e = block_sum(e, s_red);
    if (threadIdx.x == 0) {
      e += a.n_zero * fabs(base - a.sc->p_zero);
      a.sc->dangling[(a.iter + 1) & 1] = a.n_zero * base;
      a.sc->p_zero = base;
      a.sc->err = e;
      a.sc->iterations = a.iter + 1;
      if (e < a.tol) a.sc->done = 1;
      *a.done_counter = 0;
    }
  }
}

// X0 = contrib form of p0; zero-degree rows (never written by the
// iterations) hold a non-positive value in both buffers, so a gather of
// one (an arc into a vertex without out-arcs, after asymmetric updates)
// contributes fmax(x, 0) = 0 as the reference's contrib[u] = 0 does
__global__ void pr_init_k(const uint64_t* off, uint64_t n, double* x, double* x1) {
  const double p0 = 1.0 / static_cast<double>(n);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint64_t d = off[r + 1] - off[r];
    x[r] = d ? p0 / static_cast<double>(d) : -p0;
    if (!d) x1[r] = -p0;
  }
}


// p[old id] from the contrib form of the renumbered vector (zero-degree
// rows: the rank of the last executed iteration, sc->p_zero)
__global__ void pr_to_p_k(const uint64_t* off, const uint32_t* pos, uint64_t n, const double* x,
                          const PrScalars* sc, double* p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const double pz = sc->p_zero;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    const uint32_t r = pos[v];
    const uint64_t d = off[r + 1] - off[r];
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

PrRows* pr_layout(gbg_graph* g) {
  if (!g->pr_rows) {
    const uint64_t* voff = virtual_offsets(g);
    with_view(g, [&](auto view) { g->pr_rows = build_layout(g, view, voff); });
  }
  if (!g->pr_rows->grid) {
    int per_sm = 1;
    GBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pr_iter_k, kPrThreads, 0));
    g->pr_rows->grid = static_cast<uint32_t>(std::max(per_sm, 1) * g->sm_count);
    g->pr_rows->blk = dalloc<double>(g->pr_rows->grid);
  }
  return g->pr_rows;
}

// pipelined CSR builds (api.cu)
PrRows* pr_layout_rows_csr(gbg_graph* g) { return layout_rows(g, g->csr_view()); }
void pr_layout_relabel_csr(gbg_graph* g, PrRows* L, uint64_t e0, uint64_t e1) {
  layout_relabel(g, g->csr_view(), g->off, L, e0, e1);
}
void pr_layout_attach(gbg_graph* g, PrRows* L, float build_ms) {
  L->build_ms = build_ms;
  g->pr_rows = L;
}
void pr_layout_free(PrRows* L) { delete L; }

uint64_t pagerank_rows_run(gbg_graph* g, double damping, uint64_t max_iters, double tol, double* p_dev) {
  const uint64_t n = g->n;
  PrRows* L = pr_layout(g);
  double* X0 = g->ws.get<double>("pr.x0", n);
  double* X1 = g->ws.get<double>("pr.x1", n);
  PrScalars* sc = g->ws.get<PrScalars>("pr.sc", 1);
  const double p0 = 1.0 / static_cast<double>(n);
  GBG_LAUNCH(g, pr_init_k, grid_for(n, 256), 256, 0, L->off, n, X0, X1);
  // initial dangling mass: every zero-degree row holds p0
  const double n_zero = static_cast<double>(n - L->row_begin[kClasses - 1]);
  GBG_LAUNCH(g, pr_scalars_init_k, 1, 1, 0, sc, n_zero * p0, p0);
  double* X[2] = {X0, X1};
  for (uint64_t it = 0; it < max_iters; ++it) {
    PrArgs a;
    a.off = L->off;
    a.nbr = L->nbr;
    a.x_old = X[it & 1];
    a.x_new = X[(it + 1) & 1];
    a.hchunk = L->hchunk;
    a.hrow = L->hrow;
    a.heavy_partial = L->heavy_partial;
    a.heavy_counter = L->heavy_counter;
    a.blk = L->blk;
    a.done_counter = L->done_counter;
    a.sc = sc;
    std::memcpy(a.row_begin, L->row_begin, sizeof(a.row_begin));
    std::memcpy(a.unit_begin, L->unit_begin, sizeof(a.unit_begin));
    a.damping = damping;
    a.nd = static_cast<double>(n);
    a.tol = tol;
    a.iter = static_cast<int>(it);
    a.n_zero = static_cast<double>(n - L->row_begin[kClasses - 1]);
    GBG_LAUNCH(g, pr_iter_k, L->grid, kPrThreads, 0, a);
  }
  PrScalars hs;
  GBG_CUDA(cudaMemcpyAsync(g->hscalar, sc, sizeof(PrScalars), cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  std::memcpy(&hs, g->hscalar, sizeof(PrScalars));
  const uint64_t done = static_cast<uint64_t>(hs.iterations);
  // p lives in the X buffer written by the last executed iteration
  GBG_LAUNCH(g, pr_to_p_k, grid_for(n, 256), 256, 0, L->off, L->pos, n, X[done & 1], sc, p_dev);
  return done;
}

uint64_t rows_bytes(const PrRows* L) {
  if (!L) return 0;
  // relabelled CSR and both id maps (the heavy-row chunk tables are small)
  return (L->n + 1) * 8 + L->m * 4 + L->n * 8;
}

double rows_build_ms(const PrRows* L) { return L->build_ms; }
}  // namespace prrows
}  // namespace gbg

// PageRank: one fused pull kernel per power iteration.
//
// Reference: gb::pagerank (algorithms.cpp:508-555).  Per iteration the
// reference runs a serial contrib/dangling loop (528-532), the dense pull
// next[v] += contrib[u] over every v (535-542, edge_map on "everyone" with
// early exit off), then a serial finalize + L1 loop (544-551) and an early
// break when err < tolerance (552).  Here all three are one launch:
//
//   X_i[v] = p_i[v]/deg(v)  if deg(v) > 0   (the contrib the gather reads)
//          = -p_i[v]        if deg(v) = 0   (dangling mass; fmax(X,0) = 0)
//
// so a gather of fmax(X_i[u], 0) yields contrib[u], and the finalize of
// row v can emit X_{i+1}[v] directly.  The dangling sum and the L1 error
// are reduced deterministically (per-CTA partials, last-CTA fold in a fixed
// order) and published for the next launch, which computes the same base
// term (1-d)/n + d*dangling/n as algorithms.cpp:544-545.
//
// Load balance: rows are packed into row-aligned tiles of ~kTileItems
// (rows + edges) items; rows with more than kHeavy edges get their own
// tile split into kChunk-edge chunks across CTAs (deterministic two-level
// sum).  Inside a light tile the neighbour ids are streamed into shared
// memory coalesced, the fp64 contributions gathered, and each thread walks
// an equal share of the merge path (Merrill & Garland's merge-based CSR
// SpMV decomposition) with a block-wide reduce-by-key for rows that straddle
// threads.  The schedule is built once per graph and cached.
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "scan.cuh"

namespace gbg {

constexpr int kPrThreads = 256;
constexpr uint32_t kTileItems = 2048;          // light-tile budget (rows + edges)
constexpr uint32_t kHeavy = 1024;              // rows above this are split
constexpr uint32_t kTileMax = kTileItems + kHeavy + 1;
constexpr uint32_t kChunk = 4096;              // edges per heavy-row chunk

struct PrSchedule {
  uint64_t ntiles = 0, nwork = 0;
  uint32_t* tile_row = nullptr;    // [ntiles+1]
  uint32_t* work_tile = nullptr;   // [nwork]
  uint32_t* work_chunk = nullptr;  // [nwork]
  unsigned* heavy_counter = nullptr;
  double* heavy_partial = nullptr;
  double* blk = nullptr;           // [2*nwork] err, dangling partials
  unsigned* done_counter = nullptr;
  ~PrSchedule() {
    dfree(tile_row);
    dfree(work_tile);
    dfree(work_chunk);
    dfree(heavy_counter);
    dfree(heavy_partial);
    dfree(blk);
    dfree(done_counter);
  }
};

struct TileWeightIn {
  const uint64_t* voff;
  __device__ __forceinline__ uint64_t operator()(uint64_t r) const {
    uint64_t d = voff[r + 1] - voff[r];
    return d > kHeavy ? 1 : d + 1;
  }
};

__global__ void tile_flags_k(const uint64_t* voff, const uint64_t* P, uint64_t n, uint32_t* flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    bool heavy = voff[r + 1] - voff[r] > kHeavy;
    bool s = r == 0 || heavy;
    if (!s) {
      bool prev_heavy = voff[r] - voff[r - 1] > kHeavy;
      s = prev_heavy || (P[r] / kTileItems != P[r - 1] / kTileItems);
    }
    flag[r] = s ? 1u : 0u;
  }
}

struct FlagIn {
  const uint32_t* f;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return f[i]; }
};
struct TileRowOut {
  const uint32_t* f;
  uint32_t* tile_row;
  __device__ __forceinline__ void operator()(uint64_t i, uint32_t pre) const {
    if (f[i]) tile_row[pre] = static_cast<uint32_t>(i);
  }
};
struct ChunksIn {
  const uint32_t* tile_row;
  const uint64_t* voff;
  __device__ __forceinline__ uint32_t operator()(uint64_t t) const {
    uint32_t r0 = tile_row[t], r1 = tile_row[t + 1];
    uint64_t d = voff[r0 + 1] - voff[r0];
    if (r1 - r0 == 1 && d > kHeavy) return static_cast<uint32_t>((d + kChunk - 1) / kChunk);
    return 1;
  }
};
struct WorkOut {
  const uint32_t* tile_row;
  const uint64_t* voff;
  uint32_t* work_tile;
  uint32_t* work_chunk;
  __device__ __forceinline__ void operator()(uint64_t t, uint32_t pre) const {
    uint32_t c = ChunksIn{tile_row, voff}(t);
    for (uint32_t k = 0; k < c; ++k) {
      work_tile[pre + k] = static_cast<uint32_t>(t);
      work_chunk[pre + k] = k;
    }
  }
};

__global__ void set_u32_k(uint32_t* p, uint32_t v) { *p = v; }

PrSchedule* build_schedule(gbg_graph* g, const uint64_t* voff) {
  const uint64_t n = g->n;
  auto s = std::make_unique<PrSchedule>();
  uint64_t* P = g->ws.get<uint64_t>("pr.P", n + 1);
  device_scan<uint64_t>(g, TileWeightIn{voff}, ArrayOut<uint64_t>{P}, n, P + n, "pr.s1");
  uint32_t* flag = g->ws.get<uint32_t>("pr.flag", n);
  GBG_LAUNCH(g, tile_flags_k, grid_for(n, 256), 256, 0, voff, P, n, flag);
  uint32_t* cnt = g->ws.get<uint32_t>("pr.cnt", 2);
  // at most n tiles
  s->tile_row = dalloc<uint32_t>(n + 1);
  device_scan<uint32_t>(g, FlagIn{flag}, TileRowOut{flag, s->tile_row}, n, cnt, "pr.s2");
  uint32_t nt = 0;
  read_scalars(g, cnt, sizeof(nt), &nt);
  s->ntiles = nt;
  GBG_LAUNCH(g, set_u32_k, 1, 1, 0, s->tile_row + nt, static_cast<uint32_t>(n));
  device_scan<uint32_t>(g, ChunksIn{s->tile_row, voff}, NullOut{}, nt, cnt + 1, "pr.s3");
  uint32_t nw = 0;
  read_scalars(g, cnt + 1, sizeof(nw), &nw);
  s->nwork = nw;
  s->work_tile = dalloc<uint32_t>(nw);
  s->work_chunk = dalloc<uint32_t>(nw);
  device_scan<uint32_t>(g, ChunksIn{s->tile_row, voff}, WorkOut{s->tile_row, voff, s->work_tile, s->work_chunk}, nt,
                        cnt + 1, "pr.s3");
  s->heavy_counter = dalloc<unsigned>(nt);
  s->heavy_partial = dalloc<double>(nw);
  s->blk = dalloc<double>(2 * nw);
  s->done_counter = dalloc<unsigned>(1);
  GBG_CUDA(cudaMemsetAsync(s->heavy_counter, 0, nt * sizeof(unsigned), g->stream));
  GBG_CUDA(cudaMemsetAsync(s->done_counter, 0, sizeof(unsigned), g->stream));
  g->ws.release("pr.P");
  g->ws.release("pr.flag");
  return s.release();
}

// ---------------------------------------------------------------- kernels
struct PrScalars {
  double dangling[2];  // ping-pong: iteration i reads [i&1], writes [(i+1)&1]
  double err;          // L1 step difference of the last executed iteration
  int done;            // set once err < tolerance (algorithms.cpp:552)
  int iterations;      // iterations executed
};

struct PrArgs {
  const uint32_t* tile_row;
  const uint32_t* work_tile;
  const uint32_t* work_chunk;
  const uint64_t* voff;
  const double* x_old;
  double* x_new;
  double* p_out;  // written only when non-null (the last scheduled iteration)
  double* heavy_partial;
  unsigned* heavy_counter;
  double* blk;
  unsigned* done_counter;
  PrScalars* sc;
  uint64_t nwork;
  double damping, nd, tol;
  int iter;
};

struct KV {
  int64_t k;
  double v;
};

__device__ __forceinline__ KV kv_combine(KV a, KV b) { return {b.k, a.k == b.k ? a.v + b.v : b.v}; }

// Finalize row v (algorithms.cpp:544-550 for one vertex) and emit the
// next iteration's contrib form.
__device__ __forceinline__ void pr_finalize(const PrArgs& a, double base, uint32_t v, uint64_t d, double sum,
                                            double& err, double& dang) {
  const double next = base + a.damping * sum;
  const double xo = a.x_old[v];
  const double pold = d ? xo * static_cast<double>(d) : -xo;
  err += fabs(next - pold);
  if (d) {
    a.x_new[v] = next / static_cast<double>(d);
  } else {
    a.x_new[v] = -next;
    dang += next;
  }
  if (a.p_out) a.p_out[v] = next;
}

constexpr int kPerThread = (kTileMax + kPrThreads - 1) / kPrThreads;  // 13

// Persistent: CTA b owns work items b, b + grid, b + 2*grid, ... (a static
// assignment, so the err / dangling fold below is deterministic).  Each
// light tile issues all of its global loads (row ends, neighbour ids, then
// the dependent contrib gathers) as unrolled batches before one barrier, so
// every thread has ~kPerThread independent requests in flight per phase.
template <class G>
__global__ void __launch_bounds__(kPrThreads) pr_iter_k(G g, PrArgs a) {
  __shared__ double s_val[kTileMax];
  __shared__ uint32_t s_rowend[kTileMax];
  __shared__ double s_red[33];
  __shared__ KV s_warp[kPrThreads / 32];
  __shared__ int s_flag;

  if (a.sc->done) return;
  const double dcur = a.sc->dangling[a.iter & 1];
  const double base = (1.0 - a.damping) / a.nd + a.damping * dcur / a.nd;
  double err = 0.0, dang = 0.0;

  for (uint32_t w = blockIdx.x; w < a.nwork; w += gridDim.x) {
  const uint32_t t = __ldg(a.work_tile + w);
  const uint32_t r0 = __ldg(a.tile_row + t), r1 = __ldg(a.tile_row + t + 1);
  const uint64_t eb = __ldg(a.voff + r0);
  const uint64_t d0 = __ldg(a.voff + r0 + 1) - eb;
  if (r1 - r0 == 1 && d0 > kHeavy) {
    // ---- heavy row chunk
    const uint32_t c = a.work_chunk[w];
    const uint32_t nch = static_cast<uint32_t>((d0 + kChunk - 1) / kChunk);
    uint64_t b;
    uint32_t dd;
    g.seg(r0, b, dd);
    const uint64_t lo = static_cast<uint64_t>(c) * kChunk;
    const uint64_t hi = (d0 < lo + kChunk ? d0 : lo + kChunk);
    double acc = 0.0;
    constexpr int kCh = kChunk / kPrThreads;  // 16 per thread
    uint32_t ids[kCh];
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      const uint64_t k = lo + threadIdx.x + j * kPrThreads;
      ids[j] = k < hi ? g.at(b + k) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      const uint64_t k = lo + threadIdx.x + j * kPrThreads;
      const double x = k < hi ? __ldg(a.x_old + ids[j]) : 0.0;
      acc += fmax(x, 0.0);
    }
    const double s = block_sum(acc, s_red);
    if (threadIdx.x == 0) {
      a.heavy_partial[w] = s;
      __threadfence();
      s_flag = atomicAdd(a.heavy_counter + t, 1u) == nch - 1;
    }
    __syncthreads();
    if (s_flag && threadIdx.x == 0) {
      __threadfence();
      double tot = 0.0;
      const uint32_t w0 = w - c;
      for (uint32_t k = 0; k < nch; ++k) tot += ((volatile double*)a.heavy_partial)[w0 + k];
      pr_finalize(a, base, r0, d0, tot, err, dang);
      a.heavy_counter[t] = 0;
    }
  } else {
    // ---- light tile: rows [r0, r1), edges [eb, eb+E)
    const uint32_t R = r1 - r0;
    const uint32_t E = static_cast<uint32_t>(__ldg(a.voff + r1) - eb);
    uint64_t rend[kPerThread];
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const uint32_t i = threadIdx.x + j * kPrThreads;
      rend[j] = i < R ? __ldg(a.voff + r0 + i + 1) : 0;
    }
    if (G::kContiguous) {
      const uint64_t b0 = g.seg_begin(r0);
      uint32_t ids[kPerThread];
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) {
        const uint32_t k = threadIdx.x + j * kPrThreads;
        ids[j] = k < E ? g.at(b0 + k) : 0u;
      }
      double xv[kPerThread];
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) {
        const uint32_t k = threadIdx.x + j * kPrThreads;
        xv[j] = k < E ? __ldg(a.x_old + ids[j]) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) {
        const uint32_t k = threadIdx.x + j * kPrThreads;
        if (k < E) s_val[k] = fmax(xv[j], 0.0);
      }
    }
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const uint32_t i = threadIdx.x + j * kPrThreads;
      if (i < R) s_rowend[i] = static_cast<uint32_t>(rend[j] - eb);
    }
    __syncthreads();
    if (!G::kContiguous) {
      for (uint32_t k = threadIdx.x; k < E; k += kPrThreads) {
        uint32_t lo = 0, hi = R;  // first row with rowend > k
        while (lo < hi) {
          uint32_t mid = (lo + hi) >> 1;
          if (s_rowend[mid] <= k) lo = mid + 1; else hi = mid;
        }
        const uint32_t rs = lo ? s_rowend[lo - 1] : 0;
        s_val[k] = fmax(a.x_old[g.at(g.seg_begin(r0 + lo) + (k - rs))], 0.0);
      }
    }
    __syncthreads();
    // merge-path share of this thread
    const uint32_t items = R + E;
    const uint32_t ipt = (items + kPrThreads - 1) / kPrThreads;
    const uint32_t dg0 = min(threadIdx.x * ipt, items);
    const uint32_t dg1 = min(dg0 + ipt, items);
    uint32_t xmin = dg0 > E ? dg0 - E : 0, xmax = min(dg0, R);
    while (xmin < xmax) {
      uint32_t pivot = (xmin + xmax) >> 1;
      if (s_rowend[pivot] <= dg0 - pivot - 1) xmin = pivot + 1; else xmax = pivot;
    }
    uint32_t row = xmin, edge = dg0 - xmin;
    double acc = 0.0;
    int64_t first_row = -1;
    double first_val = 0.0;
    for (uint32_t dgi = dg0; dgi < dg1; ++dgi) {
      if (row < R && edge < s_rowend[row]) {
        acc += s_val[edge++];
      } else {
        if (first_row < 0) {
          first_row = row;
          first_val = acc;
        } else {
          const uint32_t deg = s_rowend[row] - (row ? s_rowend[row - 1] : 0);
          pr_finalize(a, base, r0 + row, deg, acc, err, dang);
        }
        acc = 0.0;
        ++row;
      }
    }
    // block-wide reduce-by-key of the carry-outs (keys = open row, monotone)
    KV mine{static_cast<int64_t>(row), acc};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    KV inc = mine;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      KV o{__shfl_up_sync(0xffffffffu, inc.k, dd), __shfl_up_sync(0xffffffffu, inc.v, dd)};
      if (lane >= dd) inc = kv_combine(o, inc);
    }
    KV exw{__shfl_up_sync(0xffffffffu, inc.k, 1), __shfl_up_sync(0xffffffffu, inc.v, 1)};
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
      KV run{-1, 0.0};
      for (int k = 0; k < kPrThreads / 32; ++k) {
        KV agg = s_warp[k];
        s_warp[k] = run;
        run = k == 0 ? agg : kv_combine(run, agg);
      }
    }
    __syncthreads();
    KV pre = s_warp[wid];
    if (lane > 0) pre = wid == 0 ? exw : kv_combine(pre, exw);
    if (first_row >= 0) {
      if (pre.k == first_row) first_val += pre.v;
      const uint32_t fr = static_cast<uint32_t>(first_row);
      const uint32_t deg = s_rowend[fr] - (fr ? s_rowend[fr - 1] : 0);
      pr_finalize(a, base, r0 + fr, deg, first_val, err, dang);
    }
  }
  __syncthreads();  // shared tile buffers are reused by the next work item
  }
  // ---- per-CTA partials, last CTA folds them in order
  const double be = block_sum(err, s_red);
  const double bd = block_sum(dang, s_red);
  if (threadIdx.x == 0) {
    a.blk[2 * blockIdx.x] = be;
    a.blk[2 * blockIdx.x + 1] = bd;
    __threadfence();
    s_flag = atomicAdd(a.done_counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_flag) {
    __threadfence();
    double e = 0.0, dg = 0.0;
    for (uint64_t k = threadIdx.x; k < gridDim.x; k += kPrThreads) {
      e += __ldcg(a.blk + 2 * k);
      dg += __ldcg(a.blk + 2 * k + 1);
    }
    e = block_sum(e, s_red);
    dg = block_sum(dg, s_red);
    if (threadIdx.x == 0) {
      a.sc->dangling[(a.iter + 1) & 1] = dg;
      a.sc->err = e;
      a.sc->iterations = a.iter + 1;
      if (e < a.tol) a.sc->done = 1;
      *a.done_counter = 0;
    }
  }
}

template <class G>
__global__ void pr_init_k(G g, uint64_t n, double* x) {
  const double p0 = 1.0 / static_cast<double>(n);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t d = g.degree(static_cast<uint32_t>(v));
    x[v] = d ? p0 / static_cast<double>(d) : -p0;
  }
}

template <class G>
struct DanglingIn {
  G g;
  double p0;
  __device__ __forceinline__ double operator()(uint64_t v) const {
    return g.degree(static_cast<uint32_t>(v)) ? 0.0 : p0;
  }
};

template <class G>
__global__ void pr_to_p_k(G g, uint64_t n, const double* x, double* p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t d = g.degree(static_cast<uint32_t>(v));
    p[v] = d ? x[v] * static_cast<double>(d) : -x[v];
  }
}

__global__ void pr_scalars_init_k(PrScalars* sc, const double* dangling0) {
  sc->dangling[0] = *dangling0;
  sc->dangling[1] = 0.0;
  sc->err = 0.0;
  sc->done = 0;
  sc->iterations = 0;
}

template <class G>
uint64_t pagerank_run(gbg_graph* g, G view, double damping, uint64_t max_iters, double tol, double* p_dev) {
  const uint64_t n = g->n;
  const uint64_t* voff = g->kind == GBG_KIND_CSR ? g->off : virtual_offsets(g);
  if (!g->pr) g->pr = build_schedule(g, voff);
  PrSchedule* s = g->pr;
  double* X0 = g->ws.get<double>("pr.x0", n);
  double* X1 = g->ws.get<double>("pr.x1", n);
  double* d0 = g->ws.get<double>("pr.d0", 1);
  PrScalars* sc = g->ws.get<PrScalars>("pr.sc", 1);
  const double p0 = 1.0 / static_cast<double>(n);
  GBG_LAUNCH(g, pr_init_k<G>, grid_for(n, 256), 256, 0, view, n, X0);
  device_scan<double>(g, DanglingIn<G>{view, p0}, NullOut{}, n, d0, "pr.dang");
  GBG_LAUNCH(g, pr_scalars_init_k, 1, 1, 0, sc, d0);
  double* X[2] = {X0, X1};
  int per_sm = 1;
  GBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pr_iter_k<G>, kPrThreads, 0));
  const uint64_t grid = std::min<uint64_t>(s->nwork, static_cast<uint64_t>(std::max(per_sm, 1)) * g->sm_count);
  for (uint64_t it = 0; it < max_iters; ++it) {
    PrArgs a{s->tile_row, s->work_tile, s->work_chunk, voff, X[it & 1], X[(it + 1) & 1],
             it + 1 == max_iters ? p_dev : nullptr, s->heavy_partial, s->heavy_counter, s->blk,
             s->done_counter, sc, s->nwork, damping, static_cast<double>(n), tol, static_cast<int>(it)};
    GBG_LAUNCH(g, pr_iter_k<G>, static_cast<unsigned>(grid), kPrThreads, 0, view, a);
  }
  PrScalars hs;
  GBG_CUDA(cudaMemcpyAsync(g->hscalar, sc, sizeof(PrScalars), cudaMemcpyDeviceToHost, g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  std::memcpy(&hs, g->hscalar, sizeof(PrScalars));
  const uint64_t done = static_cast<uint64_t>(hs.iterations);
  if (done < max_iters) {
    // stopped early: p lives in the X buffer written by the last iteration
    GBG_LAUNCH(g, pr_to_p_k<G>, grid_for(n, 256), 256, 0, view, n, X[done & 1], p_dev);
  }
  return done;
}

}  // namespace gbg

void gbg_graph::invalidate_derived() {
  delete pr;
  pr = nullptr;
  voff_valid = false;
}

using namespace gbg;

namespace {
gbg_status pagerank_entry(gbg_graph* g, double damping, uint64_t max_iters, double tol, double* out, bool host,
                          uint64_t* iterations) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!out) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
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
      GBG_CUDA(cudaStreamSynchronize(g->stream));
    } else {
      with_view(g, [&](auto view) { done = pagerank_run(g, view, damping, max_iters, tol, p); });
    }
    if (host) {
      GBG_CUDA(cudaMemcpyAsync(out, p, g->n * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    }
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
}

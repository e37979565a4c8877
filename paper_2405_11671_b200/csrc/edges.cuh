// Balanced all-edges traversal: the "map_neighbors over every vertex"
// loop of the reference (e.g. cc, algorithms.cpp:224-227) with the edge
// list cut into equal tiles instead of per-vertex tasks, so R-MAT hubs
// (max degree 406,360 at scale 24) spread over many CTAs.  The owning row
// of each edge comes from a binary search of the degree prefix (`voff`,
// the CSR offsets or the blocked container's virtual offsets).
#pragma once

#include "scan.cuh"

namespace gbg {

constexpr int kEdgeThreads = 256;
constexpr int kEdgeIPT = 8;
constexpr int kEdgeTile = kEdgeThreads * kEdgeIPT;

__device__ __forceinline__ uint32_t row_of(const uint64_t* voff, uint64_t n, uint64_t e, uint32_t lo) {
  uint64_t hi = n;  // voff[lo] <= e < voff[hi]
  uint64_t l = lo;
  while (hi - l > 1) {
    uint64_t mid = (l + hi) >> 1;
    if (voff[mid] <= e) l = mid; else hi = mid;
  }
  return static_cast<uint32_t>(l);
}

// op(u, v, e): arc u -> v, e = its index in voff order
template <class G, class Op>
__global__ void __launch_bounds__(kEdgeThreads) for_each_edge_k(G g, const uint64_t* __restrict__ voff, uint64_t m,
                                                                 Op op, uint64_t base) {
  __shared__ uint32_t s_row[kEdgeTile];
  const uint64_t e0 = base + static_cast<uint64_t>(blockIdx.x) * kEdgeTile;
  if (e0 >= m) return;
  const uint32_t len = static_cast<uint32_t>(m - e0 < kEdgeTile ? m - e0 : kEdgeTile);
  {
    const uint32_t k0 = threadIdx.x * kEdgeIPT;
    if (k0 < len) {
      uint32_t r = row_of(voff, g.n, e0 + k0, 0);
      uint64_t next = voff[r + 1];
#pragma unroll
      for (int j = 0; j < kEdgeIPT; ++j) {
        if (k0 + j >= len) break;
        if (next <= e0 + k0 + j) {
          r = row_of(voff, g.n, e0 + k0 + j, r + 1);
          next = voff[r + 1];
        }
        s_row[k0 + j] = r;
      }
    }
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < len; k += kEdgeThreads) {
    const uint32_t u = s_row[k];
    const uint64_t e = e0 + k;
    uint32_t v;
    if (G::kContiguous) {
      v = g.at(e);
    } else {
      v = g.at(g.seg_begin(u) + (e - voff[u]));
    }
    op(u, v, e);
  }
}

// Segmented expansion: op(seg, rank, flat) for every flat index in
// [0, total), where `scan` is the exclusive prefix of the segment sizes
// (scan[nseg] = total) and seg is the segment holding flat.  Same tiling as
// for_each_edge: one search per thread, then a walk; empty segments are
// skipped by re-searching.
template <class T>
__device__ __forceinline__ uint32_t seg_of(const T* scan, uint32_t nseg, uint64_t e, uint32_t lo) {
  uint32_t hi = nseg;  // scan[lo] <= e < scan[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (static_cast<uint64_t>(scan[mid]) <= e) lo = mid; else hi = mid;
  }
  return lo;
}

// The same search by a whole warp (warp-uniform e): 32 probes per round
// narrow [lo, hi) 32-fold, so ~log32(nseg) dependent loads instead of
// log2(nseg) (a 34K-segment copy: 3 rounds instead of 15).
template <class T>
__device__ __forceinline__ uint32_t warp_seg_of(const T* scan, uint32_t nseg, uint64_t e) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = nseg;  // scan[lo] <= e < scan[hi]
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t idx = lo + lane * step;
    const bool le = idx < hi && static_cast<uint64_t>(scan[idx]) <= e;
    const uint32_t mask = __ballot_sync(0xffffffffu, le);  // lane 0 always set
    const uint32_t last = 31 - __clz(mask);
    const uint32_t nlo = lo + last * step;
    hi = nlo + step < hi ? nlo + step : hi;
    lo = nlo;
  }
  return lo;
}

template <class T, class Op>
__global__ void __launch_bounds__(kEdgeThreads) expand_k(const T* __restrict__ scan, uint32_t nseg, uint64_t total,
                                                          Op op) {
  __shared__ uint32_t s_seg[kEdgeTile];
  const uint64_t e0 = static_cast<uint64_t>(blockIdx.x) * kEdgeTile;
  if (e0 >= total) return;
  const uint32_t len = static_cast<uint32_t>(total - e0 < kEdgeTile ? total - e0 : kEdgeTile);
  {
    const uint32_t k0 = threadIdx.x * kEdgeIPT;
    if (k0 < len) {
      uint32_t s = seg_of(scan, nseg, e0 + k0, 0);
      uint64_t next = scan[s + 1];
#pragma unroll
      for (int j = 0; j < kEdgeIPT; ++j) {
        if (k0 + j >= len) break;
        if (next <= e0 + k0 + j) {
          // short segments: step a few segments before searching the rest
          const uint64_t e = e0 + k0 + j;
          ++s;
          next = scan[s + 1];
#pragma unroll 1
          for (int p = 0; p < 3 && next <= e; ++p) next = scan[++s + 1];
          if (next <= e) {
            s = seg_of(scan, nseg, e, s + 1);
            next = scan[s + 1];
          }
        }
        s_seg[k0 + j] = s;
      }
    }
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < len; k += kEdgeThreads) {
    const uint32_t s = s_seg[k];
    const uint64_t e = e0 + k;
    op(s, static_cast<uint32_t>(e - scan[s]), e);
  }
}

template <class T, class Op>
void expand(gbg_graph* g, const T* scan, uint32_t nseg, uint64_t total, Op op) {
  if (total == 0 || nseg == 0) return;
  const uint64_t tiles = (total + kEdgeTile - 1) / kEdgeTile;
  GBG_LAUNCH(g, (expand_k<T, Op>), static_cast<unsigned>(tiles), kEdgeThreads, 0, scan, nseg, total, op);
}

// Segmented copy: for every flat index e in [0, total) of segment q (scan
// as in expand), dst_q[e - scan[q]] = src_q[e - scan[q]], with the
// segment's base pointers from op.bases(q, src, dst).  A warp copies 512
// consecutive flat elements, lanes strided (coalesced); when they lie in
// one segment (long lists) the base pointers are looked up once and all 16
// loads of a lane are in flight before the stores; otherwise each lane
// walks the segments forward.  (Element-wise expand costs a shared-memory
// segment index and the pointer loads per element: the 10^7-edge insert's
// staging copy 0.63 -> 0.45 ms.)
constexpr int kCopyIPT = 16;
constexpr uint32_t kCopyWarpItems = 32 * kCopyIPT;
#ifndef GBG_COPY_MINB
#define GBG_COPY_MINB 5
#endif
#ifndef GBG_COPY_WIN
#define GBG_COPY_WIN 4
#endif
constexpr int kCopyWin = GBG_COPY_WIN;  // multi-segment chunks: elements per lane in flight

template <class T, class Op>
__global__ void __launch_bounds__(256, GBG_COPY_MINB) copy_expand_k(const T* __restrict__ scan, uint32_t nseg, uint64_t total,
                                                      Op op) {
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = gw * kCopyWarpItems;
  if (w0 >= total) return;
  const uint64_t wend = w0 + kCopyWarpItems < total ? w0 + kCopyWarpItems : total;
  uint32_t q = warp_seg_of(scan, nseg, w0);
  uint64_t qs = static_cast<uint64_t>(scan[q]), qe = static_cast<uint64_t>(scan[q + 1]);
  const uint32_t* src;
  uint32_t* dst;
  op.bases(q, src, dst);
  if (qe >= wend) {
    uint32_t v[kCopyIPT];
#pragma unroll
    for (int j = 0; j < kCopyIPT; ++j) {
      const uint64_t e = w0 + lane + 32u * j;
      v[j] = e < wend ? src[e - qs] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kCopyIPT; ++j) {
      const uint64_t e = w0 + lane + 32u * j;
      if (e < wend) dst[e - qs] = v[j];
    }
    return;
  }
  // several segments (short lists): windows of 32 segments, lane i holding
  // segment qa + i's flat start and base pointers (one parallel load round);
  // each element finds its segment by a 5-step shuffle search over the
  // window (a lane walking the segments one by one paid a dependent chain
  // of scan + pointer loads per segment)
  for (uint32_t qa = q;; qa += 32) {
    const uint32_t qi = qa + lane;
    uint64_t si = total;
    const uint32_t* srci = nullptr;
    uint32_t* dsti = nullptr;
    if (qi < nseg) {
      si = static_cast<uint64_t>(scan[qi]);
      op.bases(qi, srci, dsti);
    }
    const uint64_t wlo = __shfl_sync(0xffffffffu, si, 0);
    const uint64_t whi = qa + 32 < nseg ? static_cast<uint64_t>(scan[qa + 32]) : total;  // warp-uniform
    for (int h = 0; h < kCopyIPT; h += kCopyWin) {  // kCopyWin elements at a time (registers)
      uint32_t v[kCopyWin];
      uint32_t kk[kCopyWin];
#pragma unroll
      for (int j = 0; j < kCopyWin; ++j) {
        const uint64_t e = w0 + lane + 32u * (h + j);
        const bool in = e < wend && e >= wlo && e < whi;
        uint32_t k = 0;
#pragma unroll
        for (uint32_t st = 16; st; st >>= 1) {
          const uint64_t sk = __shfl_sync(0xffffffffu, si, k + st);
          if (sk <= e) k += st;
        }
        const uint64_t sk = __shfl_sync(0xffffffffu, si, k);
        const uint32_t* sp = reinterpret_cast<const uint32_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(srci), k));
        kk[j] = k;
        v[j] = in ? sp[e - sk] : 0u;
      }
#pragma unroll
      for (int j = 0; j < kCopyWin; ++j) {
        const uint64_t e = w0 + lane + 32u * (h + j);
        const bool in = e < wend && e >= wlo && e < whi;
        const uint64_t sk = __shfl_sync(0xffffffffu, si, kk[j]);
        uint32_t* dp = reinterpret_cast<uint32_t*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dsti), kk[j]));
        if (in) dp[e - sk] = v[j];
      }
    }
    if (whi >= wend) break;
  }
}

template <class T, class Op>
void copy_expand(gbg_graph* g, const T* scan, uint32_t nseg, uint64_t total, Op op) {
  if (total == 0 || nseg == 0) return;
  const uint64_t warps = (total + kCopyWarpItems - 1) / kCopyWarpItems;
  GBG_LAUNCH(g, (copy_expand_k<T, Op>), static_cast<unsigned>((warps + 7) / 8), 256, 0, scan, nseg, total, op);
}

template <class G, class Op>
void for_each_edge(gbg_graph* g, G view, const uint64_t* voff, uint64_t m, Op op) {
  if (m == 0) return;
  const uint64_t tiles = (m + kEdgeTile - 1) / kEdgeTile;
  GBG_LAUNCH(g, (for_each_edge_k<G, Op>), static_cast<unsigned>(tiles), kEdgeThreads, 0, view, voff, m, op,
             uint64_t{0});
}

// the edges [e0, e1) only (same op(u, v, e) contract, e absolute)
template <class G, class Op>
void for_each_edge_range(gbg_graph* g, G view, const uint64_t* voff, uint64_t e0, uint64_t e1, Op op) {
  if (e1 <= e0) return;
  const uint64_t tiles = (e1 - e0 + kEdgeTile - 1) / kEdgeTile;
  GBG_LAUNCH(g, (for_each_edge_k<G, Op>), static_cast<unsigned>(tiles), kEdgeThreads, 0, view, voff, e1, op, e0);
}

// counts[u] += |{v in N(u) : pred(u, v)}| over the same balanced tiles.  A
// warp's 32 consecutive edges cover a run of rows, so each row's hits are
// summed with one match/ballot and added by one lane: a hub's tile costs a
// handful of atomics instead of one per edge.
template <class G, class Pred>
__global__ void __launch_bounds__(kEdgeThreads) row_count_k(G g, const uint64_t* __restrict__ voff, uint64_t m,
                                                             Pred pred, uint32_t* counts) {
  __shared__ uint32_t s_row[kEdgeTile];
  const uint64_t e0 = static_cast<uint64_t>(blockIdx.x) * kEdgeTile;
  if (e0 >= m) return;
  const uint32_t len = static_cast<uint32_t>(m - e0 < kEdgeTile ? m - e0 : kEdgeTile);
  {
    const uint32_t k0 = threadIdx.x * kEdgeIPT;
    if (k0 < len) {
      uint32_t r = row_of(voff, g.n, e0 + k0, 0);
      uint64_t next = voff[r + 1];
#pragma unroll
      for (int j = 0; j < kEdgeIPT; ++j) {
        if (k0 + j >= len) break;
        if (next <= e0 + k0 + j) {
          r = row_of(voff, g.n, e0 + k0 + j, r + 1);
          next = voff[r + 1];
        }
        s_row[k0 + j] = r;
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (uint32_t b = 0; b < len; b += kEdgeThreads) {  // warp-uniform trip count
    const uint32_t k = b + threadIdx.x;
    const bool valid = k < len;
    uint32_t u = 0xffffffffu;
    bool hit = false;
    if (valid) {
      u = s_row[k];
      const uint64_t e = e0 + k;
      const uint32_t v = G::kContiguous ? g.at(e) : g.at(g.seg_begin(u) + (e - voff[u]));
      hit = pred(u, v);
    }
    const uint32_t grp = __match_any_sync(0xffffffffu, u);
    const uint32_t hits = __ballot_sync(0xffffffffu, hit) & grp;
    if (valid && hits && lane == __ffs(grp) - 1) atomicAdd(counts + u, static_cast<uint32_t>(__popc(hits)));
  }
}

// Filtered adjacency: for every arc (u, v) with pred(u, v), out[ooff[u] + k]
// = v, k taken from cursor[u] (zeroed by the caller; ooff is the exclusive
// scan of row_count's counts).  Same warp grouping as row_count: one atomic
// per row run, positions by prefix popcount.  Order within a row is
// unspecified.
template <class G, class Pred>
__global__ void __launch_bounds__(kEdgeThreads) row_compact_k(G g, const uint64_t* __restrict__ voff, uint64_t m,
                                                               Pred pred, const uint64_t* __restrict__ ooff,
                                                               uint32_t* cursor, uint32_t* out) {
  __shared__ uint32_t s_row[kEdgeTile];
  const uint64_t e0 = static_cast<uint64_t>(blockIdx.x) * kEdgeTile;
  if (e0 >= m) return;
  const uint32_t len = static_cast<uint32_t>(m - e0 < kEdgeTile ? m - e0 : kEdgeTile);
  {
    const uint32_t k0 = threadIdx.x * kEdgeIPT;
    if (k0 < len) {
      uint32_t r = row_of(voff, g.n, e0 + k0, 0);
      uint64_t next = voff[r + 1];
#pragma unroll
      for (int j = 0; j < kEdgeIPT; ++j) {
        if (k0 + j >= len) break;
        if (next <= e0 + k0 + j) {
          r = row_of(voff, g.n, e0 + k0 + j, r + 1);
          next = voff[r + 1];
        }
        s_row[k0 + j] = r;
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (uint32_t b = 0; b < len; b += kEdgeThreads) {
    const uint32_t k = b + threadIdx.x;
    const bool valid = k < len;
    uint32_t u = 0xffffffffu, v = 0;
    bool hit = false;
    if (valid) {
      u = s_row[k];
      const uint64_t e = e0 + k;
      v = G::kContiguous ? g.at(e) : g.at(g.seg_begin(u) + (e - voff[u]));
      hit = pred(u, v);
    }
    const uint32_t grp = __match_any_sync(0xffffffffu, u);
    const uint32_t hits = __ballot_sync(0xffffffffu, hit) & grp;
    const int leader = __ffs(grp) - 1;
    uint32_t base = 0;
    if (valid && hits && lane == leader) base = atomicAdd(cursor + u, static_cast<uint32_t>(__popc(hits)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) out[ooff[u] + base + __popc(hits & ((1u << lane) - 1))] = v;
  }
}

template <class G, class Pred>
void row_compact(gbg_graph* g, G view, const uint64_t* voff, uint64_t m, Pred pred, const uint64_t* ooff,
                 uint32_t* cursor, uint32_t* out) {
  if (m == 0) return;
  const uint64_t tiles = (m + kEdgeTile - 1) / kEdgeTile;
  GBG_LAUNCH(g, (row_compact_k<G, Pred>), static_cast<unsigned>(tiles), kEdgeThreads, 0, view, voff, m, pred, ooff,
             cursor, out);
}

template <class G, class Pred>
void row_count(gbg_graph* g, G view, const uint64_t* voff, uint64_t m, Pred pred, uint32_t* counts) {
  if (m == 0) return;
  const uint64_t tiles = (m + kEdgeTile - 1) / kEdgeTile;
  GBG_LAUNCH(g, (row_count_k<G, Pred>), static_cast<unsigned>(tiles), kEdgeThreads, 0, view, voff, m, pred, counts);
}

}  // namespace gbg

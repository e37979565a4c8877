// Triangle counting over the degree-oriented adjacency.
//
// Not in the reference (PAPER.md:945-969 describes it in
// prose).  Built from the reference's pieces: derive_filter
// (derive.hpp:48-61) with predicate (deg u, u) < (deg v, v) produces a
// sorted oriented CSR (the filter keeps each list's order), and each
// triangle {a,b,c} is then counted exactly once as |N+(u) ∩ N+(v)| over the
// oriented arcs u -> v.  oracle/gbo.c:gbo_tc is the CPU restatement this is
// checked against.
//
//  1. flag every arc (edge-parallel), exclusive-scan the flags in CSR order
//     -> each kept arc's slot in the oriented arrays (stream compaction),
//  2. oriented offsets from the (sorted) oriented sources,
//  3. per oriented arc, intersect the two out-lists: every element of the
//     shorter list is binary-searched in the longer one; counts reduced per
//     CTA then one 64-bit atomic per CTA.
#include "edges.cuh"

namespace gbg {

__device__ __forceinline__ bool rank_less(uint32_t du, uint32_t u, uint32_t dv, uint32_t v) {
  return du < dv || (du == dv && u < v);
}

template <class G>
struct SrcOp {
  uint32_t* src;
  __device__ __forceinline__ void operator()(uint32_t u, uint32_t, uint64_t e) const { src[e] = u; }
};

struct OrientIn {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* src;
  __device__ __forceinline__ uint32_t operator()(uint64_t e) const {
    const uint32_t u = src[e], v = nbr[e];
    const uint32_t du = static_cast<uint32_t>(off[u + 1] - off[u]);
    const uint32_t dv = static_cast<uint32_t>(off[v + 1] - off[v]);
    return rank_less(du, u, dv, v);
  }
};
struct OrientOut {
  OrientIn in;
  uint32_t* osrc;
  uint32_t* onbr;
  __device__ __forceinline__ void operator()(uint64_t e, uint64_t pre) const {
    if (in(e)) {
      osrc[pre] = in.src[e];
      onbr[pre] = in.nbr[e];
    }
  }
};

__global__ void offsets_from_sorted64_k(const uint32_t* src, uint64_t m, uint64_t n, uint64_t* off) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= m; i += stride) {
    uint64_t lo = i == 0 ? 0 : (uint64_t)src[i - 1] + 1;
    uint64_t hi = i == m ? n : (uint64_t)src[i];
    for (uint64_t x = lo; x <= hi; ++x) off[x] = i;
  }
}

// first index i in [lo, len) with a[i] >= x: exponential probes from lo,
// then a binary search inside the bracket.  The elements of the shorter list
// are searched in increasing order, so each search starts where the last
// one ended and costs O(log gap) instead of O(log len).
__device__ __forceinline__ uint32_t gallop_lb(const uint32_t* a, uint32_t lo, uint32_t len, uint32_t x) {
  uint32_t r, step = 1;
  for (;;) {
    const uint32_t p = lo + step - 1;
    if (p >= len) {
      r = len;
      break;
    }
    if (__ldg(a + p) >= x) {
      r = p;
      break;
    }
    lo = p + 1;
    step <<= 1;
  }
  while (lo < r) {
    const uint32_t mid = (lo + r) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else r = mid;
  }
  return lo;
}

// |{a[i] : i = first, first + stride, ...} ∩ b| for ascending a and b
__device__ __forceinline__ uint32_t count_common(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb,
                                                 uint32_t first, uint32_t stride) {
  if (!lb) return 0;
  const uint32_t bmax = __ldg(b + lb - 1);
  uint32_t c = 0, pos = 0;
  for (uint32_t i = first; i < la; i += stride) {
    const uint32_t x = __ldg(a + i);
    if (x > bmax) break;
    pos = gallop_lb(b, pos, lb, x);
    if (pos < lb && __ldg(b + pos) == x) {
      ++c;
      ++pos;
    }
  }
  return c;
}

#ifndef GBG_TC_LANE_MAX
#define GBG_TC_LANE_MAX 128  // s20: 18.2 ms at 32, 17.1 at 128 (8-64 within 1%; s24 unchanged)
#endif
// arcs whose shorter list has more entries than this go to the whole warp
constexpr uint32_t kTcLaneMax = GBG_TC_LANE_MAX;

__global__ void __launch_bounds__(256) tc_count_k(uint64_t mo, const uint64_t* __restrict__ ooff,
                                                  const uint32_t* __restrict__ osrc, const uint32_t* __restrict__ onbr,
                                                  unsigned long long* total) {
  __shared__ unsigned long long s_red[33];
  unsigned long long cnt = 0;
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // one arc per lane; arcs whose shorter list exceeds kTcLaneMax entries are then
  // intersected by the whole warp (32 binary searches at a time)
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < mo; base += stride) {
    const uint64_t e = base + threadIdx.x;
    const uint32_t* a = onbr;
    const uint32_t* b = onbr;
    uint32_t la = 0, lb = 0;
    if (e < mo) {
      const uint32_t u = osrc[e], v = onbr[e];
      const uint64_t ub = ooff[u], vb = ooff[v];
      const uint32_t du = static_cast<uint32_t>(ooff[u + 1] - ub), dv = static_cast<uint32_t>(ooff[v + 1] - vb);
      a = onbr + (du <= dv ? ub : vb);
      b = onbr + (du <= dv ? vb : ub);
      la = du <= dv ? du : dv;
      lb = du <= dv ? dv : du;
    }
    if (la <= kTcLaneMax) cnt += count_common(a, la, b, lb, 0, 1);
    uint32_t hard = __ballot_sync(0xffffffffu, la > kTcLaneMax);
    while (hard) {
      const int l = __ffs(hard) - 1;
      hard &= hard - 1;
      const uint32_t* aa = reinterpret_cast<const uint32_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(a), l));
      const uint32_t* bb = reinterpret_cast<const uint32_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(b), l));
      const uint32_t na = __shfl_sync(0xffffffffu, la, l), nb = __shfl_sync(0xffffffffu, lb, l);
      cnt += count_common(aa, na, bb, nb, lane, 32);
    }
  }
  cnt = block_sum(cnt, s_red);
  if (threadIdx.x == 0 && cnt) atomicAdd(total, cnt);
}

uint64_t tc_run(gbg_graph* g) {
  const uint64_t n = g->n, m = g->m;
  if (m == 0) return 0;
  // a packed CSR view (the blocked container is gathered into one first)
  const CsrView csr = g->kind == GBG_KIND_COMPRESSED ? compressed_decoded(g) : g->csr_view();
  const uint64_t* off = csr.off;
  const uint32_t* nbr = csr.nbr;
  uint32_t* src = g->ws.get<uint32_t>("tc.src", m);
  if (g->kind == GBG_KIND_BLOCKED) {
    const uint64_t* voff = virtual_offsets(g);
    uint32_t* packed = g->ws.get<uint32_t>("tc.packed", m);
    BlockedView bv = g->blocked_view();
    for_each_edge(g, bv, voff, m, [=] __device__(uint32_t u, uint32_t v, uint64_t e) {
      packed[e] = v;
      src[e] = u;
    });
    off = voff;
    nbr = packed;
  } else {
    for_each_edge(g, csr, off, m, SrcOp<CsrView>{src});
  }
  uint32_t* osrc = g->ws.get<uint32_t>("tc.osrc", m);
  uint32_t* onbr = g->ws.get<uint32_t>("tc.onbr", m);
  uint64_t* ooff = g->ws.get<uint64_t>("tc.ooff", n + 1);
  uint64_t* cnt = g->ws.get<uint64_t>("tc.cnt", 2);
  OrientIn oin{off, nbr, src};
  device_scan<uint64_t>(g, oin, OrientOut{oin, osrc, onbr}, m, cnt, "tc.orient");
  uint64_t mo = 0;
  read_scalars(g, cnt, sizeof(mo), &mo);
  GBG_LAUNCH(g, offsets_from_sorted64_k, grid_for(mo + 1, 256), 256, 0, osrc, mo, n, ooff);
  unsigned long long* total = reinterpret_cast<unsigned long long*>(cnt + 1);
  GBG_CUDA(cudaMemsetAsync(total, 0, sizeof(unsigned long long), g->stream));
  if (mo)
    GBG_LAUNCH(g, tc_count_k, grid_for(mo, 256, g->sm_count * 8), 256, 0, mo, ooff, osrc, onbr, total);
  uint64_t t = 0;
  read_scalars(g, total, sizeof(t), &t);
  g->ws.release("tc.src");
  g->ws.release("tc.osrc");
  g->ws.release("tc.onbr");
  g->ws.release("tc.packed");
  return t;
}

}  // namespace gbg

using namespace gbg;

extern "C" gbg_status gbg_tc(gbg_graph* g, uint64_t* triangles) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!triangles) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    *triangles = tc_run(g);
  });
}

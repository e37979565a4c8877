// The dynamic blocked sorted-adjacency container and its batch update path.
//
// Reference: SetGraph<ChunkedSortedSet> with inline_k = 0 ("chunked_set",
// registry.cpp:136-137; set_graph.hpp:26-249; neighbor_sets.hpp:259-442)
// fed by prepare(GlobalSort) + apply_insert / apply_delete (batch.cpp:30-126).
//
// Layout (device): vertex v owns one allocation of cap[v] uint32 ids at
// pool[start[v]]; its deg[v] live neighbours are the ascending prefix.
// Capacities come in 16-byte blocks: power-of-two classes of 4..128 ids,
// then multiples of 128 ids (512 B) with 1/8 slack — the GPU analogue of
// ChunkedSortedSet's 128-id chunks refilled at half capacity
// (neighbor_sets.hpp:427-438), but contiguous per vertex so every traversal
// kernel reads a vertex's list with coalesced loads.  Allocations come from
// a bump pointer; when the pool runs out the live lists are compacted into a
// fresh, larger pool.
//
// Batch path (all on the device, starting from raw arcs):
//   1. key = src<<L | dst, self-loops -> sentinel; range check
//   2. radix sort (2L bits)                      prepare: sort   (batch.cpp:38)
//   3. unique, drop self-loops                   prepare: unique (batch.cpp:37-39)
//   4. per arc: binary search in src's list -> present?  keep the arcs that
//      change the container (new for insert, present for delete): the
//      applied count of insert_batch / delete_batch (neighbor_sets.hpp:339-366)
//   5. group by source; allocate grown lists (scan + bump)
//   6. stage touched lists, then merge (insert) / set-difference (delete)
//      element-parallel: each element's output slot = its rank in its own
//      list plus its rank in the other (binary search)
//   7. deg / start / cap / m updated (MetadataTracker::add_degree/add_total,
//      metadata.hpp:38-50)
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "edges.cuh"
#include "keys.cuh"
#include "rng.cuh"

namespace gbg {

__host__ __device__ __forceinline__ uint32_t cap_for(uint32_t d) {
  if (d == 0) return 0;
  if (d <= 128) {
    uint32_t c = 4;
    while (c < d) c <<= 1;
    return c;
  }
  uint64_t want = static_cast<uint64_t>(d) + d / 8;
  return static_cast<uint32_t>((want + 127) / 128 * 128);
}

// ---------------------------------------------------------------- build
struct CsrDegIn {
  const uint64_t* off;
  __device__ __forceinline__ uint64_t operator()(uint64_t v) const { return off[v + 1] - off[v]; }
};
struct CapIn {
  const uint32_t* deg;
  __device__ __forceinline__ uint64_t operator()(uint64_t v) const { return cap_for(deg[v]); }
};

__global__ void deg_cap_from_csr_k(uint64_t n, const uint64_t* off, uint32_t* deg, uint32_t* cap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t d = static_cast<uint32_t>(off[v + 1] - off[v]);
    deg[v] = d;
    cap[v] = cap_for(d);
  }
}

// warp per vertex copy of live lists between two layouts
__global__ void copy_lists_k(uint64_t n, const uint64_t* src_start, const uint32_t* src, const uint32_t* deg,
                             const uint64_t* dst_start, uint32_t* dst) {
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t v = w0; v < n; v += nw) {
    const uint32_t d = deg[v];
    const uint32_t* s = src + src_start[v];
    uint32_t* t = dst + dst_start[v];
    for (uint32_t j = lane; j < d; j += 32) t[j] = s[j];
  }
}

// Lay the live lists out afresh, each vertex at cap[v] ids (caps set by the
// caller), in a pool with room for `extra` more ids plus 50% slack.  Used at
// build (source = a packed CSR) and when the bump pool runs out (source =
// the current pool, which is then freed).
void blocked_relayout(gbg_graph* g, const uint64_t* src_start, const uint32_t* src_pool, uint64_t extra,
                      bool own_src) {
  const uint64_t n = g->n;
  uint64_t* nstart = dalloc<uint64_t>(n + 1);
  device_scan<uint64_t>(g, CapIn{g->bcap}, ArrayOut<uint64_t>{nstart}, n, nstart + n, "blk.relayout");
  uint64_t live = 0;
  read_scalars(g, nstart + n, sizeof(live), &live);
  uint64_t cap = live + extra + live / 2 + (uint64_t{1} << 20);
  cap = (cap + 3) / 4 * 4;
  uint32_t* npool = dalloc<uint32_t>(cap);
  if (n)
    GBG_LAUNCH(g, copy_lists_k, grid_for(n * 32, 256, g->sm_count * 64), 256, 0, n, src_start, src_pool, g->bdeg,
               nstart, npool);
  GBG_CUDA(cudaStreamSynchronize(g->stream));
  if (own_src) {
    dfree(g->bstart);
    dfree(g->pool);
  }
  g->bstart = nstart;
  g->pool = npool;
  g->pool_cap = cap;
  g->pool_top = live;
  g->pool_live = live;
}

void blocked_from_device_csr(gbg_graph* g, uint64_t n, const uint64_t* off, const uint32_t* nbr) {
  g->bdeg = dalloc<uint32_t>(n + 1);
  g->bcap = dalloc<uint32_t>(n + 1);
  if (n) GBG_LAUNCH(g, deg_cap_from_csr_k, grid_for(n, 256), 256, 0, n, off, g->bdeg, g->bcap);
  // the CSR offsets double as the source "start" array of a packed layout
  blocked_relayout(g, off, nbr, 0, false);
}

struct DegIn {
  const uint32_t* deg;
  __device__ __forceinline__ uint64_t operator()(uint64_t v) const { return deg[v]; }
};

const uint64_t* virtual_offsets(gbg_graph* g) {
  if (g->kind == GBG_KIND_CSR) return g->off;
  if (g->kind == GBG_KIND_COMPRESSED) return compressed_decoded(g).off;
  if (!g->voff) g->voff = dalloc<uint64_t>(g->n + 1);
  if (!g->voff_valid) {
    device_scan<uint64_t>(g, DegIn{g->bdeg}, ArrayOut<uint64_t>{g->voff}, g->n, g->voff + g->n, "blk.voff");
    g->voff_valid = true;
  }
  return g->voff;
}

// ---------------------------------------------------------------- updates
__global__ void make_keys_k(const uint32_t* pairs, uint64_t count, uint64_t n, BatchKeys bk, uint64_t* keys,
                            int* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint32_t s = pairs[2 * i], d = pairs[2 * i + 1];
    // prepare(GlobalSort) drops self-loops before anything looks at the ids
    // (batch.cpp:34-42), so only a non-loop arc can be out of range
    const bool oor = s != d && (s >= n || d >= n);
    if (oor) *bad = 1;
    // self-loops (and out-of-range arcs, which fail the call before any
    // change) become the all-ones key, itself a self-loop, dropped below
    keys[i] = s == d || oor ? bk.loop_key() : bk.make(s, d);
  }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t len, uint32_t x) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// arc membership queries: out[i] = (src,dst) present (0 for out-of-range ids)
template <class G>
__global__ void contains_k(G g, const uint32_t* pairs, uint64_t count, uint8_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint32_t s = pairs[2 * i], d = pairs[2 * i + 1];
    uint8_t r = 0;
    if (s < g.n && d < g.n) {
      uint64_t b;
      uint32_t len;
      g.seg(s, b, len);
      const uint32_t pos = lower_bound_u32(g.data() + b, len, d);
      r = pos < len && g.at(b + pos) == d;
    }
    out[i] = r;
  }
}

// presence of each prepared arc in the container (flag = changes the
// container: absent for insert, present for delete) and its rank among the
// source's current neighbours (the merge slot offset of an inserted arc)
//
// With check_sym (the container is symmetric before the batch) it also
// checks that the batch is closed under reversal: the unique (s, d) with
// s < d and the reversed unique (d, s) with s > d are the same set (equal
// counts and equal keyed hash sums).  A symmetric batch applied to a symmetric container leaves it
// symmetric (an arc is absent/present iff its reverse is), so BFS keeps
// the cached zero-degree pre-mark after R-MAT batches (bfs_premark).
// first index >= from whose element is >= x (the elements before `from`
// are < x): exponential steps from `from`, then a binary search
__device__ __forceinline__ uint32_t gallop_lb(const uint32_t* lst, uint32_t len, uint32_t x, uint32_t from) {
  uint32_t lo = from, hi = from, step = 1;
  while (hi < len && lst[hi] < x) {
    lo = hi + 1;
    hi = lo + step;
    step <<= 1;
  }
  if (hi > len) hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (lst[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Each thread takes kFlagArcs consecutive unique arcs: the first one's slot
// by binary search in its source's list, the next ones (same source,
// larger targets) by galloping on from the previous slot.  The symmetry
// check compares two keyed 64-bit hash sums: over the s < d arcs of H(s, d)
// and over the s > d arcs of H(d, s) (equal sets of unique keys give equal
// sums; unequal ones collide with probability ~2^-128), plus the counts.
__device__ __forceinline__ uint64_t sym_hash(uint64_t key, uint64_t salt) { return mix64(key * 0x9e3779b97f4a7c15ull + salt); }
// kFlagArcs = 1 for small batches, where the chain of searches of one
// thread would be the critical path
// The sorted raw keys go in directly: a duplicate of the previous key or a
// self-loop (the dropped-key sentinel included) is not applied -- the
// unique step of prepare (batch.cpp:34-42) folded into this pass, one
// scan less; U counts the unique arcs.
template <int kFlagArcs>
__global__ void apply_flags_k(const uint64_t* k, uint64_t count, unsigned long long* U_dev, BatchKeys bk,
                              const uint64_t* start, const uint32_t* deg, const uint32_t* pool, int insert,
                              uint32_t* flag, uint32_t* lb, int check_sym, unsigned long long* hsum, uint64_t* lt,
                              uint64_t* gt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * kFlagArcs;
  uint32_t nlt = 0, ngt = 0, nu = 0;
  unsigned long long h1 = 0, h2 = 0;
  for (uint64_t i0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * kFlagArcs; i0 < count; i0 += stride) {
    uint32_t ps = ~0u, ppos = 0;
#pragma unroll
    for (int j = 0; j < kFlagArcs; ++j) {
      const uint64_t i = i0 + j;
      if (i >= count) break;
      const uint64_t x = k[i];
      const uint32_t s = bk.src(x), d = bk.dst(x);
      if ((i > 0 && k[i - 1] == x) || s == d) {
        flag[i] = 0;
        continue;
      }
      ++nu;
      const uint32_t* lst = pool + start[s];
      const uint32_t len = deg[s];
      const uint32_t pos = s == ps ? gallop_lb(lst, len, d, ppos) : lower_bound_u32(lst, len, d);
      ps = s;
      ppos = pos;
      const bool present = pos < len && lst[pos] == d;
      flag[i] = insert ? !present : present;
      lb[i] = pos;
      if (check_sym) {
        if (s < d) {
          ++nlt;
          h1 += sym_hash(x, 0x243f6a8885a308d3ull);
          h2 += sym_hash(x, 0x13198a2e03707344ull);
        } else {
          ++ngt;
          const uint64_t y = bk.make(d, s);
          h1 -= sym_hash(y, 0x243f6a8885a308d3ull);
          h2 -= sym_hash(y, 0x13198a2e03707344ull);
        }
      }
    }
  }
  nu = __reduce_add_sync(0xffffffffu, nu);
  if ((threadIdx.x & 31) == 0 && nu) atomicAdd(U_dev, static_cast<unsigned long long>(nu));
  if (check_sym) {
    nlt = __reduce_add_sync(0xffffffffu, nlt);
    ngt = __reduce_add_sync(0xffffffffu, ngt);
    h1 = warp_sum(h1);
    h2 = warp_sum(h2);
    if ((threadIdx.x & 31) == 0) {
      if (nlt) atomicAdd(reinterpret_cast<unsigned long long*>(lt), nlt);
      if (ngt) atomicAdd(reinterpret_cast<unsigned long long*>(gt), ngt);
      if (h1) atomicAdd(hsum, h1);
      if (h2) atomicAdd(hsum + 1, h2);
    }
  }
}
struct ApplyOut {
  const uint32_t* flag;
  const uint64_t* k;
  const uint32_t* lb;
  uint64_t* out;
  uint32_t* out_lb;
  __device__ __forceinline__ void operator()(uint64_t i, uint32_t pre) const {
    if (flag[i]) {
      out[pre] = k[i];
      out_lb[pre] = lb[i];
    }
  }
};

// group heads over the applied arcs
struct HeadIn {
  const uint64_t* k;
  BatchKeys bk;
  const uint32_t* A;  // applied arcs (device count)
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    return i < *A && (i == 0 || bk.src(k[i - 1]) != bk.src(k[i]));
  }
};
struct HeadOut {
  const uint64_t* k;
  BatchKeys bk;
  const uint32_t* A;
  uint32_t* gstart;  // first applied arc of group
  uint32_t* gsrc;
  uint32_t* agrp;    // group of each applied arc
  __device__ __forceinline__ void operator()(uint64_t i, uint32_t pre) const {
    if (i >= *A) return;
    const bool head = HeadIn{k, bk, A}(i);
    if (head) {
      gstart[pre] = static_cast<uint32_t>(i);
      gsrc[pre] = bk.src(k[i]);
    }
    agrp[i] = head ? pre : pre - 1u;
  }
};

// per group: new degree / capacity, and whether it needs a fresh allocation
__global__ void group_plan_k(uint64_t count, const uint32_t* ng_dev, const uint32_t* A_dev, uint32_t* gstart,
                             const uint32_t* gsrc, const uint32_t* deg, const uint32_t* cap, int insert,
                             uint32_t* gcnt, uint32_t* gnewdeg, uint32_t* gnewcap, uint64_t* galloc, int* underflow) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t ng = *ng_dev, A = *A_dev;
  if (blockIdx.x == 0 && threadIdx.x == 0) gstart[ng] = A;  // closes the last group (read below only for gi + 1 < ng)
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < count; gi += stride) {
    if (gi >= ng) break;
    const uint32_t c = (gi + 1 < ng ? gstart[gi + 1] : A) - gstart[gi];
    const uint32_t s = gsrc[gi];
    const uint32_t d = deg[s];
    uint32_t nd;
    if (insert) {
      nd = d + c;
    } else {
      if (c > d) *underflow = 1;  // metadata.hpp:28-31
      nd = d - c;
    }
    gcnt[gi] = c;
    gnewdeg[gi] = nd;
    const bool grow = nd > cap[s];
    gnewcap[gi] = grow ? cap_for(nd) : cap[s];
    galloc[gi] = grow ? cap_for(nd) : 0;
  }
}

// old list sizes of touched vertices; staged_only: only the lists merged in
// place (a list that grows is merged into a fresh allocation straight from
// its old one, which stays untouched until the merge is done)
// A list merged in place keeps its elements before the first applied arc
// where they are: only [alb[first], deg) is staged.
struct OldDegIn {
  const uint32_t* gsrc;
  const uint32_t* deg;
  const uint32_t* ng;
  const uint64_t* galloc;
  const uint32_t* gstart;
  const uint32_t* alb;
  int staged_only;
  __device__ __forceinline__ uint64_t operator()(uint64_t gi) const {
    if (gi >= *ng) return 0;
    const uint32_t d = deg[gsrc[gi]];
    if (staged_only == 2) return galloc[gi] ? d : d - alb[gstart[gi]];  // every old element that may move
    if (!staged_only) return galloc[gi] ? d : 0;  // old elements of lists that grow
    return galloc[gi] ? 0 : d - alb[gstart[gi]];
  }
};

// ---- merge by group windows
// The old elements that may move, group by group, form a flat space
// (mscan: grown list -> all d old elements, read from its old allocation;
// list merged in place -> [p0, d) from p0 = its first applied arc's slot,
// read from the staging copy).  A warp takes 512 consecutive flat elements:
// it loads the metadata of the (up to 32 per window) groups they span into
// shared memory once, then each lane places its elements: old element p of
// a group goes to p + #{applied arcs with slot <= p} (insert) or, unless it
// is deleted, p - #{deleted arcs before it} (delete), the count by a binary
// search over the group's applied-arc slots (alb, ascending).  No per-
// segment metadata arrays (the segment form wrote 28 bytes per segment and
// walked ~5-element segments one global lookup at a time).
constexpr uint32_t kMergeChunk = 512;
// batches of at least this many applied arcs merge by group windows (their
// segments average ~6 old elements: 10^7-edge insert 4.55 -> 4.0 ms);
// smaller ones keep the segment form, whose segments are long hub tails
// (10^4 .. 10^6 edges: 3-9% faster there)
#ifndef GBG_MERGE_WINDOW_MIN_ARCS
#define GBG_MERGE_WINDOW_MIN_ARCS (1u << 22)
#endif
constexpr uint32_t kMergeWindowMinArcs = GBG_MERGE_WINDOW_MIN_ARCS;

__global__ void merge_chunk_first_k(const uint64_t* mscan, uint32_t ng, uint32_t* first) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ng; gi += stride) {
    const uint64_t s = mscan[gi], e = mscan[gi + 1];
    for (uint64_t c = (s + kMergeChunk - 1) / kMergeChunk; c * kMergeChunk < e; ++c) first[c] = gi;
  }
}

struct MergeArgs {
  const uint64_t* mscan;
  uint32_t ng;
  uint64_t total;
  const uint32_t* first;
  const uint32_t* gsrc;
  const uint32_t* gstart;  // [ng + 1]
  const uint64_t* galloc;
  const uint32_t* alb;
  const uint32_t* deg;
  const uint64_t* start;
  const uint64_t* newstart;
  const uint64_t* sscan;
  const uint32_t* staged;
  uint32_t* pool;
  int insert;
};

__global__ void __launch_bounds__(256) merge_chunks_k(MergeArgs a) {
  __shared__ uint64_t s_ms[8][33];
  __shared__ const uint32_t* s_src[8][32];
  __shared__ uint32_t* s_dst[8][32];
  __shared__ uint32_t s_a0[8][32], s_a1[8][32], s_p0[8][32];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t c = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t w0 = c * kMergeChunk;
  if (w0 >= a.total) return;
  const uint64_t wend = w0 + kMergeChunk < a.total ? w0 + kMergeChunk : a.total;
  uint32_t g0 = a.first[c];
  uint64_t e0 = w0;  // first flat element not yet placed
  while (e0 < wend) {
    // window: groups g0 .. g0 + 31
    const uint32_t gk = g0 + lane;
    if (gk < a.ng) {
      const uint32_t sv = a.gsrc[gk];
      const uint32_t a0 = a.gstart[gk];
      const bool grows = a.galloc[gk] != 0;
      const uint32_t p0 = grows ? 0u : a.alb[a0];
      s_ms[wib][lane] = a.mscan[gk];
      s_a0[wib][lane] = a0;
      s_a1[wib][lane] = a.gstart[gk + 1];
      s_p0[wib][lane] = p0;
      s_src[wib][lane] = grows ? a.pool + a.start[sv] : a.staged + a.sscan[gk] - p0;
      s_dst[wib][lane] = a.pool + a.newstart[sv];
    }
    const uint32_t nw = a.ng - g0 < 32 ? a.ng - g0 : 32;
    if (lane == 0) s_ms[wib][nw] = a.mscan[g0 + nw];
    __syncwarp();
    const uint64_t wlim = s_ms[wib][nw] < wend ? s_ms[wib][nw] : wend;  // elements this window covers
    for (uint64_t e = e0 + lane; e < wlim; e += 32) {
      // group of e inside the window: last k with s_ms[k] <= e
      uint32_t lo = 0, hi = nw;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_ms[wib][mid] <= e) lo = mid; else hi = mid;
      }
      const uint32_t p = s_p0[wib][lo] + static_cast<uint32_t>(e - s_ms[wib][lo]);
      // applied arcs of the group with slot <= p (insert) / < p (delete)
      const uint32_t a0 = s_a0[wib][lo], a1 = s_a1[wib][lo];
      uint32_t l = a0, h = a1;
      while (l < h) {
        const uint32_t mid = (l + h) >> 1;
        const uint32_t v = a.alb[mid];
        if (a.insert ? v <= p : v < p) l = mid + 1; else h = mid;
      }
      const bool deleted = !a.insert && l < a1 && a.alb[l] == p;
      if (!deleted) {
        const uint32_t r = l - a0;
        const uint32_t val = s_src[wib][lo][p];
        s_dst[wib][lo][a.insert ? p + r : p - r] = val;
      }
    }
    __syncwarp();
    e0 = wlim;
    g0 += nw;
  }
}

// inserted arc j of group gi -> slot (j - first arc of gi) + (old neighbours below it)
__global__ void merge_new_k(uint32_t A, const uint32_t* agrp, const uint32_t* gstart, const uint32_t* gsrc,
                            const uint64_t* akeys, const uint32_t* alb, BatchKeys bk, const uint64_t* newstart,
                            uint32_t* pool) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < A; j += stride) {
    const uint32_t gi = agrp[j];
    pool[newstart[gsrc[gi]] + (j - gstart[gi]) + alb[j]] = bk.dst(akeys[j]);
  }
}

// Staging, merge and set difference run on the balanced segmented
// expansion (edges.cuh: expand) over the touched groups.
struct StageOp {  // segments = lists merged in place, from their first applied arc's position on
  const uint32_t* gsrc;
  const uint64_t* start;
  const uint32_t* pool;
  const uint32_t* gstart;
  const uint32_t* alb;
  uint32_t* staged;
  const uint64_t* sscan;
  __device__ __forceinline__ void bases(uint32_t gi, const uint32_t*& src, uint32_t*& dst) const {
    src = pool + start[gsrc[gi]] + alb[gstart[gi]];
    dst = staged + sscan[gi];
  }
};

// The old elements of a touched list, cut at the applied arcs' positions in
// it: segment q covers old elements [begin, begin + len) of group grp, and
// all of them move by the same shift -- +r (insert: the r applied arcs of
// the group that sort before them) or -r (delete: the r deleted elements
// before them, which no segment covers).  Arc i of group gi owns segment
// i + gi (the old elements just before it), and group gi's tail segment is
// gstart[gi + 1] + gi.  One balanced expansion over the segments then moves
// every old element with no search (traversal of neighbor_sets.hpp:339-366's
// merge / set difference, done element-parallel).
__global__ void merge_segments_k(uint32_t A, uint32_t ng, const uint32_t* agrp, const uint32_t* gstart,
                                 const uint32_t* gsrc, const uint32_t* alb, const uint32_t* deg,
                                 const uint64_t* galloc, const uint64_t* start, const uint64_t* newstart,
                                 const uint64_t* sscan, const uint32_t* staged, uint32_t* pool, int insert,
                                 uint64_t* seg_len, uint32_t* seg_begin, const uint32_t** seg_src,
                                 uint32_t** seg_dst) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < A + ng; t += stride) {
    uint32_t q, gi, begin, end, r;
    if (t < A) {  // the segment before applied arc t
      gi = agrp[t];
      r = t - gstart[gi];
      q = t + gi;
      begin = r == 0 ? 0u : alb[t - 1] + (insert ? 0u : 1u);
      end = alb[t];
    } else {  // group tail
      gi = t - A;
      const uint32_t last = gstart[gi + 1] - 1;
      r = gstart[gi + 1] - gstart[gi];
      q = gstart[gi + 1] + gi;
      begin = alb[last] + (insert ? 0u : 1u);
      end = deg[gsrc[gi]];
    }
    const uint32_t s = gsrc[gi];
    const bool grows = galloc[gi] != 0;
    // a list merged in place: its elements before the first applied arc
    // stay (and are not staged)
    if (t < A && r == 0 && !grows) begin = end;
    seg_len[q] = end - begin;
    seg_begin[q] = begin;
    // old element oi of the segment: src[oi] -> dst[oi]
    seg_src[q] = grows ? pool + start[s] : staged + sscan[gi] - alb[gstart[gi]];
    seg_dst[q] = pool + newstart[s] + (insert ? static_cast<int64_t>(r) : -static_cast<int64_t>(r));
  }
}
struct MergeSegOp {
  const uint32_t* seg_begin;
  const uint32_t* const* seg_src;
  uint32_t* const* seg_dst;
  __device__ __forceinline__ void bases(uint32_t q, const uint32_t*& src, uint32_t*& dst) const {
    src = seg_src[q] + seg_begin[q];
    dst = seg_dst[q] + seg_begin[q];
  }
};


// destination of each touched list: in place, or a fresh bump allocation
__global__ void plan_dest_k(uint32_t ng, const uint32_t* gsrc, const uint64_t* galloc_scan, const uint64_t* galloc,
                            uint64_t pool_top, const uint64_t* start, uint64_t* newstart) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ng; gi += stride) {
    const uint32_t s = gsrc[gi];
    newstart[s] = galloc[gi] ? pool_top + galloc_scan[gi] : start[s];
  }
}

__global__ void finish_groups_k(uint32_t ng, const uint32_t* gsrc, const uint32_t* gnewdeg, const uint32_t* gnewcap,
                                const uint64_t* newstart, uint64_t* start, uint32_t* deg, uint32_t* cap) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ng; gi += stride) {
    const uint32_t s = gsrc[gi];
    start[s] = newstart[s];
    deg[s] = gnewdeg[gi];
    cap[s] = gnewcap[gi];
  }
}

__global__ void refresh_caps_k(uint64_t n, const uint32_t* deg, uint32_t* cap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) cap[v] = cap_for(deg[v]);
}

// Scan inputs / outputs over a prefix whose length lives in device memory
// (the scans are sized by the raw arc count, an upper bound).
template <class T, class N>
struct BoundedIn {
  const T* a;
  const N* n;
  __device__ __forceinline__ T operator()(uint64_t i) const { return i < *n ? a[i] : T(0); }
};
template <class T, class N>
struct BoundedOut {  // writes [0, n]: the exclusive prefix at n is the total (scan count + 1 elements)
  T* a;
  const N* n;
  __device__ __forceinline__ void operator()(uint64_t i, T v) const {
    if (i <= *n) a[i] = v;
  }
};

// Device-side scalars of one batch, read back to the host once.
struct UpdScalars {
  uint64_t U;     // unique, self-loop-free arcs (prepare)
  uint64_t need;  // pool ids the grown lists allocate
  uint64_t mtot;  // old elements that may move (grown lists: all; in place: from the first applied arc)
  uint64_t stot;  // old elements staged: lists merged in place, from their first applied arc on
  uint32_t A;     // applied arcs
  uint32_t ng;    // touched sources
  int bad;        // an endpoint >= n
  int under;      // metadata underflow
  unsigned long long hsum[2];  // symmetry hash sums: zero when every unique (s, d) has its reverse
  uint64_t lt, gt;  // unique arcs with s < d / s > d
};

// Grow the pool when the batch's allocations do not fit (rare): the live
// lists are compacted into a larger pool and the allocation plan redone.
static void plan_allocations(gbg_graph* g, uint64_t count, uint32_t* gstart, const uint32_t* gsrc, bool insert,
                             UpdScalars* sc, uint32_t* gcnt, uint32_t* gnewdeg, uint32_t* gnewcap, uint64_t* galloc,
                             uint64_t* gascan) {
  GBG_LAUNCH(g, group_plan_k, grid_for(count, 256, g->sm_count * 16), 256, 0, count, &sc->ng, &sc->A, gstart, gsrc,
             g->bdeg, g->bcap, insert ? 1 : 0, gcnt, gnewdeg, gnewcap, galloc, &sc->under);
  device_scan<uint64_t>(g, BoundedIn<uint64_t, uint32_t>{galloc, &sc->ng},
                        BoundedOut<uint64_t, uint32_t>{gascan, &sc->ng}, count + 1, &sc->need, "upd.alloc");
}

// The whole batch up to the staging step runs without a host round trip:
// every stage is sized by the raw arc count (an upper bound of U, A and
// the group count) and reads the actual counts from device memory; one
// readback then brings U, A, the group count, the allocation need, the
// staging size and the error flags (out-of-range ids were turned into
// dropped keys, so nothing before the readback can fault), and errors are
// raised before the container is touched.  A 10^4-edge batch went from
// eight host synchronisations to one.
uint64_t apply_batch(gbg_graph* g, const uint32_t* pairs_dev, uint64_t count, bool insert) {
  if (g->kind != GBG_KIND_BLOCKED)
    fail(GBG_ERR_UNSUPPORTED, insert ? "container is static: batch insert not supported"
                                     : "container is static: batch delete not supported");
  if (count == 0) return 0;
  if (count > 0xffffffffull) fail(GBG_ERR_INVALID_ARGUMENT, "batch too large (max 2^32-1 arcs)");
  const BatchKeys bk{key_bits(g->n)};
  PhaseTrace tr(g->stream, insert ? "insert_batch" : "delete_batch");
  UpdScalars* sc = g->ws.get<UpdScalars>("upd.sc", 1);
  GBG_CUDA(cudaMemsetAsync(sc, 0, sizeof(UpdScalars), g->stream));
  // prepare(GlobalSort): keys, radix sort, unique (batch.cpp:34-42)
  uint64_t* keys = g->ws.get<uint64_t>("upd.keys", count);
  uint64_t* sorted = g->ws.get<uint64_t>("upd.sorted", count);
  GBG_LAUNCH(g, make_keys_k, grid_for(count, 256), 256, 0, pairs_dev, count, g->n, bk, keys, &sc->bad);
  uint64_t* srt = radix_sort_u64(g, keys, sorted, count, 2 * bk.L, "upd");
  uint64_t* akeys = srt == keys ? sorted : keys;  // receives the applied arcs
  tr.mark("prepare");
  // presence of each unique arc -> the applied arcs and their merge slots
  uint32_t* flag = g->ws.get<uint32_t>("upd.flag", count);
  uint32_t* lb = g->ws.get<uint32_t>("upd.lb", count);
  uint32_t* alb = g->ws.get<uint32_t>("upd.alb", count);
  if (count >= (1u << 21))
    GBG_LAUNCH(g, apply_flags_k<4>, grid_for(count / 4 + 1, 256, g->sm_count * 16), 256, 0, srt, count,
               reinterpret_cast<unsigned long long*>(&sc->U), bk,
               g->bstart, g->bdeg, g->pool, insert ? 1 : 0, flag, lb, g->symmetric ? 1 : 0, sc->hsum, &sc->lt,
               &sc->gt);
  else
    GBG_LAUNCH(g, apply_flags_k<1>, grid_for(count, 256, g->sm_count * 16), 256, 0, srt, count,
               reinterpret_cast<unsigned long long*>(&sc->U), bk,
               g->bstart, g->bdeg, g->pool, insert ? 1 : 0, flag, lb, g->symmetric ? 1 : 0, sc->hsum, &sc->lt,
               &sc->gt);
  device_scan<uint32_t>(g, ArrayIn<uint32_t>{flag}, ApplyOut{flag, srt, lb, akeys, alb}, count, &sc->A, "upd.apply");
  // groups by source
  uint32_t* gstart = g->ws.get<uint32_t>("upd.gstart", count + 1);
  uint32_t* gsrc = g->ws.get<uint32_t>("upd.gsrc", count);
  uint32_t* agrp = g->ws.get<uint32_t>("upd.agrp", count);
  device_scan<uint32_t>(g, HeadIn{akeys, bk, &sc->A}, HeadOut{akeys, bk, &sc->A, gstart, gsrc, agrp}, count, &sc->ng,
                        "upd.heads");
  tr.mark("presence+groups");
  uint32_t* gcnt = g->ws.get<uint32_t>("upd.gcnt", count);
  uint32_t* gnewdeg = g->ws.get<uint32_t>("upd.gnewdeg", count);
  uint32_t* gnewcap = g->ws.get<uint32_t>("upd.gnewcap", count);
  uint64_t* galloc = g->ws.get<uint64_t>("upd.galloc", count);
  uint64_t* gascan = g->ws.get<uint64_t>("upd.gascan", count + 1);
  plan_allocations(g, count, gstart, gsrc, insert, sc, gcnt, gnewdeg, gnewcap, galloc, gascan);
  // mscan: every old element that may move (grown list: all d; merged in
  // place: its staged tail), sscan: the staged tails alone
  uint64_t* mscan = g->ws.get<uint64_t>("upd.mscan", count + 1);
  uint64_t* sscan = g->ws.get<uint64_t>("upd.sscan", count + 1);
  auto scan_moves = [&] {
    device_scan<uint64_t>(g, OldDegIn{gsrc, g->bdeg, &sc->ng, galloc, gstart, alb, 2},
                          BoundedOut<uint64_t, uint32_t>{mscan, &sc->ng}, count + 1, &sc->mtot, "upd.mscan");
    device_scan<uint64_t>(g, OldDegIn{gsrc, g->bdeg, &sc->ng, galloc, gstart, alb, 1},
                          BoundedOut<uint64_t, uint32_t>{sscan, &sc->ng}, count + 1, &sc->stot, "upd.sscan");
  };
  scan_moves();
  UpdScalars h;
  read_scalars(g, sc, sizeof(h), &h);
  tr.mark("plan");
  if (PhaseTrace::enabled())
    std::fprintf(stderr, "[gbg trace] batch: count %llu U %llu A %u ng %u need %llu mtot %llu stot %llu\n",
                 (unsigned long long)count, (unsigned long long)h.U, h.A, h.ng, (unsigned long long)h.need,
                 (unsigned long long)h.mtot, (unsigned long long)h.stot);
  if (h.bad) fail(GBG_ERR_OUT_OF_RANGE, "edge endpoint out of range");
  if (h.U == 0 || h.A == 0) return 0;
  if (h.under) fail(GBG_ERR_LOGIC, "metadata underflow: tracker and container diverged");
  const uint32_t A = h.A, ng = h.ng;
  if (g->pool_top + h.need > g->pool_cap) {
    // compact into a larger pool (caps refreshed to the current degrees),
    // then plan again against the new capacities
    GBG_LAUNCH(g, refresh_caps_k, grid_for(g->n, 256), 256, 0, g->n, g->bdeg, g->bcap);
    blocked_relayout(g, g->bstart, g->pool, 2 * h.need, true);
    plan_allocations(g, count, gstart, gsrc, insert, sc, gcnt, gnewdeg, gnewcap, galloc, gascan);
    scan_moves();
    read_scalars(g, sc, sizeof(h), &h);
    if (g->pool_top + h.need > g->pool_cap) fail(GBG_ERR_OOM, "blocked pool exhausted after compaction");
  }
  // stage the touched old lists that are merged in place
  uint32_t* staged = g->ws.get<uint32_t>("upd.staged", h.stot ? h.stot : 1);
  copy_expand(g, sscan, ng, h.stot, StageOp{gsrc, g->bstart, g->pool, gstart, alb, staged, sscan});
  tr.mark("stage");
  // destinations
  uint64_t* newstart = g->ws.get<uint64_t>("upd.newstart", g->n);
  GBG_LAUNCH(g, plan_dest_k, grid_for(ng, 256), 256, 0, ng, gsrc, gascan, galloc, g->pool_top, g->bstart, newstart);
  if (A < kMergeWindowMinArcs) {
    // segment form (long segments: the tails of the touched hub lists)
    const uint32_t nseg = A + ng;
    uint64_t* seg_len = g->ws.get<uint64_t>("upd.seglen", nseg);
    uint64_t* seg_scan = g->ws.get<uint64_t>("upd.segscan", nseg + 1);
    uint32_t* seg_begin = g->ws.get<uint32_t>("upd.segbegin", nseg);
    const uint32_t** seg_src = g->ws.get<const uint32_t*>("upd.segsrc", nseg);
    uint32_t** seg_dst = g->ws.get<uint32_t*>("upd.segdst", nseg);
    GBG_LAUNCH(g, merge_segments_k, grid_for(nseg, 256), 256, 0, A, ng, agrp, gstart, gsrc, alb, g->bdeg, galloc,
               g->bstart, newstart, sscan, staged, g->pool, insert ? 1 : 0, seg_len, seg_begin, seg_src, seg_dst);
    device_scan<uint64_t>(g, ArrayIn<uint64_t>{seg_len}, ArrayOut<uint64_t>{seg_scan}, nseg, seg_scan + nseg,
                          "upd.segs");
    // old elements that move: all of them (insert), all but the A deleted,
    // less those that stay in place ahead of a list's first applied arc
    const uint64_t moved = h.mtot - (insert ? 0 : A);
    copy_expand(g, seg_scan, nseg, moved, MergeSegOp{seg_begin, seg_src, seg_dst});
  } else {
    // flat space of every old element that may move, then one warp per
    // 512 of them (group windows); the inserted arcs by a thread each
    const uint64_t mtot = h.mtot;
    if (mtot) {
      const uint64_t chunks = (mtot + kMergeChunk - 1) / kMergeChunk;
      uint32_t* first = g->ws.get<uint32_t>("upd.mfirst", chunks);
      GBG_LAUNCH(g, merge_chunk_first_k, grid_for(ng, 256), 256, 0, mscan, ng, first);
      MergeArgs ma{mscan, ng, mtot, first, gsrc, gstart, galloc, alb, g->bdeg, g->bstart, newstart, sscan, staged,
                   g->pool, insert ? 1 : 0};
      GBG_LAUNCH(g, merge_chunks_k, static_cast<unsigned>((chunks + 7) / 8), 256, 0, ma);
    }
  }
  if (insert) GBG_LAUNCH(g, merge_new_k, grid_for(A, 256), 256, 0, A, agrp, gstart, gsrc, akeys, alb, bk, newstart, g->pool);
  GBG_LAUNCH(g, finish_groups_k, grid_for(ng, 256), 256, 0, ng, gsrc, gnewdeg, gnewcap, newstart, g->bstart, g->bdeg,
             g->bcap);
  tr.mark("merge");
  g->pool_top += h.need;
  if (insert) {
    g->m += A;
  } else {
    g->m -= A;
  }
  g->invalidate_derived();
  // a symmetric batch keeps a symmetric container symmetric; anything else
  // is re-verified lazily (graph_is_symmetric)
  const bool keeps = g->symmetric && h.hsum[0] == 0 && h.hsum[1] == 0 && h.lt == h.gt;
  g->symmetric = keeps;
  g->sym_checked = keeps;
  return A;
}

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_blocked_create(uint64_t n, const uint32_t* arcs, uint64_t m, gbg_graph** out) {
  return guard([&] {
    if (!out || (m && !arcs)) fail(GBG_ERR_INVALID_ARGUMENT, "gbg_blocked_create: null argument");
    *out = nullptr;
    // validate through the CSR builder (sorted, unique, in range), then lay out
    gbg_graph* csr = nullptr;
    gbg_status st = gbg_csr_from_arcs(n, arcs, m, &csr);
    if (st != GBG_OK) fail(st, gbg_last_error());
    std::unique_ptr<gbg_graph> hold_csr(csr);
    gbg_graph* g = new_handle(GBG_KIND_BLOCKED, n);
    std::unique_ptr<gbg_graph> hold(g);
    AllocStream as(g->stream);
    DeviceScope ds(g->device);
    g->m = m;
    GBG_CUDA(cudaStreamSynchronize(csr->stream));
    blocked_from_device_csr(g, n, csr->off, csr->nbr);
    GBG_CUDA(cudaStreamSynchronize(g->stream));
    *out = hold.release();
  });
}

gbg_status gbg_blocked_from_csr(gbg_graph* csr, gbg_graph** out) {
  return guard([&] {
    GBG_HANDLE(csr);
    if (!out) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (csr->kind != GBG_KIND_CSR) fail(GBG_ERR_INVALID_ARGUMENT, "gbg_blocked_from_csr: not a CSR handle");
    *out = nullptr;
    GBG_CUDA(cudaStreamSynchronize(csr->stream));
    gbg_graph* g = new_handle(GBG_KIND_BLOCKED, csr->n);
    std::unique_ptr<gbg_graph> hold(g);
    AllocStream as(g->stream);
    g->m = csr->m;
    blocked_from_device_csr(g, csr->n, csr->off, csr->nbr);
    GBG_CUDA(cudaStreamSynchronize(g->stream));
    *out = hold.release();
  });
}

static gbg_status batch_entry(gbg_graph* g, const uint32_t* arcs, uint64_t count, uint64_t* applied, bool insert,
                              bool host) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!applied || (count && !arcs)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (g->kind != GBG_KIND_BLOCKED)
      fail(GBG_ERR_UNSUPPORTED, insert ? "container is static: batch insert not supported"
                                       : "container is static: batch delete not supported");
    const uint32_t* dev = arcs;
    if (host && count) {
      uint32_t* buf = g->ws.get<uint32_t>("upd.host", 2 * count);
      GBG_CUDA(cudaMemcpyAsync(buf, arcs, 2 * count * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream));
      dev = buf;
    }
    *applied = apply_batch(g, dev, count, insert);
  });
}

gbg_status gbg_insert_batch(gbg_graph* g, const uint32_t* arcs, uint64_t count, uint64_t* applied) {
  return batch_entry(g, arcs, count, applied, true, true);
}
gbg_status gbg_delete_batch(gbg_graph* g, const uint32_t* arcs, uint64_t count, uint64_t* applied) {
  return batch_entry(g, arcs, count, applied, false, true);
}
gbg_status gbg_insert_batch_device(gbg_graph* g, const uint32_t* arcs_dev, uint64_t count, uint64_t* applied) {
  return batch_entry(g, arcs_dev, count, applied, true, false);
}
gbg_status gbg_delete_batch_device(gbg_graph* g, const uint32_t* arcs_dev, uint64_t count, uint64_t* applied) {
  return batch_entry(g, arcs_dev, count, applied, false, false);
}

static gbg_status single_arc(gbg_graph* g, uint32_t src, uint32_t dst, int* changed, bool insert) {
  return guard([&] {
    if (!g || !changed) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (g->kind != GBG_KIND_BLOCKED)
      fail(GBG_ERR_UNSUPPORTED, insert ? "container is static: insert not supported"
                                       : "container is static: delete not supported");
    // set_graph.hpp:144-149 (check_arc)
    if (src >= g->n || dst >= g->n) fail(GBG_ERR_OUT_OF_RANGE, "edge endpoint out of range");
    if (src == dst) fail(GBG_ERR_INVALID_ARGUMENT, "self-loops are rejected at ingestion");
    uint32_t pair[2] = {src, dst};
    uint64_t applied = 0;
    gbg_status st = batch_entry(g, pair, 1, &applied, insert, true);
    if (st != GBG_OK) fail(st, gbg_last_error());
    *changed = applied ? 1 : 0;
  });
}

gbg_status gbg_insert_edge(gbg_graph* g, uint32_t src, uint32_t dst, int* changed) {
  return single_arc(g, src, dst, changed, true);
}
gbg_status gbg_delete_edge(gbg_graph* g, uint32_t src, uint32_t dst, int* changed) {
  return single_arc(g, src, dst, changed, false);
}

gbg_status gbg_contains_device(gbg_graph* g, const uint32_t* arcs_dev, uint64_t count, uint8_t* out_dev) {
  return guard([&] {
    GBG_HANDLE(g);
    if (count && (!arcs_dev || !out_dev)) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    with_view(g, [&](auto view) {
      GBG_LAUNCH(g, contains_k<decltype(view)>, grid_for(count, 256, g->sm_count * 16), 256, 0, view, arcs_dev, count,
                 out_dev);
    });
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"

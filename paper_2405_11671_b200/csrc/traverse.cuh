// vertex_subset conversions and the two edge_map engines as device
// templates over a read view (CsrView / BlockedView) and an operator:
//
//   struct Op {
//     __device__ bool cond(uint32_t v);            // EdgeMapSpec::cond
//     __device__ bool claim(uint32_t v);           // push dedup (AtomicBitset::try_claim)
//     __device__ bool update(uint32_t u, uint32_t v);  // EdgeMapSpec::update
//     __device__ void dense_word(uint64_t w, uint32_t emitted_mask);  // pull: word owner hook
//   };
//
// Reference semantics: traversal.cpp:16-46 (sparse push: cond, claim, then
// update; at most one update per destination), traversal.cpp:48-95 (dense
// pull over every v with cond(v), scanning N(v) against the frontier
// bitmap, early exit at the first frontier neighbour whose update returns
// true), traversal.cpp:101-111 (switch).  Ops used with early exit must
// return true from update (BFS and the test op do).
//
// Bitmaps are uint32 words, bit v&31 of word v>>5 — byte-identical on
// little-endian to the reference's uint64 LSB-first words
// (vertex_subset.hpp:10-14).
#pragma once

#include <type_traits>
#include <utility>

#include "scan.cuh"

#ifndef GBG_PB_INLINE
#define GBG_PB_INLINE __forceinline__
#endif
#ifndef GBG_PW_INLINE
#define GBG_PW_INLINE __forceinline__
#endif

namespace gbg {

__device__ __forceinline__ bool bit_test(const uint32_t* bm, uint32_t v) {
  return (__ldg(bm + (v >> 5)) >> (v & 31)) & 1u;
}

// ---------------------------------------------------------------- subsets
__global__ void list_to_bitmap_k(const uint32_t* ids, uint64_t k, uint32_t* bm);

struct PopcIn {
  const uint32_t* bm;
  __device__ __forceinline__ uint32_t operator()(uint64_t w) const { return __popc(bm[w]); }
};
struct BitsToIdsOut {
  const uint32_t* bm;
  uint32_t* ids;
  __device__ __forceinline__ void operator()(uint64_t w, uint32_t pre) const {
    uint32_t bits = bm[w];
    while (bits) {
      int b = __ffs(bits) - 1;
      ids[pre++] = static_cast<uint32_t>(w * 32 + b);
      bits &= bits - 1;
    }
  }
};

// ascending compaction of a bitmap into an id list; *count_dev = size
inline void bitmap_to_list(gbg_graph* g, const uint32_t* bm, uint64_t nwords, uint32_t* ids, uint32_t* count_dev) {
  device_scan<uint32_t>(g, PopcIn{bm}, BitsToIdsOut{bm, ids}, nwords, count_dev, "b2l");
}

// Frontier counters packed into one 64-bit word, (count << 36) | degree sum,
// so a single atomic hands an emitting warp both its list slots and its
// offsets in the next level's edge space: the push output is its own
// exclusive degree prefix and the next sparse level needs no scan.
constexpr int kPackShift = 36;
constexpr uint64_t kPackMask = (uint64_t{1} << kPackShift) - 1;
__host__ __device__ __forceinline__ uint64_t pack_count(uint64_t p) { return p >> kPackShift; }
__host__ __device__ __forceinline__ uint64_t pack_degsum(uint64_t p) { return p & kPackMask; }

// bitmap -> ascending id list plus the exclusive prefix of the members'
// degrees (one scan over words of packed (popc, sum of degrees))
template <class G>
struct PopcDegIn {
  G g;
  const uint32_t* bm;
  __device__ __forceinline__ uint64_t operator()(uint64_t w) const {
    uint32_t bits = bm[w];
    uint64_t d = 0;
    const uint64_t c = __popc(bits);
    while (bits) {
      d += g.degree(static_cast<uint32_t>(w * 32 + __ffs(bits) - 1));
      bits &= bits - 1;
    }
    return (c << kPackShift) | d;
  }
};
template <class G>
struct BitsToIdsDscanOut {
  G g;
  const uint32_t* bm;
  uint32_t* ids;
  uint64_t* dscan;
  __device__ __forceinline__ void operator()(uint64_t w, uint64_t pre) const {
    uint32_t bits = bm[w];
    uint64_t c = pack_count(pre), d = pack_degsum(pre);
    while (bits) {
      const uint32_t v = static_cast<uint32_t>(w * 32 + __ffs(bits) - 1);
      ids[c] = v;
      dscan[c] = d;
      d += g.degree(v);
      ++c;
      bits &= bits - 1;
    }
  }
};

// ---------------------------------------------------------------- push
constexpr int kPushThreads = 256;
constexpr int kPushIPT = 8;
constexpr int kPushTile = kPushThreads * kPushIPT;
// edge count of a push from which emissions are aggregated per CTA (one
// atomic per CTA and step) instead of per warp
constexpr uint64_t kPushCtaAggregate = 1ull << 16;

template <class G>
struct FrontierDegIn {
  G g;
  const uint32_t* F;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return g.degree(F[i]); }
};

// Load-balanced expansion over the frontier's edges: tile t owns edges
// [t*kPushTile, (t+1)*kPushTile) of the concatenated neighbour lists; the
// owning frontier slot of each edge comes from a per-thread binary search
// of the exclusive degree scan, then edges are walked with consecutive
// threads on consecutive neighbours (coalesced within a list).  Emitted
// vertices are appended to `out` with their degree prefix in `out_dscan`
// (packed counter, see pack_count) and set in the bitmap `out_bm`.
// Frontier data (list, prefix, bitmaps) may have been written earlier in
// the same launch by the persistent BFS kernel, so it is read with plain
// (coherent) loads; only the graph itself goes through the read-only path.
// Edges per thread (tile = kPushThreads * ipt edges): the full kPushIPT
// when the frontier's edges fill the grid, fewer when they do not — a
// thread walks its edges one dependent chain after another, so a small
// frontier on large tiles would leave most of the grid idle while a few
// CTAs walk 8 chains each.
__host__ __device__ __forceinline__ uint32_t push_ipt(uint64_t E, uint64_t ctas) {
  const uint64_t per = (E + ctas * kPushThreads - 1) / (ctas * kPushThreads);
  return per < 1 ? 1u : (per > static_cast<uint64_t>(kPushIPT) ? static_cast<uint32_t>(kPushIPT) : static_cast<uint32_t>(per));
}
__host__ __device__ __forceinline__ uint64_t push_tiles(uint64_t E, uint32_t ipt) {
  return (E + static_cast<uint64_t>(kPushThreads) * ipt - 1) / (static_cast<uint64_t>(kPushThreads) * ipt);
}
// resident CTAs a one-shot push launch can count on (8 per SM)
constexpr uint64_t kPushCtasPerSm = 8;

template <class G, class Op>
__device__ __forceinline__ void push_tile(G g, const uint32_t* F, uint32_t nf, const uint64_t* dscan, uint64_t E,
                                          Op op, uint32_t* out, uint64_t* out_dscan, uint32_t* out_bm,
                                          unsigned long long* packed, uint64_t tile, uint32_t* s_idx,
                                          uint32_t ipt = kPushIPT) {
  const uint32_t tile_len = kPushThreads * ipt;
  const uint64_t e0 = tile * tile_len;
  if (e0 >= E) return;
  const uint32_t len = static_cast<uint32_t>(E - e0 < tile_len ? E - e0 : tile_len);
  // The tile's slot range [tlo, thi) first, by a CTA-wide 128-ary search
  // (each half of the CTA narrows one end per barrier): a per-thread binary
  // search over a large frontier is ~20 dependent loads, this is ~3 rounds,
  // and the per-thread searches below then stay inside the tile's slice.
  uint32_t tlo = 0, thi = nf;
  if (nf > 64) {
    const uint32_t half = threadIdx.x >> 7, t = threadIdx.x & 127;
    const uint64_t key = half ? e0 + len - 1 : e0;
    uint32_t lo = 0, hi = nf;  // dscan[lo] <= key < dscan[hi] (dscan[nf] := E)
    while (true) {
      const bool more = hi - lo > 32;
      const uint32_t step = (hi - lo + 127) / 128;
      const uint32_t p = lo + t * step;
      const bool le = more && p < hi && dscan[p] <= key;
      const uint32_t c_lo = __syncthreads_count(le && !half);
      const uint32_t c_hi = __syncthreads_count(le && half);
      const uint32_t c = half ? c_hi : c_lo;
      if (!__syncthreads_or(more)) break;
      if (more) {
        lo = lo + (c - 1) * step;
        hi = lo + step < hi ? lo + step : hi;
      }
    }
    if (t == 0) s_idx[half] = half ? hi : lo;
    __syncthreads();
    tlo = s_idx[0];
    thi = s_idx[1];
    __syncthreads();
  }
  {
    const uint32_t k0 = threadIdx.x * ipt;
    if (k0 < len) {
      const uint64_t e = e0 + k0;
      uint32_t lo = tlo, hi = thi;  // dscan[lo] <= e < dscan[hi]
      while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (dscan[mid] <= e) lo = mid; else hi = mid;
      }
      uint32_t i = lo;
      uint64_t next = i + 1 < nf ? dscan[i + 1] : E;
#pragma unroll
      for (int j = 0; j < kPushIPT; ++j) {
        if (j >= static_cast<int>(ipt) || k0 + j >= len) break;
        while (next <= e + j) {
          ++i;
          next = i + 1 < nf ? dscan[i + 1] : E;
          if (next <= e + j) {  // a run of empty / short segments: search it instead of walking it
            uint32_t l2 = i + 1, h2 = nf;  // dscan[l2] <= e + j < dscan[h2]
            while (h2 - l2 > 1) {
              const uint32_t mid = (l2 + h2) >> 1;
              if (dscan[mid] <= e + j) l2 = mid; else h2 = mid;
            }
            i = l2;
            next = i + 1 < nf ? dscan[i + 1] : E;
          }
        }
        s_idx[k0 + j] = i;
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  __shared__ unsigned long long s_agg[kPushThreads / 32];
  for (uint32_t base = 0; base < len; base += kPushThreads) {
    const uint32_t k = base + threadIdx.x;
    bool emit = false;
    uint32_t v = 0;
    if (k < len) {
      const uint32_t i = s_idx[k];
      const uint32_t u = F[i];
      uint64_t b;
      uint32_t d;
      g.seg(u, b, d);
      v = g.at(b + (e0 + k - dscan[i]));
      emit = op.cond(v) && op.claim(v) && op.update(u, v);
    }
    if (E < kPushCtaAggregate) {
      // small levels: one warp-aggregated atomic per warp and step
      const uint32_t mask = __ballot_sync(0xffffffffu, emit);
      if (mask) {
        const uint64_t dv = emit ? g.degree(v) : 0;
        const uint64_t dinc = warp_inclusive_scan(dv);
        const uint64_t dtot = __shfl_sync(0xffffffffu, dinc, 31);
        const int leader = __ffs(mask) - 1;
        uint64_t old = 0;
        if (lane == leader)
          old = atomicAdd(packed, (static_cast<unsigned long long>(__popc(mask)) << kPackShift) | dtot);
        old = __shfl_sync(0xffffffffu, old, leader);
        if (emit) {
          const uint64_t pos = pack_count(old) + __popc(mask & ((1u << lane) - 1));
          out[pos] = v;
          if (out_dscan) out_dscan[pos] = pack_degsum(old) + dinc - dv;
          if (out_bm) atomicOr(out_bm + (v >> 5), 1u << (v & 31));
        }
      }
      continue;
    }
    // large levels: one atomic on the packed (count, degree sum) counter
    // per CTA and step.  The counter is one address, and a level that emits
    // most of its edges (the push from a hub: 406 K emissions at scale 24
    // level 0) was bound by the rate of same-address atomics (27 -> 21 us)
    if (!__syncthreads_or(emit)) continue;  // also orders the previous step's s_agg reads before this step's writes
    const uint32_t mask = __ballot_sync(0xffffffffu, emit);
    const uint64_t dv = emit ? g.degree(v) : 0;
    const uint64_t dinc = warp_inclusive_scan(dv);
    const uint64_t dtot = __shfl_sync(0xffffffffu, dinc, 31);
    const int warp = threadIdx.x >> 5;
    if (lane == 0) s_agg[warp] = (static_cast<unsigned long long>(__popc(mask)) << kPackShift) | dtot;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long mine = lane < kPushThreads / 32 ? s_agg[lane] : 0ull;
      const unsigned long long inc = warp_inclusive_scan(mine);
      const unsigned long long tot = __shfl_sync(0xffffffffu, inc, 31);
      unsigned long long old = 0;
      if (lane == 0 && tot) old = atomicAdd(packed, tot);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (lane < kPushThreads / 32) s_agg[lane] = old + inc - mine;
    }
    __syncthreads();
    if (emit) {
      const unsigned long long old = s_agg[warp];
      const uint64_t pos = pack_count(old) + __popc(mask & ((1u << lane) - 1));
      out[pos] = v;
      if (out_dscan) out_dscan[pos] = pack_degsum(old) + dinc - dv;
      if (out_bm) atomicOr(out_bm + (v >> 5), 1u << (v & 31));
    }
  }
}

template <class G, class Op>
__global__ void __launch_bounds__(kPushThreads)
    push_k(G g, const uint32_t* __restrict__ F, uint32_t nf, const uint64_t* __restrict__ dscan,
           uint64_t E, Op op, uint32_t* __restrict__ out, uint64_t* __restrict__ out_dscan,
           uint32_t* __restrict__ out_bm, unsigned long long* packed, uint32_t ipt) {
  __shared__ uint32_t s_idx[kPushTile];
  push_tile(g, F, nf, dscan, E, op, out, out_dscan, out_bm, packed, blockIdx.x, s_idx, ipt);
}

// one push over a frontier list with its degree prefix (E = total degree)
template <class G, class Op>
inline void push_list(gbg_graph* g, G view, const uint32_t* F, uint64_t nf, const uint64_t* dscan, uint64_t E, Op op,
                      uint32_t* out, uint64_t* out_dscan, unsigned long long* packed) {
  if (!nf || !E) return;
  const uint32_t ipt = push_ipt(E, static_cast<uint64_t>(g->sm_count) * kPushCtasPerSm);
  GBG_LAUNCH(g, (push_k<G, Op>), static_cast<unsigned>(push_tiles(E, ipt)), kPushThreads, 0, view, F,
             static_cast<uint32_t>(nf), dscan, E, op, out, out_dscan, nullptr, packed, ipt);
}

// Select the vertices with pred(v) into an ascending-by-warp id list with
// its degree prefix (packed counter, as push_tile emits).
template <class G, class Pred>
__global__ void select_k(G g, Pred pred, uint32_t* list, uint64_t* dscan, unsigned long long* packed) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < g.n; base += stride) {
    const uint64_t v = base + threadIdx.x;
    const bool take = v < g.n && pred(static_cast<uint32_t>(v));
    const uint32_t mask = __ballot_sync(0xffffffffu, take);
    if (!mask) continue;
    const uint64_t dv = take ? g.degree(static_cast<uint32_t>(v)) : 0;
    const uint64_t dinc = warp_inclusive_scan(dv);
    const uint64_t dtot = __shfl_sync(0xffffffffu, dinc, 31);
    const int leader = __ffs(mask) - 1;
    unsigned long long old = 0;
    if (lane == leader) old = atomicAdd(packed, (static_cast<unsigned long long>(__popc(mask)) << kPackShift) | dtot);
    old = __shfl_sync(0xffffffffu, old, leader);
    if (take) {
      const uint64_t pos = pack_count(old) + __popc(mask & ((1u << lane) - 1));
      list[pos] = static_cast<uint32_t>(v);
      dscan[pos] = pack_degsum(old) + dinc - dv;
    }
  }
}

// ---------------------------------------------------------------- pull
constexpr int kPullThreads = 256;
constexpr uint32_t kPullSerial = 8;  // neighbours a lane scans before the warp helps
// largest member degree a bitmap-driven push (push_bitmap) takes on: one
// warp walks such a list 32 entries per step
constexpr uint32_t kBitmapPushMaxDeg = 1024;

// One warp per 32-vertex bitmap word (so output / visited words need no
// atomics).  Each lane first scans up to kPullSerial neighbours of its own
// vertex; vertices still unresolved with longer lists are then scanned by
// the whole warp, 32 neighbours per step, ballot on frontier hits, stopping
// at the first hit in list order when early exit applies.
__device__ __forceinline__ bool frontier_bit(const uint32_t* bm, uint32_t v) { return (bm[v >> 5] >> (v & 31)) & 1u; }

// `first` (optional, early-exit pulls only): every vertex's first neighbour
// in one dense array (kNoFirst when isolated), so the test that settles
// most vertices of a dense level reads 4 coalesced bytes instead of a
// 32-byte sector of a list scattered through memory (at scale 24 level 1,
// 82% of the unvisited vertices with edges hit on their first neighbour).
constexpr uint32_t kNoFirst = 0xffffffffu;

constexpr uint64_t kCwBatch = 8;  // words per warp batch of the bitmap-driven loops
#ifndef GBG_PH1
#define GBG_PH1 4
#endif
constexpr uint32_t kPh1 = GBG_PH1;  // words whose first-neighbour tests are in flight at once

// The first-neighbour table of early-exit pulls: per vertex one 64-bit word
// (degree << 32) | first neighbour (first = kNoFirst when isolated), so one
// coalesced 8-byte load gives both the test that settles most vertices of a
// dense level and the degree the next frontier's degree sum needs; the row
// offsets are read only for vertices that miss.
__device__ __forceinline__ uint32_t fd_first(uint64_t x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t fd_deg(uint64_t x) { return static_cast<uint32_t>(x >> 32); }

// One vertex of an early-exit pull per lane (c = the lane holds a live
// vertex v).  kFirst: test the cached first neighbour first (counted in
// ex); otherwise v is known to have missed there and to have d > 1.  Then
// up to kPullSerial list entries by the lane itself, then the whole warp 32
// entries per step for each lane still unresolved (ballot on frontier hits,
// the first hit in list order wins).  Warp-uniform entry; returns whether
// v was reached, its degree in d.
template <bool kFirst, class G, class Op>
__device__ __forceinline__ bool pull_vertex(G g, const uint32_t* fb, Op op, const uint64_t* fd, bool c, uint32_t v,
                                            uint32_t& d, unsigned long long& ex) {
  const int lane = threadIdx.x & 31;
  uint64_t b = 0;
  d = 0;
  bool found = false;
  uint32_t lim = 0;
  if (c) {
    if (kFirst) {
      const uint64_t x = __ldg(fd + v);
      d = fd_deg(x);
      if (d && frontier_bit(fb, fd_first(x)) && op.update(fd_first(x), v)) found = true;
      ex += d ? 1 : 0;
    }
    if (!found) {
      g.seg(v, b, d);
      lim = d < kPullSerial ? d : kPullSerial;
    }
  }
  for (uint32_t k = 1; k < lim; ++k) {
    const uint32_t u = g.at(b + k);
    ++ex;
    if (frontier_bit(fb, u) && op.update(u, v)) {
      found = true;
      break;
    }
  }
  uint32_t hard = __ballot_sync(0xffffffffu, c && d > kPullSerial && !found);
  while (hard) {
    const int l = __ffs(hard) - 1;
    hard &= hard - 1;
    const uint64_t bb = __shfl_sync(0xffffffffu, b, l);
    const uint32_t dd = __shfl_sync(0xffffffffu, d, l);
    const uint32_t vv = __shfl_sync(0xffffffffu, v, l);
    bool fl = false;
    for (uint32_t j0 = kPullSerial; j0 < dd; j0 += 32) {
      const uint32_t jj = j0 + lane;
      uint32_t u = 0;
      const bool hit = jj < dd && frontier_bit(fb, u = g.at(bb + jj));
      const uint32_t hm = __ballot_sync(0xffffffffu, hit);
      if (!hm) continue;
      const int fi = __ffs(hm) - 1;
      bool r = false;
      if (lane == fi) r = op.update(u, vv);
      if (__shfl_sync(0xffffffffu, r, fi)) {
        fl = true;
        if (lane == l) ex += j0 + fi + 1 - kPullSerial;
        break;
      }
    }
    if (lane == l) {
      if (fl) found = true;
      else ex += dd - kPullSerial;
    }
  }
  return found;
}

// Word of a packed position: the largest k < kBatch with excl_k <= t, by a
// binary search over the lanes' exclusive popcount prefixes (log2(kBatch)
// shuffles).  Lanes past the batch hold excl == total > t, and an empty
// word shares its prefix with the next one, so the word found is non-empty
// for every t < total.
template <uint32_t kBatch>
__device__ __forceinline__ uint32_t packed_word(uint32_t excl, uint32_t t) {
  uint32_t j = 0;
#pragma unroll
  for (uint32_t s = kBatch / 2; s > 0; s >>= 1) {
    const uint32_t e = __shfl_sync(0xffffffffu, excl, j + s);
    if (e <= t) j += s;
  }
  return j;
}

// Hand out the set bits of the lanes' words (lane k < B holds word wb + k
// in `w`, exclusive prefix of the popcounts in `excl`) to the lanes: lane
// t of round r0 gets bit number r0 + t; returns its word index j and bit.
template <uint32_t kBatch>
__device__ __forceinline__ void packed_bit(uint32_t w, uint32_t excl, uint32_t t, uint32_t& j, uint32_t& bit) {
  j = packed_word<kBatch>(excl, t);
  const uint32_t ej = __shfl_sync(0xffffffffu, excl, j);
  const uint32_t wj = __shfl_sync(0xffffffffu, w, j);
  bit = __fns(wj, 0, static_cast<int>(t - ej + 1));
}

// Early-exit pull for operators whose cond is a bitmap (Op::cond_word(w):
// the 32 cond bits of word w).  Each warp takes strided batches of up to 8
// words and reads a batch's cond words in one coalesced load.
//  * A batch with at most 32 live vertices (sparse cond, e.g. the second
//    dense BFS level) is packed onto the lanes and resolved in one round:
//    one dependent chain for the whole batch.
//  * Denser batches run in two phases: the first-neighbour test of every
//    live vertex, four words' (first, degree) loads and then four words'
//    frontier-bit loads in flight at once; then the vertices that missed
//    (18% at scale 24 level 1) packed onto the lanes, 32 per round, for
//    the list scan from entry 1.
// The level is issue-bound as much as latency-bound (ncu at scale 24 level
// 1: 50% issue-slot use), so the per-word bookkeeping is kept off the
// inner loops: found bits of the packed rounds are OR-ed into a per-warp
// shared-memory word each (one ATOMS per round instead of a warp reduction
// per word), the found count is the popcount of the finished words, and
// per-batch bases replace 64-bit index arithmetic per word.  The owning
// warp writes the output word and publishes the visited bits.
template <class G, class Op>
__device__ __forceinline__ void pull_words_cw(G g, const uint32_t* fb, Op op, uint32_t* nb, uint64_t nwords64,
                                              unsigned long long* packed, const uint64_t* fd,
                                              unsigned long long* examined, unsigned* heavy) {
  constexpr int kWarps = (kPullThreads > kPushThreads ? kPullThreads : kPushThreads) / 32;  // callers' CTA sizes
  __shared__ uint32_t s_fw[kWarps][kCwBatch];       // found bits of the packed rounds, per warp and batch word
  __shared__ uint8_t s_miss[kWarps][kCwBatch * 32];  // phase-1 misses of a batch in order: word << 5 | bit
  const int lane = threadIdx.x & 31;
  const uint32_t lbit = 1u << lane;
  uint32_t* sf = s_fw[threadIdx.x >> 5];
  uint8_t* sm = s_miss[threadIdx.x >> 5];
  // word indices fit 32 bits (ids are uint32: at most 2^27 words)
  const uint32_t nwords = static_cast<uint32_t>(nwords64);
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t tail = (g.n & 31) ? (1u << (g.n & 31)) - 1u : 0xffffffffu;  // live bits of the last word
  // strided batches of B words (B <= kCwBatch): a warp's batches spread
  // over the whole id range, which balances the per-word work (static
  // contiguous runs left a 10-40 us tail of late CTAs before the barrier;
  // a shared batch counter costs more in contention than it recovers)
  const uint32_t per = (nwords + nwarps - 1) / nwarps;
  const uint32_t B = per < kCwBatch ? (per ? per : 1) : static_cast<uint32_t>(kCwBatch);
  const uint64_t stride = static_cast<uint64_t>(nwarps) * B;
  unsigned long long cnt = 0, degsum = 0, ex = 0;
  uint32_t dmax = 0;
  if (lane < static_cast<int>(kCwBatch)) sf[lane] = 0;
  __syncwarp();
  for (uint64_t wb64 = static_cast<uint64_t>(gwarp) * B; wb64 < nwords; wb64 += stride) {
    const uint32_t wb = static_cast<uint32_t>(wb64);
    const uint32_t wl = wb + lane;
    const bool mine = lane < static_cast<int>(B) && wl < nwords;
    uint32_t cw = 0;  // lanes past the batch keep 0: their words have no live vertex
    if (mine) {
      cw = op.cond_word(wl);
      if (wl == nwords - 1) cw &= tail;
    }
    uint32_t fword = 0;  // lane k < B: found bits of word wb + k
    uint32_t exb = 0;
    const uint32_t total = __reduce_add_sync(0xffffffffu, __popc(cw));
    const uint32_t v0 = wb * 32;
    bool rounds = total != 0;
    if (total > 32) {
      // phase 1: first-neighbour tests, 4 words at a time; the misses go
      // to the warp's shared list in (word, bit) order
      const uint64_t* fdl = fd + static_cast<uint64_t>(wb) * 32 + lane;
      uint32_t nmiss = 0;
#pragma unroll
      for (uint32_t k0 = 0; k0 < kCwBatch; k0 += kPh1) {
        if (k0 >= B) break;
        uint64_t x[kPh1];
        bool c[kPh1];
#pragma unroll
        for (uint32_t q = 0; q < kPh1; ++q) {
          c[q] = (__shfl_sync(0xffffffffu, cw, k0 + q) & lbit) != 0;
          x[q] = c[q] ? __ldg(fdl + (k0 + q) * 32) : 0ull;
        }
        bool h[kPh1];
#pragma unroll
        for (uint32_t q = 0; q < kPh1; ++q) h[q] = fd_deg(x[q]) && frontier_bit(fb, fd_first(x[q]));
#pragma unroll
        for (uint32_t q = 0; q < kPh1; ++q) {
          const uint32_t d = fd_deg(x[q]);  // 0 for a lane without a live vertex
          if (h[q] && !op.update(fd_first(x[q]), v0 + (k0 + q) * 32 + lane)) h[q] = false;
          exb += d ? 1 : 0;
          if (h[q]) {
            degsum += d;
            dmax = max(dmax, d);
          }
          const uint32_t fm = __ballot_sync(0xffffffffu, h[q]);
          const uint32_t mm = __ballot_sync(0xffffffffu, !h[q] && d > 1);
          if (lane == static_cast<int>(k0 + q)) fword = fm;
          if (mm & lbit) sm[nmiss + __popc(mm & (lbit - 1u))] = static_cast<uint8_t>((k0 + q) * 32 + lane);
          nmiss += __popc(mm);
        }
      }
      __syncwarp();
      for (uint32_t r0 = 0; r0 < nmiss; r0 += 32) {
        const uint32_t t = r0 + lane;
        const bool c = t < nmiss;
        const uint32_t pos = c ? sm[t] : 0u;
        uint32_t d;
        if (pull_vertex<false>(g, fb, op, fd, c, v0 + pos, d, ex)) {
          atomicOr(sf + (pos >> 5), 1u << (pos & 31));
          degsum += d;
          dmax = max(dmax, d);
        }
      }
      rounds = nmiss != 0;
    } else if (total) {
      // at most 32 live vertices: one packed round, first neighbours included
      const uint32_t pc = __popc(cw);
      const uint32_t excl = warp_inclusive_scan(pc) - pc;
      const bool c = static_cast<uint32_t>(lane) < total;
      uint32_t j, bit;
      packed_bit<kCwBatch>(cw, excl, lane, j, bit);
      if (!c) bit = 0;
      uint32_t d;
      if (pull_vertex<true>(g, fb, op, fd, c, v0 + j * 32 + bit, d, ex)) {
        atomicOr(sf + j, 1u << bit);
        degsum += d;
        dmax = max(dmax, d);
      }
    }
    if (rounds) {
      __syncwarp();
      if (lane < static_cast<int>(kCwBatch)) {
        fword |= sf[lane];
        sf[lane] = 0;
      }
      __syncwarp();
    }
    ex += exb;
    cnt += __popc(fword);
    if (mine) {
      nb[wl] = fword;
      if (fword) op.dense_word(wl, fword);
    }
  }
  if (heavy && __any_sync(0xffffffffu, dmax > kBitmapPushMaxDeg) && lane == 0) *heavy = 1u;
  cnt = warp_sum(cnt);
  degsum = warp_sum(degsum);
  if (lane == 0 && cnt) atomicAdd(packed, (static_cast<unsigned long long>(cnt) << kPackShift) | degsum);
  if (examined) {
    ex = warp_sum(ex);
    if (lane == 0 && ex) atomicAdd(examined, ex);
  }
}

template <class Op, class = void>
struct HasCondWord : std::false_type {};
template <class Op>
struct HasCondWord<Op, decltype(void(std::declval<const Op&>().cond_word(uint64_t{0})))> : std::true_type {};

// `examined` (optional): adds the arcs a serial scan in list order would
// inspect (up to and including the first hit under early exit).
template <class G, class Op, bool kEarly>
__device__ __forceinline__ void pull_words(G g, const uint32_t* fb, Op op, uint32_t* nb, uint64_t nwords,
                                           unsigned long long* packed, const uint64_t* first = nullptr,
                                           unsigned long long* examined = nullptr, unsigned* heavy = nullptr) {
  if constexpr (kEarly && HasCondWord<Op>::value) {
    if (first) {
      pull_words_cw(g, fb, op, nb, nwords, packed, first, examined, heavy);
      return;
    }
  }
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  unsigned long long cnt = 0, degsum = 0, ex = 0;
  for (uint64_t w = warp0; w < nwords; w += nwarps) {
    const uint64_t v64 = w * 32 + lane;
    const uint32_t v = static_cast<uint32_t>(v64);
    const bool c = v64 < g.n && op.cond(v);
    uint64_t b = 0;
    uint32_t d = 0;
    bool found = false;
    if (c) {
      uint32_t j0 = 0;
      if (kEarly && first) {
        const uint32_t f = fd_first(__ldg(first + v));
        g.seg(v, b, d);
        if (d && frontier_bit(fb, f) && op.update(f, v)) found = true;
        j0 = 1;
        ex += d ? 1 : 0;
      } else {
        g.seg(v, b, d);
      }
      const uint32_t lim = found ? 0 : (d < kPullSerial ? d : kPullSerial);
      for (uint32_t j = j0; j < lim; ++j) {
        const uint32_t u = g.at(b + j);
        ++ex;
        if (frontier_bit(fb, u) && op.update(u, v)) {
          found = true;
          if (kEarly) break;
        }
      }
    }
    uint32_t hard = __ballot_sync(0xffffffffu, c && d > kPullSerial && !(kEarly && found));
    while (hard) {
      const int l = __ffs(hard) - 1;
      hard &= hard - 1;
      const uint64_t bb = __shfl_sync(0xffffffffu, b, l);
      const uint32_t dd = __shfl_sync(0xffffffffu, d, l);
      const uint32_t vv = static_cast<uint32_t>(w * 32 + l);
      bool fl = false;
      for (uint32_t j0 = kPullSerial; j0 < dd; j0 += 32) {
        const uint32_t j = j0 + lane;
        uint32_t u = 0;
        const bool hit = j < dd && frontier_bit(fb, u = g.at(bb + j));
        const uint32_t hm = __ballot_sync(0xffffffffu, hit);
        if (!hm) continue;
        if (kEarly) {
          const int f = __ffs(hm) - 1;
          bool r = false;
          if (lane == f) r = op.update(u, vv);
          if (__shfl_sync(0xffffffffu, r, f)) {
            fl = true;
            if (lane == l) ex += j0 + f + 1 - kPullSerial;
            break;
          }
        } else {
          bool r = hit && op.update(u, vv);
          if (__ballot_sync(0xffffffffu, r)) fl = true;
        }
      }
      if (lane == l && fl) found = true;
      if (lane == l && !(kEarly && fl)) ex += dd - kPullSerial;
    }
    const uint32_t fm = __ballot_sync(0xffffffffu, found);
    if (lane == 0) nb[w] = fm;  // every word written: no clearing pass needed
    if (fm) {
      if (lane == 0) op.dense_word(w, fm);
      cnt += __popc(fm);
      if (found) degsum += d;
    }
  }
  degsum = warp_sum(degsum);
  if (lane == 0 && cnt) atomicAdd(packed, (static_cast<unsigned long long>(cnt) << kPackShift) | degsum);
  if (examined) {
    ex = warp_sum(ex);
    if (lane == 0 && ex) atomicAdd(examined, ex);
  }
}

template <class G, class Op, bool kEarly>
__global__ void __launch_bounds__(kPullThreads)
    pull_k(G g, const uint32_t* __restrict__ fb, Op op, uint32_t* __restrict__ nb, uint64_t nwords,
           unsigned long long* packed, const uint64_t* __restrict__ first, unsigned long long* examined) {
  pull_words<G, Op, kEarly>(g, fb, op, nb, nwords, packed, first, examined);
}

// ---------------------------------------------------------------- bitmap push
// Frontier words per warp batch of push_bitmap: 16 (scale 24 level 3:
// 47.5 -> 43.6 us against 8; the pull keeps 8, where 16 cost level 2 40%).
constexpr uint64_t kPushBatch = 16;
// Warp-aggregated emission of the push output (as push_tile): one packed
// atomic per warp step hands out list slots and degree-prefix offsets.
template <class G>
__device__ __forceinline__ void emit_warp(G g, bool emit, uint32_t v, uint32_t* out, uint64_t* out_dscan,
                                          uint32_t* out_bm, unsigned long long* packed) {
  const int lane = threadIdx.x & 31;
  const uint32_t mask = __ballot_sync(0xffffffffu, emit);
  if (!mask) return;
  const uint64_t dv = emit ? g.degree(v) : 0;
  const uint64_t dinc = warp_inclusive_scan(dv);
  const uint64_t dtot = __shfl_sync(0xffffffffu, dinc, 31);
  const int leader = __ffs(mask) - 1;
  unsigned long long old = 0;
  if (lane == leader) old = atomicAdd(packed, (static_cast<unsigned long long>(__popc(mask)) << kPackShift) | dtot);
  old = __shfl_sync(0xffffffffu, old, leader);
  if (emit) {
    const uint64_t pos = pack_count(old) + __popc(mask & ((1u << lane) - 1));
    out[pos] = v;
    out_dscan[pos] = pack_degsum(old) + dinc - dv;
    atomicOr(out_bm + (v >> 5), 1u << (v & 31));
  }
}

// Sparse push straight from a frontier bitmap (the dense -> sparse
// transition), with no id list or degree prefix built first: each warp
// takes strided batches of up to kPushBatch (16) frontier words, packs the batch's
// members onto the lanes 32 per round, and every lane walks its member's
// list in lock-step with the warp (one step = one neighbour per lane, an
// aggregated emission per step); lists longer than kPullSerial finish
// warp-cooperatively, 32 neighbours per step.  Semantics as push_tile
// (traversal.cpp:16-46: cond, claim, update, emit).  Callers guarantee
// every member's degree is at most kBitmapPushMaxDeg (the dense level that
// built the bitmap flags larger ones, and then the list path runs).  At
// scale 24 this replaces the level-3 compaction (two passes over the
// bitmap with a scattered degree lookup per member, a grid barrier and a
// scan) and the per-tile searches over the 841K-member list.
template <class G, class Op>
__device__ GBG_PB_INLINE void push_bitmap(G g, const uint32_t* fbm, uint64_t nwords, Op op, uint32_t* out,
                                            uint64_t* out_dscan, uint32_t* out_bm, unsigned long long* packed) {
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t per = (nwords + nwarps - 1) / nwarps;
  const uint32_t B = static_cast<uint32_t>(per < kPushBatch ? (per ? per : 1) : kPushBatch);
  for (uint64_t wb = gwarp * B; wb < nwords; wb += nwarps * B) {
    const uint64_t wl = wb + lane;
    const uint32_t fw = wl < wb + B && wl < nwords ? fbm[wl] : 0u;
    const uint32_t pc = __popc(fw);
    const uint32_t excl = warp_inclusive_scan(pc) - pc;
    const uint32_t total = __shfl_sync(0xffffffffu, excl + pc, 31);
    for (uint32_t r0 = 0; r0 < total; r0 += 32) {
      const uint32_t t = r0 + lane;
      const bool c = t < total;
      const uint32_t j = packed_word<kPushBatch>(excl, t);
      const uint32_t ej = __shfl_sync(0xffffffffu, excl, j);
      const uint32_t fwj = __shfl_sync(0xffffffffu, fw, j);
      const uint32_t u = c ? static_cast<uint32_t>((wb + j) * 32 + __fns(fwj, 0, static_cast<int>(t - ej + 1))) : 0u;
      uint64_t b = 0;
      uint32_t d = 0;
      if (c) g.seg(u, b, d);
      const uint32_t ds = d < kPullSerial ? d : kPullSerial;
      uint32_t steps = ds;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) steps = max(steps, __shfl_xor_sync(0xffffffffu, steps, o));
      // four list entries and then their cond tests in flight at once: a
      // round is one dependent chain per warp (bitmap word -> row bounds ->
      // entries -> cond), and the level has only a few rounds per warp
      for (uint32_t k0 = 0; k0 < steps; k0 += 4) {
        uint32_t v[4];
        bool ok[4];
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) v[q] = k0 + q < ds ? g.at(b + k0 + q) : 0u;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) ok[q] = k0 + q < ds && op.cond(v[q]);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          if (k0 + q >= steps) break;
          const bool emit = ok[q] && op.claim(v[q]) && op.update(u, v[q]);
          emit_warp(g, emit, v[q], out, out_dscan, out_bm, packed);
        }
      }
      uint32_t hard = __ballot_sync(0xffffffffu, d > kPullSerial);
      while (hard) {
        const int l = __ffs(hard) - 1;
        hard &= hard - 1;
        const uint64_t bb = __shfl_sync(0xffffffffu, b, l);
        const uint32_t dd = __shfl_sync(0xffffffffu, d, l);
        const uint32_t uu = __shfl_sync(0xffffffffu, u, l);
        for (uint32_t j0 = kPullSerial; j0 < dd; j0 += 32) {
          const uint32_t jj = j0 + lane;
          uint32_t v = 0;
          bool emit = false;
          if (jj < dd) {
            v = g.at(bb + jj);
            emit = op.cond(v) && op.claim(v) && op.update(uu, v);
          }
          emit_warp(g, emit, v, out, out_dscan, out_bm, packed);
        }
      }
    }
  }
}

}  // namespace gbg

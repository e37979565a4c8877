// Device-wide exclusive scan / compaction building block (reduce-then-scan,
// three launches).  Input and output are functors so the same code serves
// degree prefix sums (frontier work, CSR offsets, tile schedules) and
// stream compaction (scatter inside the output functor).
#pragma once

#include "gbg_internal.cuh"

namespace gbg {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr uint64_t kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Exclusive scan across the block; every thread gets its exclusive prefix
// and the block total.  smem: >= 33 T.  Contains __syncthreads.
template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nwarps ? smem[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < nwarps) smem[lane] = wi - w;
    if (lane == nwarps - 1) smem[32] = wi;
  }
  __syncthreads();
  T res = smem[warp] + inc - v;
  total = smem[32];
  __syncthreads();
  return res;
}

// Deterministic block sum (fixed tree).  smem >= 33 T.
template <class T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nwarps ? smem[lane] : T(0);
    w = warp_sum(w);
    if (lane == 0) smem[32] = w;
  }
  __syncthreads();
  T r = smem[32];
  __syncthreads();
  return r;
}

// Tile t covers items [t * kScanTile, (t + 1) * kScanTile).  Loads are
// warp-striped: warp w owns the 512 consecutive items from t * kScanTile +
// w * 512, read as 16 rounds of 32 consecutive items (one coalesced load per
// round), so the input functors (which often read neighbouring elements)
// touch each sector once.
template <class T, class In>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_k(In in, uint64_t count, T* sums) {
  __shared__ T sm[33];
  const uint64_t base = blockIdx.x * kScanTile + threadIdx.x;
  T acc = 0;
#pragma unroll 4
  for (int j = 0; j < kScanItems; ++j)
    if (base + j * kScanThreads < count) acc += in(base + j * kScanThreads);
  T t = block_sum<T>(acc, sm);
  if (threadIdx.x == 0) sums[blockIdx.x] = t;
}

template <class T>
__global__ void __launch_bounds__(1024) scan_sums_k(T* sums, uint64_t nb, T* total) {
  __shared__ T sm[33];
  uint64_t per = (nb + blockDim.x - 1) / blockDim.x;
  uint64_t b = threadIdx.x * per, e = b + per < nb ? b + per : nb;
  T acc = 0;
  for (uint64_t i = b; i < e; ++i) acc += sums[i];
  T tot;
  T pre = block_exclusive_scan<T>(acc, sm, tot);
  for (uint64_t i = b; i < e; ++i) {
    T s = sums[i];
    sums[i] = pre;
    pre += s;
  }
  if (threadIdx.x == 0 && total) *total = tot;
}

template <class T, class In, class Out>
__global__ void __launch_bounds__(kScanThreads) scan_down_k(In in, Out out, uint64_t count, const T* sums) {
  __shared__ T sm[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t sub = blockIdx.x * kScanTile + static_cast<uint64_t>(warp) * (32 * kScanItems);
  T vals[kScanItems];
  T acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const uint64_t i = sub + j * 32 + lane;
    vals[j] = i < count ? in(i) : T(0);
    acc += vals[j];
  }
  // the warp's total, then the warps' exclusive prefixes across the block
  const T wtot = warp_sum(acc);
  T tot;
  T pre = block_exclusive_scan<T>(lane == 0 ? wtot : T(0), sm, tot);
  pre = __shfl_sync(0xffffffffu, pre, 0) + sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const T inc = warp_inclusive_scan(vals[j]);
    const uint64_t i = sub + j * 32 + lane;
    if (i < count) out(i, pre + inc - vals[j]);
    pre += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// Single-pass scan (decoupled look-back): tiles in processing order from
// an atomic counter; a tile publishes its aggregate as soon as it has
// summed its items, then warp 0 looks back over the preceding tiles' states
// 32 at a time (lane k reads tile t-1-k) until it finds an inclusive
// prefix, and the tile publishes its own.  The inputs are read once (the
// reduce-then-scan form reads them twice).  State word: flag in the top 2
// bits (1 = aggregate, 2 = inclusive prefix), value below.
constexpr uint64_t kScanAgg = 1ull << 62, kScanPre = 2ull << 62, kScanVal = (1ull << 62) - 1;

template <class T, class In, class Out>
__global__ void __launch_bounds__(kScanThreads) scan_onepass_k(In in, Out out, uint64_t count, uint64_t* state,
                                                              unsigned* tile_ctr, T* total) {
  __shared__ T sm[33];
  __shared__ uint32_t s_tile;
  __shared__ T s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t sub = static_cast<uint64_t>(tile) * kScanTile + static_cast<uint64_t>(warp) * (32 * kScanItems);
  T vals[kScanItems];
  T acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const uint64_t i = sub + j * 32 + lane;
    vals[j] = i < count ? in(i) : T(0);
    acc += vals[j];
  }
  const T wtot = warp_sum(acc);
  T tot;
  T pre = block_exclusive_scan<T>(lane == 0 ? wtot : T(0), sm, tot);
  if (warp == 0) {
    volatile uint64_t* st = state + tile;
    if (lane == 0) *st = (tile == 0 ? kScanPre : kScanAgg) | static_cast<uint64_t>(tot);
    uint64_t excl = 0;
    if (tile > 0) {
      int64_t t = static_cast<int64_t>(tile) - 1;
      for (;;) {
        const int64_t mine = t - lane;
        uint64_t v = mine >= 0 ? *(const volatile uint64_t*)(state + mine) : kScanPre;
        uint32_t need, pre_m;
        for (;;) {  // every state up to the nearest published prefix must be in
          pre_m = __ballot_sync(0xffffffffu, (v >> 62) == 2);
          need = pre_m ? (2u << (__ffs(pre_m) - 1)) - 1u : 0xffffffffu;
          if ((__ballot_sync(0xffffffffu, (v >> 62) == 0) & need) == 0) break;
          if ((v >> 62) == 0) v = *(const volatile uint64_t*)(state + mine);
        }
        uint64_t add = ((need >> lane) & 1u) ? (v & kScanVal) : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) add += __shfl_xor_sync(0xffffffffu, add, d);
        excl += add;
        if (pre_m) break;
        t -= 32;
      }
      if (lane == 0) *st = kScanPre | (excl + static_cast<uint64_t>(tot));
    }
    if (lane == 0) s_excl = static_cast<T>(excl);
  }
  __syncthreads();
  pre = __shfl_sync(0xffffffffu, pre, 0) + s_excl;
  if (threadIdx.x == 0 && total && (static_cast<uint64_t>(tile) + 1) * kScanTile >= count)
    *total = s_excl + tot;  // the last tile
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const T inc = warp_inclusive_scan(vals[j]);
    const uint64_t i = sub + j * 32 + lane;
    if (i < count) out(i, pre + inc - vals[j]);
    pre += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// Small scans (count <= kSmallScan): one CTA of 1024 threads walks the
// items in tiles of 16K (same warp-striped rounds as scan_down_k) and
// carries the running prefix -- one launch instead of three, for the
// latency-bound scans of small update batches and small graphs.
constexpr int kSmallScanThreads = 1024;
constexpr uint64_t kSmallScanTile = static_cast<uint64_t>(kSmallScanThreads) * kScanItems;
#ifndef GBG_SMALL_SCAN
#define GBG_SMALL_SCAN 0  // off: the one-pass scan's few CTAs beat one CTA at 20K items (10^4 batch 0.388 -> 0.355 ms)
#endif
constexpr uint64_t kSmallScan = GBG_SMALL_SCAN;

template <class T, class In, class Out>
__global__ void __launch_bounds__(kSmallScanThreads) scan_small_k(In in, Out out, uint64_t count, T* total) {
  __shared__ T sm[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T carry = 0;
  for (uint64_t t0 = 0; t0 < count; t0 += kSmallScanTile) {
    const uint64_t sub = t0 + static_cast<uint64_t>(warp) * (32 * kScanItems);
    T vals[kScanItems];
    T acc = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      const uint64_t i = sub + j * 32 + lane;
      vals[j] = i < count ? in(i) : T(0);
      acc += vals[j];
    }
    const T wtot = warp_sum(acc);
    T tot;
    T pre = block_exclusive_scan<T>(lane == 0 ? wtot : T(0), sm, tot);
    pre = __shfl_sync(0xffffffffu, pre, 0) + carry;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      const T inc = warp_inclusive_scan(vals[j]);
      const uint64_t i = sub + j * 32 + lane;
      if (i < count) out(i, pre + inc - vals[j]);
      pre += __shfl_sync(0xffffffffu, inc, 31);
    }
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// Exclusive scan of in(0..count) delivered to out(i, prefix); the grand total
// lands in *total_dev (device pointer, may be null).  No host sync.
template <class T, class In, class Out>
void device_scan(gbg_graph* g, In in, Out out, uint64_t count, T* total_dev, const char* tag = "scan") {
  if (count <= kSmallScan) {
    GBG_LAUNCH(g, (scan_small_k<T, In, Out>), 1, kSmallScanThreads, 0, in, out, count, total_dev);
    return;
  }
#ifndef GBG_SCAN_TWO_PASS
  {
    const uint64_t nt = (count + kScanTile - 1) / kScanTile;
    uint64_t* st = g->ws.get<uint64_t>(std::string(tag) + ".lb", nt + 1);
    unsigned* ctr = reinterpret_cast<unsigned*>(st + nt);
    GBG_CUDA(cudaMemsetAsync(st, 0, (nt + 1) * sizeof(uint64_t), g->stream));
    GBG_LAUNCH(g, (scan_onepass_k<T, In, Out>), static_cast<unsigned>(nt), kScanThreads, 0, in, out, count, st, ctr,
               total_dev);
    return;
  }
#endif
  uint64_t nb = (count + kScanTile - 1) / kScanTile;
  if (nb == 0) nb = 1;
  T* sums = g->ws.get<T>(std::string(tag) + ".sums", nb);
  GBG_LAUNCH(g, (scan_reduce_k<T, In>), (unsigned)nb, kScanThreads, 0, in, count, sums);
  GBG_LAUNCH(g, scan_sums_k<T>, 1, 1024, 0, sums, nb, total_dev);
  GBG_LAUNCH(g, (scan_down_k<T, In, Out>), (unsigned)nb, kScanThreads, 0, in, out, count, sums);
}

// Common functors
struct NullOut {
  template <class T>
  __device__ __forceinline__ void operator()(uint64_t, T) const {}
};
template <class T>
struct ArrayIn {
  const T* a;
  __device__ __forceinline__ T operator()(uint64_t i) const { return a[i]; }
};
template <class T>
struct ArrayOut {
  T* a;
  __device__ __forceinline__ void operator()(uint64_t i, T v) const { a[i] = v; }
};

}  // namespace gbg

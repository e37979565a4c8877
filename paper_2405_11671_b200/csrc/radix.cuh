// Stable LSD radix sort of uint64 keys over their low `bits` bits, 8-bit
// digits, three launches per digit pass:
//
//   radix_hist_k     per 4096-key tile: digit histogram -> counts[digit][tile]
//   device_scan      exclusive scan of the digit-major counts -> global slot
//                    of (digit, tile)
//   radix_scatter_k  per tile: stable rank of every key among the tile's keys
//                    with the same digit (16 rounds of 256 keys; within a
//                    warp __match_any_sync finds the peers, across warps a
//                    per-round digit count table), keys staged in shared
//                    memory in digit order, then written out so that
//                    consecutive threads store consecutive slots of a digit
//                    bucket.
//
// Used by the batch-update "prepare" (batch.cpp:34-42: sort the raw arcs)
// and the R-MAT generator's normalisation (generators.cpp:22-23).
#pragma once

#include "scan.cuh"

namespace gbg {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr uint32_t kSortTile = kSortThreads * kSortRounds;  // 4096 keys
constexpr int kRadixBits = 8;
constexpr uint32_t kRadix = 1u << kRadixBits;

static __global__ void __launch_bounds__(kSortThreads) radix_hist_k(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                             uint32_t ntiles, uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[kRadix];
  for (uint32_t d = threadIdx.x; d < kRadix; d += kSortThreads) h[d] = 0;
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < kRadix; d += kSortThreads) counts[d * ntiles + blockIdx.x] = h[d];
}

static __global__ void __launch_bounds__(kSortThreads) radix_scatter_k(const uint64_t* __restrict__ in,
                                                                uint64_t* __restrict__ out, uint64_t n, int shift,
                                                                uint32_t ntiles, const uint32_t* __restrict__ offs) {
  __shared__ uint64_t s_keys[kSortTile];
  __shared__ uint32_t s_base[kRadix];       // global slot of this tile's first key of each digit
  __shared__ uint32_t s_start[kRadix];      // first slot of each digit inside the digit-sorted tile
  __shared__ uint32_t s_run[kRadix];        // keys of each digit ranked so far (earlier rounds)
  __shared__ uint32_t s_wcnt[kSortThreads / 32][kRadix];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile;

  // tile histogram -> exclusive start of each digit inside the tile
  for (uint32_t d = threadIdx.x; d < kRadix; d += kSortThreads) {
    s_run[d] = 0;
    s_base[d] = offs[d * ntiles + blockIdx.x];
  }
  __syncthreads();
  uint64_t k[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base + r * kSortThreads + threadIdx.x;
    k[r] = i < n ? in[i] : ~0ull;
    if (i < n) atomicAdd(&s_run[(k[r] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    // exclusive scan of the 256 tile counts by one warp (8 per lane)
    uint32_t c[kRadix / 32], sum = 0;
#pragma unroll
    for (int j = 0; j < static_cast<int>(kRadix / 32); ++j) {
      c[j] = s_run[lane * (kRadix / 32) + j];
      sum += c[j];
    }
    uint32_t inc = warp_inclusive_scan(sum), pre = inc - sum;
#pragma unroll
    for (int j = 0; j < static_cast<int>(kRadix / 32); ++j) {
      s_start[lane * (kRadix / 32) + j] = pre;
      pre += c[j];
    }
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < kRadix; d += kSortThreads) s_run[d] = 0;

  // stable ranks, round by round (tile order = round-major, thread-minor)
  const uint32_t lt = (1u << lane) - 1;
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base + r * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    const uint32_t d = valid ? static_cast<uint32_t>((k[r] >> shift) & (kRadix - 1)) : kRadix + lane;
    for (uint32_t x = lane; x < kRadix; x += 32) s_wcnt[warp][x] = 0;
    __syncwarp();
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank_w = __popc(peers & lt);
    if (valid && rank_w == 0) s_wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pre = 0;
      for (int w = 0; w < warp; ++w) pre += s_wcnt[w][d];
      s_keys[s_start[d] + s_run[d] + pre + rank_w] = k[r];
    }
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < kRadix; x += kSortThreads) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < kSortThreads / 32; ++w) t += s_wcnt[w][x];
      s_run[x] += t;
    }
    __syncthreads();
  }
  // coalesced write-out: slot j of the digit-sorted tile goes to
  // s_base[digit] + (j - s_start[digit])
  const uint32_t len = static_cast<uint32_t>(n - base < kSortTile ? n - base : kSortTile);
  for (uint32_t j = threadIdx.x; j < len; j += kSortThreads) {
    const uint64_t key = s_keys[j];
    const uint32_t d = static_cast<uint32_t>((key >> shift) & (kRadix - 1));
    out[s_base[d] + (j - s_start[d])] = key;
  }
}

// Sorts keys[0..n) by their low `bits` bits (stable); scratch must hold n
// keys.  Returns the buffer holding the result (keys or scratch).
inline uint64_t* radix_sort_u64(gbg_graph* g, uint64_t* keys, uint64_t* scratch, uint64_t n, int bits,
                                const char* tag) {
  if (n <= 1 || bits <= 0) return keys;
  if (n > 0xffffffffull) fail(GBG_ERR_INVALID_ARGUMENT, "radix sort: more than 2^32-1 keys");
  const uint32_t ntiles = static_cast<uint32_t>((n + kSortTile - 1) / kSortTile);
  const uint64_t ncounts = static_cast<uint64_t>(ntiles) * kRadix;
  uint32_t* counts = g->ws.get<uint32_t>(std::string(tag) + ".cnt", ncounts + 1);
  uint64_t* src = keys;
  uint64_t* dst = scratch;
  for (int shift = 0; shift < bits; shift += kRadixBits) {
    GBG_LAUNCH(g, radix_hist_k, ntiles, kSortThreads, 0, src, n, shift, ntiles, counts);
    device_scan<uint32_t>(g, ArrayIn<uint32_t>{counts}, ArrayOut<uint32_t>{counts}, ncounts, counts + ncounts,
                          (std::string(tag) + ".scan").c_str());
    GBG_LAUNCH(g, radix_scatter_k, ntiles, kSortThreads, 0, src, dst, n, shift, ntiles, counts);
    std::swap(src, dst);
  }
  return src;
}

}  // namespace gbg

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
static_assert(kSortThreads == static_cast<int>(kRadix), "one thread per digit in the tile scan");

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
  constexpr int kWarps = kSortThreads / 32;
  constexpr uint32_t kSub = kSortTile / kWarps;  // 512 consecutive keys per warp
  __shared__ uint64_t s_keys[kSortTile];
  __shared__ uint32_t s_base[kRadix];    // global slot of this tile's first key of each digit
  __shared__ uint32_t s_start[kRadix];   // first slot of each digit inside the digit-sorted tile
  __shared__ uint32_t s_cnt[kWarps][kRadix];  // per-warp digit counts, then per-warp running slots
  __shared__ uint32_t s_red[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile + static_cast<uint64_t>(warp) * kSub;
  const uint32_t lt = (1u << lane) - 1;

  for (uint32_t x = lane; x < kRadix; x += 32) s_cnt[warp][x] = 0;
  for (uint32_t d = threadIdx.x; d < kRadix; d += kSortThreads) s_base[d] = offs[d * ntiles + blockIdx.x];
  __syncwarp();
  // 1. each warp: its keys (coalesced, kept in registers) and digit counts
  uint64_t k[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base + r * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? in[i] : ~0ull;
    const uint32_t d = valid ? static_cast<uint32_t>((k[r] >> shift) & (kRadix - 1)) : kRadix + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 2. digit totals -> tile start of each digit; per-warp start inside it
  {
    const uint32_t d = threadIdx.x;  // kSortThreads == kRadix
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += s_cnt[w][d];
    uint32_t all;
    const uint32_t start = block_exclusive_scan(tot, s_red, all);
    s_start[d] = start;
    uint32_t run = start;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_cnt[w][d];
      s_cnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
  // 3. each warp ranks its keys in order (stable) into the staged tile
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const bool valid = base + r * 32 + lane < n;
    const uint32_t d = valid ? static_cast<uint32_t>((k[r] >> shift) & (kRadix - 1)) : kRadix + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (valid) s_keys[s_cnt[warp][d] + __popc(peers & lt)] = k[r];
    __syncwarp();
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 4. coalesced write-out: slot j of the digit-sorted tile goes to
  // s_base[digit] + (j - s_start[digit])
  const uint64_t tile0 = static_cast<uint64_t>(blockIdx.x) * kSortTile;
  const uint32_t len = static_cast<uint32_t>(n - tile0 < kSortTile ? n - tile0 : kSortTile);
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

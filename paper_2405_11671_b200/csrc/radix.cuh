// Stable LSD radix sort of uint64 keys over their low `bits` bits, 8-bit
// digits, one launch per digit pass (the "onesweep" structure):
//
//   radix_global_hist_k  one read of the keys: the histogram of every digit
//                        pass at once -> the global bucket base of each digit
//   radix_onesweep_k     per 4096-key tile (tiles taken in order from an
//                        atomic counter): digit counts of the tile, published
//                        at once; the tile's exclusive prefix per digit from a
//                        decoupled look-back over the preceding tiles'
//                        published counts / prefixes; stable rank of every
//                        key among the tile's keys with the same digit (within
//                        a warp __match_any_sync finds the peers, across warps
//                        per-warp digit counts), keys staged in shared memory
//                        in digit order, then written so that consecutive
//                        threads store consecutive slots of a digit bucket.
//
// So a pass reads and writes the keys once (the former separate histogram
// pass and count scan are gone).  Used by the batch-update "prepare"
// (batch.cpp:34-42: sort the raw arcs) and the R-MAT generator's
// normalisation (generators.cpp:22-23).
#pragma once

#include "scan.cuh"

namespace gbg {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr uint32_t kSortTile = kSortThreads * kSortRounds;  // 4096 keys
constexpr int kRadixBits = 8;
constexpr uint32_t kRadix = 1u << kRadixBits;
static_assert(kSortThreads == static_cast<int>(kRadix), "one thread per digit in the tile scan");

constexpr int kMaxPasses = 8;
constexpr uint64_t kLbAgg = 1ull << 62;   // published: the tile's own count
constexpr uint64_t kLbPre = 2ull << 62;   // published: inclusive prefix through the tile
constexpr uint64_t kLbVal = (1ull << 62) - 1;

static __global__ void __launch_bounds__(kSortThreads) radix_global_hist_k(const uint64_t* __restrict__ keys,
                                                                           uint64_t n, int passes,
                                                                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kMaxPasses][kRadix];
  for (int p = 0; p < passes; ++p) h[p][threadIdx.x] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint64_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (p * kRadixBits)) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int p = 0; p < passes; ++p)
    if (h[p][threadIdx.x]) atomicAdd(hist + p * kRadix + threadIdx.x, h[p][threadIdx.x]);
}

// per pass: exclusive scan of the 256 digit counts -> bucket bases (in place)
static __global__ void __launch_bounds__(kSortThreads) radix_bases_k(uint32_t* hist, int passes) {
  __shared__ uint32_t s_red[33];
  for (int p = 0; p < passes; ++p) {
    uint32_t all;
    const uint32_t c = hist[p * kRadix + threadIdx.x];
    const uint32_t e = block_exclusive_scan(c, s_red, all);
    __syncthreads();
    hist[p * kRadix + threadIdx.x] = e;
    __syncthreads();
  }
}

// the register-resident pass: only for sorts the small path cannot take
// (n <= kSmallMax with more than 51 key bits)
static __global__ void __launch_bounds__(kSortThreads, 3) radix_onesweep_k(const uint64_t* __restrict__ in,
                                                                        uint64_t* __restrict__ out, uint64_t n,
                                                                        int shift, const uint32_t* __restrict__ base,
                                                                        uint64_t* state, unsigned int* tile_ctr) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr uint32_t kSub = kSortTile / kWarps;  // 512 consecutive keys per warp
  __shared__ uint64_t s_keys[kSortTile];
  __shared__ uint32_t s_base[kRadix];    // global slot of this tile's first key of each digit
  __shared__ uint32_t s_start[kRadix];   // first slot of each digit inside the digit-sorted tile
  __shared__ uint32_t s_cnt[kWarps][kRadix];  // per-warp digit counts, then per-warp running slots
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);  // processing order == tile order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t x = lane; x < kRadix; x += 32) s_cnt[warp][x] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base0 = static_cast<uint64_t>(tile) * kSortTile + static_cast<uint64_t>(warp) * kSub;
  const uint32_t lt = (1u << lane) - 1;
  // 1. each warp: its keys (coalesced) and digit counts
  uint64_t k[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base0 + r * 32 + lane;
    const bool valid = i < n;
    const uint64_t key = valid ? in[i] : ~0ull;
    k[r] = key;
    const uint32_t d = valid ? static_cast<uint32_t>((key >> shift) & (kRadix - 1)) : kRadix + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 2. digit totals: publish them, tile start of each digit, per-warp starts
  {
    const uint32_t d = threadIdx.x;  // kSortThreads == kRadix
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += s_cnt[w][d];
    volatile uint64_t* st = state + static_cast<uint64_t>(tile) * kRadix + d;
    if (tile == 0) {
      *st = kLbPre | tot;
    } else {
      *st = kLbAgg | tot;
    }
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
    // 3. decoupled look-back: the tile's exclusive prefix of digit d
    uint64_t excl = 0;
    for (int64_t t = static_cast<int64_t>(tile) - 1; t >= 0; --t) {
      const volatile uint64_t* q = state + static_cast<uint64_t>(t) * kRadix + d;
      uint64_t v;
      while (((v = *q) >> 62) == 0) {
      }
      excl += v & kLbVal;
      if ((v >> 62) == 2) break;
    }
    if (tile > 0) *st = kLbPre | (excl + tot);
    s_base[d] = base[d] + static_cast<uint32_t>(excl);
  }
  __syncthreads();
  // 4. each warp ranks its keys in order (stable) into the staged tile
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base0 + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? static_cast<uint32_t>((k[r] >> shift) & (kRadix - 1)) : kRadix + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (valid) s_keys[s_cnt[warp][d] + __popc(peers & lt)] = k[r];
    __syncwarp();
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 5. coalesced write-out: slot j of the digit-sorted tile goes to
  // s_base[digit] + (j - s_start[digit])
  const uint64_t tile0 = static_cast<uint64_t>(tile) * kSortTile;
  const uint32_t len = static_cast<uint32_t>(n - tile0 < kSortTile ? n - tile0 : kSortTile);
  for (uint32_t j = threadIdx.x; j < len; j += kSortThreads) {
    const uint64_t key = s_keys[j];
    const uint32_t d = static_cast<uint32_t>((key >> shift) & (kRadix - 1));
    out[s_base[d] + (j - s_start[d])] = key;
  }
}

// Sorts above the small path: the same pass with the tile staged in shared
// memory by one 1-D bulk copy (no key registers: 3 CTAs per SM), in-warp
// ranking by bit-sliced ballots (eight votes give each key the mask of the
// round's lanes with its digit), the digit-ordered tile in a second shared
// buffer, and a look-back that reads four predecessor states per step.
// 18.5M 44-bit keys: 150 us per pass against 195 us for the match_any /
// reload pass (profiles/sort_bench.cu).
__device__ __forceinline__ uint32_t radix_smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr size_t kSortBulkSmem = 2ull * kSortTile * sizeof(uint64_t);
#ifndef GBG_SORT_BULK_MIN
#define GBG_SORT_BULK_MIN 0  // every sort above the small path (10^5-edge batch: 0.76 -> 0.71 ms)
#endif

static __global__ void __launch_bounds__(kSortThreads, 3) radix_onesweep_bulk_k(
    const uint64_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t n, int shift,
    const uint32_t* __restrict__ base, uint64_t* state, unsigned int* tile_ctr) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr uint32_t kSub = kSortTile / kWarps;
  extern __shared__ __align__(16) uint64_t s_sort_dyn[];
  uint64_t* s_in = s_sort_dyn;
  uint64_t* s_out = s_sort_dyn + kSortTile;
  __shared__ uint32_t s_base[kRadix];
  __shared__ uint32_t s_start[kRadix];
  __shared__ uint32_t s_cnt[kWarps][kRadix];
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_tile;
  __shared__ __align__(8) uint64_t s_bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(tile_ctr, 1u);  // processing order == tile order
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(radix_smem_addr(&s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (uint32_t x = lane; x < kRadix; x += 32) s_cnt[warp][x] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tile0 = static_cast<uint64_t>(tile) * kSortTile;
  const uint32_t len = static_cast<uint32_t>(n - tile0 < kSortTile ? n - tile0 : kSortTile);
  if (threadIdx.x == 0) {
    const uint32_t b16 = (len * 8u) & ~15u;  // bulk copies move multiples of 16 bytes
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(radix_smem_addr(&s_bar)), "r"(b16)
                 : "memory");
    if (b16)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       radix_smem_addr(s_in)),
                   "l"(in + tile0), "r"(b16), "r"(radix_smem_addr(&s_bar))
                   : "memory");
    if (len & 1u) s_in[len - 1] = in[tile0 + len - 1];  // odd tail key
  }
  {
    uint32_t done;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(radix_smem_addr(&s_bar))
          : "memory");
    } while (!done);
  }
  __syncthreads();  // the odd tail key
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t w0 = warp * kSub;
  uint32_t pm[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint32_t i = w0 + r * 32 + lane;
    const bool valid = i < len;
    const uint32_t d = static_cast<uint32_t>((s_in[i] >> shift) & (kRadix - 1));
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
      const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bb : ~bb;
    }
    pm[r] = peers;
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const uint32_t d = threadIdx.x;  // kSortThreads == kRadix
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += s_cnt[w][d];
    volatile uint64_t* st = state + static_cast<uint64_t>(tile) * kRadix + d;
    *st = (tile == 0 ? kLbPre : kLbAgg) | tot;
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
    uint64_t excl = 0;
    for (int64_t t = static_cast<int64_t>(tile) - 1; t >= 0; t -= 4) {
      uint64_t v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        v[q] = t - q >= 0 ? *(const volatile uint64_t*)(state + static_cast<uint64_t>(t - q) * kRadix + d) : kLbPre;
      bool stop = false;
      for (int q = 0; q < 4 && t - q >= 0; ++q) {
        uint64_t x = v[q];
        while ((x >> 62) == 0) x = *(const volatile uint64_t*)(state + static_cast<uint64_t>(t - q) * kRadix + d);
        excl += x & kLbVal;
        if ((x >> 62) == 2) {
          stop = true;
          break;
        }
      }
      if (stop) break;
    }
    if (tile > 0) *st = kLbPre | (excl + tot);
    s_base[d] = base[d] + static_cast<uint32_t>(excl);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint32_t i = w0 + r * 32 + lane;
    const bool valid = i < len;
    const uint64_t key = s_in[i];
    const uint32_t d = static_cast<uint32_t>((key >> shift) & (kRadix - 1));
    const uint32_t peers = pm[r];
    if (valid) s_out[s_cnt[warp][d] + __popc(peers & lt)] = key;
    __syncwarp();
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < len; j += kSortThreads) {
    const uint64_t key = s_out[j];
    const uint32_t d = static_cast<uint32_t>((key >> shift) & (kRadix - 1));
    out[s_base[d] + (j - s_start[d])] = key;
  }
}

// ---- small sorts (n <= kSmallMax): two launches instead of a histogram
// pass and one onesweep launch per digit (a 10^4-edge update batch sorts
// 2 * 10^4 keys, where the digit passes are pure launch + look-back
// latency).  Tiles of 4096 keys are bitonic-sorted in shared memory as
// (masked key << tile bits | index in tile) -- the index makes the order stable;
// then every CTA loads all sorted tiles into shared memory and places each
// key of its tile by binary searches in the other tiles (keys of earlier
// tiles first on ties).
#ifndef GBG_SMALL_SORT_TILE
#define GBG_SMALL_SORT_TILE 1024  // 1024-key tiles: 10^4 batch 0.388 -> 0.351 ms against 4096
#endif
constexpr uint32_t kSmallTile = GBG_SMALL_SORT_TILE;
constexpr int kSmallTileBits = kSmallTile == 4096 ? 12 : kSmallTile == 2048 ? 11 : 10;
static_assert(kSmallTile == (1u << kSmallTileBits), "small sort tile: 1024, 2048 or 4096 keys");
constexpr uint32_t kSmallMax = 24576;  // all keys in the merge CTA's shared memory (192 KB)
constexpr int kSmallThreads = 1024;

static __global__ void __launch_bounds__(kSmallThreads) small_sort_tiles_k(const uint64_t* __restrict__ in,
                                                                          uint64_t n, uint64_t mask,
                                                                          uint64_t* __restrict__ tmp) {
  __shared__ uint64_t s[kSmallTile];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSmallTile;
  const uint32_t len = static_cast<uint32_t>(n - base < kSmallTile ? n - base : kSmallTile);
  for (uint32_t i = threadIdx.x; i < kSmallTile; i += kSmallThreads)
    s[i] = i < len ? ((in[base + i] & mask) << kSmallTileBits) | i : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= kSmallTile; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < kSmallTile; i += kSmallThreads) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = s[i], b = s[ixj];
          if ((a > b) == ((i & k) == 0)) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < len; i += kSmallThreads) tmp[base + i] = s[i];
}

static __global__ void __launch_bounds__(kSmallThreads) small_merge_k(const uint64_t* __restrict__ tmp,
                                                                     const uint64_t* __restrict__ in, uint64_t n,
                                                                     uint64_t* __restrict__ out) {
  extern __shared__ uint64_t s_all[];
  for (uint32_t i = threadIdx.x; i < n; i += kSmallThreads) s_all[i] = tmp[i];
  __syncthreads();
  const uint32_t ntiles = static_cast<uint32_t>((n + kSmallTile - 1) / kSmallTile);
  const uint32_t c = blockIdx.x;
  const uint32_t base = c * kSmallTile;
  const uint32_t len = static_cast<uint32_t>(n - base < kSmallTile ? n - base : kSmallTile);
  for (uint32_t i = threadIdx.x; i < len; i += kSmallThreads) {
    const uint64_t v = s_all[base + i];
    const uint64_t key = v >> kSmallTileBits;
    uint32_t pos = i;
    for (uint32_t o = 0; o < ntiles; ++o) {
      if (o == c) continue;
      uint32_t lo = o * kSmallTile;
      uint32_t hi = lo + static_cast<uint32_t>(n - lo < kSmallTile ? n - lo : kSmallTile);
      const uint32_t t0 = lo;
      // count of keys < key (later tiles) or <= key (earlier tiles)
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint64_t km = s_all[mid] >> kSmallTileBits;
        if (o < c ? km <= key : km < key) lo = mid + 1;
        else hi = mid;
      }
      pos += lo - t0;
    }
    out[pos] = in[base + (v & (kSmallTile - 1))];
  }
}

// Sorts keys[0..n) by their low `bits` bits (stable); scratch must hold n
// keys.  Returns the buffer holding the result (keys or scratch).
inline uint64_t* radix_sort_u64(gbg_graph* g, uint64_t* keys, uint64_t* scratch, uint64_t n, int bits,
                                const char* tag) {
  if (n <= 1 || bits <= 0) return keys;
  if (n > 0xffffffffull) fail(GBG_ERR_INVALID_ARGUMENT, "radix sort: more than 2^32-1 keys");
  const int passes = (bits + kRadixBits - 1) / kRadixBits;
  if (passes > kMaxPasses) fail(GBG_ERR_LOGIC, "radix sort: too many digit passes");
  static bool attr = [] {
    cudaFuncSetAttribute(small_merge_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmallMax * sizeof(uint64_t)));
    cudaFuncSetAttribute(radix_onesweep_bulk_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSortBulkSmem));
    return true;
  }();
  (void)attr;
  if (n <= kSmallMax && bits <= 51) {
    uint64_t* tmp = g->ws.get<uint64_t>(std::string(tag) + ".small", n);
    const unsigned nt = static_cast<unsigned>((n + kSmallTile - 1) / kSmallTile);
    GBG_LAUNCH(g, small_sort_tiles_k, nt, kSmallThreads, 0, keys, n, (uint64_t{1} << bits) - 1, tmp);
    GBG_LAUNCH(g, small_merge_k, nt, kSmallThreads, n * sizeof(uint64_t), tmp, keys, n, scratch);
    return scratch;
  }
  const uint32_t ntiles = static_cast<uint32_t>((n + kSortTile - 1) / kSortTile);
  const std::string t(tag);
  uint32_t* hist = g->ws.get<uint32_t>(t + ".hist", kMaxPasses * kRadix);
  uint64_t* state = g->ws.get<uint64_t>(t + ".lb", static_cast<uint64_t>(ntiles) * kRadix);
  unsigned int* ctr = g->ws.get<unsigned int>(t + ".ctr", kMaxPasses);
  GBG_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), g->stream));
  GBG_CUDA(cudaMemsetAsync(ctr, 0, kMaxPasses * sizeof(unsigned int), g->stream));
  GBG_LAUNCH(g, radix_global_hist_k, grid_for(n, kSortThreads, static_cast<unsigned>(g->sm_count) * 4u),
             kSortThreads, 0, keys, n, passes, hist);
  GBG_LAUNCH(g, radix_bases_k, 1, kSortThreads, 0, hist, passes);
  uint64_t* src = keys;
  uint64_t* dst = scratch;
  for (int p = 0; p < passes; ++p) {
    GBG_CUDA(cudaMemsetAsync(state, 0, static_cast<uint64_t>(ntiles) * kRadix * sizeof(uint64_t), g->stream));
    if (n > GBG_SORT_BULK_MIN)
      GBG_LAUNCH(g, radix_onesweep_bulk_k, ntiles, kSortThreads, kSortBulkSmem, src, dst, n, p * kRadixBits,
                 hist + p * kRadix,
                 state, ctr + p);
    else
      GBG_LAUNCH(g, radix_onesweep_k, ntiles, kSortThreads, 0, src, dst, n, p * kRadixBits, hist + p * kRadix,
                 state, ctr + p);
    std::swap(src, dst);
  }
  return src;
}

}  // namespace gbg

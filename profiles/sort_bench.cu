// Stand-alone timing of one LSD radix pass over uint64 keys (analysis only):
// the library's onesweep passes (radix.cuh) against the experimental
// variants that led to the bulk-staged pass (ballot ranking; v2 = what
// radix_onesweep_bulk_k now is).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_11671_b200/csrc \
//        profiles/sort_bench.cu -o profiles/sort_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "radix.cuh"

using namespace gbg;

// ---- variant: ballot ranking, keys kept in registers
template <int kRounds, bool kNoLB = false>
static __global__ void __launch_bounds__(kSortThreads, 2) onesweep_ballot_k(const uint64_t* __restrict__ in,
                                                                           uint64_t* __restrict__ out, uint64_t n,
                                                                           int shift, const uint32_t* __restrict__ base,
                                                                           uint64_t* state, unsigned int* tile_ctr) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr uint32_t kTile = kSortThreads * kRounds;
  constexpr uint32_t kSub = kTile / kWarps;
  __shared__ uint64_t s_keys[kTile];
  __shared__ uint32_t s_base[kRadix];
  __shared__ uint32_t s_start[kRadix];
  __shared__ uint32_t s_cnt[kWarps][kRadix];
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t x = lane; x < kRadix; x += 32) s_cnt[warp][x] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base0 = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * kSub;
  const uint32_t lt = (1u << lane) - 1;
  uint64_t k[kRounds];
  uint32_t pm[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint64_t i = base0 + r * 32 + lane;
    k[r] = i < n ? in[i] : ~0ull;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint64_t i = base0 + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = static_cast<uint32_t>((k[r] >> shift) & (kRadix - 1));
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
    const uint32_t d = threadIdx.x;
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
    if (kNoLB) {
      excl = static_cast<uint64_t>(tile) * tot;  // timing experiment only: wrong bases
    } else {
    for (int64_t t = static_cast<int64_t>(tile) - 1; t >= 0; --t) {
      const volatile uint64_t* q = state + static_cast<uint64_t>(t) * kRadix + d;
      uint64_t v;
      while (((v = *q) >> 62) == 0) {
      }
      excl += v & kLbVal;
      if ((v >> 62) == 2) break;
    }
    }
    if (tile > 0) *st = kLbPre | (excl + tot);
    s_base[d] = kNoLB ? static_cast<uint32_t>((static_cast<uint64_t>(tile) * kTile) % (n - 2 * kTile))
                      : base[d] + static_cast<uint32_t>(excl);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint64_t i = base0 + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = static_cast<uint32_t>((k[r] >> shift) & (kRadix - 1));
    const uint32_t peers = pm[r];
    if (valid) s_keys[s_cnt[warp][d] + __popc(peers & lt)] = k[r];
    __syncwarp();
    if (valid && (peers & lt) == 0) s_cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const uint64_t tile0 = static_cast<uint64_t>(tile) * kTile;
  const uint32_t len = static_cast<uint32_t>(n - tile0 < kTile ? n - tile0 : kTile);
  for (uint32_t j = threadIdx.x; j < len; j += kSortThreads) {
    const uint64_t key = s_keys[j];
    const uint32_t d = static_cast<uint32_t>((key >> shift) & (kRadix - 1));
    out[s_base[d] + (j - s_start[d])] = key;
  }
}


// ---- variant v2: tile keys staged in shared memory by a 1-D bulk copy,
// ballot ranking, two shared buffers (in / digit-ordered out), 3 CTAs per
// SM, look-back reading 4 predecessor states at once.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int kRounds>
static __global__ void __launch_bounds__(kSortThreads, 3) onesweep_v2_k(const uint64_t* __restrict__ in,
                                                                       uint64_t* __restrict__ out, uint64_t n,
                                                                       int shift, const uint32_t* __restrict__ base,
                                                                       uint64_t* state, unsigned int* tile_ctr) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr uint32_t kTile = kSortThreads * kRounds;
  constexpr uint32_t kSub = kTile / kWarps;
  extern __shared__ __align__(16) uint64_t s_dyn[];
  uint64_t* s_in = s_dyn;
  uint64_t* s_out = s_dyn + kTile;
  __shared__ uint32_t s_base[kRadix];
  __shared__ uint32_t s_start[kRadix];
  __shared__ uint32_t s_cnt[kWarps][kRadix];
  __shared__ uint32_t s_red[33];
  __shared__ uint32_t s_tile;
  __shared__ __align__(8) uint64_t s_bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(tile_ctr, 1u);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (uint32_t x = lane; x < kRadix; x += 32) s_cnt[warp][x] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tile0 = static_cast<uint64_t>(tile) * kTile;
  const uint32_t len = static_cast<uint32_t>(n - tile0 < kTile ? n - tile0 : kTile);
  if (threadIdx.x == 0) {
    const uint32_t bytes = len * 8;  // multiple of 8; bulk copies need 16: pad with one key below
    const uint32_t b16 = (bytes + 15) & ~15u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&s_bar)), "r"(b16) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(s_in)),
                 "l"(in + tile0), "r"(b16), "r"(smem_addr(&s_bar))
                 : "memory");
  }
  {
    uint32_t done;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done)
                   : "r"(smem_addr(&s_bar))
                   : "memory");
    } while (!done);
  }
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t w0 = warp * kSub;
  uint32_t pm[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
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
    const uint32_t d = threadIdx.x;
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
    // look-back, 4 predecessor states per step
    uint64_t excl = 0;
    int64_t t = static_cast<int64_t>(tile) - 1;
    while (t >= 0) {
      uint64_t v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        v[q] = t - q >= 0 ? *(const volatile uint64_t*)(state + static_cast<uint64_t>(t - q) * kRadix + d) : kLbPre;
      bool stop = false;
      int q = 0;
      for (; q < 4 && t - q >= 0; ++q) {
        uint64_t x = v[q];
        while ((x >> 62) == 0) x = *(const volatile uint64_t*)(state + static_cast<uint64_t>(t - q) * kRadix + d);
        excl += x & kLbVal;
        if ((x >> 62) == 2) {
          stop = true;
          break;
        }
      }
      if (stop) break;
      t -= 4;
    }
    if (tile > 0) *st = kLbPre | (excl + tot);
    s_base[d] = base[d] + static_cast<uint32_t>(excl);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
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

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);               \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 18500000;
  const int bits = 44;
  std::vector<uint64_t> h(n);
  uint64_t s = 88172645463325252ull;
  for (auto& x : h) {  // skewed high bits (R-MAT-like sources), uniform low bits
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const uint64_t src = (s >> 40) & ((1u << 22) - 1);
    const uint64_t sk = src & (src >> 3) & (src >> 7);  // denser at small ids
    x = (sk << 22) | (s & ((1u << 22) - 1));
  }
  uint64_t *d_in, *d_out, *d_state;
  uint32_t *d_hist;
  unsigned *d_ctr;
  const int passes = (bits + 7) / 8;
  CK(cudaMalloc(&d_in, n * 8));
  CK(cudaMalloc(&d_out, n * 8));
  const uint32_t maxtiles = (n + 1023) / 1024;
  CK(cudaMalloc(&d_state, (uint64_t)maxtiles * kRadix * 8));
  CK(cudaMalloc(&d_hist, kMaxPasses * kRadix * 4));
  CK(cudaMalloc(&d_ctr, 64 * 4));
  CK(cudaMemcpy(d_in, h.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_hist, 0, kMaxPasses * kRadix * 4));
  radix_global_hist_k<<<148 * 4, kSortThreads>>>(d_in, n, passes, d_hist);
  radix_bases_k<<<1, kSortThreads>>>(d_hist, passes);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, uint32_t tile) {
    const uint32_t ntiles = (n + tile - 1) / tile;
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      // a full sort, one pass per launch; time the middle pass (digit 2)
      CK(cudaMemcpy(d_in, h.data(), n * 8, cudaMemcpyHostToDevice));
      uint64_t *src = d_in, *dst = d_out;
      for (int p = 0; p < passes; ++p) {
        CK(cudaMemset(d_state, 0, (uint64_t)ntiles * kRadix * 8));
        CK(cudaMemset(d_ctr, 0, 4));
        if (p == 2) cudaEventRecord(e0);
        launch(ntiles, src, dst, p * 8, d_hist + p * kRadix);
        if (p == 2) cudaEventRecord(e1);
        std::swap(src, dst);
      }
      CK(cudaDeviceSynchronize());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
      if (it == 0) {  // check: sorted by the low 48 bits and a permutation (sum)
        std::vector<uint64_t> r(n);
        CK(cudaMemcpy(r.data(), src, n * 8, cudaMemcpyDeviceToHost));
        bool ok = std::is_sorted(r.begin(), r.end());
        uint64_t a = 0, b = 0;
        for (uint64_t i = 0; i < n; ++i) { a += h[i]; b += r[i]; }
        printf("%s: %s\n", name, ok && a == b ? "sorted ok" : "WRONG");
      }
    }
    printf("%s: pass %.1f us = %.2f TB/s (read+write)\n", name, best * 1e3, 16.0 * n / (best * 1e-3) / 1e12);
  };
  run("library onesweep (small sorts: match_any, keys in registers)", [&](uint32_t nt, uint64_t* a, uint64_t* b, int sh, const uint32_t* bs) {
    radix_onesweep_k<<<nt, kSortThreads>>>(a, b, n, sh, bs, d_state, d_ctr);
  }, kSortTile);
  cudaFuncSetAttribute(radix_onesweep_bulk_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortBulkSmem);
  run("library onesweep (large sorts: bulk-staged tile, ballot ranking)", [&](uint32_t nt, uint64_t* a, uint64_t* b, int sh, const uint32_t* bs) {
    radix_onesweep_bulk_k<<<nt, kSortThreads, kSortBulkSmem>>>(a, b, n, sh, bs, d_state, d_ctr);
  }, kSortTile);
  run("ballot ranking, 16 rounds", [&](uint32_t nt, uint64_t* a, uint64_t* b, int sh, const uint32_t* bs) {
    onesweep_ballot_k<16><<<nt, kSortThreads>>>(a, b, n, sh, bs, d_state, d_ctr);
  }, kSortThreads * 16);
  run("ballot ranking, 8 rounds", [&](uint32_t nt, uint64_t* a, uint64_t* b, int sh, const uint32_t* bs) {
    onesweep_ballot_k<8><<<nt, kSortThreads>>>(a, b, n, sh, bs, d_state, d_ctr);
  }, kSortThreads * 8);
  cudaFuncSetAttribute(onesweep_v2_k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4096 * 8);
  run("v2: bulk-staged tile, ballot ranking, 3 CTAs/SM, 4-wide look-back", [&](uint32_t nt, uint64_t* a, uint64_t* b, int sh, const uint32_t* bs) {
    onesweep_v2_k<16><<<nt, kSortThreads, 2 * 4096 * 8>>>(a, b, n, sh, bs, d_state, d_ctr);
  }, kSortThreads * 16);
  run("ballot, 16 rounds, NO look-back (timing only)", [&](uint32_t nt, uint64_t* a, uint64_t* b, int sh, const uint32_t* bs) {
    onesweep_ballot_k<16, true><<<nt, kSortThreads>>>(a, b, n, sh, bs, d_state, d_ctr);
  }, kSortThreads * 16);
  return 0;
}

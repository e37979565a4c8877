// Packed arc keys and the device "prepare" steps shared by the R-MAT
// generator (generators.cpp:9-29: sort + unique) and the batch update path
// (batch.cpp:34-42: drop self-loops, sort, unique).
//
// An arc (s,d) with ids < 2^L packs into the 2L-bit key s<<L | d, whose
// numeric order is the reference's lexicographic Edge order
// (types.hpp:21-25), so sorting keys == std::sort on Edges.
#pragma once

#include <cub/device/device_radix_sort.cuh>

#include "scan.cuh"

namespace gbg {

struct BatchKeys {
  int L;
  __host__ __device__ __forceinline__ uint64_t make(uint32_t s, uint32_t d) const {
    return (static_cast<uint64_t>(s) << L) | d;
  }
  __host__ __device__ __forceinline__ uint32_t src(uint64_t k) const { return static_cast<uint32_t>(k >> L); }
  __host__ __device__ __forceinline__ uint32_t dst(uint64_t k) const {
    return static_cast<uint32_t>(k & ((uint64_t{1} << L) - 1));
  }
  // self-loops are encoded as this key (itself a self-loop) and dropped
  __host__ __device__ __forceinline__ uint64_t loop_key() const {
    return make((1u << L) - 1, (1u << L) - 1);
  }
};

inline int key_bits(uint64_t n) {
  int L = 1;
  while ((uint64_t{1} << L) < n) ++L;
  return L;
}

// first of each run of equal keys, self-loops excluded
struct UniqueIn {
  const uint64_t* k;
  BatchKeys bk;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    const uint64_t x = k[i];
    return (i == 0 || k[i - 1] != x) && bk.src(x) != bk.dst(x);
  }
};
struct UniqueOut {
  const uint64_t* k;
  BatchKeys bk;
  uint64_t* out;
  __device__ __forceinline__ void operator()(uint64_t i, uint64_t pre) const {
    if (UniqueIn{k, bk}(i)) out[pre] = k[i];
  }
};

// LSD radix sort of `count` keys over 2L bits (CUB onesweep), then unique.
// keys_in is clobbered; returns the unique count, result in *out.
inline uint64_t sort_unique_keys(gbg_graph* g, uint64_t* keys_in, uint64_t* scratch, uint64_t count, BatchKeys bk,
                                 uint64_t* out, const char* tag) {
  size_t temp = 0;
  GBG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, keys_in, scratch, count, 0, 2 * bk.L, g->stream));
  void* tmp = g->ws.get(std::string(tag) + ".cubtmp", temp);
  GBG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, temp, keys_in, scratch, count, 0, 2 * bk.L, g->stream));
  g->launches += static_cast<uint64_t>((2 * bk.L + 7) / 8) + 1;
  uint64_t* cnt = g->ws.get<uint64_t>(std::string(tag) + ".ucnt", 1);
  device_scan<uint64_t>(g, UniqueIn{scratch, bk}, UniqueOut{scratch, bk, out}, count, cnt,
                        (std::string(tag) + ".uniq").c_str());
  uint64_t U = 0;
  read_scalars(g, cnt, sizeof(U), &U);
  g->ws.release(std::string(tag) + ".cubtmp");
  return U;
}

}  // namespace gbg

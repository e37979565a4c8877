// Packed arc keys and the device "prepare" steps shared by the R-MAT
// generator (generators.cpp:9-29: sort + unique) and the batch update path
// (batch.cpp:34-42: drop self-loops, sort, unique).
//
// An arc (s,d) with ids < 2^L packs into the 2L-bit key s<<L | d, whose
// numeric order is the reference's lexicographic Edge order
// (types.hpp:21-25), so sorting keys == std::sort on Edges.
#pragma once

#include "radix.cuh"

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
    const uint32_t all = static_cast<uint32_t>((uint64_t{1} << L) - 1);  // L may be 32
    return make(all, all);
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

// Stable LSD radix sort of `count` keys over 2L bits (radix.cuh), then
// unique.  a and b are both clobbered; returns the buffer (a or b) that
// holds the *U_out unique keys — the other one is free scratch afterwards.
inline uint64_t* sort_unique_keys(gbg_graph* g, uint64_t* a, uint64_t* b, uint64_t count, BatchKeys bk,
                                  uint64_t* U_out, const char* tag) {
  uint64_t* sorted = radix_sort_u64(g, a, b, count, 2 * bk.L, tag);
  uint64_t* other = sorted == a ? b : a;
  uint64_t* cnt = g->ws.get<uint64_t>(std::string(tag) + ".ucnt", 1);
  device_scan<uint64_t>(g, UniqueIn{sorted, bk}, UniqueOut{sorted, bk, other}, count, cnt,
                        (std::string(tag) + ".uniq").c_str());
  read_scalars(g, cnt, sizeof(*U_out), U_out);
  return other;
}

}  // namespace gbg

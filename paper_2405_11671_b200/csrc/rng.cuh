// Counter-based splitmix64 streams, restating rng.hpp:11-29 of the
// reference: every (seed, stream, counter) triple maps to an independent
// value, so device threads draw the reference's exact numbers.
#pragma once

#include <cstdint>

namespace gbg {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
  return mix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}
__host__ __device__ __forceinline__ uint64_t rng_u64(uint64_t seed, uint64_t stream, uint64_t counter) {
  return mix64(hash_combine(hash_combine(seed, stream), counter));
}

}  // namespace gbg

// L2 residency control for the gather-heavy kernels: streamed arrays
// (neighbour ids, offsets) are loaded with an evict_first policy so they do
// not push the gathered vector (evict_last) out of the 126 MB L2.
#pragma once

#include <stdint.h>

namespace gbg {

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* a, uint64_t pol) {
  uint64_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep_f64(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
// hot gathers: keep in L1 as well; cold gathers: do not allocate in L1 (so
// they cannot evict the hot lines)
__device__ __forceinline__ double ld_hot_f64(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_cold_f64(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}

}  // namespace gbg

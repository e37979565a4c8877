// Counter-based splitmix64 streams, restating rng.hpp:11-29 of the
// reference: every (seed, stream, counter) triple maps to an independent
// value, so device threads draw the reference's exact numbers.
#pragma once

#include <math_constants.h>

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

// rng.hpp:27-29: top 53 bits times 2^-53
__host__ __device__ __forceinline__ double rng_double(uint64_t seed, uint64_t stream, uint64_t counter) {
  return static_cast<double>(rng_u64(seed, stream, counter) >> 11) * 0x1.0p-53;
}

// log1p exactly as the reference's C library computes it on the hosts this
// image runs on: glibc's double log1p (the classic fdlibm argument
// reduction, 2^k * (1 + f), with the Estrin-ordered degree-14 polynomial in
// s = f / (2 + f)), in the operation order and fused multiply-adds of its
// x86-64 FMA build.  Every product/sum is an explicit _rn intrinsic so nvcc
// cannot contract differently; validated bit-for-bit against the host libm
// (tests/test_gpu_ldd.py).  rng_exponential's shifts feed a floor(), so a
// 1-ulp difference could move a vertex's start round.
__device__ __forceinline__ double libm_log1p(double x) {
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  constexpr double two54 = 1.80143985094819840000e+16;
  constexpr double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
                   Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                   Lp7 = 1.479819860511658591e-01;
  const int32_t hx = static_cast<int32_t>(__double2hiint(x));
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {  // x < 0.41422
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (__dadd_rn(two54, x) > 0.0 && ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= static_cast<int32_t>(0xbfd2bec3)) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return __dadd_rn(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double dk = static_cast<double>(k);
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) return k == 0 ? 0.0 : __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    const double R = __dmul_rn(hfsq, __fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double R = __fma_rn(z6, R4, __fma_rn(z4, R3, __fma_rn(z, Lp1, __dmul_rn(z2, R2))));
  const double t = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(t, __fma_rn(dk, ln2_lo, c))), f));
}

// rng.hpp:31-35
__device__ __forceinline__ double rng_exponential(uint64_t seed, uint64_t stream, uint64_t counter, double rate) {
  const double u = rng_double(seed, stream, counter);
  return __ddiv_rn(-libm_log1p(-u), rate);
}

}  // namespace gbg

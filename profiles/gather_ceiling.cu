// Gather-ceiling microbenchmark for the PageRank pull:
// how fast can one B200 do the pull's unavoidable work -- one 8-byte gather
// of the degree-ordered contribution vector per arc -- if it did nothing
// else?  No row sums, no finalize: each thread streams arc source ids
// (4 B, coalesced, evict_first) and gathers T[id] (8 B, evict_last so the
// hot part of T stays in L2), summing into a per-warp total.  A streaming
// kernel over the same byte count (ids + one contiguous 8-byte word per
// arc) gives the HBM reference.  Build (profiles/gather_ceiling.py does it):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC \
//        -o profiles/_gather/libgather.so profiles/gather_ceiling.cu
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_ids(const uint4* a, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned long long ld_gather(const unsigned long long* a, uint64_t pol) {
  unsigned long long v;
  asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// each thread: 8 ids per step (two 16-byte loads), then 8 gathers in flight
__global__ void __launch_bounds__(256) gather_k(const uint32_t* ids, uint64_t m, const unsigned long long* T,
                                                unsigned long long* out) {
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t nq = m / 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint4 a = ld_ids(reinterpret_cast<const uint4*>(ids) + 2 * q, pf);
    const uint4 b = ld_ids(reinterpret_cast<const uint4*>(ids) + 2 * q + 1, pf);
    const uint32_t u[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    unsigned long long x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = ld_gather(T + u[k], pl);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
  }
  for (uint64_t e = nq * 8 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += stride) s += T[ids[e]];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// same bytes, no gather: ids + one contiguous 8-byte word per arc
__global__ void __launch_bounds__(256) stream_k(const uint32_t* ids, uint64_t m, const unsigned long long* V,
                                                unsigned long long* out) {
  const uint64_t pf = pol_first();
  const uint64_t nq = m / 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint4 a = ld_ids(reinterpret_cast<const uint4*>(ids) + 2 * q, pf);
    const uint4 b = ld_ids(reinterpret_cast<const uint4*>(ids) + 2 * q + 1, pf);
    s += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = ld_ids(reinterpret_cast<const uint4*>(V) + 4 * q + k, pf);
      s += v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}
}  // namespace

extern "C" int gc_run(int kind, const uint32_t* ids, uint64_t m, const unsigned long long* T, unsigned long long* out,
                      int reps, float* ms) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fn = kind == 0 ? (void*)gather_k : (void*)stream_k;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0);
  const int grid = sms * per;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) {
    if (kind == 0) gather_k<<<grid, 256>>>(ids, m, T, out);
    else stream_k<<<grid, 256>>>(ids, m, T, out);
  }
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) {
    if (kind == 0) gather_k<<<grid, 256>>>(ids, m, T, out);
    else stream_k<<<grid, 256>>>(ids, m, T, out);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  *ms /= reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return static_cast<int>(cudaGetLastError());
}

// Grid-barrier cost on B200: cooperative_groups grid.sync() at several
// grid shapes vs a two-level barrier (one arrival per CTA on a per-group
// counter, then one per group on the root).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_bench gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void cg_sync_k(int iters, unsigned long long* out) {
  cg::grid_group grid = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

// sense-reversing barrier: counters[0..G) per group of CTAs, counters[G] root, flag at [G+1]
__device__ __forceinline__ void tree_sync(unsigned* ctr, unsigned ngroups, unsigned per_group, unsigned& sense) {
  __syncthreads();
  if (threadIdx.x == 0) {
    sense ^= 1u;
    const unsigned grp = blockIdx.x / per_group;
    const unsigned gsize = min(per_group, gridDim.x - grp * per_group);
    volatile unsigned* flag = ctr + ngroups + 1;
    __threadfence();
    if (atomicAdd(ctr + grp, 1u) == gsize - 1) {
      ctr[grp] = 0;
      if (atomicAdd(ctr + ngroups, 1u) == ngroups - 1) {
        ctr[ngroups] = 0;
        __threadfence();
        *flag = sense;
      }
    }
    while (*flag != sense) {
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void tree_sync_k(int iters, unsigned* ctr, unsigned per_group, unsigned long long* out) {
  const unsigned ngroups = (gridDim.x + per_group - 1) / per_group;
  unsigned sense = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) tree_sync(ctr, ngroups, per_group, sense);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  unsigned* ctr;
  cudaMalloc(&d, 8);
  cudaMalloc(&ctr, 4096);
  const int iters = 2000;
  struct Shape { int per_sm, threads; } shapes[] = {{8, 256}, {4, 256}, {2, 1024}, {1, 1024}, {1, 256}};
  for (auto sh : shapes) {
    int grid = sms * sh.per_sm;
    void* args[] = {(void*)&iters, (void*)&d};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)cg_sync_k, grid, sh.threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)cg_sync_k, grid, sh.threads, args, 0, 0);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync   %4d x %4d: %.3f us/sync (%s)\n", grid, sh.threads, ms * 1000 / iters, cudaGetErrorString(e));
    for (unsigned pg : {8u, 16u, 37u}) {
      cudaMemset(ctr, 0, 4096);
      void* a2[] = {(void*)&iters, (void*)&ctr, (void*)&pg, (void*)&d};
      cudaLaunchCooperativeKernel((void*)tree_sync_k, grid, sh.threads, a2, 0, 0);
      cudaMemset(ctr, 0, 4096);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)tree_sync_k, grid, sh.threads, a2, 0, 0);
      cudaEventRecord(b);
      e = cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("tree_sync/%2u %4d x %4d: %.3f us/sync (%s)\n", pg, grid, sh.threads, ms * 1000 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}

// Low-diameter decomposition (randomised ball growing).
//
// Reference: gb::ldd (algorithms.cpp:114-188).  Every vertex draws a start
// shift Exponential(beta) from the counter RNG (rng_exponential(seed, v, 0),
// rng.hpp:31-35) and starts its own cluster at round
// floor(max_shift - shift) unless a wavefront reached it first; rounds are
// synchronous, ties go to the lowest centre id, and each joined vertex
// records its round and a tree parent (the smallest same-cluster neighbour
// from an earlier round; itself at centres).  Everything is min-based and
// order-independent, so the device rounds give the reference's exact
// labels, parents and rounds — provided the shifts are bit-identical, which
// libm_log1p (rng.cuh) guarantees.
//
// Per round r on the device:
//   join   one pass over the unlabeled vertices: candidate (min arriving
//          centre) or, when start <= r, the vertex itself; joined vertices
//          form the next frontier (id list + degree prefix, packed emission)
//   grow   one balanced push over the frontier's arcs (v -> u) does both
//          what the reference does at the end of round r (parent of v: min
//          u with label[u] == label[v] and round[u] < r) and at the start
//          of round r + 1 (arrival: candidate[u] = min(candidate[u],
//          label[v]) for unlabeled u) — the conditions are disjoint and
//          labels do not change in between.
#include <cstdio>

#include "rng.cuh"
#include "traverse.cuh"

namespace gbg {

namespace {

constexpr uint32_t kNone = 0xffffffffu;  // kNoVertex

__global__ void ldd_shift_k(uint64_t n, uint64_t seed, double beta, double* shift, unsigned long long* max_bits) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double local = 0.0;  // algorithms.cpp:130: max_shift starts at 0.0
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    const double s = rng_exponential(seed, v, 0, beta);
    shift[v] = s;
    local = s > local ? s : local;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_xor_sync(0xffffffffu, local, o);
    local = other > local ? other : local;
  }
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(local)));
}

__global__ void ldd_init_k(uint64_t n, const double* shift, const unsigned long long* max_bits, uint64_t* start,
                           uint32_t* label, uint32_t* cand, uint32_t* parent, uint64_t* rounds) {
  const double max_shift = __longlong_as_double(static_cast<long long>(*max_bits));
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    start[v] = static_cast<uint64_t>(floor(__dsub_rn(max_shift, shift[v])));
    label[v] = kNone;
    cand[v] = kNone;
    parent[v] = kNone;
    rounds[v] = 0;
  }
}

// join pass: label the unlabeled vertices that have a candidate (or whose
// start has come), emit them as the next frontier
template <class G>
__global__ void ldd_join_k(G g, uint64_t r, const uint64_t* start, uint32_t* label, const uint32_t* cand,
                           uint64_t* rounds, uint32_t* list, uint64_t* dscan, unsigned long long* packed) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < g.n; base += stride) {
    const uint64_t v = base + threadIdx.x;
    bool take = false;
    uint64_t dv = 0;
    if (v < g.n && label[v] == kNone) {
      uint32_t c = cand[v];
      if (start[v] <= r && static_cast<uint32_t>(v) < c) c = static_cast<uint32_t>(v);
      if (c != kNone) {
        label[v] = c;
        rounds[v] = r;
        take = true;
        dv = g.degree(static_cast<uint32_t>(v));
      }
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, take);
    if (!mask) continue;
    const uint64_t dinc = warp_inclusive_scan(dv);
    const uint64_t dtot = __shfl_sync(0xffffffffu, dinc, 31);
    const int leader = __ffs(mask) - 1;
    unsigned long long old = 0;
    if (lane == leader) old = atomicAdd(packed, (static_cast<unsigned long long>(__popc(mask)) << kPackShift) | dtot);
    old = __shfl_sync(0xffffffffu, old, leader);
    if (take) {
      const uint64_t pos = pack_count(old) + __popc(mask & ((1u << lane) - 1));
      list[pos] = static_cast<uint32_t>(v);
      dscan[pos] = pack_degsum(old) + dinc - dv;
    }
  }
}

// grow: arrivals for round r + 1 and tree parents of round r's joiners
struct LddGrowOp {
  const uint32_t* label;
  uint32_t* cand;
  uint32_t* parent;
  const uint64_t* rounds;
  uint64_t r;
  __device__ __forceinline__ bool cond(uint32_t) const { return true; }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t v, uint32_t u) const {
    const uint32_t lu = label[u], lv = label[v];
    if (lu == kNone) {
      atomicMin(cand + u, lv);
    } else if (lu == lv && rounds[u] < r) {
      atomicMin(parent + v, u);
    }
    return false;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

__global__ void ldd_centres_k(const uint32_t* list, uint64_t k, const uint32_t* label, uint32_t* parent) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
    const uint32_t v = list[i];
    if (label[v] == v && parent[v] == kNone) parent[v] = v;
  }
}

template <class G>
void ldd_run(gbg_graph* g, G view, double beta, uint64_t seed, uint32_t* label, uint32_t* parent, uint64_t* rounds) {
  const uint64_t n = g->n;
  double* shift = g->ws.get<double>("ldd.shift", n);
  uint64_t* start = g->ws.get<uint64_t>("ldd.start", n);
  uint32_t* cand = g->ws.get<uint32_t>("ldd.cand", n);
  uint32_t* list = g->ws.get<uint32_t>("ldd.list", n + 1);
  uint64_t* dscan = g->ws.get<uint64_t>("ldd.dscan", n + 1);
  unsigned long long* sc = g->ws.get<unsigned long long>("ldd.sc", 2);  // [0] max shift bits, [1] packed
  PhaseTrace tr(g->stream, "ldd");
  GBG_CUDA(cudaMemsetAsync(sc, 0, 2 * sizeof(unsigned long long), g->stream));
  const unsigned grid = grid_for(n, 256, static_cast<unsigned>(g->sm_count) * 8u);
  GBG_LAUNCH(g, ldd_shift_k, grid, 256, 0, n, seed, beta, shift, sc);
  GBG_LAUNCH(g, ldd_init_k, grid, 256, 0, n, shift, sc, start, label, cand, parent, rounds);
  tr.mark("shifts");
  uint64_t labeled = 0, r = 0;
  while (labeled < n) {
    GBG_CUDA(cudaMemsetAsync(sc + 1, 0, sizeof(unsigned long long), g->stream));
    GBG_LAUNCH(g, ldd_join_k<G>, grid, 256, 0, view, r, start, label, cand, rounds, list, dscan, sc + 1);
    unsigned long long p = 0;
    read_scalars(g, sc + 1, sizeof(p), &p);
    const uint64_t k = pack_count(p), E = pack_degsum(p);
    labeled += k;
    if (k) {
      push_list(g, view, list, k, dscan, E, LddGrowOp{label, cand, parent, rounds, r}, nullptr, nullptr, sc);
      GBG_LAUNCH(g, ldd_centres_k, grid_for(k, 256), 256, 0, list, k, label, parent);
    }
    ++r;
  }
  tr.mark("rounds");
  if (PhaseTrace::enabled()) std::fprintf(stderr, "[gbg] ldd: %llu rounds\n", (unsigned long long)r);
}

__global__ void log1p_k(const double* x, uint64_t n, double* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) out[i] = libm_log1p(x[i]);
}

}  // namespace

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_ldd(gbg_graph* g, double beta, uint64_t seed, uint32_t* labels, uint32_t* parents, uint64_t* rounds) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!(beta > 0.0 && beta <= 1.0)) fail(GBG_ERR_INVALID_ARGUMENT, "ldd: beta must be in (0, 1]");
    if (!labels && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    if (!g->n) return;
    const uint64_t n = g->n;
    uint32_t* dl = g->ws.get<uint32_t>("ldd.label", n);
    uint32_t* dp = g->ws.get<uint32_t>("ldd.parent", n);
    uint64_t* dr = g->ws.get<uint64_t>("ldd.rounds", n);
    with_view(g, [&](auto view) { ldd_run(g, view, beta, seed, dl, dp, dr); });
    GBG_CUDA(cudaMemcpyAsync(labels, dl, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    if (parents) GBG_CUDA(cudaMemcpyAsync(parents, dp, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    if (rounds) GBG_CUDA(cudaMemcpyAsync(rounds, dr, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_selftest_log1p(const double* x, uint64_t n, double* out) {
  return guard([&] {
    if (!n) return;
    if (!x || !out) fail(GBG_ERR_INVALID_ARGUMENT, "null buffer");
    double *dx = nullptr, *dy = nullptr;
    GBG_CUDA(cudaMalloc(&dx, n * sizeof(double)));
    GBG_CUDA(cudaMalloc(&dy, n * sizeof(double)));
    GBG_CUDA(cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice));
    log1p_k<<<grid_for(n, 256), 256>>>(dx, n, dy);
    GBG_CUDA(cudaGetLastError());
    GBG_CUDA(cudaMemcpy(out, dy, n * sizeof(double), cudaMemcpyDeviceToHost));
    GBG_CUDA(cudaFree(dx));
    GBG_CUDA(cudaFree(dy));
  });
}

}  // extern "C"

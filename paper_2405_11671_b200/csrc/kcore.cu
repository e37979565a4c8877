// k-core decomposition (coreness per vertex).
//
// Reference: gb::kcore (algorithms.cpp:330-374) over the monotone bucket
// queue gb::Buckets (buckets.cpp:7-59): peel the lowest non-empty degree
// bucket k, decrement the remaining degree of not-yet-peeled neighbours,
// move them to bucket max(k, remaining).  Coreness is unique (the peel is
// monotone), so any peeling order gives the reference's output.
//
// Device version, level by level:
//   select  a pass over the alive list peels every vertex with remaining
//           degree <= k (coreness := k) into a frontier list with its
//           degree prefix (packed emission, traverse.cuh), compacts the
//           survivors into the next alive list and takes their minimum
//           remaining degree (the next non-empty level when nothing peels);
//   push    rounds over the frontier decrement alive neighbours; one whose
//           remaining degree crosses k+1 -> k is peeled at this level and
//           emitted into the next round's frontier.
// Compacting the alive list makes the selects cost sum_v coreness(v)
// instead of levels * n.  All levels run inside one persistent cooperative
// launch with grid barriers between steps (the BFS pattern, bfs.cu); a
// launch-per-step host loop is the fallback.
#include <cooperative_groups.h>

#include <cstdio>
#include <vector>

#include "traverse.cuh"

namespace gbg {

namespace {

constexpr int64_t kUnset = -1;

template <class G>
__global__ void kcore_init_k(G g, int32_t* deg, int64_t* core) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < g.n; v += stride) {
    deg[v] = static_cast<int32_t>(g.degree(static_cast<uint32_t>(v)));
    core[v] = kUnset;
  }
}

// Step counters: [0] packed frontier (count << 36 | degree sum), [1]
// survivors, [2] minimum survivor degree (reset to all-ones).
constexpr int kSlot = 4;

__device__ __forceinline__ void reset_slot(unsigned long long* c) {
  c[0] = 0;
  c[1] = 0;
  c[2] = ~0ull;
}

// One select pass (grid-stride): items [0, na) of `alive` (or the identity
// when alive == nullptr).
template <class G>
__device__ void kcore_select(G g, int32_t* deg, int64_t* core, int64_t k, const uint32_t* alive, uint64_t na,
                             uint32_t* survivors, uint32_t* list, uint64_t* dscan, unsigned long long* c) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long local_min = ~0ull;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < na; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool take = false, keep = false;
    uint32_t v = 0;
    uint64_t dv = 0;
    if (i < na) {
      v = alive ? __ldcg(alive + i) : static_cast<uint32_t>(i);
      if (__ldcg(core + v) == kUnset) {  // L2 loads: written by other CTAs in earlier steps
        const int d = __ldcg(deg + v);
        if (d <= k) {
          take = true;
          core[v] = k;
          dv = g.degree(v);
        } else {
          keep = true;
          if (static_cast<unsigned long long>(d) < local_min) local_min = static_cast<unsigned long long>(d);
        }
      }
    }
    const uint32_t tmask = __ballot_sync(0xffffffffu, take);
    if (tmask) {
      const uint64_t dinc = warp_inclusive_scan(dv);
      const uint64_t dtot = __shfl_sync(0xffffffffu, dinc, 31);
      const int leader = __ffs(tmask) - 1;
      unsigned long long old = 0;
      if (lane == leader) old = atomicAdd(c, (static_cast<unsigned long long>(__popc(tmask)) << kPackShift) | dtot);
      old = __shfl_sync(0xffffffffu, old, leader);
      if (take) {
        const uint64_t pos = pack_count(old) + __popc(tmask & ((1u << lane) - 1));
        list[pos] = v;
        dscan[pos] = pack_degsum(old) + dinc - dv;
      }
    }
    const uint32_t kmask = __ballot_sync(0xffffffffu, keep);
    if (kmask) {
      const int leader = __ffs(kmask) - 1;
      unsigned long long old = 0;
      if (lane == leader) old = atomicAdd(c + 1, static_cast<unsigned long long>(__popc(kmask)));
      old = __shfl_sync(0xffffffffu, old, leader);
      if (keep) survivors[old + __popc(kmask & ((1u << lane) - 1))] = v;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, local_min, o);
    local_min = other < local_min ? other : local_min;
  }
  if (lane == 0 && local_min != ~0ull) atomicMin(c + 2, local_min);
}

template <class G>
__global__ void kcore_select_k(G g, int32_t* deg, int64_t* core, int64_t k, const uint32_t* alive, uint64_t na,
                               uint32_t* survivors, uint32_t* list, uint64_t* dscan, unsigned long long* c) {
  kcore_select(g, deg, core, k, alive, na, survivors, list, dscan, c);
}

// push operator: decrement alive neighbours; emit (and peel at level k) the
// ones crossing k+1 -> k
struct KcoreOp {
  int32_t* deg;
  int64_t* core;
  int64_t k;
  __device__ __forceinline__ bool cond(uint32_t v) const {
    return *reinterpret_cast<volatile int64_t*>(core + v) == kUnset;
  }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t, uint32_t v) const {
    const int32_t old = atomicSub(deg + v, 1);
    if (old == k + 1) {
      core[v] = k;
      return true;
    }
    return false;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

struct KcoreCoop {
  int32_t* deg;
  int64_t* core;
  uint32_t* alive[2];
  uint32_t* list[2];
  uint64_t* dscan[2];
  unsigned long long* slot;   // [3][kSlot] step counters, ring of three
  unsigned long long* stats;  // [0] levels peeled, [1] steps
};

// Step s writes slot s % 3, reads slot (s - 1) % 3 after the barrier, and
// resets slot (s + 1) % 3 (last read at the start of step s - 1).
template <class G>
__global__ void __launch_bounds__(kPushThreads, 4) kcore_coop_k(G g, KcoreCoop s) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ uint32_t s_idx[kPushTile];
  const bool t0 = blockIdx.x == 0 && threadIdx.x == 0;
  uint64_t step = 0, levels = 0, na = g.n;
  int ca = 0, cf = 0;
  bool identity = true;
  int64_t k = 0;
  for (;;) {
    unsigned long long* c = s.slot + (step % 3) * kSlot;
    if (t0) reset_slot(s.slot + ((step + 1) % 3) * kSlot);
    kcore_select(g, s.deg, s.core, k, identity ? nullptr : s.alive[ca], na, s.alive[ca ^ 1], s.list[cf],
                 s.dscan[cf], c);
    grid.sync();
    unsigned long long p = *reinterpret_cast<volatile unsigned long long*>(c);
    na = *reinterpret_cast<volatile unsigned long long*>(c + 1);
    const unsigned long long minv = *reinterpret_cast<volatile unsigned long long*>(c + 2);
    identity = false;
    ca ^= 1;
    ++step;
    if (pack_count(p) == 0) {
      if (na == 0) break;
      k = static_cast<int64_t>(minv);  // no vertex at this level: jump to the lowest remaining degree
      continue;
    }
    ++levels;
    const KcoreOp op{s.deg, s.core, k};
    while (pack_count(p) > 0) {
      const uint64_t size = pack_count(p), degsum = pack_degsum(p);
      c = s.slot + (step % 3) * kSlot;
      if (t0) reset_slot(s.slot + ((step + 1) % 3) * kSlot);
      const uint32_t ipt = push_ipt(degsum, gridDim.x);
      const uint64_t tiles = push_tiles(degsum, ipt);
      for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        push_tile(g, s.list[cf], static_cast<uint32_t>(size), s.dscan[cf], degsum, op, s.list[cf ^ 1],
                  s.dscan[cf ^ 1], static_cast<uint32_t*>(nullptr), c, t, s_idx, ipt);
        __syncthreads();
      }
      grid.sync();
      p = *reinterpret_cast<volatile unsigned long long*>(c);
      cf ^= 1;
      ++step;
    }
    if (na == 0) break;
    ++k;
  }
  if (t0) {
    s.stats[0] = levels;
    s.stats[1] = step;
  }
}

template <class G>
void kcore_run(gbg_graph* g, G view, int64_t* core) {
  const uint64_t n = g->n;
  int32_t* deg = g->ws.get<int32_t>("kc.deg", n);
  uint32_t* alive[2] = {g->ws.get<uint32_t>("kc.a0", n), g->ws.get<uint32_t>("kc.a1", n)};
  uint32_t* list[2] = {g->ws.get<uint32_t>("kc.l0", n + 1), g->ws.get<uint32_t>("kc.l1", n + 1)};
  uint64_t* dscan[2] = {g->ws.get<uint64_t>("kc.d0", n + 1), g->ws.get<uint64_t>("kc.d1", n + 1)};
  unsigned long long* slot = g->ws.get<unsigned long long>("kc.slot", 3 * kSlot + 2);
  PhaseTrace tr(g->stream, "kcore");
  GBG_LAUNCH(g, kcore_init_k<G>, grid_for(n, 256), 256, 0, view, deg, core);
  std::vector<unsigned long long> init(3 * kSlot + 2, 0);
  for (int i = 0; i < 3; ++i) init[i * kSlot + 2] = ~0ull;
  GBG_CUDA(cudaMemcpyAsync(slot, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                           g->stream));
  GBG_CUDA(cudaStreamSynchronize(g->stream));  // `init` is pageable and goes out of scope

  int per_sm = 0;
  const int coop = coop_enabled(g->device) ? 1 : 0;
  GBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kcore_coop_k<G>, kPushThreads, 0));
  if (coop && per_sm > 0) {
    KcoreCoop s{deg, core, {alive[0], alive[1]}, {list[0], list[1]}, {dscan[0], dscan[1]}, slot, slot + 3 * kSlot};
    void* args[] = {&view, &s};
    GBG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kcore_coop_k<G>),
                                         static_cast<unsigned>(per_sm * g->sm_count), kPushThreads, args, 0,
                                         g->stream));
    g->launches++;
    tr.mark("peel");
    if (PhaseTrace::enabled()) {
      unsigned long long st[2];
      read_scalars(g, slot + 3 * kSlot, sizeof(st), st);
      std::fprintf(stderr, "[gbg] kcore: %llu levels, %llu steps (cooperative)\n", st[0], st[1]);
    }
    return;
  }
  // fallback: the same steps, one launch each, counters read back by the host
  const unsigned grid = grid_for(n, 256, static_cast<unsigned>(g->sm_count) * 8u);
  const unsigned long long reset[kSlot] = {0, 0, ~0ull, 0};
  uint64_t na = n;
  int ca = 0, cf = 0;
  bool identity = true;
  int64_t k = 0;
  for (;;) {
    GBG_CUDA(cudaMemcpyAsync(slot, reset, sizeof(reset), cudaMemcpyHostToDevice, g->stream));
    GBG_LAUNCH(g, kcore_select_k<G>, grid, 256, 0, view, deg, core, k, identity ? nullptr : alive[ca], na,
               alive[ca ^ 1], list[cf], dscan[cf], slot);
    unsigned long long h[3];
    read_scalars(g, slot, sizeof(h), h);
    na = h[1];
    identity = false;
    ca ^= 1;
    uint64_t size = pack_count(h[0]), E = pack_degsum(h[0]);
    if (size == 0) {
      if (na == 0) break;
      k = static_cast<int64_t>(h[2]);
      continue;
    }
    while (size > 0) {
      GBG_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned long long), g->stream));
      push_list(g, view, list[cf], size, dscan[cf], E, KcoreOp{deg, core, k}, list[cf ^ 1], dscan[cf ^ 1], slot);
      unsigned long long p = 0;
      read_scalars(g, slot, sizeof(p), &p);
      size = pack_count(p);
      E = pack_degsum(p);
      cf ^= 1;
    }
    if (na == 0) break;
    ++k;
  }
  tr.mark("peel");
}

}  // namespace

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_kcore(gbg_graph* g, uint64_t* coreness) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!coreness && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    if (!g->n) return;
    int64_t* d = g->ws.get<int64_t>("kc.core", g->n);
    with_view(g, [&](auto view) { kcore_run(g, view, d); });
    GBG_CUDA(cudaMemcpyAsync(coreness, d, g->n * sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"

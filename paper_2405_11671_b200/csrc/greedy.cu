// Priority-order greedy algorithms: maximal independent set and coloring.
//
// Reference: gb::mis (algorithms.cpp:434-504) and gb::coloring
// (algorithms.cpp:376-432).  Both fix a total priority order ("beats") and
// resolve vertices in rounds: waiting[v] counts the neighbours that beat v,
// a vertex is ready when the count reaches zero, and resolving a vertex
// releases (decrements) its lower-priority neighbours.  The result is the
// sequential greedy answer in priority order (lexicographically-first MIS
// under (rank, id); first-fit coloring in largest-log-degree-first order),
// so it is independent of the schedule and the device output is identical.
//
// Device rounds are the reference's rounds: a frontier list with its degree
// prefix (packed emission, traverse.cuh), the knock-out / release steps as
// load-balanced pushes (push_list) whose update returns true exactly when a
// neighbour's waiting count hits zero, and the initial waiting counts from
// one balanced pass over all edges (row_count, edges.cuh).
//
// Both need every arc's reverse: on a directed graph the reference's own
// result depends on the OpenMP schedule (mis) or reads uncoloured
// neighbours (coloring), so asymmetric input is rejected.
#include <cooperative_groups.h>

#include <cstdio>

#include "edges.cuh"
#include "rng.cuh"
#include "traverse.cuh"

namespace gbg {

namespace {

constexpr uint32_t kUndecided = 0, kIn = 1, kOut = 2;
constexpr uint32_t kUncolored = 0xffffffffu;

// mis: lower (rank, id) wins (algorithms.cpp:438-440)
struct RankBeats {
  const uint64_t* rank;
  __device__ __forceinline__ bool operator()(uint32_t a, uint32_t b) const {
    const uint64_t ra = rank[a], rb = rank[b];
    return ra != rb ? ra < rb : a < b;
  }
};
// coloring: higher bit_width(degree) first, ties to the lower id
// (algorithms.cpp:378-385)
struct LlfBeats {
  const uint8_t* llf;
  __device__ __forceinline__ bool operator()(uint32_t a, uint32_t b) const {
    const uint32_t la = llf[a], lb = llf[b];
    return la != lb ? la > lb : a < b;
  }
};
// row_count predicate: neighbour v beats row u
template <class Beats>
struct BeatenBy {
  Beats beats;
  __device__ __forceinline__ bool operator()(uint32_t u, uint32_t v) const { return beats(v, u); }
};
struct Ready {
  const uint32_t* waiting;
  __device__ __forceinline__ bool operator()(uint32_t v) const { return waiting[v] == 0; }
};

__global__ void mis_init_k(uint64_t n, uint64_t seed, uint64_t* rank, uint32_t* status, uint32_t* waiting) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    rank[v] = rng_u64(seed, 7, v);  // algorithms.cpp:437
    status[v] = kUndecided;
    waiting[v] = 0;
  }
}

template <class G>
__global__ void coloring_init_k(G g, uint8_t* llf, uint32_t* colors, uint32_t* waiting) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < g.n; v += stride) {
    const uint64_t d = g.degree(static_cast<uint32_t>(v));
    llf[v] = static_cast<uint8_t>(d ? 64 - __clzll(d) : 0);  // std::bit_width
    colors[v] = kUncolored;
    waiting[v] = 0;
  }
}

__global__ void mark_in_k(const uint32_t* list, uint64_t k, uint32_t* status) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) status[list[i]] = kIn;
}

__global__ void mis_out_k(uint64_t n, const uint32_t* status, uint8_t* in_set) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    in_set[v] = status[v] == kIn ? 1 : 0;
}

// joiners knock their undecided neighbours out (algorithms.cpp:468-476)
struct KnockOutOp {
  uint32_t* status;
  __device__ __forceinline__ bool cond(uint32_t v) const {
    return *reinterpret_cast<volatile uint32_t*>(status + v) == kUndecided;
  }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t, uint32_t v) const {
    return atomicCAS(status + v, kUndecided, kOut) == kUndecided;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

// a decided vertex releases its undecided lower-priority neighbours; the
// one that drops a count to zero emits it (algorithms.cpp:481-491)
struct MisReleaseOp {
  RankBeats beats;
  const uint32_t* status;
  uint32_t* waiting;
  __device__ __forceinline__ bool cond(uint32_t v) const { return status[v] == kUndecided; }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t u, uint32_t v) const {
    return beats(u, v) && atomicSub(waiting + v, 1u) == 1u;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

// a coloured vertex releases every neighbour it is not beaten by
// (algorithms.cpp:418-422; a self-loop decrements its own count, as there)
struct ColorReleaseOp {
  LlfBeats beats;
  uint32_t* waiting;
  __device__ __forceinline__ bool cond(uint32_t) const { return true; }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t u, uint32_t v) const {
    return !beats(v, u) && atomicSub(waiting + v, 1u) == 1u;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

// First-fit colour of each ready vertex: the smallest colour not used by a
// neighbour that beats it (algorithms.cpp:406-417), read from the
// precomputed beater lists (boff / bnbr: only the neighbours that beat v,
// all coloured by the time v is ready), so a hub scans its few beaters
// instead of its whole adjacency.  A lane takes a vertex with < 64 beaters
// alone with a 64-bit used-mask (the answer is below 64); longer lists go
// to a heavy list that color_heavy_k scans with a whole CTA per vertex into
// a shared bitmap window, sliding the window while every colour in it is
// taken.  Rounds are short chains of mid-degree vertices, so the heavy scan
// must not be one warp's serial loop.
constexpr int kColorThreads = 256;
constexpr uint32_t kLightBeaters = 64;
constexpr uint32_t kHeavyWindow = 4096;  // colours per shared bitmap pass

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// true when v was coloured; false when it has too many beaters for a lane
__device__ __forceinline__ bool color_light(uint32_t v, const uint64_t* __restrict__ boff,
                                            const uint32_t* __restrict__ bnbr, uint32_t* colors) {
  const uint64_t b = boff[v], d = boff[v + 1] - b;
  if (d >= kLightBeaters) return false;
  uint64_t used = 0;
#pragma unroll 4
  for (uint32_t j = 0; j < d; ++j) {
    const uint32_t c = __ldcg(colors + bnbr[b + j]);  // coloured by other CTAs in earlier rounds
    if (c < 64) used |= uint64_t{1} << c;
  }
  colors[v] = static_cast<uint32_t>(__ffsll(static_cast<long long>(~used)) - 1);
  return true;
}

// whole-CTA first fit for one heavy vertex (called by every thread)
__device__ void color_heavy(uint32_t x, const uint64_t* __restrict__ boff, const uint32_t* __restrict__ bnbr,
                            uint32_t* colors, uint32_t* s_bm, uint32_t* s_first) {
  const uint64_t b = boff[x], d = boff[x + 1] - b;
  for (uint32_t window = 0;; window += kHeavyWindow) {
    for (uint32_t w = threadIdx.x; w < kHeavyWindow / 32; w += blockDim.x) s_bm[w] = 0;
    if (threadIdx.x == 0) *s_first = 0xffffffffu;
    __syncthreads();
    uint64_t j = threadIdx.x;
    for (; j + 3 * blockDim.x < d; j += 4 * blockDim.x) {  // four gathers in flight per thread
      uint32_t u[4], c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = bnbr[b + j + q * blockDim.x];
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] = colors[u[q]] - window;  // below the window wraps past it
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c[q] < kHeavyWindow) atomicOr(&s_bm[c[q] >> 5], 1u << (c[q] & 31));
    }
    for (; j < d; j += blockDim.x) {
      const uint32_t c = colors[bnbr[b + j]] - window;
      if (c < kHeavyWindow) atomicOr(&s_bm[c >> 5], 1u << (c & 31));
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < kHeavyWindow / 32; w += blockDim.x)
      if (s_bm[w] != 0xffffffffu) atomicMin(s_first, w * 32 + (__ffs(~s_bm[w]) - 1));
    __syncthreads();
    const uint32_t first = *s_first;
    __syncthreads();
    if (first != 0xffffffffu) {
      if (threadIdx.x == 0) colors[x] = window + first;
      return;
    }
  }
}

__global__ void __launch_bounds__(kColorThreads)
    color_light_k(const uint32_t* __restrict__ F, uint32_t nf, const uint64_t* __restrict__ boff,
                  const uint32_t* __restrict__ bnbr, uint32_t* colors, uint32_t* heavy, uint32_t* nheavy) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nf; i += stride) {
    const uint32_t v = F[i];
    if (!color_light(v, boff, bnbr, colors)) heavy[atomicAdd(nheavy, 1u)] = v;
  }
}

__global__ void __launch_bounds__(kColorThreads)
    color_heavy_k(const uint32_t* __restrict__ heavy, const uint32_t* __restrict__ nheavy,
                  const uint64_t* __restrict__ boff, const uint32_t* __restrict__ bnbr, uint32_t* colors) {
  __shared__ uint32_t s_bm[kHeavyWindow / 32];
  __shared__ uint32_t s_first;
  const uint32_t nh = *nheavy;
  for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) color_heavy(heavy[h], boff, bnbr, colors, s_bm, &s_first);
}

// Release with colouring on emission: the lane whose decrement makes v
// ready colours it at once when it has < 64 beaters (all coloured in
// earlier rounds: a beater is coloured before it releases), so the next
// round only releases; heavier vertices are queued for a CTA-wide colouring
// step after the round's barrier.
struct ColorReleaseFusedOp {
  LlfBeats beats;
  uint32_t* waiting;
  const uint64_t* boff;
  const uint32_t* bnbr;
  uint32_t* colors;
  uint32_t* heavy;
  uint32_t* nheavy;
  __device__ __forceinline__ bool cond(uint32_t) const { return true; }
  __device__ __forceinline__ bool claim(uint32_t) const { return true; }
  __device__ __forceinline__ bool update(uint32_t u, uint32_t v) const {
    if (beats(v, u) || atomicSub(waiting + v, 1u) != 1u) return false;
    if (color_light(v, boff, bnbr, colors)) return true;
    heavy[atomicAdd(nheavy, 1u)] = v;
    return false;
  }
  __device__ __forceinline__ void dense_word(uint64_t, uint32_t) const {}
};

// All rounds in one persistent cooperative launch (the BFS pattern,
// bfs.cu): per round, the release push over the vertices coloured last
// round colours the light vertices it makes ready and emits them as the
// next list; after a grid barrier, CTAs colour the heavy ones and append
// them to the same list (a second barrier only in rounds that have heavy
// vertices).  Counters rotate through a ring of three (reset two rounds
// after use).
struct ColorCoop {
  uint32_t* list[2];
  uint64_t* dscan[2];
  unsigned long long* packed;  // [3]
  uint32_t* nheavy;            // [3]
  uint32_t* heavy;
  const uint64_t* boff;
  const uint32_t* bnbr;
  uint32_t* colors;
  LlfBeats beats;
  uint32_t* waiting;
  unsigned long long* rounds;  // [0] rounds, [1] ns in releases, [2] ns in heavy steps (CTA 0)
};

// the initially ready vertices have no beaters: colour 0 (first fit)
__global__ void color_zero_k(const uint32_t* list, const unsigned long long* packed, uint32_t* colors) {
  const uint64_t k = pack_count(*packed);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) colors[list[i]] = 0;
}

template <class G>
__global__ void __launch_bounds__(kPushThreads, 4) color_coop_k(G g, ColorCoop s) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ uint32_t s_idx[kPushTile];
  __shared__ uint32_t s_bm[kHeavyWindow / 32];
  __shared__ uint32_t s_first;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int cur = 0;
  uint64_t r = 0;
  unsigned long long t_rel = 0, t_heavy = 0, t0 = globaltimer_ns();
  for (;; ++r) {
    const unsigned long long p = *reinterpret_cast<volatile unsigned long long*>(s.packed + r % 3);
    const uint64_t size = pack_count(p), degsum = pack_degsum(p);
    if (size == 0) break;
    if (tid == 0) {
      s.packed[(r + 2) % 3] = 0;  // last read two rounds ago
      s.nheavy[(r + 1) % 3] = 0;
    }
    uint32_t* nh_ctr = s.nheavy + r % 3;
    unsigned long long* next_ctr = s.packed + (r + 1) % 3;
    const int nxt = cur ^ 1;
    const ColorReleaseFusedOp op{s.beats, s.waiting, s.boff, s.bnbr, s.colors, s.heavy, nh_ctr};
    const uint32_t ipt = push_ipt(degsum, gridDim.x);
    const uint64_t tiles = push_tiles(degsum, ipt);
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      push_tile(g, s.list[cur], static_cast<uint32_t>(size), s.dscan[cur], degsum, op, s.list[nxt], s.dscan[nxt],
                static_cast<uint32_t*>(nullptr), next_ctr, t, s_idx, ipt);
      __syncthreads();
    }
    grid.sync();
    unsigned long long t1 = globaltimer_ns();
    t_rel += t1 - t0;
    t0 = t1;
    const uint32_t nh = *reinterpret_cast<volatile uint32_t*>(nh_ctr);
    if (nh) {
      for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const uint32_t v = s.heavy[h];
        color_heavy(v, s.boff, s.bnbr, s.colors, s_bm, &s_first);
        if (threadIdx.x == 0) {
          const uint64_t dv = g.degree(v);
          const unsigned long long old = atomicAdd(next_ctr, (1ull << kPackShift) | dv);
          s.list[nxt][pack_count(old)] = v;
          s.dscan[nxt][pack_count(old)] = pack_degsum(old);
        }
      }
      grid.sync();
      t1 = globaltimer_ns();
      t_heavy += t1 - t0;
      t0 = t1;
    }
    cur = nxt;
  }
  if (tid == 0) {
    s.rounds[0] = r;
    s.rounds[1] = t_rel;
    s.rounds[2] = t_heavy;
  }
}

struct WideIn {
  const uint32_t* a;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};

struct Lists {
  uint32_t* id[3];
  uint64_t* dscan[3];
};

Lists frontier_lists(gbg_graph* g, const char* tag) {
  Lists l;
  const std::string t(tag);
  for (int i = 0; i < 3; ++i) {
    l.id[i] = g->ws.get<uint32_t>(t + ".l" + char('0' + i), g->n + 1);
    l.dscan[i] = g->ws.get<uint64_t>(t + ".d" + char('0' + i), g->n + 1);
  }
  return l;
}

template <class G>
void mis_run(gbg_graph* g, G view, uint64_t seed, uint8_t* in_set) {
  const uint64_t n = g->n;
  uint64_t* rank = g->ws.get<uint64_t>("mis.rank", n);
  uint32_t* status = g->ws.get<uint32_t>("mis.status", n);
  uint32_t* waiting = g->ws.get<uint32_t>("mis.wait", n);
  unsigned long long* sc = g->ws.get<unsigned long long>("mis.sc", 2);
  Lists L = frontier_lists(g, "mis");
  const RankBeats beats{rank};
  GBG_LAUNCH(g, mis_init_k, grid_for(n, 256), 256, 0, n, seed, rank, status, waiting);
  row_count(g, view, virtual_offsets(g), g->m, BeatenBy<RankBeats>{beats}, waiting);
  GBG_CUDA(cudaMemsetAsync(sc, 0, 2 * sizeof(unsigned long long), g->stream));
  GBG_LAUNCH(g, (select_k<G, Ready>), grid_for(n, 256, static_cast<unsigned>(g->sm_count) * 8u), 256, 0, view,
             Ready{waiting}, L.id[0], L.dscan[0], sc);
  unsigned long long p[2];
  read_scalars(g, sc, sizeof(p), p);
  int J = 0, O = 1, N = 2;
  uint64_t nj = pack_count(p[0]), ej = pack_degsum(p[0]);
  while (nj > 0) {
    GBG_LAUNCH(g, mark_in_k, grid_for(nj, 256), 256, 0, L.id[J], nj, status);
    GBG_CUDA(cudaMemsetAsync(sc, 0, 2 * sizeof(unsigned long long), g->stream));
    push_list(g, view, L.id[J], nj, L.dscan[J], ej, KnockOutOp{status}, L.id[O], L.dscan[O], sc + 1);
    read_scalars(g, sc + 1, sizeof(p[1]), &p[1]);
    const uint64_t no = pack_count(p[1]), eo = pack_degsum(p[1]);
    const MisReleaseOp rel{beats, status, waiting};
    push_list(g, view, L.id[J], nj, L.dscan[J], ej, rel, L.id[N], L.dscan[N], sc);
    push_list(g, view, L.id[O], no, L.dscan[O], eo, rel, L.id[N], L.dscan[N], sc);
    read_scalars(g, sc, sizeof(p[0]), &p[0]);
    nj = pack_count(p[0]);
    ej = pack_degsum(p[0]);
    std::swap(J, N);
  }
  GBG_LAUNCH(g, mis_out_k, grid_for(n, 256), 256, 0, n, status, in_set);
}

template <class G>
void coloring_run(gbg_graph* g, G view, uint32_t* colors) {
  const uint64_t n = g->n;
  uint8_t* llf = g->ws.get<uint8_t>("col.llf", n);
  uint32_t* waiting = g->ws.get<uint32_t>("col.wait", n);
  // [0..2] packed ready counters, [3..6] rounds + step times, [7..8] heavy counters (u32 x3)
  unsigned long long* sc = g->ws.get<unsigned long long>("col.sc", 9);
  uint32_t* nheavy = reinterpret_cast<uint32_t*>(sc + 7);
  Lists L = frontier_lists(g, "col");
  const LlfBeats beats{llf};
  PhaseTrace tr(g->stream, "coloring");
  GBG_LAUNCH(g, coloring_init_k<G>, grid_for(n, 256), 256, 0, view, llf, colors, waiting);
  const uint64_t* voff = virtual_offsets(g);
  row_count(g, view, voff, g->m, BeatenBy<LlfBeats>{beats}, waiting);
  // beater lists: the neighbours that beat v, gathered once
  uint64_t* boff = g->ws.get<uint64_t>("col.boff", n + 1);
  device_scan<uint64_t>(g, WideIn{waiting}, ArrayOut<uint64_t>{boff}, n, boff + n, "col.scan");
  uint64_t nbeat = 0;
  read_scalars(g, boff + n, sizeof(nbeat), &nbeat);
  uint32_t* bnbr = g->ws.get<uint32_t>("col.bnbr", nbeat);
  uint32_t* cursor = g->ws.get<uint32_t>("col.cursor", n);
  GBG_CUDA(cudaMemsetAsync(cursor, 0, n * sizeof(uint32_t), g->stream));
  row_compact(g, view, voff, g->m, BeatenBy<LlfBeats>{beats}, boff, cursor, bnbr);
  uint32_t* heavy = g->ws.get<uint32_t>("col.heavy", n);
  GBG_CUDA(cudaMemsetAsync(sc, 0, 9 * sizeof(unsigned long long), g->stream));
  GBG_LAUNCH(g, (select_k<G, Ready>), grid_for(n, 256, static_cast<unsigned>(g->sm_count) * 8u), 256, 0, view,
             Ready{waiting}, L.id[0], L.dscan[0], sc);
  tr.mark("setup");
  const ColorReleaseOp rel{beats, waiting};

  int per_sm = 0;
  const int coop = coop_enabled(g->device) ? 1 : 0;
  GBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, color_coop_k<G>, kPushThreads, 0));
  uint64_t rounds = 0;
  if (coop && per_sm > 0) {
    GBG_LAUNCH(g, color_zero_k, grid_for(n, 256), 256, 0, L.id[0], sc, colors);
    ColorCoop cs{{L.id[0], L.id[1]}, {L.dscan[0], L.dscan[1]}, sc, nheavy, heavy, boff, bnbr, colors, beats, waiting,
                 sc + 3};
    void* args[] = {&view, &cs};
    GBG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(color_coop_k<G>),
                                         static_cast<unsigned>(per_sm * g->sm_count), kPushThreads, args, 0,
                                         g->stream));
    g->launches++;
    if (PhaseTrace::enabled()) {
      unsigned long long h[3];
      read_scalars(g, sc + 3, sizeof(h), h);
      rounds = h[0];
      std::fprintf(stderr, "[gbg] coloring: %llu rounds (cooperative): releases %.2f ms, heavy steps %.2f ms\n",
                   h[0], h[1] * 1e-6, h[2] * 1e-6);
    }
  } else {
    unsigned long long p = 0;
    read_scalars(g, sc, sizeof(p), &p);
    int F = 0, N = 1;
    uint64_t nf = pack_count(p), ef = pack_degsum(p);
    while (nf > 0) {
      ++rounds;
      GBG_CUDA(cudaMemsetAsync(nheavy, 0, sizeof(uint32_t), g->stream));
      GBG_LAUNCH(g, color_light_k, grid_for(nf, kColorThreads), kColorThreads, 0, L.id[F], static_cast<uint32_t>(nf),
                 boff, bnbr, colors, heavy, nheavy);
      GBG_LAUNCH(g, color_heavy_k, static_cast<unsigned>(g->sm_count) * 4u, kColorThreads, 0, heavy, nheavy, boff,
                 bnbr, colors);
      GBG_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), g->stream));
      push_list(g, view, L.id[F], nf, L.dscan[F], ef, rel, L.id[N], L.dscan[N], sc);
      read_scalars(g, sc, sizeof(p), &p);
      nf = pack_count(p);
      ef = pack_degsum(p);
      std::swap(F, N);
    }
  }
  tr.mark("rounds");
  if (PhaseTrace::enabled())
    std::fprintf(stderr, "[gbg] coloring: %llu rounds (%s)\n", (unsigned long long)rounds,
                 coop && per_sm > 0 ? "cooperative" : "host loop");
}

void require_symmetric(gbg_graph* g, const char* what) {
  if (!graph_is_symmetric(g))
    fail(GBG_ERR_INVALID_ARGUMENT,
         std::string(what) + " needs a symmetric graph (every arc's reverse present)");
}

}  // namespace

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_mis(gbg_graph* g, uint64_t seed, uint8_t* in_set) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!in_set && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    if (!g->n) return;
    require_symmetric(g, "mis");
    uint8_t* d = g->ws.get<uint8_t>("mis.out", g->n);
    with_view(g, [&](auto view) { mis_run(g, view, seed, d); });
    GBG_CUDA(cudaMemcpyAsync(in_set, d, g->n, cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

gbg_status gbg_coloring(gbg_graph* g, uint32_t* colors) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!colors && g->n) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    if (!g->n) return;
    require_symmetric(g, "coloring");
    uint32_t* d = g->ws.get<uint32_t>("col.out", g->n);
    with_view(g, [&](auto view) { coloring_run(g, view, d); });
    GBG_CUDA(cudaMemcpyAsync(colors, d, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"

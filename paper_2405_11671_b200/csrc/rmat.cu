// Device R-MAT: gb::generate_update_batch and gb::generate_rmat, bit-exact.
//
// Reference: generate_update_batch (batch.cpp:128-154) draws, for i in
// [0, size) and level in [0, log2_n), r = rng_double(seed, i, level)
// (rng.hpp:22-29: splitmix64 counter hash, top 53 bits * 2^-53) and picks a
// quadrant with r < a / a+b / a+b+c, shifting bits of (u, v) MSB first;
// each draw is emitted as (u,v) then (v,u).  generate_rmat
// (generators.cpp:67-72) then normalizes (generators.cpp:9-29): drop
// self-loops, add reverses, sort, unique, n = 2^log2_n.  All of it is
// integer arithmetic plus double compares of exactly-representable values,
// so the device result is bit-identical; the thresholds a+b and a+b+c are
// evaluated on the host in the reference's left-to-right order.
#include <memory>

#include "keys.cuh"
#include "rng.cuh"

namespace gbg {

struct RmatParams {
  double t1, t2, t3;  // a, a+b, a+b+c
  uint32_t log2_n;
  uint64_t seed;
};

__device__ __forceinline__ void rmat_draw(const RmatParams& p, uint64_t i, uint32_t& u, uint32_t& v) {
  const uint64_t h = hash_combine(p.seed, i);
  uint32_t uu = 0, vv = 0;
  for (uint32_t level = 0; level < p.log2_n; ++level) {
    const double r = static_cast<double>(mix64(hash_combine(h, level)) >> 11) * 0x1.0p-53;
    uu <<= 1;
    vv <<= 1;
    if (r < p.t1) {
    } else if (r < p.t2) {
      vv |= 1;
    } else if (r < p.t3) {
      uu |= 1;
    } else {
      uu |= 1;
      vv |= 1;
    }
  }
  u = uu;
  v = vv;
}

__global__ void rmat_batch_k(RmatParams p, uint64_t size, uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += stride) {
    uint32_t u, v;
    rmat_draw(p, i, u, v);
    reinterpret_cast<uint4*>(out)[i] = make_uint4(u, v, v, u);
  }
}

__global__ void rmat_keys_k(RmatParams p, uint64_t size, BatchKeys bk, uint64_t* keys) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += stride) {
    uint32_t u, v;
    rmat_draw(p, i, u, v);
    const bool loop = u == v;
    keys[2 * i] = loop ? bk.loop_key() : bk.make(u, v);
    keys[2 * i + 1] = loop ? bk.loop_key() : bk.make(v, u);
  }
}

__global__ void split_keys_k(const uint64_t* keys, uint64_t m, BatchKeys bk, uint32_t* src, uint32_t* dst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint64_t k = keys[i];
    src[i] = bk.src(k);
    dst[i] = bk.dst(k);
  }
}

RmatParams make_params(uint32_t log2_n, double a, double b, double c, uint64_t seed) {
  if (log2_n < 1 || log2_n > 31) fail(GBG_ERR_CONFIG, "rmat: log2_n must be in [1, 31]");
  RmatParams p;
  p.t1 = a;
  p.t2 = a + b;
  p.t3 = a + b + c;
  p.log2_n = log2_n;
  p.seed = seed;
  return p;
}

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_update_batch_device(uint32_t log2_n, double a, double b, double c, uint64_t size, uint64_t seed,
                                   uint32_t* arcs_dev) {
  return guard([&] {
    if (size < 1) fail(GBG_ERR_CONFIG, "update batch size must be >= 1");  // batch.cpp:130
    if (!arcs_dev) fail(GBG_ERR_INVALID_ARGUMENT, "null output");
    RmatParams p = make_params(log2_n, a, b, c, seed);
    std::unique_ptr<gbg_graph> h(new_handle(GBG_KIND_CSR, 0));
    AllocStream as(h->stream);
    GBG_LAUNCH(h.get(), rmat_batch_k, grid_for(size, 256, h->sm_count * 16), 256, 0, p, size, arcs_dev);
    GBG_CUDA(cudaStreamSynchronize(h->stream));
  });
}

gbg_status gbg_rmat_create(uint32_t log2_n, uint64_t arcs, double a, double b, double c, uint64_t seed, int kind,
                           gbg_graph** out) {
  return guard([&] {
    if (!out) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (kind != GBG_KIND_CSR && kind != GBG_KIND_BLOCKED && kind != GBG_KIND_COMPRESSED)
      fail(GBG_ERR_CONFIG, "rmat: unknown container kind");
    *out = nullptr;
    RmatParams p = make_params(log2_n, a, b, c, seed);
    const uint64_t n = uint64_t{1} << log2_n;
    std::unique_ptr<gbg_graph> g(new_handle(GBG_KIND_CSR, n));
    AllocStream as(g->stream);
    const BatchKeys bk{static_cast<int>(log2_n)};
    const uint64_t count = 2 * arcs;
    uint64_t m = 0;
    {
      uint64_t* keys = dalloc<uint64_t>(count);
      uint64_t* scratch = dalloc<uint64_t>(count);
      try {
        if (arcs) GBG_LAUNCH(g.get(), rmat_keys_k, grid_for(arcs, 256, g->sm_count * 16), 256, 0, p, arcs, bk, keys);
        uint64_t* uniq = keys;
        if (arcs) uniq = sort_unique_keys(g.get(), keys, scratch, count, bk, &m, "rmat");
        g->m = m;
        g->off = dalloc<uint64_t>(n + 1);
        g->nbr = dalloc<uint32_t>(m);
        uint32_t* src = reinterpret_cast<uint32_t*>(uniq == keys ? scratch : keys);  // the free buffer
        if (m) GBG_LAUNCH(g.get(), split_keys_k, grid_for(m, 256, g->sm_count * 16), 256, 0, uniq, m, bk, src, g->nbr);
        build_csr_offsets_from_sorted_src(g.get(), src, m, g->off);
        GBG_CUDA(cudaStreamSynchronize(g->stream));
      } catch (...) {
        dfree(keys);
        dfree(scratch);
        throw;
      }
      dfree(keys);
      dfree(scratch);
    }
    g->symmetric = true;
    g->ws.release("rmat.uniq.sums");
    if (kind == GBG_KIND_BLOCKED) {
      std::unique_ptr<gbg_graph> b(new_handle(GBG_KIND_BLOCKED, n));
      AllocStream bas(b->stream);
      b->m = m;
      b->symmetric = true;
      blocked_from_device_csr(b.get(), n, g->off, g->nbr);
      GBG_CUDA(cudaStreamSynchronize(b->stream));
      *out = b.release();
    } else if (kind == GBG_KIND_COMPRESSED) {
      gbg_graph* z = nullptr;
      const gbg_status st = gbg_compressed_from(g.get(), &z);
      if (st != GBG_OK) fail(st, gbg_last_error());
      *out = z;
    } else {
      *out = g.release();
    }
  });
}

}  // extern "C"

// Compressed CSR container: gap-compressed neighbour lists in the
// reference's byte code, encoded and decoded on the device.
//
// Reference: gb::CompressedCsrGraph (compressed_csr.hpp:12-46,
// compressed_csr.cpp:5-51) over the byte code of bytecode.hpp:11-62: per
// vertex, the first neighbour as a zig-zag signed difference from the
// vertex id, then unsigned gaps, each a base-128 varint (low 7 bits first,
// high bit = continuation); byte_offsets[n+1] delimit the segments.  The
// device copy holds exactly those two arrays (bytes padded by 8 so decoders
// may over-read) plus each vertex's degree (4 B/vertex; the reference
// decodes to count).  Static like the reference (no batch updates; no
// parallel maps: capabilities {1,1,1,0,0,0}).
//
// Encode: one warp per vertex, 32 neighbours per step — values and varint
// lengths per lane, a warp scan of the lengths places every varint.
// Decode (warp-parallel varint decode): a warp reads 32 bytes of a
// segment; terminators (high bit clear) come from one ballot, each
// terminator lane assembles its varint from up to four preceding lanes by
// shuffles, a warp scan of the decoded gaps (the first one zig-zag, relative
// to the vertex id) yields the ids, and the window advances to just past the
// last complete varint (a varint is at most 5 bytes for 32-bit ids, so
// every window completes at least six).
//
// Traversals on a compressed handle decode it once per API call into a
// transient CSR (released when the call returns) and run the CSR engines:
// decode streams the segments at HBM speed, while decoding inside the
// frontier engines would put a serial varint dependency in every random
// neighbour access.
#include <memory>

#include "gbg_internal.cuh"
#include "scan.cuh"

namespace gbg {

namespace {

constexpr int kCzThreads = 256;

__device__ __forceinline__ uint32_t varint_len(uint64_t x) {
  const uint32_t bits = 64 - __clzll(x | 1);
  return (bits + 6) / 7;
}
__device__ __forceinline__ uint64_t zigzag_encode(int64_t x) {  // bytecode.hpp:19-22
  return x >= 0 ? 2 * static_cast<uint64_t>(x) : 2 * static_cast<uint64_t>(-(x + 1)) + 1;
}
__device__ __forceinline__ int64_t zigzag_decode(uint64_t z) {  // bytecode.hpp:24-27
  return (z & 1) ? -static_cast<int64_t>(z >> 1) - 1 : static_cast<int64_t>(z >> 1);
}

// the varint value of neighbour i of v (i > 0: gap to the predecessor)
template <class G>
__device__ __forceinline__ uint64_t code_value(G g, uint32_t v, uint64_t b, uint32_t i) {
  const uint32_t x = g.at(b + i);
  if (i == 0) return zigzag_encode(static_cast<int64_t>(x) - static_cast<int64_t>(v));
  return static_cast<uint64_t>(x - g.at(b + i - 1));
}

__device__ __forceinline__ uint64_t warp_excl_scan_u64(uint64_t x, uint64_t& total) {
  const int lane = threadIdx.x & 31;
  uint64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - x;
}

// pass 1: bytes per vertex (warp per vertex) + degrees
template <class G>
__global__ void __launch_bounds__(kCzThreads) cz_len_k(G g, uint64_t* len, uint32_t* deg) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t v = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); v < g.n; v += warps) {
    uint64_t b;
    uint32_t d;
    g.seg(static_cast<uint32_t>(v), b, d);
    uint64_t sum = 0;
    for (uint32_t i = lane; i < d; i += 32) sum += varint_len(code_value(g, static_cast<uint32_t>(v), b, i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      len[v] = sum;
      deg[v] = d;
    }
  }
}

// pass 2: write the byte code (warp per vertex, 32 varints per step)
template <class G>
__global__ void __launch_bounds__(kCzThreads) cz_write_k(G g, const uint64_t* coff, uint8_t* bytes) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t v = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); v < g.n; v += warps) {
    uint64_t b;
    uint32_t d;
    g.seg(static_cast<uint32_t>(v), b, d);
    uint64_t pos = coff[v];
    for (uint32_t base = 0; base < d; base += 32) {
      const uint32_t i = base + lane;
      uint64_t val = 0;
      uint32_t len = 0;
      if (i < d) {
        val = code_value(g, static_cast<uint32_t>(v), b, i);
        len = varint_len(val);
      }
      uint64_t total;
      const uint64_t at = pos + warp_excl_scan_u64(len, total);
      for (uint32_t k = 0; k < len; ++k) {
        bytes[at + k] = static_cast<uint8_t>((val & 0x7f) | (k + 1 < len ? 0x80 : 0));
        val >>= 7;
      }
      pos += total;
    }
  }
}

struct WideIn {
  const uint32_t* a;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};
struct U64In {
  const uint64_t* a;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};

// warp-parallel decode of vertex v's segment into out[0 .. deg)
__device__ __forceinline__ void cz_decode_vertex(uint32_t v, const uint8_t* __restrict__ bytes, uint64_t p,
                                                 uint64_t end, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1;
  int64_t cur = v;
  uint64_t k = 0;
  bool first = true;
  while (p < end) {
    const bool in = p + lane < end;
    const uint32_t c = in ? bytes[p + lane] : 0x80u;
    const bool term = in && !(c & 0x80u);
    const uint32_t tm = __ballot_sync(0xffffffffu, term);
    if (!tm) return;  // malformed (cannot happen for encoder output)
    const uint32_t prev = tm & below;
    const int start = prev ? 32 - __clz(prev) : 0;  // first byte of this lane's varint
    uint64_t val = c & 0x7fu;  // this lane's byte is the varint's most significant
#pragma unroll
    for (int d = 1; d <= 4; ++d) {  // shift in the earlier (less significant) bytes
      const uint32_t cd = __shfl_up_sync(0xffffffffu, c, d);
      if (lane - d >= start) val = (val << 7) | (cd & 0x7fu);
    }
    int64_t contrib = 0;
    if (term) {
      const uint64_t z = val;
      const bool is_first = first && prev == 0;
      contrib = is_first ? zigzag_decode(z) : static_cast<int64_t>(z);
    }
    int64_t inc = contrib;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (term) out[k + __popc(prev)] = static_cast<uint32_t>(cur + inc);
    cur += __shfl_sync(0xffffffffu, inc, 31);
    k += __popc(tm);
    first = false;
    p += 32 - __clz(tm);  // just past the last complete varint
  }
}

__global__ void __launch_bounds__(kCzThreads)
    cz_decode_k(uint64_t n, const uint64_t* __restrict__ coff, const uint8_t* __restrict__ bytes,
                const uint64_t* __restrict__ dst_off, uint32_t* out) {
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t v = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); v < n; v += warps)
    cz_decode_vertex(static_cast<uint32_t>(v), bytes, coff[v], coff[v + 1], out + dst_off[v]);
}

__global__ void cz_decode_one_k(uint32_t v, const uint64_t* coff, const uint8_t* bytes, uint32_t* out) {
  cz_decode_vertex(v, bytes, coff[v], coff[v + 1], out);
}

template <class G>
void encode_into(gbg_graph* dst, G view) {
  const uint64_t n = dst->n;
  uint64_t* len = dst->ws.get<uint64_t>("cz.len", n);
  dst->coff = dalloc<uint64_t>(n + 1);
  dst->cdeg = dalloc<uint32_t>(n ? n : 1);
  const unsigned grid = grid_for(n * 32, kCzThreads, static_cast<unsigned>(dst->sm_count) * 16u);
  GBG_LAUNCH(dst, cz_len_k<G>, grid, kCzThreads, 0, view, len, dst->cdeg);
  device_scan<uint64_t>(dst, U64In{len}, ArrayOut<uint64_t>{dst->coff}, n, dst->coff + n, "cz.scan");
  read_scalars(dst, dst->coff + n, sizeof(dst->cbytes_len), &dst->cbytes_len);
  dst->cbytes = dalloc<uint8_t>(dst->cbytes_len + 8);
  GBG_CUDA(cudaMemsetAsync(dst->cbytes + dst->cbytes_len, 0x80, 8, dst->stream));
  GBG_LAUNCH(dst, cz_write_k<G>, grid, kCzThreads, 0, view, dst->coff, dst->cbytes);
  dst->ws.release("cz.len");
}

}  // namespace

// The decoded CSR of a compressed handle, built on first use within the
// current API call (released by TransientScope when the call returns).
CsrView compressed_decoded(gbg_graph* g) {
  if (!g->cz_ready) {
    const uint64_t n = g->n;
    uint64_t* off = g->ws.get<uint64_t>("cz.off", n + 1);
    uint32_t* nbr = g->ws.get<uint32_t>("cz.nbr", g->m ? g->m : 1);
    device_scan<uint64_t>(g, WideIn{g->cdeg}, ArrayOut<uint64_t>{off}, n, off + n, "cz.dscan");
    GBG_LAUNCH(g, cz_decode_k, grid_for(n * 32, kCzThreads, static_cast<unsigned>(g->sm_count) * 16u), kCzThreads, 0,
               n, g->coff, g->cbytes, off, nbr);
    g->cz_ready = true;
  }
  return {g->n, static_cast<const uint64_t*>(g->ws.get("cz.off", 0)),
          static_cast<const uint32_t*>(g->ws.get("cz.nbr", 0))};
}

void release_transient(gbg_graph* g) {
  if (g->kind != GBG_KIND_COMPRESSED || !g->cz_ready) return;
  g->ws.release("cz.off");
  g->ws.release("cz.nbr");
  g->cz_ready = false;
}

// One vertex's neighbours into device memory (read API).
void compressed_neighbors(gbg_graph* g, uint32_t v, uint32_t* out_dev) {
  cz_decode_one_k<<<1, 32, 0, g->stream>>>(v, g->coff, g->cbytes, out_dev);
  cuda_check(cudaGetLastError(), "cz_decode_one_k");
  g->launches++;
}

}  // namespace gbg

using namespace gbg;

extern "C" {

gbg_status gbg_compressed_from(gbg_graph* src, gbg_graph** out) {
  return guard([&] {
    if (!out) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    GBG_HANDLE(src);
    std::unique_ptr<gbg_graph> g(new_handle(GBG_KIND_COMPRESSED, src->n));
    g->m = src->m;
    g->symmetric = src->symmetric;
    g->sym_checked = src->sym_checked;
    // the new handle's stream must see src's data: finish src's work first
    // (including the decode of a compressed source, cached for this call)
    if (src->kind == GBG_KIND_COMPRESSED) compressed_decoded(src);
    GBG_CUDA(cudaStreamSynchronize(src->stream));
    {
      AllocStream as(g->stream);
      with_view(src, [&](auto view) { encode_into(g.get(), view); });
      GBG_CUDA(cudaStreamSynchronize(g->stream));
    }
    *out = g.release();
  });
}

gbg_status gbg_compressed_create(uint64_t n, uint64_t m, const uint64_t* offsets, const uint32_t* neighbors,
                                 gbg_graph** out) {
  return guard([&] {
    if (!out) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    gbg_graph* csr = nullptr;
    gbg_status st = gbg_csr_create(n, m, offsets, neighbors, &csr);  // validated like csr.cpp:14-18
    if (st != GBG_OK) fail(st, gbg_last_error());
    std::unique_ptr<gbg_graph> hold(csr);
    st = gbg_compressed_from(csr, out);
    if (st != GBG_OK) fail(st, gbg_last_error());
  });
}

gbg_status gbg_compressed_bytes(gbg_graph* g, uint64_t* byte_offsets, uint8_t* bytes, uint64_t* nbytes) {
  return guard([&] {
    GBG_HANDLE(g);
    if (!nbytes) fail(GBG_ERR_INVALID_ARGUMENT, "null argument");
    if (g->kind != GBG_KIND_COMPRESSED) fail(GBG_ERR_UNSUPPORTED, "not a compressed container");
    *nbytes = g->cbytes_len;
    if (byte_offsets)
      GBG_CUDA(cudaMemcpyAsync(byte_offsets, g->coff, (g->n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                               g->stream));
    if (bytes && g->cbytes_len)
      GBG_CUDA(cudaMemcpyAsync(bytes, g->cbytes, g->cbytes_len, cudaMemcpyDeviceToHost, g->stream));
    GBG_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"

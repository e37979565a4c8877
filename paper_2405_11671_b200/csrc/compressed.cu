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

// Bytes of the varints of neighbours [i0, i1) of v (warp-cooperative).
template <class G>
__device__ __forceinline__ uint64_t cz_len_range(G g, uint32_t v, uint64_t b, uint32_t i0, uint32_t i1) {
  const int lane = threadIdx.x & 31;
  uint64_t sum = 0;
  for (uint32_t i = i0 + lane; i < i1; i += 32) sum += varint_len(code_value(g, v, b, i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return sum;
}

// Write the varints of neighbours [i0, i1) of v from byte `pos` on.
template <class G>
__device__ __forceinline__ void cz_write_range(G g, uint32_t v, uint64_t b, uint32_t i0, uint32_t i1, uint64_t pos,
                                               uint8_t* bytes) {
  const int lane = threadIdx.x & 31;
  for (uint32_t base = i0; base < i1; base += 32) {
    const uint32_t i = base + lane;
    uint64_t val = 0;
    uint32_t len = 0;
    if (i < i1) {
      val = code_value(g, v, b, i);
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

// Decode the varints that START in [p, p1) (p at a varint start; bytes are
// read up to seg_end).  kWrite: out[k] = id; otherwise only count / sum.
// Ids are VertexId (uint32) arithmetic like bytecode_decode_each
// (bytecode.hpp:50-58), so the running sums are taken mod 2^32.
template <bool kWrite>
__device__ __forceinline__ void cz_decode_range(const uint8_t* __restrict__ bytes, uint64_t origin, uint64_t p,
                                                uint64_t p1, uint64_t seg_end, uint32_t cur, bool first,
                                                uint32_t* out, uint64_t& count, uint32_t& sum) {
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1;
  while (p < p1) {
    const bool in = p + lane < seg_end;
    const uint32_t c = in ? bytes[p + lane - origin] : 0x80u;
    const bool term = in && !(c & 0x80u);
    const uint32_t tm = __ballot_sync(0xffffffffu, term);
    const uint32_t prev = tm & below;
    const int start = prev ? 32 - __clz(prev) : 0;  // first byte of this lane's varint
    const bool incl = term && p + start < p1;       // a prefix of the terminators
    const uint32_t im = __ballot_sync(0xffffffffu, incl);
    if (!im) return;
    uint64_t val = c & 0x7fu;  // this lane's byte is the varint's most significant
#pragma unroll
    for (int d = 1; d <= 4; ++d) {  // shift in the earlier (less significant) bytes
      const uint32_t cd = __shfl_up_sync(0xffffffffu, c, d);
      if (lane - d >= start) val = (val << 7) | (cd & 0x7fu);
    }
    uint32_t inc = 0;
    if (incl) inc = (first && prev == 0) ? static_cast<uint32_t>(zigzag_decode(val)) : static_cast<uint32_t>(val);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (kWrite && incl) out[count + __popc(prev)] = cur + inc;
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    cur += tot;
    sum += tot;
    count += __popc(im);
    first = false;
    p += 32 - __clz(im);  // just past the last included varint
  }
}

// Stage bytes [p, e) of the code into a per-warp shared buffer with
// independent 32-bit loads (all in flight at once) so the window walk reads
// shared memory instead of paying a global-load latency per window.
// Returns the origin: buf[q - origin] == bytes[q] for q in [p, e).
constexpr uint32_t kStageBytes = 4096 + 16;
__device__ __forceinline__ uint64_t cz_stage(const uint8_t* __restrict__ bytes, uint64_t p, uint64_t e,
                                             uint32_t* buf) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = p >> 2, w1 = (e + 3) >> 2;  // the code is 256-byte aligned and padded by 8
  const uint32_t* src = reinterpret_cast<const uint32_t*>(bytes);
  for (uint64_t w = w0 + lane; w < w1; w += 32) buf[w - w0] = __ldg(src + w);
  __syncwarp();
  return w0 << 2;
}

// One short segment decoded by one lane (the serial loop of
// bytecode_decode_each, bytecode.hpp:40-58).
__device__ __forceinline__ void cz_decode_lane(const uint8_t* __restrict__ bytes, uint64_t p, uint64_t e, uint32_t v,
                                               uint32_t* out) {
  uint32_t cur = v, k = 0;
  uint64_t val = 0;
  int shift = 0;
  bool first = true;
  for (; p < e; ++p) {
    const uint32_t c = bytes[p];
    val |= static_cast<uint64_t>(c & 0x7fu) << shift;
    if (c & 0x80u) {
      shift += 7;
      continue;
    }
    cur = first ? v + static_cast<uint32_t>(zigzag_decode(val)) : cur + static_cast<uint32_t>(val);
    out[k++] = cur;
    first = false;
    val = 0;
    shift = 0;
  }
}

// Segments longer than these are cut into chunks handled by separate
// warps (a 406K-neighbour hub is ~600 KB of code): encode by neighbours,
// decode by bytes with a count/sum pre-pass and a segmented scan.
constexpr uint32_t kEncChunk = 1024;  // neighbours
constexpr uint32_t kDecChunk = 4096;  // bytes

// pass 1: bytes per light vertex (warp per vertex) + degrees
template <class G>
__global__ void __launch_bounds__(kCzThreads) cz_len_k(G g, uint64_t* len, uint32_t* deg) {
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t v = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); v < g.n; v += warps) {
    uint64_t b;
    uint32_t d;
    g.seg(static_cast<uint32_t>(v), b, d);
    const uint64_t sum = d > kEncChunk ? 0 : cz_len_range(g, static_cast<uint32_t>(v), b, 0, d);
    if ((threadIdx.x & 31) == 0) {
      len[v] = sum;
      deg[v] = d;
    }
  }
}

template <class G>
__global__ void __launch_bounds__(kCzThreads) cz_write_k(G g, const uint64_t* coff, uint8_t* bytes) {
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t v = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); v < g.n; v += warps) {
    uint64_t b;
    uint32_t d;
    g.seg(static_cast<uint32_t>(v), b, d);
    if (d <= kEncChunk) cz_write_range(g, static_cast<uint32_t>(v), b, 0, d, coff[v], bytes);
  }
}

// heavy vertices and their chunk prefix
struct HeavyChunks {
  const uint32_t* list;  // heavy vertex ids
  uint32_t nh;
  const uint64_t* cbase;  // [nh + 1] first chunk of each heavy vertex
  uint64_t nchunks;
};

__device__ __forceinline__ uint32_t chunk_owner(const HeavyChunks& h, uint64_t c) {
  uint32_t lo = 0, hi = h.nh;  // cbase[lo] <= c < cbase[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (h.cbase[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// encode chunk lengths (warp per chunk)
template <class G>
__global__ void __launch_bounds__(kCzThreads) cz_chunk_len_k(G g, HeavyChunks h, uint64_t* clen) {
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t c = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); c < h.nchunks; c += warps) {
    const uint32_t hv = chunk_owner(h, c);
    const uint32_t v = h.list[hv];
    uint64_t b;
    uint32_t d;
    g.seg(v, b, d);
    const uint32_t i0 = static_cast<uint32_t>(c - h.cbase[hv]) * kEncChunk;
    const uint32_t i1 = i0 + kEncChunk < d ? i0 + kEncChunk : d;
    const uint64_t sum = cz_len_range(g, v, b, i0, i1);
    if ((threadIdx.x & 31) == 0) clen[c] = sum;
  }
}

// per heavy vertex: total bytes into len[v]
__global__ void cz_heavy_total_k(HeavyChunks h, const uint64_t* cpos, uint64_t* len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < h.nh; i += stride)
    len[h.list[i]] = cpos[h.cbase[i + 1]] - cpos[h.cbase[i]];
}

template <class G>
__global__ void __launch_bounds__(kCzThreads)
    cz_chunk_write_k(G g, HeavyChunks h, const uint64_t* cpos, const uint64_t* coff, uint8_t* bytes) {
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t c = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); c < h.nchunks; c += warps) {
    const uint32_t hv = chunk_owner(h, c);
    const uint32_t v = h.list[hv];
    uint64_t b;
    uint32_t d;
    g.seg(v, b, d);
    const uint32_t i0 = static_cast<uint32_t>(c - h.cbase[hv]) * kEncChunk;
    const uint32_t i1 = i0 + kEncChunk < d ? i0 + kEncChunk : d;
    cz_write_range(g, v, b, i0, i1, coff[v] + cpos[c] - cpos[h.cbase[hv]], bytes);
  }
}

// decode of the segments up to kDecChunk bytes: lane i of a warp owns
// vertex base + i; segments up to kLaneBytes are decoded by their lane,
// longer ones by the whole warp in turn
constexpr uint32_t kLaneBytes = 24;

__global__ void __launch_bounds__(kCzThreads)
    cz_decode_k(uint64_t n, const uint64_t* __restrict__ coff, const uint8_t* __restrict__ bytes,
                const uint64_t* __restrict__ dst_off, uint32_t* out) {
  __shared__ uint32_t s_buf[kCzThreads / 32][kStageBytes / 4];
  uint32_t* buf = s_buf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const uint64_t step = (uint64_t)gridDim.x * kCzThreads;
  for (uint64_t base = ((uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5)) * 32; base < n; base += step) {
    const uint64_t v = base + lane;
    uint64_t p = 0, e = 0;
    if (v < n) {
      p = coff[v];
      e = coff[v + 1];
    }
    const uint64_t len = e - p;
    if (len && len <= kLaneBytes) cz_decode_lane(bytes, p, e, static_cast<uint32_t>(v), out + dst_off[v]);
    uint32_t wide = __ballot_sync(0xffffffffu, len > kLaneBytes && len <= kDecChunk);
    while (wide) {
      const int src = __ffs(wide) - 1;
      wide &= wide - 1;
      const uint64_t xp = __shfl_sync(0xffffffffu, p, src), xe = __shfl_sync(0xffffffffu, e, src);
      const uint32_t xv = static_cast<uint32_t>(base + src);
      uint64_t cnt = 0;
      uint32_t sum = 0;
      const uint64_t origin = cz_stage(bytes, xp, xe, buf);
      cz_decode_range<true>(reinterpret_cast<const uint8_t*>(buf), origin, xp, xe, xe, xv, true, out + dst_off[xv],
                            cnt, sum);
      __syncwarp();
    }
  }
}

// first varint start at or after p0 within [seg_begin, seg_end)
__device__ __forceinline__ uint64_t cz_align(const uint8_t* bytes, uint64_t seg_begin, uint64_t p0,
                                             uint64_t seg_end) {
  if (p0 == seg_begin || !(bytes[p0 - 1] & 0x80u)) return p0;
  const int lane = threadIdx.x & 31;
  const bool term = p0 + lane < seg_end && !(bytes[p0 + lane] & 0x80u);
  const uint32_t tm = __ballot_sync(0xffffffffu, term);
  return tm ? p0 + __ffs(tm) : seg_end;
}

// decode chunks: pass A (count / sum) and pass C (write at the scanned bases)
template <bool kWrite>
__global__ void __launch_bounds__(kCzThreads)
    cz_decode_chunks_k(HeavyChunks h, const uint64_t* __restrict__ coff, const uint8_t* __restrict__ bytes,
                       uint64_t* ccnt, uint64_t* csum, const uint64_t* dst_off, uint32_t* out) {
  __shared__ uint32_t s_buf[kCzThreads / 32][kStageBytes / 4];
  uint32_t* buf = s_buf[threadIdx.x >> 5];
  const uint64_t warps = (uint64_t)gridDim.x * (kCzThreads / 32);
  for (uint64_t c = (uint64_t)blockIdx.x * (kCzThreads / 32) + (threadIdx.x >> 5); c < h.nchunks; c += warps) {
    const uint32_t hv = chunk_owner(h, c);
    const uint32_t v = h.list[hv];
    const uint64_t sb = coff[v], se = coff[v + 1];
    const uint64_t j = c - h.cbase[hv];
    const uint64_t p0 = sb + j * kDecChunk;
    const uint64_t p1 = p0 + kDecChunk < se ? p0 + kDecChunk : se;
    const uint64_t s0 = cz_align(bytes, sb, p0, se);
    // the last varint starting before p1 ends at most 4 bytes later
    const uint64_t stage_end = p1 + 4 < se ? p1 + 4 : se;
    const uint64_t origin = cz_stage(bytes, s0, stage_end, buf);
    const uint8_t* sbuf = reinterpret_cast<const uint8_t*>(buf);
    uint64_t cnt = 0;
    uint32_t sum = 0;
    if (kWrite) {
      const uint64_t first_c = h.cbase[hv];
      const uint64_t base_cnt = ccnt[c] - ccnt[first_c];
      const uint32_t base_sum = static_cast<uint32_t>(csum[c] - csum[first_c]);  // mod 2^32
      cz_decode_range<true>(sbuf, origin, s0, p1, stage_end, v + base_sum, j == 0, out + dst_off[v] + base_cnt, cnt,
                            sum);
    } else {
      cz_decode_range<false>(sbuf, origin, s0, p1, stage_end, 0, j == 0, nullptr, cnt, sum);
      if ((threadIdx.x & 31) == 0) {
        ccnt[c] = cnt;
        csum[c] = sum;
      }
    }
    __syncwarp();
  }
}

__global__ void cz_decode_one_k(uint32_t v, const uint64_t* coff, const uint8_t* bytes, uint32_t* out) {
  uint64_t cnt = 0;
  uint32_t sum = 0;
  cz_decode_range<true>(bytes, 0, coff[v], coff[v + 1], coff[v + 1], v, true, out, cnt, sum);
}

struct WideIn {
  const uint32_t* a;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};
struct U64In {
  const uint64_t* a;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};
// heavy selection + chunk counts
struct HeavyDeg {
  const uint32_t* deg;
  __device__ __forceinline__ bool operator()(uint32_t v) const { return deg[v] > kEncChunk; }
};
struct HeavyBytes {
  const uint64_t* coff;
  __device__ __forceinline__ bool operator()(uint32_t v) const { return coff[v + 1] - coff[v] > kDecChunk; }
};
struct EncChunksIn {
  const uint32_t* list;
  const uint32_t* deg;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    return (deg[list[i]] + kEncChunk - 1) / kEncChunk;
  }
};
struct DecChunksIn {
  const uint32_t* list;
  const uint64_t* coff;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    const uint32_t v = list[i];
    return (coff[v + 1] - coff[v] + kDecChunk - 1) / kDecChunk;
  }
};

template <class Pred>
__global__ void cz_select_k(uint64_t n, Pred pred, uint32_t* list, unsigned int* count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    if (pred(static_cast<uint32_t>(v))) list[atomicAdd(count, 1u)] = static_cast<uint32_t>(v);
}

// heavy list (order irrelevant) and its chunk prefix; returns the chunk count
template <class Pred, class ChunksIn>
HeavyChunks heavy_chunks(gbg_graph* g, Pred pred, ChunksIn chunks_of, const char* tag) {
  const std::string t(tag);
  uint32_t* list = g->ws.get<uint32_t>(t + ".heavy", g->n);
  unsigned int* cnt = g->ws.get<unsigned int>(t + ".nheavy", 1);
  GBG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned int), g->stream));
  GBG_LAUNCH(g, cz_select_k<Pred>, grid_for(g->n, 256), 256, 0, g->n, pred, list, cnt);
  unsigned int nh = 0;
  read_scalars(g, cnt, sizeof(nh), &nh);
  HeavyChunks h{list, nh, nullptr, 0};
  if (!nh) return h;
  chunks_of.list = list;
  uint64_t* cbase = g->ws.get<uint64_t>(t + ".cbase", nh + 1);
  device_scan<uint64_t>(g, chunks_of, ArrayOut<uint64_t>{cbase}, nh, cbase + nh, (t + ".cscan").c_str());
  read_scalars(g, cbase + nh, sizeof(h.nchunks), &h.nchunks);
  h.cbase = cbase;
  return h;
}

inline unsigned warp_grid(gbg_graph* g, uint64_t items) {
  return grid_for(items * 32, kCzThreads, static_cast<unsigned>(g->sm_count) * 16u);
}

template <class G>
void encode_into(gbg_graph* dst, G view) {
  const uint64_t n = dst->n;
  uint64_t* len = dst->ws.get<uint64_t>("cz.len", n);
  dst->coff = dalloc<uint64_t>(n + 1);
  dst->cdeg = dalloc<uint32_t>(n ? n : 1);
  GBG_LAUNCH(dst, cz_len_k<G>, warp_grid(dst, n), kCzThreads, 0, view, len, dst->cdeg);
  const HeavyChunks h = heavy_chunks(dst, HeavyDeg{dst->cdeg}, EncChunksIn{nullptr, dst->cdeg}, "cz.enc");
  uint64_t* cpos = nullptr;
  if (h.nchunks) {
    uint64_t* clen = dst->ws.get<uint64_t>("cz.clen", h.nchunks);
    cpos = dst->ws.get<uint64_t>("cz.cpos", h.nchunks + 1);
    GBG_LAUNCH(dst, cz_chunk_len_k<G>, warp_grid(dst, h.nchunks), kCzThreads, 0, view, h, clen);
    device_scan<uint64_t>(dst, U64In{clen}, ArrayOut<uint64_t>{cpos}, h.nchunks, cpos + h.nchunks, "cz.cposscan");
    GBG_LAUNCH(dst, cz_heavy_total_k, grid_for(h.nh, 256), 256, 0, h, cpos, len);
  }
  device_scan<uint64_t>(dst, U64In{len}, ArrayOut<uint64_t>{dst->coff}, n, dst->coff + n, "cz.scan");
  read_scalars(dst, dst->coff + n, sizeof(dst->cbytes_len), &dst->cbytes_len);
  dst->cbytes = dalloc<uint8_t>(dst->cbytes_len + 8);
  GBG_CUDA(cudaMemsetAsync(dst->cbytes + dst->cbytes_len, 0x80, 8, dst->stream));
  GBG_LAUNCH(dst, cz_write_k<G>, warp_grid(dst, n), kCzThreads, 0, view, dst->coff, dst->cbytes);
  if (h.nchunks)
    GBG_LAUNCH(dst, cz_chunk_write_k<G>, warp_grid(dst, h.nchunks), kCzThreads, 0, view, h, cpos, dst->coff,
               dst->cbytes);
  for (const char* b : {"cz.len", "cz.clen", "cz.cpos", "cz.enc.heavy", "cz.enc.cbase"}) dst->ws.release(b);
}

}  // namespace

// The decoded CSR of a compressed handle, built on first use within the
// current API call (released by TransientScope when the call returns).
CsrView compressed_decoded(gbg_graph* g) {
  if (!g->cz_ready) {
    const uint64_t n = g->n;
    uint64_t* off = g->ws.get<uint64_t>("cz.off", n + 1);
    uint32_t* nbr = g->ws.get<uint32_t>("cz.nbr", g->m ? g->m : 1);
    PhaseTrace tr(g->stream, "decode");
    device_scan<uint64_t>(g, WideIn{g->cdeg}, ArrayOut<uint64_t>{off}, n, off + n, "cz.dscan");
    tr.mark("offsets");
    GBG_LAUNCH(g, cz_decode_k, warp_grid(g, n), kCzThreads, 0, n, g->coff, g->cbytes, off, nbr);
    tr.mark("light");
    const HeavyChunks h = heavy_chunks(g, HeavyBytes{g->coff}, DecChunksIn{nullptr, g->coff}, "cz.dec");
    if (h.nchunks) {
      uint64_t* ccnt = g->ws.get<uint64_t>("cz.ccnt", h.nchunks);
      uint64_t* csum = g->ws.get<uint64_t>("cz.csum", h.nchunks);
      uint64_t* cnt_pre = g->ws.get<uint64_t>("cz.cntpre", h.nchunks + 1);
      uint64_t* sum_pre = g->ws.get<uint64_t>("cz.sumpre", h.nchunks + 1);
      GBG_LAUNCH(g, cz_decode_chunks_k<false>, warp_grid(g, h.nchunks), kCzThreads, 0, h, g->coff, g->cbytes, ccnt,
                 csum, nullptr, nullptr);
      device_scan<uint64_t>(g, U64In{ccnt}, ArrayOut<uint64_t>{cnt_pre}, h.nchunks, cnt_pre + h.nchunks,
                            "cz.cntscan");
      device_scan<uint64_t>(g, U64In{csum}, ArrayOut<uint64_t>{sum_pre}, h.nchunks, sum_pre + h.nchunks,
                            "cz.sumscan");  // differences of prefixes are exact mod 2^32
      GBG_LAUNCH(g, cz_decode_chunks_k<true>, warp_grid(g, h.nchunks), kCzThreads, 0, h, g->coff, g->cbytes, cnt_pre,
                 sum_pre, off, nbr);
    }
    tr.mark("heavy");
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

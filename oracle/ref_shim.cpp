// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (BYO `graphbench`,
// /root/reference/proj/src/*.cpp compiled in place by oracle/Makefile into
// oracle/_ref/libgbref.so).  Only tests/, __graft_entry__.smoke() and the
// bench.py cpu-baseline / --impl reference legs load it.  Every entry point
// forwards to the reference's own public API:
//
//   gbref_rmat            gb::generate_rmat            (generators.cpp:67-72)
//   gbref_er / gbref_t4   gb::generate_er / tiny_fixture_graph (generators.cpp:31-78)
//   gbref_normalize       gb::normalize_arcs           (generators.cpp:9-29)
//   gbref_csr_*           gb::CsrGraph::build          (csr.cpp:9-25)
//   gbref_bfs             gb::bfs                      (algorithms.cpp:29-58)
//   gbref_bfs_trace       gb::edge_map loop w/ mode_out (traversal.cpp:101-111)
//   gbref_pagerank        gb::pagerank                 (algorithms.cpp:508-555)
//   gbref_cc              gb::cc                       (algorithms.cpp:194-234)
//   gbref_kcore           gb::kcore                    (algorithms.cpp:330-374)
//   gbref_coloring        gb::coloring                 (algorithms.cpp:376-432)
//   gbref_mis             gb::mis                      (algorithms.cpp:434-504)
//   gbref_ldd             gb::ldd                      (algorithms.cpp:114-188)
//   gbref_compressed      gb::CompressedCsrGraph::build (compressed_csr.cpp:5-17)
//   gbref_log1p           std::log1p of the reference's C library (rng.hpp:33)
//   gbref_update_batch    gb::generate_update_batch    (batch.cpp:128-154)
//   gbref_prepare_global  gb::prepare(GlobalSort)      (batch.cpp:30-42)
//   gbref_chunked_*       registry "chunked_set" + apply_insert/apply_delete
//                         (registry.cpp:136-137, batch.cpp:105-126)
//   gbref_edge_map_*      gb::edge_map_sparse / edge_map_dense (traversal.cpp:16-95)
//
// Exceptions never cross the C boundary: every call returns 0 on success or
// a nonzero code (1 out_of_range, 2 invalid_argument, 3 unsupported,
// 4 config, 5 format, 6 logic, 9 other) and the message is kept for
// gbref_last_error().

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "gb/algorithms.hpp"
#include "gb/batch.hpp"
#include "gb/compressed_csr.hpp"
#include "gb/csr.hpp"
#include "gb/facade.hpp"
#include "gb/generators.hpp"
#include "gb/io.hpp"
#include "gb/parallel.hpp"
#include "gb/registry.hpp"
#include "gb/rng.hpp"
#include "gb/traversal.hpp"

using namespace gb;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const unsupported_operation& e) {
    g_err = e.what();
    return 3;
  } catch (const config_error& e) {
    g_err = e.what();
    return 4;
  } catch (const format_error& e) {
    g_err = e.what();
    return 5;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

std::vector<Edge> pairs_to_edges(const uint32_t* pairs, uint64_t count) {
  std::vector<Edge> out(count);
  for (uint64_t i = 0; i < count; ++i) out[i] = {pairs[2 * i], pairs[2 * i + 1]};
  return out;
}

void edges_to_pairs(const std::vector<Edge>& e, uint32_t* out) {
  for (size_t i = 0; i < e.size(); ++i) {
    out[2 * i] = e[i].src;
    out[2 * i + 1] = e[i].dst;
  }
}

// CsrGraph from caller CSR arrays, through the reference's validated build.
CsrGraph csr_from_arrays(uint64_t n, const uint64_t* off, const uint32_t* nbr) {
  std::vector<Edge> arcs;
  arcs.reserve(off[n]);
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t k = off[v]; k < off[v + 1]; ++k)
      arcs.push_back({static_cast<VertexId>(v), nbr[k]});
  return CsrGraph::build(n, arcs);
}

void export_container(const GraphContainer& c, uint64_t* off, uint32_t* nbr) {
  GraphView view(c);
  uint64_t n = view.num_vertices();
  uint64_t pos = 0;
  off[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    c.map_neighbors(static_cast<VertexId>(v), [&](VertexId u) { nbr[pos++] = u; });
    off[v + 1] = pos;
  }
}

}  // namespace

extern "C" {

const char* gbref_last_error() { return g_err.c_str(); }

void gbref_set_threads(int t) { set_num_workers(t); }
int gbref_num_threads() { return num_workers(); }

uint64_t gbref_hash_combine(uint64_t a, uint64_t b) { return hash_combine(a, b); }
uint64_t gbref_mix64(uint64_t x) { return mix64(x); }
double gbref_rng_double(uint64_t s, uint64_t st, uint64_t c) { return rng_double(s, st, c); }

// ---- GraphData handles ----
void* gbref_rmat(uint64_t log2_n, uint64_t arcs, double a, double b, double c,
                 uint64_t seed) {
  void* out = nullptr;
  int rc = guard([&] {
    RmatParams p;
    p.a = a;
    p.b = b;
    p.c = c;
    p.log2_n = log2_n;
    out = new GraphData(generate_rmat(p, arcs, seed));
  });
  return rc == 0 ? out : nullptr;
}

void* gbref_er(uint64_t n, double p, uint64_t seed) {
  void* out = nullptr;
  guard([&] { out = new GraphData(generate_er({n, p}, seed)); });
  return out;
}

void* gbref_t4() { return new GraphData(tiny_fixture_graph()); }

void* gbref_normalize(const uint32_t* pairs, uint64_t count, uint64_t min_n) {
  void* out = nullptr;
  guard([&] { out = new GraphData(normalize_arcs(pairs_to_edges(pairs, count), min_n)); });
  return out;
}

uint64_t gbref_graph_n(void* h) { return static_cast<GraphData*>(h)->n; }
uint64_t gbref_graph_m(void* h) { return static_cast<GraphData*>(h)->arcs.size(); }
void gbref_graph_arcs(void* h, uint32_t* out) {
  edges_to_pairs(static_cast<GraphData*>(h)->arcs, out);
}
void gbref_graph_free(void* h) { delete static_cast<GraphData*>(h); }

int gbref_graph_csr(void* h, uint64_t* off, uint32_t* nbr) {
  return guard([&] {
    const GraphData& g = *static_cast<GraphData*>(h);
    CsrGraph c = CsrGraph::build(g.n, g.arcs);
    std::memcpy(off, c.offsets().data(), (g.n + 1) * sizeof(uint64_t));
    std::memcpy(nbr, c.neighbors().data(), c.neighbors().size() * sizeof(uint32_t));
  });
}

// ---- CSR handles (for repeated algorithm calls on one graph) ----
void* gbref_csr_create(uint64_t n, const uint64_t* off, const uint32_t* nbr) {
  void* out = nullptr;
  guard([&] { out = new CsrGraph(csr_from_arrays(n, off, nbr)); });
  return out;
}

// From sorted, deduplicated arc pairs (CsrGraph::build validation applies).
void* gbref_csr_from_pairs(uint64_t n, const uint32_t* pairs, uint64_t count) {
  void* out = nullptr;
  guard([&] { out = new CsrGraph(CsrGraph::build(n, pairs_to_edges(pairs, count))); });
  return out;
}

void gbref_csr_free(void* h) { delete static_cast<CsrGraph*>(h); }

// gb::save_binary / gb::load_binary_csr (io.cpp:75-110)
int gbref_save_binary(void* csr, const char* path) {
  return guard([&] { save_binary(*static_cast<CsrGraph*>(csr), path); });
}
void* gbref_load_binary(const char* path) {
  void* out = nullptr;
  guard([&] { out = new CsrGraph(load_binary_csr(path)); });
  return out;
}
uint64_t gbref_csr_n(void* csr) { return static_cast<CsrGraph*>(csr)->num_vertices(); }
uint64_t gbref_csr_m(void* csr) { return static_cast<CsrGraph*>(csr)->num_edges(); }
void gbref_csr_arrays(void* csr, uint64_t* off, uint32_t* nbr) {
  const CsrGraph& c = *static_cast<CsrGraph*>(csr);
  std::memcpy(off, c.offsets().data(), c.offsets().size() * sizeof(uint64_t));
  std::memcpy(nbr, c.neighbors().data(), c.neighbors().size() * sizeof(uint32_t));
}

// BFS depths as int32 (-1 unreached), the BASELINE narrowing of
// gb::bfs(...).distances (UINT64_MAX -> -1).
int gbref_bfs(void* csr, uint32_t src, int32_t* depth) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    BfsResult r = bfs(view, src);
    for (size_t v = 0; v < r.distances.size(); ++v)
      depth[v] = r.distances[v] == kInfiniteDistance ? -1 : static_cast<int32_t>(r.distances[v]);
  });
}

// Same BFS loop as algorithms.cpp:29-58 but recording, per level, the mode
// edge_map chose (0 sparse, 1 dense) and the input frontier size.
int gbref_bfs_trace(void* csr, uint32_t src, int32_t* modes, uint64_t* sizes,
                    uint64_t cap, uint64_t* levels) {
  return guard([&] {
    const GraphContainer& c = *static_cast<CsrGraph*>(csr);
    GraphView g(c);
    uint64_t n = g.num_vertices();
    std::vector<std::atomic<VertexId>> parent(n);
    for (auto& p : parent) p.store(kNoVertex, std::memory_order_relaxed);
    parent[src].store(src);
    VertexSubset frontier = VertexSubset::singleton(n, src);
    uint64_t lvl = 0;
    while (frontier.size() > 0) {
      auto update = [&](VertexId u, VertexId v) {
        parent[v].store(u, std::memory_order_relaxed);
        return true;
      };
      auto cond = [&](VertexId v) {
        return parent[v].load(std::memory_order_relaxed) == kNoVertex;
      };
      EdgeMapMode mode;
      EdgeMapSpec spec{update, cond};
      spec.mode_out = &mode;
      if (lvl < cap) sizes[lvl] = frontier.size();
      frontier = edge_map(g, frontier, spec);
      if (lvl < cap) modes[lvl] = mode == EdgeMapMode::Dense ? 1 : 0;
      ++lvl;
    }
    *levels = lvl;
  });
}

int gbref_pagerank(void* csr, double damping, uint64_t iters, double tol, double* out) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    std::vector<double> p = pagerank(view, damping, iters, tol);
    std::memcpy(out, p.data(), p.size() * sizeof(double));
  });
}

// gb::bc (algorithms.cpp:60-103): single-source Brandes dependencies
int gbref_bc(void* csr, uint32_t src, double* out) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    std::vector<double> d = bc(view, src);
    std::memcpy(out, d.data(), d.size() * sizeof(double));
  });
}

int gbref_cc(void* csr, uint32_t* labels) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    std::vector<VertexId> l = cc(view);
    std::memcpy(labels, l.data(), l.size() * sizeof(uint32_t));
  });
}

int gbref_kcore(void* csr, uint64_t* out) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    std::vector<uint64_t> c = kcore(view);
    std::memcpy(out, c.data(), c.size() * sizeof(uint64_t));
  });
}

int gbref_coloring(void* csr, uint32_t* out) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    std::vector<uint32_t> c = coloring(view);
    std::memcpy(out, c.data(), c.size() * sizeof(uint32_t));
  });
}

int gbref_mis(void* csr, uint64_t seed, uint8_t* out) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    std::vector<uint8_t> s = mis(view, seed);
    std::memcpy(out, s.data(), s.size());
  });
}

int gbref_ldd(void* csr, double beta, uint64_t seed, uint32_t* labels, uint32_t* parents, uint64_t* rounds) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    LddResult r = ldd(view, beta, seed);
    std::memcpy(labels, r.labels.data(), r.labels.size() * sizeof(uint32_t));
    std::memcpy(parents, r.parents.data(), r.parents.size() * sizeof(uint32_t));
    std::memcpy(rounds, r.rounds.data(), r.rounds.size() * sizeof(uint64_t));
  });
}

// byte_offsets[n+1] and the concatenated segments; *nbytes in/out (pass
// bytes == nullptr to query the size)
int gbref_compressed(void* csr, uint64_t* byte_offsets, uint8_t* bytes, uint64_t* nbytes) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(csr);
    CompressedCsrGraph c = CompressedCsrGraph::build(g);
    uint64_t pos = 0;
    for (VertexId v = 0; v < g.num_vertices(); ++v) {
      auto seg = c.segment(v);
      if (byte_offsets) byte_offsets[v] = pos;
      if (bytes) std::memcpy(bytes + pos, seg.data(), seg.size());
      pos += seg.size();
    }
    if (byte_offsets) byte_offsets[g.num_vertices()] = pos;
    *nbytes = pos;
  });
}

void gbref_log1p(const double* x, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = std::log1p(x[i]);
}

// One edge_map call with a membership cond given as a byte mask (cond[v] !=
// 0) and update always true.  mode: 0 sparse, 1 dense, 2 auto (edge_map).
// Frontier given as sorted-or-not id list.  Output: membership bytes.
int gbref_edge_map(void* csr, const uint32_t* ids, uint64_t nids,
                   const uint8_t* cond, int mode, int early_exit,
                   uint8_t* out_member, uint64_t* out_updates, int* mode_out) {
  return guard([&] {
    const GraphContainer& c = *static_cast<CsrGraph*>(csr);
    GraphView g(c);
    uint64_t n = g.num_vertices();
    VertexSubset frontier(n, std::vector<VertexId>(ids, ids + nids));
    std::atomic<uint64_t> updates{0};
    auto update = [&](VertexId, VertexId) {
      updates.fetch_add(1);
      return true;
    };
    auto cnd = [&](VertexId v) { return cond[v] != 0; };
    EdgeMapSpec spec{update, cnd};
    spec.allow_dense_early_exit = early_exit != 0;
    EdgeMapMode chosen;
    spec.mode_out = &chosen;
    VertexSubset out = mode == 0   ? edge_map_sparse(g, frontier, spec)
                       : mode == 1 ? edge_map_dense(g, frontier, spec)
                                   : edge_map(g, frontier, spec);
    std::memset(out_member, 0, n);
    out.for_each([&](VertexId v) { out_member[v] = 1; });
    *out_updates = updates.load();
    if (mode_out) *mode_out = mode == 2 ? (chosen == EdgeMapMode::Dense ? 1 : 0) : mode;
  });
}

// vertex_filter (traversal.cpp:117-131), pred(v) = keep[v] != 0.  words ==
// nullptr: sparse input ids[k] -> out_ids[*out_k] in the reference's order;
// else dense input -> out_words (and *out_k = member count).  *out_dense
// reports the output representation.
int gbref_vertex_filter(uint64_t n, const uint32_t* ids, uint64_t k, const uint64_t* words,
                        const uint8_t* keep, uint32_t* out_ids, uint64_t* out_words,
                        uint64_t* out_k, int* out_dense) {
  return guard([&] {
    VertexSubset s = words ? VertexSubset(n, std::vector<uint64_t>(words, words + (n + 63) / 64),
                                          VertexSubset::Repr::Dense)
                           : VertexSubset(n, std::vector<VertexId>(ids, ids + k));
    VertexSubset r = vertex_filter(s, [&](VertexId v) { return keep[v] != 0; });
    *out_dense = r.is_dense() ? 1 : 0;
    *out_k = r.size();
    if (r.is_dense())
      std::copy(r.words().begin(), r.words().end(), out_words);
    else
      std::copy(r.ids().begin(), r.ids().end(), out_ids);
  });
}

// ---- batches ----
int gbref_update_batch(uint64_t log2_n, double a, double b, double c,
                       uint64_t size, uint64_t seed, uint32_t* out_pairs) {
  return guard([&] {
    RmatParams p;
    p.a = a;
    p.b = b;
    p.c = c;
    p.log2_n = log2_n;
    EdgeBatch eb = generate_update_batch(p, size, seed);
    edges_to_pairs(eb.updates, out_pairs);
  });
}

// prepare(GlobalSort); returns the prepared count through *out_count.
int gbref_prepare_global(const uint32_t* pairs, uint64_t count, uint32_t* out_pairs,
                         uint64_t* out_count) {
  return guard([&] {
    EdgeBatch eb{pairs_to_edges(pairs, count)};
    PreparedBatch pb = prepare(eb, BatchForm::GlobalSort);
    edges_to_pairs(pb.arcs, out_pairs);
    *out_count = pb.arcs.size();
  });
}

// ---- the dynamic reference container (config 5): "chunked_set" ----
void* gbref_chunked_build(uint64_t n, const uint32_t* pairs, uint64_t count) {
  void* out = nullptr;
  guard([&] {
    GraphData g;
    g.n = n;
    g.arcs = pairs_to_edges(pairs, count);
    out = container_by_name("chunked_set").build(g).release();
  });
  return out;
}

void gbref_container_free(void* c) { delete static_cast<GraphContainer*>(c); }

int gbref_chunked_apply(void* c, const uint32_t* pairs, uint64_t count, int insert,
                        uint64_t* applied) {
  return guard([&] {
    GraphContainer& g = *static_cast<GraphContainer*>(c);
    EdgeBatch eb{pairs_to_edges(pairs, count)};
    PreparedBatch pb = prepare(eb, g.preferred_batch_form());
    *applied = insert ? apply_insert(g, pb) : apply_delete(g, pb);
  });
}

uint64_t gbref_container_m(void* c) { return static_cast<GraphContainer*>(c)->num_edges(); }
uint64_t gbref_container_n(void* c) { return static_cast<GraphContainer*>(c)->num_vertices(); }
uint64_t gbref_container_degree(void* c, uint32_t v) {
  return static_cast<GraphContainer*>(c)->degree(v);
}

int gbref_container_export(void* c, uint64_t* off, uint32_t* nbr) {
  return guard([&] { export_container(*static_cast<GraphContainer*>(c), off, nbr); });
}

int gbref_container_bfs(void* c, uint32_t src, int32_t* depth) {
  return guard([&] {
    GraphView view(*static_cast<GraphContainer*>(c));
    BfsResult r = bfs(view, src);
    for (size_t v = 0; v < r.distances.size(); ++v)
      depth[v] = r.distances[v] == kInfiniteDistance ? -1 : static_cast<int32_t>(r.distances[v]);
  });
}

// ---- timed calls for bench.py's CPU legs: steady_clock around the
// reference call alone, as bench.cpp times a trial (bench.cpp:88-103) and
// an update (prepare + apply, bench.cpp:171-186); conversions stay outside
namespace {
double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

int gbref_time_pagerank(void* csr, double damping, uint64_t iters, double tol, double* seconds,
                        double* rank_sum) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    auto t0 = std::chrono::steady_clock::now();
    std::vector<double> p = pagerank(view, damping, iters, tol);
    *seconds = seconds_since(t0);
    double s = 0.0;
    for (double x : p) s += x;
    *rank_sum = s;
  });
}

int gbref_time_bfs(void* csr, uint32_t src, double* seconds, uint64_t* reached) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    auto t0 = std::chrono::steady_clock::now();
    BfsResult r = bfs(view, src);
    *seconds = seconds_since(t0);
    uint64_t k = 0;
    for (uint64_t d : r.distances) k += d != kInfiniteDistance;
    *reached = k;
  });
}

int gbref_time_cc(void* csr, double* seconds, uint64_t* components) {
  return guard([&] {
    GraphView view(*static_cast<CsrGraph*>(csr));
    auto t0 = std::chrono::steady_clock::now();
    std::vector<VertexId> l = cc(view);
    *seconds = seconds_since(t0);
    uint64_t k = 0;
    for (size_t v = 0; v < l.size(); ++v) k += l[v] == v;
    *components = k;
  });
}

int gbref_chunked_apply_timed(void* c, const uint32_t* pairs, uint64_t count, int insert, uint64_t* applied,
                              double* seconds) {
  return guard([&] {
    GraphContainer& g = *static_cast<GraphContainer*>(c);
    EdgeBatch eb{pairs_to_edges(pairs, count)};
    auto t0 = std::chrono::steady_clock::now();
    PreparedBatch pb = prepare(eb, g.preferred_batch_form());
    *applied = insert ? apply_insert(g, pb) : apply_delete(g, pb);
    *seconds = seconds_since(t0);
  });
}

int gbref_container_bfs_timed(void* c, uint32_t src, double* seconds, uint64_t* reached) {
  return guard([&] {
    GraphView view(*static_cast<GraphContainer*>(c));
    auto t0 = std::chrono::steady_clock::now();
    BfsResult r = bfs(view, src);
    *seconds = seconds_since(t0);
    uint64_t k = 0;
    for (uint64_t d : r.distances) k += d != kInfiniteDistance;
    *reached = k;
  });
}

}  // extern "C"

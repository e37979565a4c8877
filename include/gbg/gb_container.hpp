// gb_container.hpp — lifts libgbg handles into the reference's plugin
// surface, gb::GraphContainer (graph_container.hpp:36-87), so the reference
// harness drives the device containers unchanged: registry-style
// ContainerInfo factories (registry.hpp:15-19) for
// VerifyOptions::extra_containers (bench.hpp:79-83), apply_insert /
// apply_delete (batch.cpp:105-126), and run_benchmark's MaskedGraph wrapper
// (bench.cpp:78-81).
//
// Reads served to CPU callers (map_neighbors & co.) come from a host mirror
// of the adjacency, fetched once from the device (gbg_export_csr) and
// refreshed after every update; the device algorithms (gbg::bfs, pagerank,
// cc, bc, ldd, kcore, coloring, mis, triangle_count below) run on the device copy.  Errors come back as the
// reference's exception types.
//
// Header-only; needs the reference include tree (-I <reference>/include) and
// libgbg.so at link time.
#pragma once

#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gb/algorithms.hpp"
#include "gb/graph_container.hpp"
#include "gb/graph_data.hpp"
#include "gb/registry.hpp"
#include "gbg_c.h"

namespace gbg {

// gbg_status -> the reference exception it mirrors (types.hpp:43-62).
inline void check(gbg_status s) {
  if (s == GBG_OK) return;
  std::string msg = gbg_last_error();
  switch (s) {
    case GBG_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case GBG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case GBG_ERR_UNSUPPORTED: throw gb::unsupported_operation(msg);
    case GBG_ERR_CONFIG: throw gb::config_error(msg);
    case GBG_ERR_FORMAT: throw gb::format_error(msg);
    case GBG_ERR_LOGIC: throw std::logic_error(msg);
    case GBG_ERR_OOM: throw std::bad_alloc();
    default: throw std::runtime_error("gbg: " + msg);
  }
}

static_assert(sizeof(gb::Edge) == 2 * sizeof(uint32_t), "gb::Edge must be two packed uint32 ids");

class GpuGraph : public gb::GraphContainer {
 public:
  explicit GpuGraph(gbg_graph* h) : h_(h) {}
  ~GpuGraph() override { gbg_graph_destroy(h_); }
  GpuGraph(const GpuGraph&) = delete;
  GpuGraph& operator=(const GpuGraph&) = delete;

  gbg_graph* handle() const { return h_; }

  uint64_t num_vertices() const override {
    uint64_t n = 0;
    check(gbg_num_vertices(h_, &n));
    return n;
  }
  uint64_t num_edges() const override {
    uint64_t m = 0;
    check(gbg_num_edges(h_, &m));
    return m;
  }
  uint64_t degree(gb::VertexId i) const override {
    range(i);
    const Mirror& mm = mirror();
    return mm.off[i + 1] - mm.off[i];
  }
  void map_neighbors(gb::VertexId i, gb::NeighborFn f) const override {
    range(i);
    const Mirror& mm = mirror();
    for (uint64_t k = mm.off[i]; k < mm.off[i + 1]; ++k) f(mm.nbr[k]);
  }
  void map_neighbors_early_exit(gb::VertexId i, gb::NeighborStopFn f) const override {
    range(i);
    const Mirror& mm = mirror();
    for (uint64_t k = mm.off[i]; k < mm.off[i + 1]; ++k)
      if (f(mm.nbr[k])) return;
  }
  void parallel_map_neighbors(gb::VertexId i, gb::NeighborFn f) const override { map_neighbors(i, f); }
  void parallel_map_neighbors_early_exit(gb::VertexId i, gb::NeighborStopFn f) const override {
    map_neighbors_early_exit(i, f);
  }

  gb::Capabilities capabilities() const override {
    gbg_caps c{};
    check(gbg_capabilities(h_, &c));
    return {c.has_num_edges != 0, c.has_degree != 0, c.has_map_early_exit != 0, c.has_parallel_map != 0,
            c.has_parallel_map_early_exit != 0, c.has_batch_updates != 0};
  }

  bool insert_edge(gb::Edge e) override {
    int changed = 0;
    check(gbg_insert_edge(h_, e.src, e.dst, &changed));
    invalidate();
    return changed != 0;
  }
  bool delete_edge(gb::Edge e) override {
    int changed = 0;
    check(gbg_delete_edge(h_, e.src, e.dst, &changed));
    invalidate();
    return changed != 0;
  }
  // The device path re-prepares (sort + dedup) anyway, so any form is fine.
  uint64_t insert_sorted_batch(std::span<const gb::Edge> batch) override {
    uint64_t applied = 0;
    check(gbg_insert_batch(h_, reinterpret_cast<const uint32_t*>(batch.data()), batch.size(), &applied));
    invalidate();
    return applied;
  }
  uint64_t delete_sorted_batch(std::span<const gb::Edge> batch) override {
    uint64_t applied = 0;
    check(gbg_delete_batch(h_, reinterpret_cast<const uint32_t*>(batch.data()), batch.size(), &applied));
    invalidate();
    return applied;
  }
  gb::BatchForm preferred_batch_form() const override { return gb::BatchForm::GlobalSort; }

  uint64_t memory_bytes() const override {
    uint64_t b = 0;
    check(gbg_memory_bytes(h_, &b));
    return b;
  }

 private:
  struct Mirror {
    std::vector<uint64_t> off;
    std::vector<uint32_t> nbr;
  };
  void range(gb::VertexId i) const {
    if (i >= num_vertices()) throw std::out_of_range("vertex out of range");
  }
  const Mirror& mirror() const {
    std::lock_guard<std::mutex> lk(mu_);
    if (!mirror_) {
      auto m = std::make_unique<Mirror>();
      m->off.resize(num_vertices() + 1);
      m->nbr.resize(num_edges() + 1);
      check(gbg_export_csr(h_, m->off.data(), m->nbr.data()));
      mirror_ = std::move(m);
    }
    return *mirror_;
  }
  void invalidate() {
    std::lock_guard<std::mutex> lk(mu_);
    mirror_.reset();
  }

  gbg_graph* h_;
  mutable std::mutex mu_;
  mutable std::unique_ptr<Mirror> mirror_;
};

// gb::CsrGraph on the device (csr.hpp:12-53); rejects updates.
class GpuCsrGraph final : public GpuGraph {
 public:
  using GpuGraph::GpuGraph;
  static std::unique_ptr<GpuCsrGraph> build(uint64_t n, std::span<const gb::Edge> arcs) {
    gbg_graph* h = nullptr;
    check(gbg_csr_from_arcs(n, reinterpret_cast<const uint32_t*>(arcs.data()), arcs.size(), &h));
    return std::make_unique<GpuCsrGraph>(h);
  }
};

// The dynamic blocked container in the chunked_set role (registry.cpp:136-137).
class GpuBlockedGraph final : public GpuGraph {
 public:
  using GpuGraph::GpuGraph;
  static std::unique_ptr<GpuBlockedGraph> build(uint64_t n, std::span<const gb::Edge> arcs) {
    gbg_graph* h = nullptr;
    check(gbg_blocked_create(n, reinterpret_cast<const uint32_t*>(arcs.data()), arcs.size(), &h));
    return std::make_unique<GpuBlockedGraph>(h);
  }
};

// gb::CompressedCsrGraph (compressed_csr.hpp:12-46) on the device; static,
// no parallel maps (its capabilities say so, like the reference's).
class GpuCompressedGraph final : public GpuGraph {
 public:
  using GpuGraph::GpuGraph;
  static std::unique_ptr<GpuCompressedGraph> build(uint64_t n, std::span<const gb::Edge> arcs) {
    gbg_graph* csr = nullptr;
    check(gbg_csr_from_arcs(n, reinterpret_cast<const uint32_t*>(arcs.data()), arcs.size(), &csr));
    gbg_graph* h = nullptr;
    const gbg_status st = gbg_compressed_from(csr, &h);
    gbg_graph_destroy(csr);
    check(st);
    return std::make_unique<GpuCompressedGraph>(h);
  }
};

// Factories in the shape of the reference registry (registry.cpp:112-142),
// for VerifyOptions::extra_containers.
inline const std::vector<gb::ContainerInfo>& gpu_containers() {
  static const std::vector<gb::ContainerInfo> list = {
      {"gpu_csr", false,
       [](const gb::GraphData& g) -> gb::GraphContainerPtr { return GpuCsrGraph::build(g.n, g.arcs); }},
      {"gpu_blocked", true,
       [](const gb::GraphData& g) -> gb::GraphContainerPtr { return GpuBlockedGraph::build(g.n, g.arcs); }},
      {"gpu_compressed", false,
       [](const gb::GraphData& g) -> gb::GraphContainerPtr { return GpuCompressedGraph::build(g.n, g.arcs); }},
  };
  return list;
}

// ---- device algorithms with the reference's result shapes -------------
inline const GpuGraph& device_of(const gb::GraphView& view) {
  auto* g = dynamic_cast<const GpuGraph*>(&view.container());
  if (!g) throw gb::unsupported_operation("gbg: view is not backed by a device container (no CPU fallback)");
  return *g;
}

// gb::bfs(...).distances (algorithms.cpp:29-58): kInfiniteDistance when unreached.
inline std::vector<uint64_t> bfs_distances(const GpuGraph& g, gb::VertexId source) {
  std::vector<int32_t> d(g.num_vertices());
  check(gbg_bfs(g.handle(), source, d.data(), nullptr));
  std::vector<uint64_t> out(d.size());
  for (size_t v = 0; v < d.size(); ++v) out[v] = d[v] < 0 ? gb::kInfiniteDistance : static_cast<uint64_t>(d[v]);
  return out;
}

inline std::vector<double> pagerank(const GpuGraph& g, double damping, uint64_t max_iters, double tolerance) {
  std::vector<double> p(g.num_vertices());
  check(gbg_pagerank(g.handle(), damping, max_iters, tolerance, p.data(), nullptr));
  return p;
}

inline std::vector<gb::VertexId> cc(const GpuGraph& g) {
  std::vector<gb::VertexId> l(g.num_vertices());
  check(gbg_cc(g.handle(), l.data()));
  return l;
}

// gb::bc (algorithms.cpp:60-103)
inline std::vector<double> bc(const GpuGraph& g, gb::VertexId source) {
  std::vector<double> d(g.num_vertices());
  check(gbg_bc(g.handle(), source, d.data()));
  return d;
}

// gb::kcore (algorithms.cpp:330-374)
inline std::vector<uint64_t> kcore(const GpuGraph& g) {
  std::vector<uint64_t> c(g.num_vertices());
  check(gbg_kcore(g.handle(), c.data()));
  return c;
}

// gb::coloring (algorithms.cpp:376-432); symmetric graphs
inline std::vector<uint32_t> coloring(const GpuGraph& g) {
  std::vector<uint32_t> c(g.num_vertices());
  check(gbg_coloring(g.handle(), c.data()));
  return c;
}

// gb::mis (algorithms.cpp:434-504); symmetric graphs
inline std::vector<uint8_t> mis(const GpuGraph& g, uint64_t seed) {
  std::vector<uint8_t> f(g.num_vertices());
  check(gbg_mis(g.handle(), seed, f.data()));
  return f;
}

// gb::ldd (algorithms.cpp:114-188), the reference's result struct
inline gb::LddResult ldd(const GpuGraph& g, double beta, uint64_t seed) {
  gb::LddResult r;
  const uint64_t n = g.num_vertices();
  r.labels.resize(n);
  r.parents.resize(n);
  r.rounds.resize(n);
  check(gbg_ldd(g.handle(), beta, seed, r.labels.data(), r.parents.data(), r.rounds.data()));
  return r;
}

inline uint64_t triangle_count(const GpuGraph& g) {
  uint64_t t = 0;
  check(gbg_tc(g.handle(), &t));
  return t;
}

// AlgorithmInfo-shaped entries (registry.hpp:26-29) running on the device
// when the view's container is a GpuGraph (an unmasked view).
inline const std::vector<gb::AlgorithmInfo>& gpu_algorithms() {
  static const std::vector<gb::AlgorithmInfo> list = {
      {"bfs",
       [](const gb::GraphView& v, const gb::AlgoParams& p) {
         gb::CanonicalOutput out;
         out.ints = bfs_distances(device_of(v), p.source);
         return out;
       }},
      {"bc",
       [](const gb::GraphView& v, const gb::AlgoParams& p) {
         gb::CanonicalOutput out;
         out.reals = bc(device_of(v), p.source);
         return out;
       }},
      {"cc",
       [](const gb::GraphView& v, const gb::AlgoParams&) {
         gb::CanonicalOutput out;
         for (gb::VertexId l : cc(device_of(v))) out.ints.push_back(l);
         return out;
       }},
      {"ldd",
       [](const gb::GraphView& v, const gb::AlgoParams& p) {
         gb::CanonicalOutput out;
         for (gb::VertexId l : ldd(device_of(v), p.beta, p.seed).labels) out.ints.push_back(l);
         return out;
       }},
      {"kcore",
       [](const gb::GraphView& v, const gb::AlgoParams&) {
         gb::CanonicalOutput out;
         out.ints = kcore(device_of(v));
         return out;
       }},
      {"coloring",
       [](const gb::GraphView& v, const gb::AlgoParams&) {
         gb::CanonicalOutput out;
         for (uint32_t c : coloring(device_of(v))) out.ints.push_back(c);
         return out;
       }},
      {"mis",
       [](const gb::GraphView& v, const gb::AlgoParams& p) {
         gb::CanonicalOutput out;
         for (uint8_t f : mis(device_of(v), p.seed)) out.ints.push_back(f);
         return out;
       }},
      {"pagerank",
       [](const gb::GraphView& v, const gb::AlgoParams& p) {
         gb::CanonicalOutput out;
         out.reals = pagerank(device_of(v), p.damping, p.max_iters, p.tolerance);
         return out;
       }},
  };
  return list;
}

}  // namespace gbg

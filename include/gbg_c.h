/*
 * gbg_c.h — C ABI of the B200-native frontier-traversal + batch-update
 * library (paper_2405_11671_b200/libgbg.so).
 *
 * This is the drop-in boundary for the hot path of BYO's `graphbench`
 * (reference: /root/reference/proj).  The reference exposes no C ABI: its
 * surface is the C++ virtual class gb::GraphContainer
 * (include/gb/graph_container.hpp:36-87) plus free algorithm / traversal
 * functions (include/gb/algorithms.hpp:28-76, include/gb/traversal.hpp:37-56)
 * and the batch pipeline (include/gb/batch.hpp:32-56).  Each entry point
 * below names the reference interface it replaces.  The C++ adapter in
 * include/gbg/gb_container.hpp lifts these handles back into
 * gb::GraphContainer so the reference harness (run_benchmark,
 * verify_graph's extra_containers, apply_insert/apply_delete) drives them
 * unchanged; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "host" buffers are ordinary CPU memory
 *    owned by the caller; "_device" variants take/produce device pointers
 *    on the handle's CUDA device.
 *  - Every call returns gbg_status; on failure gbg_last_error() (thread
 *    local) holds the message.  Status codes map 1:1 onto the reference's
 *    exception types (types.hpp:43-62 and the std:: exceptions listed in
 *    SURVEY §8b): OUT_OF_RANGE -> std::out_of_range, INVALID_ARGUMENT ->
 *    std::invalid_argument, UNSUPPORTED -> gb::unsupported_operation,
 *    CONFIG -> gb::config_error, FORMAT -> gb::format_error, LOGIC ->
 *    std::logic_error.
 *  - Calls on one handle are serialised by a per-handle mutex and run on the
 *    handle's own CUDA stream (gbg_stream()); read calls are safe from many
 *    threads (graph_container.hpp:31-35), updates are phased by the caller.
 *  - Vertex ids are uint32 (types.hpp:11); arcs are (src,dst) uint32 pairs,
 *    the byte layout of gb::Edge (types.hpp:18-26).
 */
#ifndef GBG_C_H
#define GBG_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gbg_status {
  GBG_OK = 0,
  GBG_ERR_CUDA = 1,
  GBG_ERR_OOM = 2,
  GBG_ERR_OUT_OF_RANGE = 3,
  GBG_ERR_INVALID_ARGUMENT = 4,
  GBG_ERR_UNSUPPORTED = 5,
  GBG_ERR_CONFIG = 6,
  GBG_ERR_FORMAT = 7,
  GBG_ERR_LOGIC = 8
} gbg_status;

typedef struct gbg_graph gbg_graph;

/* Mirrors gb::Capabilities (capabilities.hpp:14-48). */
typedef struct gbg_caps {
  int has_num_edges;
  int has_degree;
  int has_map_early_exit;
  int has_parallel_map;
  int has_parallel_map_early_exit;
  int has_batch_updates;
} gbg_caps;

enum { GBG_KIND_CSR = 0, GBG_KIND_BLOCKED = 1, GBG_KIND_COMPRESSED = 2 };
enum { GBG_MODE_SPARSE = 0, GBG_MODE_DENSE = 1, GBG_MODE_AUTO = 2 };

#define GBG_MAX_LEVELS 64
/* Per-level record of a BFS run (the reference's EdgeMapSpec::mode_out,
 * traversal.hpp:32, plus the work the direction switch saw). */
typedef struct gbg_bfs_stats {
  uint64_t levels;                       /* edge_map calls made            */
  int32_t mode[GBG_MAX_LEVELS];          /* GBG_MODE_SPARSE / _DENSE       */
  uint64_t frontier[GBG_MAX_LEVELS];     /* |F| fed to level i             */
  uint64_t degree_sum[GBG_MAX_LEVELS];   /* sum deg(F) fed to level i      */
  uint64_t reached;                      /* vertices with depth >= 0       */
  float level_ms[GBG_MAX_LEVELS];        /* device time of level i; persistent path: only with GBG_BFS_LEVEL_TIMES=1, else 0 */
  uint64_t examined[GBG_MAX_LEVELS];     /* arcs inspected by level i in the reference's
                                            order: sum deg(F) for a push, and for an
                                            early-exit pull each vertex's list up to
                                            its first frontier hit (SURVEY §8(d) E_scan) */
} gbg_bfs_stats;

/* ---- errors / runtime ---------------------------------------------- */
const char* gbg_last_error(void);
/* Select the CUDA device used by handles created afterwards on this thread. */
gbg_status gbg_set_device(int device);
/* Number of library kernels launched on this handle since creation. */
uint64_t gbg_launch_count(const gbg_graph* g);
/* The handle's cudaStream_t (as void*), for event timing by callers. */
void* gbg_stream(const gbg_graph* g);
gbg_status gbg_synchronize(gbg_graph* g);

/* ---- containers ----------------------------------------------------- */
/* gb::CsrGraph::build from CSR arrays (csr.cpp:9-25): offsets[n+1],
 * neighbors[m] host arrays; rejects out-of-range ids and non-increasing
 * segments with GBG_ERR_FORMAT, like csr.cpp:14-18. */
gbg_status gbg_csr_create(uint64_t n, uint64_t m, const uint64_t* offsets,
                          const uint32_t* neighbors, gbg_graph** out);
/* gbg_csr_create with build flags.  GBG_CREATE_PAGERANK_LAYOUT also builds
 * the degree-ordered PageRank layout while the neighbour ids upload (it is
 * otherwise built by the first gbg_pagerank call).  The upload is chunked
 * and overlapped with validation either way; pinned host buffers make it
 * asynchronous. */
enum { GBG_CREATE_PAGERANK_LAYOUT = 1 };
gbg_status gbg_csr_create_ex(uint64_t n, uint64_t m, const uint64_t* offsets,
                             const uint32_t* neighbors, uint32_t flags, gbg_graph** out);
/* gb::CsrGraph::build(n, arcs) from sorted, deduplicated (src,dst) pairs. */
gbg_status gbg_csr_from_arcs(uint64_t n, const uint32_t* arcs, uint64_t m, gbg_graph** out);
/* The dynamic blocked sorted-adjacency container: the role of
 * SetGraph<ChunkedSortedSet> with inline_k = 0 ("chunked_set",
 * registry.cpp:136-137) built by insert_sorted_batch(g.arcs)
 * (registry.cpp:16-21).  arcs: GlobalSort-prepared pairs. */
gbg_status gbg_blocked_create(uint64_t n, const uint32_t* arcs, uint64_t m, gbg_graph** out);
/* Device-side copy of a CSR handle into a new blocked container. */
gbg_status gbg_blocked_from_csr(gbg_graph* csr, gbg_graph** out);
/* gb::generate_rmat (generators.cpp:67-72) on the device, bit-exact:
 * `arcs` recursive-quadrant draws with rng_double(seed, i, level)
 * (batch.cpp:128-154), symmetrised, self-loops dropped, deduplicated;
 * n = 2^log2_n.  kind = GBG_KIND_CSR or GBG_KIND_BLOCKED. */
gbg_status gbg_rmat_create(uint32_t log2_n, uint64_t arcs, double a, double b, double c,
                           uint64_t seed, int kind, gbg_graph** out);
gbg_status gbg_graph_destroy(gbg_graph* g);
/* gb::CompressedCsrGraph::build (compressed_csr.cpp:5-17) on the device:
 * the byte code of bytecode.hpp:11-62 (zig-zag first delta from the vertex
 * id, then gaps, base-128 varints) with byte_offsets[n+1].  Static
 * (updates -> GBG_ERR_UNSUPPORTED), capabilities {1,1,1,0,0,0}
 * (compressed_csr.hpp:27-29).  _from encodes any handle's lists; _create
 * takes host CSR arrays validated like gbg_csr_create. */
gbg_status gbg_compressed_from(gbg_graph* src, gbg_graph** out);
gbg_status gbg_compressed_create(uint64_t n, uint64_t m, const uint64_t* offsets,
                                 const uint32_t* neighbors, gbg_graph** out);
/* The raw encoding: byte_offsets[n+1] and bytes[*nbytes] (either may be
 * NULL to query *nbytes first) — CompressedCsrGraph::segment's data. */
gbg_status gbg_compressed_bytes(gbg_graph* g, uint64_t* byte_offsets, uint8_t* bytes, uint64_t* nbytes);
/* GBCSR1 binary graph files (io.cpp:75-114; README.md:134-138): magic
 * "GBCSR1\0\0", n and m as little-endian uint64, n+1 uint64 offsets, m uint32
 * neighbour ids.  load = load_binary_csr (validated like csr.cpp:14-18 and
 * io.cpp:91-108, GBG_ERR_FORMAT otherwise) straight into a device container
 * of `kind`; save = save_binary from any container (lists ascending). */
gbg_status gbg_load_gbcsr1(const char* path, int kind, gbg_graph** out);
gbg_status gbg_save_gbcsr1(gbg_graph* g, const char* path);

/* ---- read API (graph_container.hpp:39-60, csr.hpp:19-33) ------------ */
gbg_status gbg_kind(const gbg_graph* g, int* kind);
gbg_status gbg_num_vertices(const gbg_graph* g, uint64_t* n);
gbg_status gbg_num_edges(const gbg_graph* g, uint64_t* m);
gbg_status gbg_degree(gbg_graph* g, uint32_t v, uint64_t* deg);
/* All degrees, host uint64[n]. */
gbg_status gbg_degrees(gbg_graph* g, uint64_t* out);
/* map_neighbors(v) materialised: up to `cap` ids in ascending order into
 * host `out`; *deg receives the full degree. */
gbg_status gbg_neighbors(gbg_graph* g, uint32_t v, uint32_t* out, uint64_t cap, uint64_t* deg);
/* Whole adjacency as CSR into host offsets[n+1], neighbors[m] (the host
 * mirror the C++ adapter serves map_neighbors from). */
gbg_status gbg_export_csr(gbg_graph* g, uint64_t* offsets, uint32_t* neighbors);
gbg_status gbg_capabilities(const gbg_graph* g, gbg_caps* caps);
/* graph_container.hpp:86: bytes of device memory holding the topology. */
gbg_status gbg_memory_bytes(const gbg_graph* g, uint64_t* bytes);

/* ---- vertex_subset (vertex_subset.hpp:15-77) ------------------------- */
/* to_dense (vertex_subset.cpp:32-37): ids[k] (any order, duplicates ok) ->
 * ceil(n/64) uint64 words, bit v = vertex v, LSB first.  Host buffers. */
gbg_status gbg_subset_to_dense(uint64_t n, const uint32_t* ids, uint64_t k, uint64_t* words);
/* to_sparse (vertex_subset.cpp:39-45): words -> ascending ids; *k = size. */
gbg_status gbg_subset_to_sparse(uint64_t n, const uint64_t* words, uint32_t* ids, uint64_t* k);
/* vertex_filter (traversal.cpp:117-131) with pred(v) = keep[v] != 0, in the
 * input's representation: sparse ids[k] -> out[*out_k] (ascending and
 * unique, as VertexSubset's constructor makes them, vertex_subset.cpp:8-15;
 * out holds k entries), dense words -> out_words.  vertex_map (traversal.cpp:113-115) applies a
 * host callback per member and has nothing to offload. */
gbg_status gbg_vertex_filter_sparse(uint64_t n, const uint32_t* ids, uint64_t k, const uint8_t* keep,
                                    uint32_t* out, uint64_t* out_k);
gbg_status gbg_vertex_filter_dense(uint64_t n, const uint64_t* words, const uint8_t* keep, uint64_t* out_words);

/* ---- edge_map (traversal.hpp:37-56 / traversal.cpp:16-111) ---------- */
/* One edge_map over frontier ids[k] with cond(v) = cond_mask[v] != 0 and an
 * update that always returns true; mode GBG_MODE_SPARSE (edge_map_sparse,
 * claim-then-update), _DENSE (edge_map_dense, early exit when early_exit)
 * or _AUTO (edge_map's |F| + sum deg(F) > m/20 switch).  out_member[v] = 1
 * for output members; *updates counts update() calls; *mode_out = chosen. */
gbg_status gbg_edge_map(gbg_graph* g, const uint32_t* ids, uint64_t k, const uint8_t* cond_mask,
                        int mode, int early_exit, uint8_t* out_member, uint64_t* updates,
                        int* mode_out);

/* ---- algorithms (algorithms.hpp) ------------------------------------ */
/* gb::bfs (algorithms.cpp:29-58), direction-optimising with the reference
 * switch; depth int32[n], -1 = unreached (kInfiniteDistance). */
gbg_status gbg_bfs(gbg_graph* g, uint32_t source, int32_t* depth, gbg_bfs_stats* stats);
/* gbg_bfs_device: depths stay in device memory.  With stats == NULL nothing
 * returns to the host and the call is asynchronous on the handle's stream
 * (gbg_stream(); gbg_synchronize() or stream-ordered work before reading
 * depth_dev); with stats the call synchronises to fill them. */
gbg_status gbg_bfs_device(gbg_graph* g, uint32_t source, int32_t* depth_dev, gbg_bfs_stats* stats);
/* gb::pagerank (algorithms.cpp:508-555): fp64, uniform dangling
 * redistribution, stop at max_iters or L1 step < tolerance.  damping must be
 * in (0,1) and tolerance > 0 (GBG_ERR_INVALID_ARGUMENT otherwise). */
gbg_status gbg_pagerank(gbg_graph* g, double damping, uint64_t max_iters, double tolerance,
                        double* ranks, uint64_t* iterations);
gbg_status gbg_pagerank_device(gbg_graph* g, double damping, uint64_t max_iters, double tolerance,
                               double* ranks_dev, uint64_t* iterations);
/* Build (or fetch) the handle's cached PageRank layout — the graph
 * renumbered by degree, see pagerank.cu — ahead of the first gbg_pagerank
 * call; *build_ms = its one-time device build time.  Invalidated by updates. */
gbg_status gbg_pagerank_prepare(gbg_graph* g, double* build_ms);
/* Device bytes held by the handle's cached PageRank indexes (0 when not
 * built): the tiled index gbg_pagerank_prepare builds and the relabelled row
 * layout one-shot calls build.  Both are derived data, dropped on updates. */
gbg_status gbg_pagerank_index_bytes(const gbg_graph* g, uint64_t* tiled, uint64_t* rows);
/* gb::cc (algorithms.cpp:194-234): labels = minimum vertex id of each
 * component. */
gbg_status gbg_cc(gbg_graph* g, uint32_t* labels);
gbg_status gbg_cc_device(gbg_graph* g, uint32_t* labels_dev);
/* gb::bc (algorithms.cpp:60-103): single-source Brandes dependencies over
 * the BFS levels; delta[n] fp64, 0 for unreached vertices. */
gbg_status gbg_bc(gbg_graph* g, uint32_t source, double* delta);
gbg_status gbg_bc_device(gbg_graph* g, uint32_t source, double* delta_dev);
/* gb::kcore (algorithms.cpp:330-374, buckets.cpp:7-59): coreness[n] under
 * out-degree peeling (remaining degree of v drops when a peeled vertex has
 * v as a neighbour).  Coreness is order-independent, so it is exact on any
 * graph. */
gbg_status gbg_kcore(gbg_graph* g, uint64_t* coreness);
/* gb::coloring (algorithms.cpp:376-432): first-fit colours in
 * largest-log-degree-first order, ties to the lower id.  Symmetric graphs
 * only (GBG_ERR_INVALID_ARGUMENT otherwise). */
gbg_status gbg_coloring(gbg_graph* g, uint32_t* colors);
/* gb::mis (algorithms.cpp:434-504): in_set[n] 0/1, the lexicographically
 * first MIS under (rng_u64(seed, 7, v), v).  Symmetric graphs only. */
gbg_status gbg_mis(gbg_graph* g, uint64_t seed, uint8_t* in_set);
/* gb::ldd (algorithms.cpp:114-188): labels[n] (cluster centre), parents[n]
 * (tree edge; itself at centres; UINT32_MAX when none), rounds[n] (round
 * joined).  parents / rounds may be NULL.  beta outside (0, 1] ->
 * GBG_ERR_INVALID_ARGUMENT (std::invalid_argument). */
gbg_status gbg_ldd(gbg_graph* g, double beta, uint64_t seed, uint32_t* labels, uint32_t* parents, uint64_t* rounds);
/* Test hook: the device log1p behind ldd's Exponential shifts on n host
 * values (must equal the host C library's log1p bit for bit). */
gbg_status gbg_selftest_log1p(const double* x, uint64_t n, double* out);
/* Triangle count (not in the reference): orient u->v iff
 * (deg u, u) < (deg v, v) (derive_filter, derive.hpp:48-61), count
 * |N+(u) ∩ N+(v)| over oriented arcs. */
gbg_status gbg_tc(gbg_graph* g, uint64_t* triangles);

/* ---- batch updates (batch.hpp:32-56, graph_container.hpp:64-82) ----- */
/* prepare(GlobalSort) + apply_insert / apply_delete fused on the device:
 * raw arcs (src,dst pairs, may hold self-loops and duplicates) are
 * radix-sorted, self-loops dropped, deduplicated (batch.cpp:34-42) and
 * merged into / removed from the blocked container (set_graph.hpp:197-238).
 * *applied = arcs that changed the container.  Out-of-range ids ->
 * GBG_ERR_OUT_OF_RANGE (set_graph.hpp:145-146).  CSR handles ->
 * GBG_ERR_UNSUPPORTED (graph_container.hpp:71-78). */
gbg_status gbg_insert_batch(gbg_graph* g, const uint32_t* arcs, uint64_t count, uint64_t* applied);
gbg_status gbg_delete_batch(gbg_graph* g, const uint32_t* arcs, uint64_t count, uint64_t* applied);
gbg_status gbg_insert_batch_device(gbg_graph* g, const uint32_t* arcs_dev, uint64_t count,
                                   uint64_t* applied);
gbg_status gbg_delete_batch_device(gbg_graph* g, const uint32_t* arcs_dev, uint64_t count,
                                   uint64_t* applied);
/* insert_edge / delete_edge (graph_container.hpp:64-69); self-loops ->
 * GBG_ERR_INVALID_ARGUMENT (set_graph.hpp:147-148). */
gbg_status gbg_insert_edge(gbg_graph* g, uint32_t src, uint32_t dst, int* changed);
gbg_status gbg_delete_edge(gbg_graph* g, uint32_t src, uint32_t dst, int* changed);
/* Arc membership for `count` device (src,dst) pairs: out_dev[i] = 1 iff the
 * arc is present (ChunkedSortedSet::contains per source,
 * neighbor_sets.hpp:305-310); out-of-range ids give 0.  Used to keep update
 * batches disjoint from the base graph (bench.cpp:150-169). */
gbg_status gbg_contains_device(gbg_graph* g, const uint32_t* arcs_dev, uint64_t count, uint8_t* out_dev);
/* gb::generate_update_batch (batch.cpp:128-154) on the device, bit-exact:
 * writes 2*size (src,dst) pairs (draw, then its reverse) to arcs_dev. */
gbg_status gbg_update_batch_device(uint32_t log2_n, double a, double b, double c, uint64_t size,
                                   uint64_t seed, uint32_t* arcs_dev);

#ifdef __cplusplus
}
#endif
#endif /* GBG_C_H */

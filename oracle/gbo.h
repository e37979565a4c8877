/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hot
 * path (BYO graphbench, /root/reference/proj).  It is the parity checker for
 * the CUDA library and is pinned against the reference itself
 * (oracle/_ref/libgbref.so) and the golden fixtures in tests/golden/.
 * Never linked into the product.  Every function cites the reference
 * file:line it restates.  Return codes: 0 ok, 1 out_of_range, 5 format. */
#ifndef GBO_H
#define GBO_H
#include <stdint.h>

uint64_t gbo_mix64(uint64_t x);
uint64_t gbo_hash_combine(uint64_t a, uint64_t b);
double gbo_rng_double(uint64_t seed, uint64_t stream, uint64_t counter);
uint64_t gbo_rng_u64(uint64_t seed, uint64_t stream, uint64_t counter);

void gbo_update_batch(uint64_t log2_n, double a, double b, double c, uint64_t size,
                      uint64_t seed, uint32_t* out_pairs);
uint64_t gbo_normalize(const uint32_t* raw_pairs, uint64_t count, uint64_t min_n,
                       uint32_t* out_pairs, uint64_t* n_out);
uint64_t gbo_prepare_global(const uint32_t* pairs, uint64_t count, uint32_t* out_pairs);
void gbo_sort_u64(uint64_t* keys, uint64_t count);

int gbo_csr_build(uint64_t n, const uint32_t* pairs, uint64_t m, uint64_t* off, uint32_t* nbr);

int gbo_bfs(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t src, int32_t* depth,
            int32_t* modes, uint64_t* sizes, uint64_t cap, uint64_t* levels);
int gbo_pagerank(uint64_t n, const uint64_t* off, const uint32_t* nbr, double damping,
                 uint64_t iters, double tol, double* out);
uint64_t gbo_bfs_examined(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t src, uint64_t* examined,
                          uint64_t cap);
void gbo_cc(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* labels);
int gbo_bc(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t src, double* delta);
uint64_t gbo_tc(uint64_t n, const uint64_t* off, const uint32_t* nbr);
void gbo_kcore(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint64_t* coreness);
void gbo_coloring(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* colors);
int gbo_ldd(uint64_t n, const uint64_t* off, const uint32_t* nbr, double beta, uint64_t seed, uint32_t* labels,
            uint32_t* parents, uint64_t* rounds);
uint64_t gbo_bytecode_encode(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint64_t* byte_offsets,
                             uint8_t* bytes);
void gbo_mis(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint64_t seed, uint8_t* in_set);

void gbo_subset_to_dense(uint64_t n, const uint32_t* ids, uint64_t k, uint64_t* words);
uint64_t gbo_subset_to_sparse(uint64_t n, const uint64_t* words, uint32_t* ids);

int gbo_edge_map(uint64_t n, const uint64_t* off, const uint32_t* nbr, const uint32_t* ids,
                 uint64_t nids, const uint8_t* cond, int mode, int early_exit, uint8_t* out_member,
                 uint64_t* updates);

uint64_t gbo_set_apply(uint64_t n, const uint64_t* off, const uint32_t* nbr, const uint32_t* batch,
                       uint64_t bcount, int insert, uint64_t* off_out, uint32_t* nbr_out);
/* gbo_omp.c: OpenMP R-MAT generator straight into CSR, GBCSR1 writer */
uint64_t gbo_rmat_csr_omp(uint64_t log2_n, double a, double b, double c, uint64_t draws, uint64_t seed,
                          uint64_t* off, uint32_t** nbr_out);
void gbo_free(void* p);
int gbo_save_gbcsr1(const char* path, uint64_t n, const uint64_t* off, const uint32_t* nbr);
#endif

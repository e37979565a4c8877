/* TEST INFRASTRUCTURE ONLY — see gbo.h.  OpenMP restatement of the
 * reference's R-MAT graph generator, used to produce BASELINE-scale inputs
 * on the host for the CPU reference arm of bench.py (the reference's own
 * generate_rmat sorts 1.07e9 Edge values serially: ~400 s at scale 24).
 * Output is identical by construction: the same counter-based draws
 * (rng.hpp:22-29, batch.cpp:128-154) and the same normalisation
 * (generators.cpp:9-29: drop self loops, add reverses, sort, unique), only
 * the sort is replaced by a per-source bucket sort.  Pinned against
 * gb::generate_rmat in tests/test_oracle.py.  Citations are relative to
 * /root/reference/proj. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <omp.h>

#include "gbo.h"

/* ascending sort of one bucket: insertion sort below 24 keys, else
 * median-of-3 quicksort recursing into the smaller side (qsort's indirect
 * comparator dominated the generator's time) */
static void sort_u32(uint32_t* s, int64_t len) {
  while (len > 24) {
    int64_t mid = len / 2;
    uint32_t a = s[0], b = s[mid], c = s[len - 1];
    uint32_t p = a < b ? (b < c ? b : (a < c ? c : a)) : (a < c ? a : (b < c ? c : b));
    int64_t i = 0, j = len - 1;
    for (;;) {
      while (s[i] < p) ++i;
      while (s[j] > p) --j;
      if (i >= j) break;
      uint32_t t = s[i];
      s[i] = s[j];
      s[j] = t;
      ++i;
      --j;
    }
    /* [0, j] <= p <= [j+1, len) */
    int64_t left = j + 1;
    if (left < len - left) {
      sort_u32(s, left);
      s += left;
      len -= left;
    } else {
      sort_u32(s + left, len - left);
      len = left;
    }
  }
  for (int64_t k = 1; k < len; ++k) {
    uint32_t x = s[k];
    int64_t q = k - 1;
    while (q >= 0 && s[q] > x) {
      s[q + 1] = s[q];
      --q;
    }
    s[q + 1] = x;
  }
}

static inline uint64_t mix64(uint64_t x) { /* rng.hpp:11-16 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static inline uint64_t hash_combine(uint64_t a, uint64_t b) { /* rng.hpp:18-20 */
  return mix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

/* batch.cpp:137-152 for draw i (rng_double(seed, i, level) =
 * mix64(hash_combine(hash_combine(seed, i), level)) >> 11 times 2^-53).
 * The quadrant chain r < a / < a+b / < a+b+c is evaluated as three
 * comparisons against the same left-to-right sums (u gets a 1 from
 * r >= a+b, v from a <= r < a+b or r >= a+b+c): identical bits, no
 * mispredicted branches (they were ~2/3 of the generator's time). */
static inline void rmat_draw(uint64_t log2_n, double a, double b, double c, uint64_t seed, uint64_t i,
                             uint32_t* uo, uint32_t* vo) {
  const uint64_t hs = hash_combine(seed, i);
  const double ab = a + b, abc = a + b + c;
  uint32_t u = 0, v = 0;
  for (uint64_t level = 0; level < log2_n; ++level) {
    const double r = (double)(mix64(hash_combine(hs, level)) >> 11) * 0x1.0p-53;
    const uint32_t q1 = r >= a, q2 = r >= ab, q3 = r >= abc;
    u = (u << 1) | q2;
    v = (v << 1) | ((q1 & (q2 ^ 1u)) | q3);
  }
  *uo = u;
  *vo = v;
}

/* generate_rmat(params, draws, seed) (generators.cpp:67-72) as a CSR:
 * off[2^log2_n + 1] (caller-allocated), *nbr_out malloc'ed (free with
 * gbo_free).  Returns m, or UINT64_MAX when memory runs out. */
uint64_t gbo_rmat_csr_omp(uint64_t log2_n, double a, double b, double c, uint64_t draws, uint64_t seed,
                          uint64_t* off, uint32_t** nbr_out) {
  const uint64_t n = (uint64_t)1 << log2_n;
  const int T = omp_get_max_threads();
  /* per-thread arc counts per source, later per-thread write cursors:
   * the hubs would serialise shared atomic counters */
  uint32_t* cnt = (uint32_t*)calloc((size_t)T * n, sizeof(uint32_t));
  uint64_t* deg = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  if (!cnt || !deg) {
    free(cnt);
    free(deg);
    return UINT64_MAX;
  }
  /* pass 1: arcs per source, both directions, self loops dropped; thread t
   * takes draws [t*draws/T, (t+1)*draws/T) in both passes */
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    uint32_t* mine = cnt + (size_t)t * n;
    const uint64_t i0 = draws * (uint64_t)t / (uint64_t)T, i1 = draws * (uint64_t)(t + 1) / (uint64_t)T;
    /* draws in groups of 64, then the group's increments back to back:
     * the counters miss in cache, and a tight loop keeps many misses in
     * flight where one after each 24-level draw would not */
    uint32_t us[64], vs[64];
    for (uint64_t g = i0; g < i1; g += 64) {
      const int k = (int)(i1 - g < 64 ? i1 - g : 64);
      for (int j = 0; j < k; ++j) rmat_draw(log2_n, a, b, c, seed, g + (uint64_t)j, &us[j], &vs[j]);
      for (int j = 0; j < k; ++j)
        if (us[j] != vs[j]) {
          ++mine[us[j]];
          ++mine[vs[j]];
        }
    }
  }
#pragma omp parallel for schedule(static)
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t d = 0;
    for (int t = 0; t < T; ++t) d += cnt[(size_t)t * n + v];
    deg[v] = d;
  }
  uint64_t total = 0;
  for (uint64_t v = 0; v < n; ++v) {
    off[v] = total;
    total += deg[v];
  }
  off[n] = total;
  /* cursors: thread t writes source v's arcs from off[v] + sum of the
   * earlier threads' counts */
#pragma omp parallel for schedule(static)
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t run = off[v];
    for (int t = 0; t < T; ++t) {
      uint32_t k = cnt[(size_t)t * n + v];
      cnt[(size_t)t * n + v] = (uint32_t)run;
      run += k;
    }
  }
  uint32_t* tmp = (uint32_t*)malloc((total ? total : 1) * sizeof(uint32_t));
  if (!tmp || total > UINT32_MAX) {
    free(cnt);
    free(deg);
    free(tmp);
    return UINT64_MAX;
  }
  /* pass 2: the same draws scattered into per-source buckets */
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    uint32_t* cur = cnt + (size_t)t * n;
    const uint64_t i0 = draws * (uint64_t)t / (uint64_t)T, i1 = draws * (uint64_t)(t + 1) / (uint64_t)T;
    uint32_t us[64], vs[64];
    for (uint64_t g = i0; g < i1; g += 64) {
      const int k = (int)(i1 - g < 64 ? i1 - g : 64);
      for (int j = 0; j < k; ++j) rmat_draw(log2_n, a, b, c, seed, g + (uint64_t)j, &us[j], &vs[j]);
      for (int j = 0; j < k; ++j)
        if (us[j] != vs[j]) {
          tmp[cur[us[j]]++] = vs[j];
          tmp[cur[vs[j]]++] = us[j];
        }
    }
  }
  free(cnt);
  /* sort + unique each bucket in place; deg[v] = unique count */
#pragma omp parallel for schedule(dynamic, 4096)
  for (uint64_t v = 0; v < n; ++v) {
    uint32_t* s = tmp + off[v];
    uint64_t d = off[v + 1] - off[v];
    if (d > 1) sort_u32(s, (int64_t)d);
    uint64_t w = 0;
    for (uint64_t k = 0; k < d; ++k)
      if (w == 0 || s[k] != s[w - 1]) s[w++] = s[k];
    deg[v] = w;
  }
  /* compact: each bucket's unique prefix moves down to its new offset (a
   * bucket only moves towards lower addresses, so a serial pass in order
   * never overwrites an unmoved bucket) */
  uint64_t m = 0, prev_old = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t o = prev_old;
    prev_old = off[v + 1];
    off[v] = m;
    if (deg[v] && m != o) memmove(tmp + m, tmp + o, deg[v] * sizeof(uint32_t));
    m += deg[v];
  }
  off[n] = m;
  free(deg);
  uint32_t* shrunk = (uint32_t*)realloc(tmp, (m ? m : 1) * sizeof(uint32_t));
  *nbr_out = shrunk ? shrunk : tmp;
  return m;
}

void gbo_free(void* p) { free(p); }

/* io.cpp:75-85 (save_binary): "GBCSR1\0\0", u64 n, u64 m, u64 offsets[n+1],
 * u32 neighbours[m], little-endian.  Returns 0, or 5 on an I/O error. */
int gbo_save_gbcsr1(const char* path, uint64_t n, const uint64_t* off, const uint32_t* nbr) {
  FILE* f = fopen(path, "wb");
  if (!f) return 5;
  static const char magic[8] = {'G', 'B', 'C', 'S', 'R', '1', 0, 0};
  uint64_t m = off[n];
  int ok = fwrite(magic, 1, 8, f) == 8 && fwrite(&n, 8, 1, f) == 1 && fwrite(&m, 8, 1, f) == 1 &&
           fwrite(off, 8, n + 1, f) == n + 1 && (m == 0 || fwrite(nbr, 4, m, f) == m);
  ok = (fclose(f) == 0) && ok;
  return ok ? 0 : 5;
}

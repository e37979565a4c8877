/* TEST INFRASTRUCTURE ONLY — see gbo.h.  Plain-C restatement of the
 * reference hot path; serial, deliberately simple.  Citations are relative
 * to /root/reference/proj. */
#include "gbo.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* rng.hpp:11-16 (splitmix64 finalizer) */
uint64_t gbo_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:18-20 */
uint64_t gbo_hash_combine(uint64_t a, uint64_t b) {
  return gbo_mix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

/* rng.hpp:22-24 */
uint64_t gbo_rng_u64(uint64_t seed, uint64_t stream, uint64_t counter) {
  return gbo_mix64(gbo_hash_combine(gbo_hash_combine(seed, stream), counter));
}

/* rng.hpp:27-29: top 53 bits of rng_u64 times 2^-53 */
double gbo_rng_double(uint64_t seed, uint64_t stream, uint64_t counter) {
  return (double)(gbo_rng_u64(seed, stream, counter) >> 11) * 0x1.0p-53;
}

/* batch.cpp:128-154: `size` recursive-quadrant draws, each emitted as (u,v)
 * followed by (v,u).  Thresholds a, a+b, a+b+c are evaluated left to right
 * exactly as the reference writes them. */
void gbo_update_batch(uint64_t log2_n, double a, double b, double c, uint64_t size,
                      uint64_t seed, uint32_t* out) {
  for (uint64_t i = 0; i < size; ++i) {
    uint32_t u = 0, v = 0;
    for (uint64_t level = 0; level < log2_n; ++level) {
      double r = gbo_rng_double(seed, i, level);
      u <<= 1;
      v <<= 1;
      if (r < a) {
      } else if (r < a + b) {
        v |= 1;
      } else if (r < a + b + c) {
        u |= 1;
      } else {
        u |= 1;
        v |= 1;
      }
    }
    out[4 * i + 0] = u;
    out[4 * i + 1] = v;
    out[4 * i + 2] = v;
    out[4 * i + 3] = u;
  }
}

/* LSD radix sort of u64 keys, 16-bit digits (replaces std::sort on Edge,
 * whose lexicographic order (types.hpp:21-25) equals the order of
 * src<<32|dst keys). */
void gbo_sort_u64(uint64_t* keys, uint64_t count) {
  if (count < 2) return;
  uint64_t* tmp = (uint64_t*)malloc(count * sizeof(uint64_t));
  uint64_t* cnt = (uint64_t*)malloc(65536 * sizeof(uint64_t));
  uint64_t* src = keys;
  uint64_t* dst = tmp;
  for (int shift = 0; shift < 64; shift += 16) {
    memset(cnt, 0, 65536 * sizeof(uint64_t));
    for (uint64_t i = 0; i < count; ++i) cnt[(src[i] >> shift) & 0xffff]++;
    if (cnt[(src[0] >> shift) & 0xffff] == count) continue; /* digit constant */
    uint64_t sum = 0;
    for (int d = 0; d < 65536; ++d) {
      uint64_t c = cnt[d];
      cnt[d] = sum;
      sum += c;
    }
    for (uint64_t i = 0; i < count; ++i) dst[cnt[(src[i] >> shift) & 0xffff]++] = src[i];
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != keys) memcpy(keys, src, count * sizeof(uint64_t));
  free(tmp);
  free(cnt);
}

static uint64_t unique_u64(uint64_t* k, uint64_t count) {
  if (count == 0) return 0;
  uint64_t w = 1;
  for (uint64_t i = 1; i < count; ++i)
    if (k[i] != k[w - 1]) k[w++] = k[i];
  return w;
}

/* generators.cpp:9-29: drop self loops, add reverses, sort, unique;
 * n = max(min_n, 1 + max id seen, loops included). */
uint64_t gbo_normalize(const uint32_t* raw, uint64_t count, uint64_t min_n, uint32_t* out,
                       uint64_t* n_out) {
  uint64_t* k = (uint64_t*)malloc((2 * count + 1) * sizeof(uint64_t));
  uint64_t w = 0, max_id = 0;
  int any = 0;
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t s = raw[2 * i], d = raw[2 * i + 1];
    uint64_t hi = s > d ? s : d;
    if (hi > max_id) max_id = hi;
    any = 1;
    if (s == d) continue;
    k[w++] = ((uint64_t)s << 32) | d;
    k[w++] = ((uint64_t)d << 32) | s;
  }
  gbo_sort_u64(k, w);
  w = unique_u64(k, w);
  for (uint64_t i = 0; i < w; ++i) {
    out[2 * i] = (uint32_t)(k[i] >> 32);
    out[2 * i + 1] = (uint32_t)k[i];
  }
  free(k);
  uint64_t n = any ? max_id + 1 : 0;
  *n_out = n > min_n ? n : min_n;
  return w;
}

/* batch.cpp:34-42: GlobalSort prepare = drop self loops, sort (src,dst),
 * unique. */
uint64_t gbo_prepare_global(const uint32_t* pairs, uint64_t count, uint32_t* out) {
  uint64_t* k = (uint64_t*)malloc((count + 1) * sizeof(uint64_t));
  uint64_t w = 0;
  for (uint64_t i = 0; i < count; ++i)
    if (pairs[2 * i] != pairs[2 * i + 1])
      k[w++] = ((uint64_t)pairs[2 * i] << 32) | pairs[2 * i + 1];
  gbo_sort_u64(k, w);
  w = unique_u64(k, w);
  for (uint64_t i = 0; i < w; ++i) {
    out[2 * i] = (uint32_t)(k[i] >> 32);
    out[2 * i + 1] = (uint32_t)k[i];
  }
  free(k);
  return w;
}

/* csr.cpp:9-25: validated build (ids < n, strictly increasing arcs). */
int gbo_csr_build(uint64_t n, const uint32_t* p, uint64_t m, uint64_t* off, uint32_t* nbr) {
  memset(off, 0, (n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    uint32_t s = p[2 * i], d = p[2 * i + 1];
    if (s >= n || d >= n) return 5;
    if (i > 0) {
      uint64_t prev = ((uint64_t)p[2 * i - 2] << 32) | p[2 * i - 1];
      uint64_t cur = ((uint64_t)s << 32) | d;
      if (!(prev < cur)) return 5;
    }
    off[s + 1]++;
    nbr[i] = d;
  }
  for (uint64_t i = 0; i < n; ++i) off[i + 1] += off[i];
  return 0;
}

/* ---- traversal restatement --------------------------------------------- */

static int test_bit(const uint64_t* w, uint64_t v) { return (int)((w[v >> 6] >> (v & 63)) & 1); }
static void set_bit(uint64_t* w, uint64_t v) { w[v >> 6] |= (uint64_t)1 << (v & 63); }

/* vertex_subset.cpp:32-37 */
void gbo_subset_to_dense(uint64_t n, const uint32_t* ids, uint64_t k, uint64_t* words) {
  memset(words, 0, ((n + 63) / 64) * sizeof(uint64_t));
  for (uint64_t i = 0; i < k; ++i) set_bit(words, ids[i]);
}

/* vertex_subset.cpp:39-45 + for_each (vertex_subset.hpp:55-67): ascending. */
uint64_t gbo_subset_to_sparse(uint64_t n, const uint64_t* words, uint32_t* ids) {
  uint64_t k = 0;
  for (uint64_t w = 0; w < (n + 63) / 64; ++w) {
    uint64_t bits = words[w];
    while (bits) {
      ids[k++] = (uint32_t)(w * 64 + (uint64_t)__builtin_ctzll(bits));
      bits &= bits - 1;
    }
  }
  return k;
}

/* traversal.cpp:16-95 with cond = byte mask and update = always true.
 * mode 0 sparse push (claim-then-update, traversal.cpp:16-46), mode 1 dense
 * pull (traversal.cpp:48-95). ids need not be sorted; duplicates ignored. */
int gbo_edge_map(uint64_t n, const uint64_t* off, const uint32_t* nbr, const uint32_t* ids,
                 uint64_t nids, const uint8_t* cond, int mode, int early_exit, uint8_t* out,
                 uint64_t* updates) {
  uint64_t nw = (n + 63) / 64;
  uint64_t* fb = (uint64_t*)calloc(nw + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < nids; ++i) {
    if (ids[i] >= n) {
      free(fb);
      return 1;
    }
    set_bit(fb, ids[i]);
  }
  memset(out, 0, n);
  uint64_t upd = 0;
  if (mode == 0) {
    uint64_t* claimed = (uint64_t*)calloc(nw + 1, sizeof(uint64_t));
    for (uint64_t u = 0; u < n; ++u) {
      if (!test_bit(fb, u)) continue;
      for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
        uint32_t v = nbr[k];
        if (!cond[v] || test_bit(claimed, v)) continue;
        set_bit(claimed, v);
        upd++;
        out[v] = 1;
      }
    }
    free(claimed);
  } else {
    for (uint64_t v = 0; v < n; ++v) {
      if (!cond[v]) continue;
      for (uint64_t k = off[v]; k < off[v + 1]; ++k) {
        if (test_bit(fb, nbr[k])) {
          upd++;
          out[v] = 1;
          if (early_exit) break;
        }
      }
    }
  }
  free(fb);
  *updates = upd;
  return 0;
}

/* algorithms.cpp:29-58 (bfs) over edge_map (traversal.cpp:101-111):
 * dense iff |F| + sum deg(F) > m/20.  Records per-level mode and input
 * frontier size; depth -1 = unreached (the BASELINE int32 narrowing). */
int gbo_bfs(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t src, int32_t* depth,
            int32_t* modes, uint64_t* sizes, uint64_t cap, uint64_t* levels) {
  if (src >= n) return 1;
  uint64_t m = off[n];
  uint64_t nw = (n + 63) / 64;
  uint32_t* cur = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  uint32_t* nxt = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  uint64_t* fb = (uint64_t*)calloc(nw + 1, sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) depth[v] = -1;
  depth[src] = 0;
  uint64_t fsize = 1, lvl = 0;
  cur[0] = src;
  int32_t d = 0;
  while (fsize > 0) {
    ++d;
    uint64_t degsum = 0;
    for (uint64_t i = 0; i < fsize; ++i) degsum += off[cur[i] + 1] - off[cur[i]];
    int dense = (double)(fsize + degsum) > (1.0 / 20.0) * (double)m;
    if (lvl < cap) {
      modes[lvl] = dense;
      sizes[lvl] = fsize;
    }
    uint64_t k = 0;
    if (!dense) {
      /* the reference sorts each sparse subset (vertex_subset.cpp:10-11);
       * cur[] is kept ascending below, so push visits in the same order */
      for (uint64_t i = 0; i < fsize; ++i) {
        uint32_t u = cur[i];
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
          uint32_t v = nbr[e];
          if (depth[v] != -1) continue;
          depth[v] = d;
          nxt[k++] = v;
        }
      }
      /* ascending order, like the VertexSubset constructor */
      uint64_t* tmp = (uint64_t*)malloc((k + 1) * sizeof(uint64_t));
      for (uint64_t i = 0; i < k; ++i) tmp[i] = nxt[i];
      gbo_sort_u64(tmp, k);
      for (uint64_t i = 0; i < k; ++i) nxt[i] = (uint32_t)tmp[i];
      free(tmp);
    } else {
      memset(fb, 0, nw * sizeof(uint64_t));
      for (uint64_t i = 0; i < fsize; ++i) set_bit(fb, cur[i]);
      for (uint64_t v = 0; v < n; ++v) {
        if (depth[v] != -1) continue;
        for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
          if (test_bit(fb, nbr[e])) {
            nxt[k++] = (uint32_t)v; /* ascending by construction */
            break;
          }
        }
      }
      for (uint64_t i = 0; i < k; ++i) depth[nxt[i]] = d;
    }
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
    fsize = k;
    ++lvl;
  }
  *levels = lvl;
  free(cur);
  free(nxt);
  free(fb);
  return 0;
}

/* algorithms.cpp:508-555: power iteration, uniform dangling redistribution,
 * dense pull summing in sorted-neighbour order, L1 stop rule. */
int gbo_pagerank(uint64_t n, const uint64_t* off, const uint32_t* nbr, double damping,
                 uint64_t iters, double tol, double* out) {
  if (!(damping > 0.0 && damping < 1.0)) return 2;
  if (!(tol > 0.0)) return 2;
  if (n == 0) return 0;
  double* p = out;
  double* contrib = (double*)malloc(n * sizeof(double));
  double* next = (double*)malloc(n * sizeof(double));
  for (uint64_t v = 0; v < n; ++v) p[v] = 1.0 / (double)n;
  for (uint64_t it = 0; it < iters; ++it) {
    double dangling = 0.0;
    for (uint64_t v = 0; v < n; ++v) {
      uint64_t dg = off[v + 1] - off[v];
      contrib[v] = dg ? p[v] / (double)dg : 0.0;
      if (dg == 0) dangling += p[v];
    }
    for (uint64_t v = 0; v < n; ++v) {
      double s = 0.0;
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) s += contrib[nbr[e]];
      next[v] = s;
    }
    double base = (1.0 - damping) / (double)n + damping * dangling / (double)n;
    double err = 0.0;
    for (uint64_t v = 0; v < n; ++v) {
      next[v] = base + damping * next[v];
      err += fabs(next[v] - p[v]);
    }
    memcpy(p, next, n * sizeof(double));
    if (err < tol) break;
  }
  free(contrib);
  free(next);
  return 0;
}

/* algorithms.cpp:60-103: single-source Brandes dependencies.  Path counts
 * pulled level by level from the previous layer, dependencies pulled from
 * the next layer in reverse level order, each sum in sorted-neighbour order.
 * Unreached vertices get 0. */
int gbo_bc(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t src, double* delta) {
  if (src >= n) return 1;
  int32_t* dist = (int32_t*)malloc((n + 1) * sizeof(int32_t));
  uint64_t levels = 0;
  int32_t mode[1];
  uint64_t size[1];
  gbo_bfs(n, off, nbr, src, dist, mode, size, 0, &levels);
  int32_t maxd = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (dist[v] > maxd) maxd = dist[v];
  double* sigma = (double*)calloc(n + 1, sizeof(double));
  sigma[src] = 1.0;
  for (int32_t d = 1; d <= maxd; ++d)
    for (uint64_t v = 0; v < n; ++v) {
      if (dist[v] != d) continue;
      double t = 0.0;
      for (uint64_t e = off[v]; e < off[v + 1]; ++e)
        if (dist[nbr[e]] == d - 1) t += sigma[nbr[e]];
      sigma[v] = t;
    }
  for (uint64_t v = 0; v < n; ++v) delta[v] = 0.0;
  for (int32_t d = maxd - 1; d >= 0; --d)
    for (uint64_t v = 0; v < n; ++v) {
      if (dist[v] != d) continue;
      double t = 0.0;
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        uint32_t w = nbr[e];
        if (dist[w] == d + 1) t += (sigma[v] / sigma[w]) * (1.0 + delta[w]);
      }
      delta[v] = t;
    }
  free(dist);
  free(sigma);
  return 0;
}

/* algorithms.cpp:194-234 semantics: components labelled by their minimum
 * vertex id (union by smaller root, full compression at the end). */
void gbo_cc(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* lab) {
  for (uint64_t v = 0; v < n; ++v) lab[v] = (uint32_t)v;
  for (uint64_t u = 0; u < n; ++u) {
    for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t a = (uint32_t)u, b = nbr[e];
      while (lab[a] != a) a = lab[a] = lab[lab[a]];
      while (lab[b] != b) b = lab[b] = lab[lab[b]];
      if (a == b) continue;
      if (a < b) lab[b] = a; else lab[a] = b;
    }
  }
  for (uint64_t v = 0; v < n; ++v) {
    uint32_t r = (uint32_t)v;
    while (lab[r] != r) r = lab[r];
    lab[v] = r;
  }
}

/* Triangle counting — NOT in the reference; restated from
 * PAPER.md:945-969 on the reference's primitives: derive_filter
 * (derive.hpp:48-61) keeps arc (u,v) iff (deg u, u) < (deg v, v), giving a
 * sorted oriented CSR; then |N+(u) ∩ N+(v)| per oriented arc by merge
 * intersection of neighbor_segment()s (csr.hpp:40-42), summed in uint64. */
uint64_t gbo_tc(uint64_t n, const uint64_t* off, const uint32_t* nbr) {
  uint64_t* o2 = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  uint64_t m = off[n];
  uint32_t* a2 = (uint32_t*)malloc((m + 1) * sizeof(uint32_t));
  uint64_t w = 0;
  for (uint64_t u = 0; u < n; ++u) {
    uint64_t du = off[u + 1] - off[u];
    o2[u] = w;
    for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t v = nbr[e];
      uint64_t dv = off[v + 1] - off[v];
      if (du < dv || (du == dv && u < v)) a2[w++] = v;
    }
  }
  o2[n] = w;
  uint64_t total = 0;
  for (uint64_t u = 0; u < n; ++u) {
    for (uint64_t e = o2[u]; e < o2[u + 1]; ++e) {
      uint32_t v = a2[e];
      uint64_t i = o2[u], j = o2[v];
      while (i < o2[u + 1] && j < o2[v + 1]) {
        if (a2[i] < a2[j]) ++i;
        else if (a2[i] > a2[j]) ++j;
        else { ++total; ++i; ++j; }
      }
    }
  }
  free(o2);
  free(a2);
  return total;
}

/* SetGraph<ChunkedSortedSet>::apply_batch (set_graph.hpp:197-238) over
 * ChunkedSortedSet::insert_batch / delete_batch (neighbor_sets.hpp:339-366):
 * per source, merge+unique (insert) or set difference (delete) of the sorted
 * neighbour list with the batch's sorted destinations.  `batch` must be a
 * GlobalSort-prepared arc list.  Returns the applied arc count. */
uint64_t gbo_set_apply(uint64_t n, const uint64_t* off, const uint32_t* nbr, const uint32_t* batch,
                       uint64_t bcount, int insert, uint64_t* off_out, uint32_t* nbr_out) {
  uint64_t applied = 0, w = 0, b = 0;
  off_out[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t i = off[v], ie = off[v + 1];
    uint64_t bs = b;
    while (b < bcount && batch[2 * b] == v) ++b;
    uint64_t j = bs, je = b;
    while (i < ie || j < je) {
      if (j >= je || (i < ie && nbr[i] < batch[2 * j + 1])) {
        nbr_out[w++] = nbr[i++];
      } else if (i >= ie || batch[2 * j + 1] < nbr[i]) {
        if (insert) {
          nbr_out[w++] = batch[2 * j + 1];
          ++applied;
        }
        ++j;
      } else { /* equal */
        if (insert) nbr_out[w++] = nbr[i];
        else ++applied;
        ++i;
        ++j;
      }
    }
    off_out[v + 1] = w;
  }
  return applied;
}

/* algorithms.cpp:330-374 + buckets.cpp:7-59: peel the lowest bucket k;
 * each peeled vertex decrements the remaining degree of the neighbours still
 * in a bucket above k, which move to bucket max(k, remaining).  Restated as
 * the serial bin-sort peel (vertices in nondecreasing remaining degree; a
 * neighbour only drops while above the current level), which visits the
 * same bucket sequence one vertex at a time. */
void gbo_kcore(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint64_t* core) {
  if (!n) return;
  uint64_t md = 0;
  uint64_t* rem = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) {
    rem[v] = off[v + 1] - off[v];
    if (rem[v] > md) md = rem[v];
  }
  uint64_t* bin = (uint64_t*)calloc(md + 2, sizeof(uint64_t));
  uint64_t* pos = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint32_t* vert = (uint32_t*)malloc(n * sizeof(uint32_t));
  for (uint64_t v = 0; v < n; ++v) ++bin[rem[v]];
  uint64_t start = 0;
  for (uint64_t d = 0; d <= md; ++d) {
    uint64_t c = bin[d];
    bin[d] = start;
    start += c;
  }
  for (uint64_t v = 0; v < n; ++v) {
    pos[v] = bin[rem[v]]++;
    vert[pos[v]] = (uint32_t)v;
  }
  for (uint64_t d = md; d > 0; --d) bin[d] = bin[d - 1];
  bin[0] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t v = vert[i];
    core[v] = rem[v];
    for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
      uint32_t u = nbr[e];
      if (rem[u] > rem[v]) {
        uint64_t du = rem[u], pu = pos[u], pw = bin[du];
        uint32_t w = vert[pw];
        if (u != w) {
          pos[u] = pw;
          vert[pw] = u;
          pos[w] = pu;
          vert[pu] = w;
        }
        ++bin[du];
        --rem[u];
      }
    }
  }
  free(rem);
  free(bin);
  free(pos);
  free(vert);
}

static unsigned gbo_bit_width(uint64_t x) {
  unsigned b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

/* algorithms.cpp:376-432: waiting[v] = neighbours beating v (higher
 * bit_width(degree), ties to the lower id); ready vertices take the smallest
 * colour unused by the neighbours beating them, then release the others.
 * Rounds run serially, in frontier order. */
void gbo_coloring(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* colors) {
  if (!n) return;
  unsigned* llf = (unsigned*)malloc(n * sizeof(unsigned));
  int64_t* waiting = (int64_t*)calloc(n, sizeof(int64_t));
  uint32_t* cur = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* nxt = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint64_t md = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t d = off[v + 1] - off[v];
    llf[v] = gbo_bit_width(d);
    if (d > md) md = d;
    colors[v] = UINT32_MAX;
  }
#define GBO_BEATS(a, b) (llf[a] != llf[b] ? llf[a] > llf[b] : (a) < (b))
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t e = off[v]; e < off[v + 1]; ++e)
      if (GBO_BEATS(nbr[e], (uint32_t)v)) ++waiting[v];
  uint64_t nc = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (waiting[v] == 0) cur[nc++] = (uint32_t)v;
  unsigned char* used = (unsigned char*)malloc(md + 2);
  while (nc) {
    uint64_t nn = 0;
    for (uint64_t i = 0; i < nc; ++i) {
      uint32_t v = cur[i];
      uint64_t d = off[v + 1] - off[v];
      memset(used, 0, d + 1);
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        uint32_t u = nbr[e];
        if (GBO_BEATS(u, v) && colors[u] <= d) used[colors[u]] = 1;
      }
      uint32_t c = 0;
      while (used[c]) ++c;
      colors[v] = c;
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        uint32_t u = nbr[e];
        if (GBO_BEATS(u, v)) continue;
        if (--waiting[u] == 0) nxt[nn++] = u;
      }
    }
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
    nc = nn;
  }
#undef GBO_BEATS
  free(llf);
  free(waiting);
  free(cur);
  free(nxt);
  free(used);
}

/* algorithms.cpp:434-504: rank[v] = rng_u64(seed, 7, v), lower (rank, id)
 * wins; joiners enter and knock their undecided neighbours out, then every
 * vertex decided this round releases its undecided lower-priority
 * neighbours; released vertices still undecided join next round. */
void gbo_mis(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint64_t seed, uint8_t* in_set) {
  if (!n) return;
  uint64_t* rank = (uint64_t*)malloc(n * sizeof(uint64_t));
  int64_t* waiting = (int64_t*)calloc(n, sizeof(int64_t));
  uint8_t* status = (uint8_t*)calloc(n, 1); /* 0 undecided, 1 in, 2 out */
  uint32_t* join = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* decided = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* rel = (uint32_t*)malloc(n * sizeof(uint32_t));
  for (uint64_t v = 0; v < n; ++v) rank[v] = gbo_rng_u64(seed, 7, v);
#define GBO_BEATS(a, b) (rank[a] != rank[b] ? rank[a] < rank[b] : (a) < (b))
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t e = off[v]; e < off[v + 1]; ++e)
      if (GBO_BEATS(nbr[e], (uint32_t)v)) ++waiting[v];
  uint64_t nj = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (waiting[v] == 0) join[nj++] = (uint32_t)v;
  while (nj) {
    uint64_t nd = 0;
    for (uint64_t i = 0; i < nj; ++i) {
      uint32_t v = join[i];
      status[v] = 1;
      decided[nd++] = v;
    }
    for (uint64_t i = 0; i < nj; ++i) {
      uint32_t v = join[i];
      for (uint64_t e = off[v]; e < off[v + 1]; ++e)
        if (status[nbr[e]] == 0) {
          status[nbr[e]] = 2;
          decided[nd++] = nbr[e];
        }
    }
    uint64_t nr = 0;
    for (uint64_t i = 0; i < nd; ++i) {
      uint32_t v = decided[i];
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        uint32_t u = nbr[e];
        if (GBO_BEATS(v, u) && status[u] == 0 && --waiting[u] == 0) rel[nr++] = u;
      }
    }
    nj = 0;
    for (uint64_t i = 0; i < nr; ++i)
      if (status[rel[i]] == 0) join[nj++] = rel[i];
  }
#undef GBO_BEATS
  for (uint64_t v = 0; v < n; ++v) in_set[v] = status[v] == 1;
  free(rank);
  free(waiting);
  free(status);
  free(join);
  free(decided);
  free(rel);
}

/* algorithms.cpp:114-188: shifts Exponential(beta) from rng_exponential
 * (rng.hpp:31-35, the C library's log1p), start = floor(max_shift - shift);
 * synchronous rounds: arrivals (min centre over the previous round's
 * joiners), self-starts, labelling, then each joiner's parent = smallest
 * same-cluster neighbour from an earlier round (itself at centres).
 * Returns 1 (invalid argument) unless 0 < beta <= 1. */
int gbo_ldd(uint64_t n, const uint64_t* off, const uint32_t* nbr, double beta, uint64_t seed, uint32_t* label,
            uint32_t* parent, uint64_t* rounds) {
  if (!(beta > 0.0 && beta <= 1.0)) return 1;
  if (!n) return 0;
  const uint32_t none = UINT32_MAX;
  double* shift = (double*)malloc(n * sizeof(double));
  uint64_t* start = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint32_t* cand = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* front = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* next = (uint32_t*)malloc(n * sizeof(uint32_t));
  double max_shift = 0.0;
  for (uint64_t v = 0; v < n; ++v) {
    shift[v] = -log1p(-gbo_rng_double(seed, v, 0)) / beta;
    if (shift[v] > max_shift) max_shift = shift[v];
  }
  for (uint64_t v = 0; v < n; ++v) {
    start[v] = (uint64_t)floor(max_shift - shift[v]);
    label[v] = cand[v] = parent[v] = none;
    rounds[v] = 0;
  }
  uint64_t labeled = 0, nf = 0, round = 0;
  while (labeled < n) {
    for (uint64_t i = 0; i < nf; ++i) {
      uint32_t u = front[i], c = label[u];
      for (uint64_t e = off[u]; e < off[u + 1]; ++e)
        if (label[nbr[e]] == none && c < cand[nbr[e]]) cand[nbr[e]] = c;
    }
    for (uint64_t v = 0; v < n; ++v)
      if (label[v] == none && start[v] <= round && (uint32_t)v < cand[v]) cand[v] = (uint32_t)v;
    uint64_t nn = 0;
    for (uint64_t v = 0; v < n; ++v) {
      if (label[v] != none || cand[v] == none) continue;
      label[v] = cand[v];
      rounds[v] = round;
      next[nn++] = (uint32_t)v;
    }
    for (uint64_t i = 0; i < nn; ++i) {
      uint32_t v = next[i], c = label[v], best = none;
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        uint32_t u = nbr[e];
        if (label[u] == c && rounds[u] < rounds[v] && u < best) best = u;
      }
      parent[v] = (v == c && best == none) ? v : best;
    }
    labeled += nn;
    uint32_t* t = front;
    front = next;
    next = t;
    nf = nn;
    ++round;
  }
  free(shift);
  free(start);
  free(cand);
  free(front);
  free(next);
  return 0;
}

/* bytecode.hpp:11-27 + compressed_csr.cpp:5-17: per vertex, zig-zag of the
 * first neighbour minus the vertex id, then gaps, as base-128 varints (low 7
 * bits first, high bit = more); byte_offsets[n+1].  bytes may be NULL to
 * size the encoding.  Returns the byte count. */
uint64_t gbo_bytecode_encode(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint64_t* byte_offsets,
                             uint8_t* bytes) {
  uint64_t pos = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (byte_offsets) byte_offsets[v] = pos;
    for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
      uint64_t x;
      if (e == off[v]) {
        int64_t d = (int64_t)nbr[e] - (int64_t)v;
        x = d >= 0 ? 2 * (uint64_t)d : 2 * (uint64_t)(-(d + 1)) + 1;
      } else {
        x = (uint64_t)(nbr[e] - nbr[e - 1]);
      }
      do {
        uint8_t b = (uint8_t)(x & 0x7f);
        x >>= 7;
        if (x) b |= 0x80;
        if (bytes) bytes[pos] = b;
        ++pos;
      } while (x);
    }
  }
  if (byte_offsets) byte_offsets[n] = pos;
  return pos;
}

/* Arcs the reference's traversal inspects per BFS level (SURVEY §8(d) E_scan):
 * a sparse level (edge_map_sparse, traversal.cpp:16-46) maps every
 * frontier member's whole list, sum deg(F); a dense early-exit level
 * (edge_map_dense, traversal.cpp:48-95) scans each unvisited vertex's list
 * in order up to and including its first frontier member.  Same switch rule
 * and level structure as gbo_bfs.  Returns the number of levels. */
uint64_t gbo_bfs_examined(uint64_t n, const uint64_t* off, const uint32_t* nbr, uint32_t src, uint64_t* examined,
                          uint64_t cap) {
  if (src >= n) return 0;
  uint64_t m = off[n];
  uint64_t nw = (n + 63) / 64;
  int32_t* depth = (int32_t*)malloc(n * sizeof(int32_t));
  uint32_t* cur = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  uint32_t* nxt = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  uint64_t* fb = (uint64_t*)calloc(nw + 1, sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) depth[v] = -1;
  depth[src] = 0;
  uint64_t fsize = 1, lvl = 0;
  cur[0] = src;
  int32_t d = 0;
  while (fsize > 0) {
    ++d;
    uint64_t degsum = 0, ex = 0;
    for (uint64_t i = 0; i < fsize; ++i) degsum += off[cur[i] + 1] - off[cur[i]];
    int dense = (double)(fsize + degsum) > (1.0 / 20.0) * (double)m;
    uint64_t k = 0;
    if (!dense) {
      ex = degsum;
      for (uint64_t i = 0; i < fsize; ++i) {
        uint32_t u = cur[i];
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
          uint32_t v = nbr[e];
          if (depth[v] != -1) continue;
          depth[v] = d;
          nxt[k++] = v;
        }
      }
    } else {
      memset(fb, 0, nw * sizeof(uint64_t));
      for (uint64_t i = 0; i < fsize; ++i) set_bit(fb, cur[i]);
      for (uint64_t v = 0; v < n; ++v) {
        if (depth[v] != -1) continue;
        for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
          ++ex;
          if (test_bit(fb, nbr[e])) {
            nxt[k++] = (uint32_t)v;
            break;
          }
        }
      }
      for (uint64_t i = 0; i < k; ++i) depth[nxt[i]] = d;
    }
    if (lvl < cap) examined[lvl] = ex;
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
    fsize = k;
    ++lvl;
  }
  free(depth);
  free(cur);
  free(nxt);
  free(fb);
  return lvl;
}

/* TEST INFRASTRUCTURE ONLY — the CPU restatement (oracle) of the bit-exact
 * parts of the mini-batch GCN step. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library; the product (libggb.so)
 * never does.
 *
 * Pinned against the reference itself (oracle/_ref, tests/test_oracle.py)
 * and against the known answers of the reference's own tests.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9e3779b97f4a7c15ULL

/* include/gridgnn/rng.hpp:10-15 */
uint64_t orc_splitmix64(uint64_t x) {
  x += GOLDEN;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:17-19 */
uint64_t orc_hash_combine(uint64_t a, uint64_t b) {
  return orc_splitmix64(a ^ (GOLDEN + (b << 6) + (b >> 2)));
}

/* rng.hpp:73-76 */
double orc_element_unit(uint64_t key, uint64_t i, uint64_t j) {
  uint64_t h = orc_splitmix64(orc_hash_combine(orc_hash_combine(key, i), j));
  return (double)(h >> 11) * 0x1.0p-53;
}

/* rng.hpp:22-69: counter stream */
typedef struct {
  uint64_t state;
  double spare;
  int have_spare;
} orc_stream;

static uint64_t st_next_u64(orc_stream* s) {
  s->state += GOLDEN;
  uint64_t x = s->state;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static double st_next_unit(orc_stream* s) { return (double)(st_next_u64(s) >> 11) * 0x1.0p-53; }
static uint64_t st_next_below(orc_stream* s, uint64_t bound) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t x;
  do {
    x = st_next_u64(s);
  } while (x >= limit);
  return x % bound;
}
/* next_below with the test-only extra rejection rule of
 * ggb_sample_vertices_test_reject (x % reject_mod == 0 also rejected) */
static uint64_t st_next_below_rej(orc_stream* s, uint64_t bound, uint64_t reject_mod) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t x;
  do {
    x = st_next_u64(s);
  } while (x >= limit || (reject_mod && x % reject_mod == 0));
  return x % bound;
}
static double st_next_normal(orc_stream* s) {
  if (s->have_spare) {
    s->have_spare = 0;
    return s->spare;
  }
  double u, v, q;
  do {
    u = 2.0 * st_next_unit(s) - 1.0;
    v = 2.0 * st_next_unit(s) - 1.0;
    q = u * u + v * v;
  } while (q >= 1.0 || q == 0.0);
  const double f = sqrt(-2.0 * log(q) / q);
  s->spare = v * f;
  s->have_spare = 1;
  return u * f;
}

/* include/gridgnn/comm.hpp:29-39 */
float orc_bf16_round(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) {
    uint32_t r = u & 0xffff0000u;
    if ((u & 0x007fffffu) != 0 && (r & 0x007f0000u) == 0) r |= 0x00400000u;
    float f;
    memcpy(&f, &r, 4);
    return f;
  }
  const uint32_t lsb = (u >> 16) & 1u;
  uint32_t r = (u + 0x7fffu + lsb) & 0xffff0000u;
  float f;
  memcpy(&f, &r, 4);
  return f;
}

/* include/gridgnn/model.hpp:164-171 */
uint64_t orc_dropout_key(uint64_t seed, int dp, uint64_t gstep, int layer) {
  return orc_hash_combine(
      orc_hash_combine(orc_hash_combine(orc_hash_combine(seed, 0xd509), (uint64_t)dp), gstep),
      (uint64_t)layer);
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* src/sampling.cpp:11-33. Returns 0, or 1 for invalid arguments. The
 * partial Fisher-Yates needs the full length-n permutation, as the
 * reference does. */
int orc_sample_vertices(int64_t n, int64_t b, uint64_t seed, uint64_t step, int64_t* out) {
  if (b <= 0 || b > n) return 1;
  orc_stream s = {orc_splitmix64(seed + step), 0.0, 0};
  int64_t* perm = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  if (!perm) return 2;
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = 0; i < b; ++i) {
    const int64_t j = i + (int64_t)st_next_below(&s, (uint64_t)(n - i));
    const int64_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  memcpy(out, perm, (size_t)b * sizeof(int64_t));
  free(perm);
  qsort(out, (size_t)b, sizeof(int64_t), cmp_i64);
  return 0;
}

/* src/shardsample.cpp:8-17 */
int orc_block_partition(int64_t n, int g, int64_t* out) {
  if (g < 1) return 1;
  const int64_t base = n / g, extra = n % g;
  out[0] = 0;
  for (int k = 0; k < g; ++k) out[k + 1] = out[k] + base + (k < extra ? 1 : 0);
  return 0;
}

static int64_t lower_bound_i64(const int64_t* v, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (v[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* src/shardsample.cpp:158-165 */
void orc_sample_partition(const int64_t* s, int64_t b, const int64_t* offsets, int64_t k,
                          int64_t* out) {
  for (int64_t i = 0; i < k; ++i) out[i] = lower_bound_i64(s, b, offsets[i]);
}

/* One rank's shard of the rescaled mini-batch adjacency (Alg. 2), restating
 * make_csr_shard (shardsample.cpp:19-45), locate_ranges (:47-56),
 * extract_rows (:58-87), filter_and_remap (:89-109), assemble_shard
 * (:111-122) with csr_from_triples/csr_transpose (src/csr.cpp:29-94) and
 * build_local_minibatch (:124-156).
 *
 * Entries of the sampled rows are visited in row order and, within a row, in
 * increasing column order (the global CSR is canonical), so the kept triples
 * are already the canonical CSR order csr_from_triples would produce; the
 * transpose is the stable counting sort of csr.cpp:74-94.
 *
 * Pass row_ptr==NULL to only query: meta = {row_lo,row_hi,col_lo,col_hi,
 * nnz_extracted, nnz_kept}. Otherwise a_* receive the local CSR (row_ptr
 * length rows+1) and t_* its transpose. */
int orc_local_minibatch(int64_t n, const int64_t* g_row_ptr, const int64_t* g_col,
                        const double* g_val, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                        int64_t b, uint64_t seed, uint64_t step, int64_t* meta,
                        int64_t* a_row_ptr, int64_t* a_col, double* a_val, int64_t* t_row_ptr,
                        int64_t* t_col, double* t_val) {
  if (b < 2 || b > n) return 1;
  if (r0 < 0 || r0 > r1 || r1 > n || c0 < 0 || c0 > c1 || c1 > n) return 1;
  int64_t* s = (int64_t*)malloc((size_t)b * sizeof(int64_t));
  orc_sample_vertices(n, b, seed, step, s);
  const int64_t row_lo = lower_bound_i64(s, b, r0), row_hi = lower_bound_i64(s, b, r1);
  const int64_t col_lo = lower_bound_i64(s, b, c0), col_hi = lower_bound_i64(s, b, c1);
  const double p = (double)(b - 1) / (double)(n - 1);
  const int64_t nr = row_hi - row_lo, nc = col_hi - col_lo;
  int64_t extracted = 0, kept = 0;
  if (a_row_ptr) {
    a_row_ptr[0] = 0;
    for (int64_t k = 0; k <= nc; ++k) t_row_ptr[k] = 0;
  }
  for (int64_t i = 0; i < nr; ++i) {
    const int64_t v = s[row_lo + i];
    for (int64_t e = g_row_ptr[v]; e < g_row_ptr[v + 1]; ++e) {
      const int64_t c = g_col[e];
      if (c < c0 || c >= c1) continue; /* outside the static shard's columns */
      ++extracted;
      const int64_t pos = lower_bound_i64(s + col_lo, nc, c);
      if (pos == nc || s[col_lo + pos] != c) continue;
      if (a_row_ptr) {
        a_col[kept] = pos;
        a_val[kept] = (v != c) ? g_val[e] / p : g_val[e];
        ++t_row_ptr[pos + 1];
      }
      ++kept;
    }
    if (a_row_ptr) a_row_ptr[i + 1] = kept;
  }
  if (a_row_ptr) {
    for (int64_t k = 0; k < nc; ++k) t_row_ptr[k + 1] += t_row_ptr[k];
    int64_t* cursor = (int64_t*)malloc((size_t)(nc + 1) * sizeof(int64_t));
    memcpy(cursor, t_row_ptr, (size_t)(nc + 1) * sizeof(int64_t));
    for (int64_t r = 0; r < nr; ++r)
      for (int64_t k = a_row_ptr[r]; k < a_row_ptr[r + 1]; ++k) {
        const int64_t slot = cursor[a_col[k]]++;
        t_col[slot] = r;
        t_val[slot] = a_val[k];
      }
    free(cursor);
  }
  meta[0] = row_lo;
  meta[1] = row_hi;
  meta[2] = col_lo;
  meta[3] = col_hi;
  meta[4] = extracted;
  meta[5] = kept;
  free(s);
  return 0;
}

/* ---- dataset (src/dataset.cpp) -------------------------------------------- */

/* dataset.cpp:133-150. Returns the edge count; uv (2*count) may be NULL. */
int64_t orc_synthetic_edges(int64_t n, double avg_degree, uint64_t seed, int64_t* uv) {
  orc_stream s = {orc_hash_combine(seed, 0xe0e0), 0.0, 0};
  const uint64_t target = (uint64_t)(avg_degree * (double)n / 2.0);
  int64_t m = 0;
  if (n > 1)
    for (uint64_t e = 0; e < target; ++e) {
      const int64_t u = (int64_t)st_next_below(&s, (uint64_t)n);
      const int64_t v = (int64_t)st_next_below(&s, (uint64_t)n);
      if (u != v) {
        if (uv) {
          uv[2 * m] = u;
          uv[2 * m + 1] = v;
        }
        ++m;
      }
    }
  return m;
}

static int cmp_pair(const void* a, const void* b) {
  const int64_t* x = (const int64_t*)a;
  const int64_t* y = (const int64_t*)b;
  if (x[0] != y[0]) return (x[0] > y[0]) - (x[0] < y[0]);
  return (x[1] > y[1]) - (x[1] < y[1]);
}

/* dataset.cpp:47-83: D^-1/2 (A+I) D^-1/2 over the symmetrized, deduplicated
 * edges. Query with row_ptr==NULL returns nnz. Returns -1 on bad input. */
int64_t orc_normalize_adjacency(const int64_t* uv, int64_t m, int64_t n, int64_t* row_ptr,
                                int64_t* col, double* val) {
  int64_t cap = 2 * m + n, k = 0;
  int64_t* und = (int64_t*)malloc((size_t)cap * 2 * sizeof(int64_t));
  for (int64_t e = 0; e < m; ++e) {
    const int64_t u = uv[2 * e], v = uv[2 * e + 1];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      free(und);
      return -1;
    }
    if (u == v) continue;
    und[2 * k] = u;
    und[2 * k + 1] = v;
    ++k;
    und[2 * k] = v;
    und[2 * k + 1] = u;
    ++k;
  }
  for (int64_t v = 0; v < n; ++v) {
    und[2 * k] = v;
    und[2 * k + 1] = v;
    ++k;
  }
  qsort(und, (size_t)k, 2 * sizeof(int64_t), cmp_pair);
  int64_t w = 0;
  for (int64_t i = 0; i < k; ++i)
    if (w == 0 || und[2 * i] != und[2 * (w - 1)] || und[2 * i + 1] != und[2 * (w - 1) + 1]) {
      und[2 * w] = und[2 * i];
      und[2 * w + 1] = und[2 * i + 1];
      ++w;
    }
  if (row_ptr) {
    int64_t* deg = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < w; ++i) ++deg[und[2 * i]];
    row_ptr[0] = 0;
    for (int64_t v = 0; v < n; ++v) row_ptr[v + 1] = row_ptr[v] + deg[v];
    for (int64_t i = 0; i < w; ++i) {
      const int64_t u = und[2 * i], v = und[2 * i + 1];
      col[i] = v;
      val[i] = 1.0 / sqrt((double)deg[u] * (double)deg[v]);
    }
    free(deg);
  }
  free(und);
  return w;
}

/* dataset.cpp:100-102: n*d_in N(0,1) draws (Marsaglia polar) cast to float */
void orc_features(int64_t n, int64_t d_in, uint64_t seed, float* out) {
  orc_stream s = {orc_hash_combine(seed, 0xfea7), 0.0, 0};
  for (int64_t k = 0; k < n * d_in; ++k) out[k] = (float)st_next_normal(&s);
}

/* dataset.cpp:104-120: degree-quantile classes, vertices ordered by
 * (degree without self-loop, id). */
void orc_labels(int64_t n, const int64_t* row_ptr, int64_t n_classes, int32_t* labels) {
  /* counting sort by degree, stable in id == std::stable_sort by (deg, id) */
  int64_t maxd = 0;
  for (int64_t v = 0; v < n; ++v) {
    const int64_t d = row_ptr[v + 1] - row_ptr[v] - 1;
    if (d > maxd) maxd = d;
  }
  int64_t* cnt = (int64_t*)calloc((size_t)maxd + 2, sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) ++cnt[row_ptr[v + 1] - row_ptr[v] - 1 + 1];
  for (int64_t d = 0; d <= maxd; ++d) cnt[d + 1] += cnt[d];
  for (int64_t v = 0; v < n; ++v) {
    const int64_t pos = cnt[row_ptr[v + 1] - row_ptr[v] - 1]++;
    labels[v] = (int32_t)((pos * n_classes) / n);
  }
  free(cnt);
}

/* dataset.cpp:122-129 */
void orc_split(int64_t n, uint64_t seed, uint8_t* split) {
  const uint64_t key = orc_hash_combine(seed, 0x5b11);
  for (int64_t v = 0; v < n; ++v) {
    const double u = orc_element_unit(key, (uint64_t)v, 0);
    split[v] = u < 0.6 ? 0 : (u < 0.8 ? 1 : 2);
  }
}

/* model.hpp:139-149: global weight matrix rows x cols drawn from element_unit */
void orc_fill_weight(int64_t rows, int64_t cols, uint64_t key, float* out) {
  const double lim = sqrt(6.0 / (double)(rows + cols));
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j)
      out[i * cols + j] =
          (float)((2.0 * orc_element_unit(key, (uint64_t)i, (uint64_t)j) - 1.0) * lim);
}

/* Dropout keep-mask of a rows x cols block at global offset (r0, c0):
 * out[i*cols+j] = element_unit(key, r0+i, c0+j) >= rate (pmm.hpp:317-322). */
void orc_dropout_keep(uint64_t key, int64_t r0, int64_t c0, int64_t rows, int64_t cols,
                      double rate, uint8_t* out) {
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j)
      out[i * cols + j] =
          orc_element_unit(key, (uint64_t)(r0 + i), (uint64_t)(c0 + j)) >= rate ? 1 : 0;
}

/* R-MAT edge list of gendata.cu k_rmat (new code, not in the reference: the
 * BASELINE configs[0] input). Edge e descends `scale` levels; level k draws
 * u = unit(splitmix64(hash_combine(hash_combine(key, e), k))) with
 * key = hash_combine(seed, 0x7a3a7) and takes quadrant a | b | c | d. */
void orc_rmat_edges(int scale, int64_t m, double a, double b, double c, uint64_t seed, int64_t* uv) {
  const uint64_t key = orc_hash_combine(seed, 0x7a3a7);
  for (int64_t e = 0; e < m; ++e) {
    const uint64_t ke = orc_hash_combine(key, (uint64_t)e);
    int64_t u = 0, v = 0;
    for (int k = 0; k < scale; ++k) {
      const double x = (double)(orc_splitmix64(orc_hash_combine(ke, (uint64_t)k)) >> 11) * 0x1.0p-53;
      const int64_t bit = (int64_t)1 << (scale - 1 - k);
      if (x >= a + b + c) {
        u |= bit;
        v |= bit;
      } else if (x >= a + b) {
        u |= bit;
      } else if (x >= a) {
        v |= bit;
      }
    }
    uv[2 * e] = u;
    uv[2 * e + 1] = v;
  }
}

/* sample_vertices (src/sampling.cpp:11-33) with the extra rejection rule */
int orc_sample_vertices_reject(int64_t n, int64_t b, uint64_t seed, uint64_t step, uint64_t reject_mod,
                               int64_t* out) {
  if (b <= 0 || b > n) return 1;
  orc_stream s = {orc_splitmix64(seed + step), 0.0, 0};
  int64_t* perm = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  if (!perm) return 2;
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = 0; i < b; ++i) {
    const int64_t j = i + (int64_t)st_next_below_rej(&s, (uint64_t)(n - i), reject_mod);
    const int64_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  memcpy(out, perm, (size_t)b * sizeof(int64_t));
  free(perm);
  qsort(out, (size_t)b, sizeof(int64_t), cmp_i64);
  return 0;
}

/* TEST INFRASTRUCTURE ONLY — the CPU oracle (see slimsell_oracle.h).
 *
 * Plain-C restatement of the reference algorithm; each function names the
 * reference file:line (relative to /root/reference/proj) it restates. Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 */
#include "slimsell_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL

/* generator.cpp:9-13 (splitmix64 finaliser) */
uint64_t so_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* FNV-1a-64 of int32 values as the little-endian int64 bytes of their
 * sign-extended values, continuing from h (pass 0xcbf29ce484222325 first):
 * fingerprints a device-resident int32 col against the reference's int64 col
 * without a 2x host copy. Test infrastructure. */
uint64_t so_fnv1a64_i32(const int32_t* a, int64_t count, uint64_t h) {
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t v = (uint64_t)(int64_t)a[i];
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 0x100000001b3ULL;
    }
  }
  return h;
}

uint64_t so_fnv1a64(const void* data, int64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* generator.hpp:29-31 SplitMix64::split */
static uint64_t split_state(uint64_t state, uint64_t tag) {
  return so_mix64(state ^ so_mix64(tag + 0x6a09e667f3bcc909ULL));
}

/* generator.hpp:22-27 next()/next_unit() */
static uint64_t next_u64(uint64_t* s) {
  *s += GAMMA;
  return so_mix64(*s);
}
static double next_unit(uint64_t* s) { return (double)(next_u64(s) >> 11) * 0x1.0p-53; }

/* generator.cpp:60-89 gen_kronecker (candidate stage) */
int so_gen_kronecker_pairs(int64_t scale, int64_t ef, uint64_t seed,
                           const double init[4], int64_t* uv) {
  if (scale < 1 || ef < 1) return SO_EINVAL;
  double sum = init[0] + init[1] + init[2] + init[3];
  if (fabs(sum - 1.0) > 1e-9) return SO_EINVAL;
  const double ab = init[0] + init[1];
  const double abc = ab + init[2];
  uint64_t s = split_state(seed, 0x4b);
  const int64_t cand = ef << scale;
  for (int64_t e = 0; e < cand; ++e) {
    int64_t u = 0, v = 0;
    for (int64_t l = 0; l < scale; ++l) {
      double r = next_unit(&s);
      int ub = r >= ab;
      int vb = ub ? (r >= abc) : (r >= init[0]);
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    uv[2 * e] = u;
    uv[2 * e + 1] = v;
  }
  return SO_OK;
}

/* generator.cpp:15-58 gen_erdos_renyi (geometric skips over the pair index) */
int so_gen_erdos_renyi_pairs(int64_t n, double p, uint64_t seed, int64_t** uv_out,
                             int64_t* count) {
  if (n < 0 || !(p >= 0.0 && p <= 1.0)) return SO_EINVAL;
  int64_t cap = 1024, cnt = 0;
  int64_t* uv = (int64_t*)malloc(sizeof(int64_t) * 2 * cap);
  if (!uv) return SO_ENOMEM;
#define PUSH(a, b)                                                    \
  do {                                                                \
    if (cnt == cap) {                                                 \
      cap *= 2;                                                       \
      int64_t* t = (int64_t*)realloc(uv, sizeof(int64_t) * 2 * cap);  \
      if (!t) {                                                       \
        free(uv);                                                     \
        return SO_ENOMEM;                                             \
      }                                                               \
      uv = t;                                                         \
    }                                                                 \
    uv[2 * cnt] = (a);                                                \
    uv[2 * cnt + 1] = (b);                                            \
    ++cnt;                                                            \
  } while (0)
  if (p > 0.0 && n > 1) {
    if (p == 1.0) {
      for (int64_t a = 0; a < n; ++a)
        for (int64_t b = a + 1; b < n; ++b) PUSH(a, b);
    } else {
      uint64_t s = split_state(seed, 0xe5);
      const double denom = log1p(-p);
      int64_t u = 0, off = 0, row_left = n - 1;
      int done = 0;
      int64_t steps = (int64_t)floor(log(1.0 - next_unit(&s)) / denom);
      for (;;) {
        /* advance the (u, off) cursor by `steps` pairs */
        while (steps >= row_left - off) {
          steps -= row_left - off;
          ++u;
          off = 0;
          row_left = n - 1 - u;
          if (u >= n - 1) {
            done = 1;
            break;
          }
        }
        if (done) break;
        off += steps;
        PUSH(u, u + 1 + off);
        steps = 1 + (int64_t)floor(log(1.0 - next_unit(&s)) / denom);
      }
    }
  }
#undef PUSH
  *uv_out = uv;
  *count = cnt;
  return SO_OK;
}

static int cmp_pair(const void* a, const void* b) {
  const int64_t* x = (const int64_t*)a;
  const int64_t* y = (const int64_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
  return 0;
}

/* graph.cpp:65-86 Graph::from_pairs: orient u<v, drop self-loops, sort, dedup */
int64_t so_normalize_pairs(int64_t* uv, int64_t count, int64_t n, int64_t* n_out) {
  int64_t max_id = -1;
  for (int64_t i = 0; i < count; ++i) {
    int64_t a = uv[2 * i], b = uv[2 * i + 1];
    if (a < 0 || b < 0) return -SO_ERANGE;
    if (a > b) {
      uv[2 * i] = b;
      uv[2 * i + 1] = a;
      b = a;
    }
    if (b > max_id) max_id = b;
  }
  if (n < 0) n = max_id + 1;
  else if (max_id >= n) return -SO_ERANGE;
  int64_t w = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (uv[2 * i] == uv[2 * i + 1]) continue;
    uv[2 * w] = uv[2 * i];
    uv[2 * w + 1] = uv[2 * i + 1];
    ++w;
  }
  qsort(uv, (size_t)w, 2 * sizeof(int64_t), cmp_pair);
  int64_t m = 0;
  for (int64_t i = 0; i < w; ++i) {
    if (m > 0 && uv[2 * (m - 1)] == uv[2 * i] && uv[2 * (m - 1) + 1] == uv[2 * i + 1])
      continue;
    uv[2 * m] = uv[2 * i];
    uv[2 * m + 1] = uv[2 * i + 1];
    ++m;
  }
  if (n_out) *n_out = n;
  return m;
}

/* graph.cpp:212-232 to_csr: counting pass + fill pass over sorted (u<v) edges */
void so_to_csr(int64_t n, const int64_t* uv, int64_t m, int64_t* row, int64_t* col) {
  memset(row, 0, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t e = 0; e < m; ++e) {
    row[uv[2 * e] + 1]++;
    row[uv[2 * e + 1] + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) row[i + 1] += row[i];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(cur, row, sizeof(int64_t) * (size_t)n);
  for (int64_t e = 0; e < m; ++e) {
    int64_t a = uv[2 * e], b = uv[2 * e + 1];
    col[cur[a]++] = b;
    col[cur[b]++] = a;
  }
  free(cur);
}

/* ---- repr.cpp:62-82 make_sort_plan ------------------------------------ */
static const int64_t* g_len; /* qsort context (single-threaded oracle) */
static int cmp_by_len_desc_id_asc(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  if (g_len[x] != g_len[y]) return g_len[x] > g_len[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}

int so_make_sort_plan(const int64_t* lengths, int64_t n, int64_t sigma, int64_t* perm,
                      int64_t* inv_perm, int64_t* sigma_eff) {
  if (sigma <= 0) return SO_EINVAL;
  int64_t s = sigma < (n > 1 ? n : 1) ? sigma : (n > 1 ? n : 1);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  g_len = lengths;
  for (int64_t w = 0; w < n; w += s) {
    int64_t end = w + s < n ? w + s : n;
    qsort(perm + w, (size_t)(end - w), sizeof(int64_t), cmp_by_len_desc_id_asc);
  }
  for (int64_t p = 0; p < n; ++p) inv_perm[perm[p]] = p;
  *sigma_eff = s;
  return SO_OK;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y);
}

/* repr.cpp:84-131 build_slimsell */
int so_build_slimsell(int64_t n, const int64_t* row, const int64_t* col, int64_t C,
                      int64_t sigma, so_repr* r) {
  memset(r, 0, sizeof(*r));
  if (C <= 0 || sigma <= 0) return SO_EINVAL;
  int64_t* len = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t v = 0; v < n; ++v) len[v] = row[v + 1] - row[v];
  r->perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  r->inv_perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  so_make_sort_plan(len, n, sigma, r->perm, r->inv_perm, &r->sigma);
  r->C = C;
  r->n = n;
  r->n_chunks = (n + C - 1) / C;
  r->n_padded = r->n_chunks * C;
  r->nonzeros = n == 0 ? 0 : row[n];
  r->cs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(r->n_chunks ? r->n_chunks : 1));
  r->cl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(r->n_chunks ? r->n_chunks : 1));
  int64_t total = 0;
  for (int64_t i = 0; i < r->n_chunks; ++i) {
    int64_t longest = 0;
    for (int64_t p = i * C; p < (i + 1) * C && p < n; ++p)
      if (len[r->perm[p]] > longest) longest = len[r->perm[p]];
    r->cs[i] = total;
    r->cl[i] = longest;
    total += C * longest;
  }
  r->n_cells = total;
  r->col = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total ? total : 1));
  for (int64_t i = 0; i < total; ++i) r->col[i] = -1;
  int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(r->nonzeros ? r->nonzeros : 1));
  for (int64_t p = 0; p < n; ++p) {
    int64_t o = r->perm[p], d = len[o];
    for (int64_t k = 0; k < d; ++k) nb[k] = r->inv_perm[col[row[o] + k]];
    qsort(nb, (size_t)d, sizeof(int64_t), cmp_i64);
    int64_t base = r->cs[p / C] + p % C;
    for (int64_t k = 0; k < d; ++k) r->col[base + k * C] = nb[k];
  }
  r->padding = total - r->nonzeros;
  free(nb);
  free(len);
  return SO_OK;
}

void so_repr_free(so_repr* r) {
  free(r->col);
  free(r->cs);
  free(r->cl);
  free(r->perm);
  free(r->inv_perm);
  memset(r, 0, sizeof(*r));
}

/* ---- semiring.hpp:56-87 scalar ops -------------------------------------- */
static int64_t sr_zero(int v) { return v == SO_TROPICAL ? SO_KINF : 0; }
static int64_t sr_plus(int v, int64_t a, int64_t b) {
  switch (v) {
    case SO_TROPICAL: return a < b ? a : b;
    case SO_REAL: return (int64_t)((uint64_t)a + (uint64_t)b);
    case SO_BOOLEAN: return a | b;
    default: return a > b ? a : b;
  }
}
static int64_t sr_times(int v, int64_t a, int64_t b) {
  switch (v) {
    case SO_TROPICAL: return (a == SO_KINF || b == SO_KINF) ? SO_KINF : a + b;
    case SO_REAL:
    case SO_SELMAX: return (int64_t)((uint64_t)a * (uint64_t)b);
    default: return a & b;
  }
}

/* repr.cpp:20-35 slim_segment_impl: acc[lane] = plus(acc, times(x[c], edge|pad)) */
static void segment(const so_repr* r, int v, const int64_t* x, int64_t* acc, int64_t chunk,
                    int64_t cb, int64_t clen) {
  const int64_t edge = 1, pad = sr_zero(v); /* semiring.hpp:61-84: edge 1, pad == zero */
  const int64_t* cells = r->col + r->cs[chunk] + cb * r->C;
  for (int64_t j = 0; j < clen; ++j, cells += r->C)
    for (int64_t lane = 0; lane < r->C; ++lane) {
      int64_t c = cells[lane];
      acc[lane] = sr_plus(v, acc[lane], sr_times(v, x[c < 0 ? 0 : c], c < 0 ? pad : edge));
    }
}

/* repr.cpp:193-217 spmv_chunks / spmv_step */
int so_spmv_step(const so_repr* r, int variant, const int64_t* x_prev, int64_t* out,
                 int64_t cb, int64_t ce) {
  if (variant < 0 || variant > 3) return SO_EINVAL;
  if (cb < 0 || ce > r->n_chunks || cb > ce) return SO_EINVAL;
  for (int64_t i = cb; i < ce; ++i) {
    int64_t* acc = out + i * r->C;
    memcpy(acc, x_prev + i * r->C, sizeof(int64_t) * (size_t)r->C);
    segment(r, variant, x_prev, acc, i, 0, r->cl[i]);
  }
  return SO_OK;
}

/* ---- the BFS engine: bfs.cpp:53-155 + semiring.cpp:56-157 --------------- */
typedef struct {
  int64_t *x, *f, *g, *p, *d, *xprev;
} so_state;

int so_bfs_spmv(const so_repr* r, int64_t root, int variant, int slimwork, int64_t L,
                int64_t max_iterations, int want_parents, const int64_t* csr_row,
                const int64_t* csr_col, int64_t* dist, int64_t* parent,
                int64_t* parent_len, int64_t* iterations, int64_t* stats,
                int64_t stats_cap) {
  if (variant < 0 || variant > 3) return SO_EINVAL;
  const int64_t n = r->n, np = r->n_padded, C = r->C;
  /* semiring.cpp:57-60 */
  if (root < 0 || root >= n) return SO_ERANGE;
  const int filtered = variant == SO_REAL || variant == SO_BOOLEAN;
  size_t bytes = sizeof(int64_t) * (size_t)(np ? np : 1);
  so_state s;
  s.x = (int64_t*)malloc(bytes);
  s.f = (int64_t*)malloc(bytes);
  s.g = (int64_t*)malloc(bytes);
  s.p = (int64_t*)malloc(bytes);
  s.d = (int64_t*)malloc(bytes);
  s.xprev = (int64_t*)malloc(bytes);
  /* init_state (semiring.cpp:56-88) composed with permute_in (repr.cpp:239-245,
   * fills as bfs.cpp:57-61): positions move, VALUES do not (sel-max keeps
   * root+1 in original numbering — the reference's quirk). */
  const int64_t zero = sr_zero(variant);
  for (int64_t q = 0; q < np; ++q) {
    s.x[q] = zero;
    s.f[q] = variant == SO_TROPICAL ? SO_KINF : 0;
    s.d[q] = SO_KINF;
    s.g[q] = filtered && q < n ? 1 : 0;
    s.p[q] = 0;
  }
  const int64_t rp = r->inv_perm[root];
  s.d[rp] = 0;
  switch (variant) {
    case SO_TROPICAL: s.x[rp] = 0; s.f[rp] = 0; break;
    case SO_REAL:
    case SO_BOOLEAN: s.x[rp] = 1; s.f[rp] = 1; s.g[rp] = 0; break;
    default: s.x[rp] = root + 1; s.p[rp] = root + 1; s.f[rp] = 1; break;
  }
  memcpy(s.xprev, s.x, bytes);

  /* plan_subchunks (bfs.cpp:10-22): segment count per chunk */
  int64_t nseg_total = 0;
  int64_t* first = NULL;
  int64_t* partials = NULL;
  if (L > 0) {
    first = (int64_t*)malloc(sizeof(int64_t) * (size_t)(r->n_chunks + 1));
    for (int64_t i = 0; i < r->n_chunks; ++i) {
      first[i] = nseg_total;
      nseg_total += (r->cl[i] + L - 1) / L;
    }
    first[r->n_chunks] = nseg_total;
    partials = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nseg_total * C + 1));
  }

  const int64_t cap = max_iterations > 0 ? max_iterations : n + 1;
  int converged = n == 0;
  int64_t k = 0, niter = 0;
  for (k = 1; !converged && k <= cap; ++k) {
    int64_t st[7] = {k, 0, 0, 0, 0, 0, 0};
    int64_t* t = s.xprev; s.xprev = s.x; s.x = t; /* bfs.cpp:106 */
    const int64_t* in = filtered ? s.f : s.xprev;  /* bfs.cpp:109-111 */
    for (int64_t i = 0; i < r->n_chunks; ++i) {
      const int64_t r0 = i * C, r1 = (i + 1) * C < n ? (i + 1) * C : n;
      if (slimwork) {
        /* should_skip_chunk (semiring.cpp:130-150): every real row visited */
        int skip = 1;
        for (int64_t q = r0; q < r1 && skip; ++q) {
          if (variant == SO_TROPICAL) skip = s.f[q] != SO_KINF;
          else if (filtered) skip = s.g[q] == 0;
          else skip = s.p[q] != 0;
        }
        if (skip) {
          memcpy(s.x + r0, s.xprev + r0, sizeof(int64_t) * (size_t)C);
          st[3]++;
          continue;
        }
      }
      st[2]++;
      st[5] += r->cl[i];
      if (L <= 0) {
        /* run_task, whole chunk, seeded from input (bfs.cpp:157-170) */
        memcpy(s.x + r0, in + r0, sizeof(int64_t) * (size_t)C);
        segment(r, variant, in, s.x + r0, i, 0, r->cl[i]);
      } else if (first[i] == first[i + 1]) {
        memcpy(s.x + r0, in + r0, sizeof(int64_t) * (size_t)C); /* bfs.cpp:127-130 */
      } else {
        for (int64_t sg = first[i]; sg < first[i + 1]; ++sg) {
          int64_t* acc = partials + sg * C;
          int64_t cb = (sg - first[i]) * L;
          int64_t cl = r->cl[i] - cb < L ? r->cl[i] - cb : L;
          if (sg == first[i]) memcpy(acc, in + r0, sizeof(int64_t) * (size_t)C);
          else
            for (int64_t l = 0; l < C; ++l) acc[l] = zero;
          segment(r, variant, in, acc, i, cb, cl);
          st[4]++;
        }
        /* combine_chunks (bfs.cpp:205-220): fold in segment order */
        memcpy(s.x + r0, partials + first[i] * C, sizeof(int64_t) * (size_t)C);
        for (int64_t sg = first[i] + 1; sg < first[i + 1]; ++sg)
          for (int64_t l = 0; l < C; ++l)
            s.x[r0 + l] = sr_plus(variant, s.x[r0 + l], partials[sg * C + l]);
      }
    }
    /* post_process (semiring.cpp:90-128) over all padded rows */
    for (int64_t q = 0; q < np; ++q) {
      if (variant == SO_TROPICAL) {
        s.f[q] = s.x[q];
        s.d[q] = s.x[q];
      } else if (filtered) {
        int newly = s.x[q] != 0 && s.g[q] != 0;
        s.f[q] = newly;
        if (newly) { s.d[q] = k; s.g[q] = 0; }
      } else {
        int newly = s.p[q] == 0 && s.x[q] != 0;
        s.f[q] = newly;
        if (newly) { s.p[q] = s.x[q]; s.d[q] = k; }
        s.x[q] = s.x[q] != 0 ? q + 1 : 0;
      }
    }
    /* frontier size over real rows (bfs.cpp:147-153) */
    for (int64_t q = 0; q < n; ++q)
      st[6] += variant == SO_TROPICAL ? (s.xprev[q] == SO_KINF && s.x[q] != SO_KINF)
                                      : (s.f[q] != 0);
    /* is_converged (semiring.cpp:152-157) */
    converged = 1;
    if (variant == SO_TROPICAL) {
      for (int64_t q = 0; q < np && converged; ++q) converged = s.x[q] == s.xprev[q];
    } else {
      for (int64_t q = 0; q < np && converged; ++q) converged = s.f[q] == 0;
    }
    if (stats && niter < stats_cap) memcpy(stats + 7 * niter, st, sizeof(st));
    ++niter;
  }
  /* permute_out (repr.cpp:247-253) */
  for (int64_t q = 0; q < n; ++q) dist[r->perm[q]] = s.d[q];
  if (iterations) *iterations = niter;
  int rc = converged ? SO_OK : SO_ECAP;
  int64_t plen = 0;
  if (rc == SO_OK && want_parents) {
    if (variant == SO_SELMAX) {
      /* selmax_parents (bfs.cpp:94-101): the stored value is decoded as a
       * PERMUTED position even for the root's original-id encoding. */
      for (int64_t v = 0; v < n; ++v) parent[v] = -1;
      for (int64_t q = 0; q < n; ++q)
        if (s.p[q] != 0) parent[r->perm[q]] = r->perm[s.p[q] - 1];
      plen = n;
    } else if (csr_row) {
      rc = so_dp_transform(n, csr_row, csr_col, dist, parent);
      plen = rc == SO_OK ? n : 0;
    }
  }
  if (parent_len) *parent_len = plen;
  free(s.x); free(s.f); free(s.g); free(s.p); free(s.d); free(s.xprev);
  free(first);
  free(partials);
  return rc;
}

/* bfs.cpp:248-291 bfs_traditional: level-synchronous queue BFS, ascending frontier */
static int cmp_i64v(const void* a, const void* b) { return cmp_i64(a, b); }
int so_bfs_traditional(int64_t n, const int64_t* row, const int64_t* col, int64_t root,
                       int64_t* dist, int64_t* parent, int64_t* iterations) {
  if (root < 0 || root >= n) return SO_ERANGE;
  for (int64_t v = 0; v < n; ++v) { dist[v] = SO_KINF; parent[v] = -1; }
  dist[root] = 0;
  parent[root] = root;
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* nxt = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t nc = 1, k = 0;
  cur[0] = root;
  while (nc > 0) {
    ++k;
    int64_t nn = 0;
    for (int64_t i = 0; i < nc; ++i) {
      int64_t u = cur[i];
      for (int64_t e = row[u]; e < row[u + 1]; ++e) {
        int64_t w = col[e];
        if (dist[w] == SO_KINF) { dist[w] = k; parent[w] = u; nxt[nn++] = w; }
      }
    }
    qsort(nxt, (size_t)nn, sizeof(int64_t), cmp_i64v);
    int64_t* t = cur; cur = nxt; nxt = t;
    nc = nn;
  }
  *iterations = k;
  free(cur);
  free(nxt);
  return SO_OK;
}

/* semiring.cpp:159-187 dp_transform: smallest-id neighbour one level closer */
int so_dp_transform(int64_t n, const int64_t* row, const int64_t* col, const int64_t* d,
                    int64_t* parent) {
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = -1;
    if (d[v] == SO_KINF) continue;
    if (d[v] == 0) { parent[v] = v; continue; }
    for (int64_t e = row[v]; e < row[v + 1]; ++e) {
      int64_t w = col[e];
      if (d[w] != SO_KINF && d[w] == d[v] - 1) { parent[v] = w; break; }
    }
    if (parent[v] == -1) return SO_EINVAL;
  }
  return SO_OK;
}

/* cli.cpp:114-134 pick_roots (random:k form): distinct draws of
 * SplitMix64(seed).split(0x526f).next() % n */
void so_pick_roots(int64_t n, int64_t want, uint64_t seed, int64_t* roots) {
  if (want < 1) want = 1;
  if (want > n) want = n;
  unsigned char* used = (unsigned char*)calloc((size_t)n, 1);
  uint64_t s = split_state(seed, 0x526f);
  int64_t got = 0;
  while (got < want) {
    int64_t r = (int64_t)(next_u64(&s) % (uint64_t)n);
    if (!used[r]) { used[r] = 1; roots[got++] = r; }
  }
  free(used);
}

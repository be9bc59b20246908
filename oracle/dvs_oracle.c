/*
 * dvs_oracle.c -- CPU restatement of the reference's batched graph-search path.
 *
 * TEST INFRASTRUCTURE ONLY (see dvs_oracle.h).  Plain C11 + pthreads.
 * Every routine follows the reference line by line in *semantics* (same
 * accumulation order, same (dist, id) tie rules, same visited counter) but is
 * written from scratch: open-addressing visited set, qsort pools.
 *
 * Pinned by tests/test_oracle.py against oracle/_ref/libdvsref.so (the
 * reference's own sources compiled unmodified) and the tests/golden fixtures.
 */
#define _GNU_SOURCE
#include "dvs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char *dvso_last_error(void) { return g_err; }

static int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the engine behind tests/support/synthetic.hpp)               */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void dvso_mt64_seed(dvso_mt64 *g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = MT_N;
}

uint64_t dvso_mt64_next(dvso_mt64 *g) {
  if (g->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (g->mt[i] & MT_UM) | (g->mt[(i + 1) % MT_N] & MT_LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= MT_A;
      g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* synthetic.hpp:15-17 */
double dvso_uniform01(dvso_mt64 *g) { return (double)(dvso_mt64_next(g) >> 11) * 0x1.0p-53; }
/* synthetic.hpp:19-21 */
double dvso_uniform(dvso_mt64 *g, double lo, double hi) { return lo + (hi - lo) * dvso_uniform01(g); }
/* synthetic.hpp:23-28 (Box-Muller, cosine branch only) */
double dvso_gaussian(dvso_mt64 *g) {
  double u1 = dvso_uniform01(g);
  while (u1 <= 1e-300) u1 = dvso_uniform01(g);
  const double u2 = dvso_uniform01(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* synthetic.hpp:30-40 */
void dvso_random_dataset(uint64_t n, int dim, uint64_t seed, double lo, double hi, float *out) {
  dvso_mt64 g;
  dvso_mt64_seed(&g, seed);
  const uint64_t total = n * (uint64_t)dim;
  for (uint64_t i = 0; i < total; ++i) out[i] = (float)dvso_uniform(&g, lo, hi);
}

/* synthetic.hpp:50-73 */
void dvso_gaussian_mixture(uint64_t n, int dim, int components, double mean_scale,
                           double stddev, uint64_t seed, float *means_out, float *points_out,
                           int *labels_out) {
  dvso_mt64 g;
  dvso_mt64_seed(&g, seed);
  for (int c = 0; c < components; ++c)
    for (int j = 0; j < dim; ++j) means_out[(size_t)c * dim + j] = (float)(dvso_gaussian(&g) * mean_scale);
  for (uint64_t i = 0; i < n; ++i) {
    const int c = (int)(i % (uint64_t)components);
    if (labels_out) labels_out[i] = c;
    for (int j = 0; j < dim; ++j)
      points_out[i * dim + j] = (float)(means_out[(size_t)c * dim + j] + dvso_gaussian(&g) * stddev);
  }
}

/* synthetic.hpp:76-90 */
void dvso_mixture_queries(const float *means, int components, int dim, uint64_t n,
                          double stddev, uint64_t seed, float *out) {
  dvso_mt64 g;
  dvso_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < n; ++i) {
    const float *mean = means + (size_t)(i % (uint64_t)components) * dim;
    for (int j = 0; j < dim; ++j) out[i * dim + j] = (float)(mean[j] + dvso_gaussian(&g) * stddev);
  }
}

/* ------------------------------------------------------------------------ */
/* distance.cpp:19-50 -- fp64 sequential accumulation, rounded to float     */
/* ------------------------------------------------------------------------ */
float dvso_squared_l2(const float *a, const float *b, int dim) {
  double acc = 0.0;
  for (int i = 0; i < dim; ++i) {
    const double diff = (double)a[i] - (double)b[i];
    acc += diff * diff;
  }
  return (float)acc;
}

double dvso_dot(const float *a, const float *b, int dim) {
  double acc = 0.0;
  for (int i = 0; i < dim; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

double dvso_squared_norm(const float *a, int dim) {
  double acc = 0.0;
  for (int i = 0; i < dim; ++i) acc += (double)a[i] * (double)a[i];
  return acc;
}

float dvso_squared_l2_expanded(const float *a, const float *b, int dim) {
  const double d = dvso_squared_norm(a, dim) + dvso_squared_norm(b, dim) - 2.0 * dvso_dot(a, b, dim);
  return (float)(d < 0.0 ? 0.0 : d);
}

static inline float metric_dist(int metric, const float *q, const float *v, int dim) {
  if (metric == DVSO_METRIC_IP) return (float)(-dvso_dot(q, v, dim));
  return dvso_squared_l2(q, v, dim);
}

/* ------------------------------------------------------------------------ */
/* ScoredId ordering: dataset.hpp:43-46 scored_less                         */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint32_t id;
  float dist;
} scored_t;

static int scored_cmp(const void *pa, const void *pb) {
  const scored_t *a = (const scored_t *)pa, *b = (const scored_t *)pb;
  if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
  return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

static int scored_less(scored_t a, scored_t b) {
  if (a.dist != b.dist) return a.dist < b.dist;
  return a.id < b.id;
}

/* graph_index.cpp:21-44 */
int dvso_compute_entry_order(const float *data, uint64_t n, int dim, uint32_t *out) {
  if (n == 0 || dim <= 0) return fail(DVSO_EINVAL, "compute_entry_order: empty partition");
  double *sums = calloc((size_t)dim, sizeof(double));
  float *mean = malloc(sizeof(float) * (size_t)dim);
  scored_t *order = malloc(sizeof(scored_t) * n);
  if (!sums || !mean || !order) {
    free(sums); free(mean); free(order);
    return fail(DVSO_EINTERNAL, "compute_entry_order: out of memory");
  }
  for (uint64_t i = 0; i < n; ++i)
    for (int j = 0; j < dim; ++j) sums[j] += data[i * dim + j];
  for (int j = 0; j < dim; ++j) mean[j] = (float)(sums[j] / (double)n);
  for (uint64_t i = 0; i < n; ++i) {
    order[i].id = (uint32_t)i;
    order[i].dist = dvso_squared_l2(data + i * dim, mean, dim);
  }
  qsort(order, n, sizeof(scored_t), scored_cmp);
  for (uint64_t i = 0; i < n; ++i) out[i] = order[i].id;
  free(sums); free(mean); free(order);
  return DVSO_OK;
}

/* ------------------------------------------------------------------------ */
/* generic order-preserving parallel-for                                    */
/* ------------------------------------------------------------------------ */
typedef int (*range_fn)(void *ctx, uint64_t begin, uint64_t end);
typedef struct {
  range_fn fn;
  void *ctx;
  uint64_t begin, end;
  int rc;
  char err[512];
} pf_task;

static void *pf_thread(void *arg) {
  pf_task *t = (pf_task *)arg;
  t->rc = t->fn(t->ctx, t->begin, t->end);
  if (t->rc) memcpy(t->err, g_err, sizeof t->err);
  return NULL;
}

static int parallel_for(uint64_t n, int nthreads, range_fn fn, void *ctx) {
  if (nthreads <= 1 || n < 2) return fn(ctx, 0, n);
  if ((uint64_t)nthreads > n) nthreads = (int)n;
  pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
  pf_task *tasks = calloc((size_t)nthreads, sizeof(pf_task));
  /* interleaved blocks of 16 would balance better, but contiguous ranges keep
   * the restatement trivially order-preserving; outputs are per-index anyway */
  for (int t = 0; t < nthreads; ++t) {
    tasks[t].fn = fn;
    tasks[t].ctx = ctx;
    tasks[t].begin = n * (uint64_t)t / (uint64_t)nthreads;
    tasks[t].end = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
    pthread_create(&th[t], NULL, pf_thread, &tasks[t]);
  }
  int rc = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    if (tasks[t].rc && !rc) {
      rc = tasks[t].rc;
      memcpy(g_err, tasks[t].err, sizeof g_err);
    }
  }
  free(th);
  free(tasks);
  return rc;
}

/* graph_index.cpp:46-97: exact kNN rows, ties by lower id; tiny partitions
 * repeat the sorted list cyclically; a lone node pads with itself. */
typedef struct {
  const float *data;
  uint64_t n;
  int dim, dg;
  uint32_t *adj;
} build_ctx;

static int build_rows(void *vctx, uint64_t begin, uint64_t end) {
  build_ctx *c = (build_ctx *)vctx;
  const uint64_t n = c->n;
  scored_t *others = malloc(sizeof(scored_t) * (n > 1 ? n - 1 : 1));
  for (uint64_t v = begin; v < end; ++v) {
    uint32_t *row = c->adj + v * (uint64_t)c->dg;
    if (n == 1) {
      for (int j = 0; j < c->dg; ++j) row[j] = 0;
      continue;
    }
    uint64_t m = 0;
    for (uint64_t u = 0; u < n; ++u) {
      if (u == v) continue;
      others[m].id = (uint32_t)u;
      others[m].dist = dvso_squared_l2(c->data + v * c->dim, c->data + u * c->dim, c->dim);
      ++m;
    }
    qsort(others, m, sizeof(scored_t), scored_cmp);
    for (int j = 0; j < c->dg; ++j) row[j] = others[(uint64_t)j % m].id;
  }
  free(others);
  return DVSO_OK;
}

int dvso_build_graph(const float *data, uint64_t n, int dim, int out_degree,
                     uint32_t *adjacency_out, int nthreads) {
  if (n == 0) return fail(DVSO_EINVAL, "build_graph: empty partition");
  if (out_degree < 1) return fail(DVSO_EINVAL, "build_graph: out_degree must be >= 1");
  build_ctx c = {data, n, dim, out_degree, adjacency_out};
  return parallel_for(n, nthreads, build_rows, &c);
}

/* ------------------------------------------------------------------------ */
/* beam_search_stats, graph_index.cpp:105-187                               */
/* ------------------------------------------------------------------------ */
typedef struct {
  float dist;
  uint32_t local;
  uint8_t expanded;
} cand_t;

/* cand_less, graph_index.cpp:122-125 */
static int cand_cmp(const void *pa, const void *pb) {
  const cand_t *a = (const cand_t *)pa, *b = (const cand_t *)pb;
  if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
  return a->local < b->local ? -1 : (a->local > b->local ? 1 : 0);
}

/* exact visited set: open addressing on u32 ids, never forgets
 * (graph_index.cpp:133 unordered_set semantics) */
typedef struct {
  uint32_t *slots;
  uint64_t mask;
} vset;

static int vset_insert(vset *s, uint32_t id) {
  uint64_t h = ((uint64_t)id * 0x9E3779B97F4A7C15ULL) >> 20;
  for (;;) {
    h &= s->mask;
    if (s->slots[h] == UINT32_MAX) {
      s->slots[h] = id;
      return 1;
    }
    if (s->slots[h] == id) return 0;
    ++h;
  }
}

static int validate_params(const dvso_params *p) {
  if (p->iterations < 1 || p->beam_width < 1 || p->k < 1 || p->entry_count < 1)
    return fail(DVSO_EINVAL, "SearchParams: iterations, beam_width, k and entry_count must all be >= 1");
  if (p->metric != DVSO_METRIC_L2 && p->metric != DVSO_METRIC_IP)
    return fail(DVSO_EINVAL, "SearchParams: unknown metric %d", p->metric);
  return DVSO_OK;
}

int dvso_beam_search(const dvso_graph *g, const float *query, const dvso_params *p,
                     uint32_t *out_ids, float *out_dists, uint32_t *out_count,
                     uint64_t *out_visited) {
  int rc = validate_params(p);
  if (rc) return rc;
  const uint64_t n = g->n;
  if (n == 0) return fail(DVSO_EINVAL, "beam_search: empty graph");
  const int dim = g->dim, dg = g->out_degree;
  const uint64_t cap_a = 4ULL * (uint64_t)p->k;
  const uint64_t cap_b = 2ULL * (uint64_t)p->iterations * (uint64_t)p->beam_width;
  const uint64_t cap = cap_a > cap_b ? cap_a : cap_b;
  const uint64_t entries = (uint64_t)p->entry_count < n ? (uint64_t)p->entry_count : n;

  uint64_t pool_cap = cap + (uint64_t)p->beam_width * (uint64_t)dg;
  if (entries > pool_cap) pool_cap = entries;
  cand_t *pool = malloc(sizeof(cand_t) * pool_cap);
  /* visited never exceeds min(n, entries + I*w*dg) */
  uint64_t bound = entries + (uint64_t)p->iterations * (uint64_t)p->beam_width * (uint64_t)dg;
  if (bound > n) bound = n;
  uint64_t hsz = 64;
  while (hsz < 2 * bound + 1) hsz <<= 1;
  vset vs = {malloc(sizeof(uint32_t) * hsz), hsz - 1};
  uint64_t *frontier = malloc(sizeof(uint64_t) * (size_t)p->beam_width);
  if (!pool || !vs.slots || !frontier) {
    free(pool); free(vs.slots); free(frontier);
    return fail(DVSO_EINTERNAL, "beam_search: out of memory");
  }
  memset(vs.slots, 0xFF, sizeof(uint32_t) * hsz);
  uint64_t scored = 0, size = 0;

  for (uint64_t i = 0; i < entries; ++i) { /* :146-151 */
    const uint32_t local = g->entry_order[i];
    vset_insert(&vs, local);
    ++scored;
    pool[size].dist = metric_dist(p->metric, query, g->vectors + (uint64_t)local * dim, dim);
    pool[size].local = local;
    pool[size].expanded = 0;
    ++size;
  }
  qsort(pool, size, sizeof(cand_t), cand_cmp); /* shrink(), :141-144 */
  if (size > cap) size = cap;

  for (int iter = 0; iter < p->iterations; ++iter) { /* :155 */
    uint64_t nf = 0;
    for (uint64_t i = 0; i < size && nf < (uint64_t)p->beam_width; ++i)
      if (!pool[i].expanded) frontier[nf++] = i;
    if (nf == 0) break; /* :160 */
    for (uint64_t f = 0; f < nf; ++f) pool[frontier[f]].expanded = 1;
    const uint64_t before = size;
    for (uint64_t f = 0; f < nf; ++f) {
      const uint32_t *row = g->adjacency + (uint64_t)pool[frontier[f]].local * (uint64_t)dg;
      for (int j = 0; j < dg; ++j) {
        const uint32_t nb = row[j];
        if (vset_insert(&vs, nb)) {
          ++scored;
          pool[size].dist = metric_dist(p->metric, query, g->vectors + (uint64_t)nb * dim, dim);
          pool[size].local = nb;
          pool[size].expanded = 0;
          ++size;
        }
      }
    }
    if (size != before) {
      qsort(pool, size, sizeof(cand_t), cand_cmp);
      if (size > cap) size = cap;
    }
  }

  /* :173-186: global ids, re-sorted by (dist, gid), first min(k, size) */
  scored_t *all = malloc(sizeof(scored_t) * (size ? size : 1));
  for (uint64_t i = 0; i < size; ++i) {
    all[i].id = g->global_ids[pool[i].local];
    all[i].dist = pool[i].dist;
  }
  qsort(all, size, sizeof(scored_t), scored_cmp);
  const uint64_t want = (uint64_t)p->k < size ? (uint64_t)p->k : size;
  for (uint64_t i = 0; i < want; ++i) {
    out_ids[i] = all[i].id;
    out_dists[i] = all[i].dist;
  }
  *out_count = (uint32_t)want;
  *out_visited = scored;
  free(all); free(pool); free(vs.slots); free(frontier);
  return DVSO_OK;
}

typedef struct {
  const dvso_graph *g;
  const float *queries;
  const dvso_params *p;
  uint32_t *ids;
  float *dists;
  uint32_t *count;
  uint64_t *visited;
} search_ctx;

static int search_rows(void *vctx, uint64_t begin, uint64_t end) {
  search_ctx *c = (search_ctx *)vctx;
  const uint64_t k = (uint64_t)c->p->k;
  for (uint64_t q = begin; q < end; ++q) {
    int rc = dvso_beam_search(c->g, c->queries + q * (uint64_t)c->g->dim, c->p, c->ids + q * k,
                              c->dists + q * k, c->count + q, c->visited + q);
    if (rc) return rc;
  }
  return DVSO_OK;
}

int dvso_beam_search_batch(const dvso_graph *g, const float *queries, uint64_t nq,
                           const dvso_params *p, int nthreads, uint32_t *out_ids,
                           float *out_dists, uint32_t *out_count, uint64_t *out_visited) {
  int rc = validate_params(p);
  if (rc) return rc;
  search_ctx c = {g, queries, p, out_ids, out_dists, out_count, out_visited};
  return parallel_for(nq, nthreads, search_rows, &c);
}

/* ------------------------------------------------------------------------ */
/* combine_results, simulator.cpp:219-243                                   */
/* ------------------------------------------------------------------------ */
int dvso_combine_results(int nparts, const uint32_t *ids, const float *dists,
                         const uint32_t *counts, int stride, int k, uint32_t *out_ids,
                         float *out_dists, uint32_t *out_count) {
  if (k < 1) return fail(DVSO_EINVAL, "combine_results: k must be >= 1");
  uint64_t total = 0;
  for (int j = 0; j < nparts; ++j) total += counts[j];
  scored_t *merged = malloc(sizeof(scored_t) * (total ? total : 1));
  uint64_t m = 0;
  for (int j = 0; j < nparts; ++j) {
    const uint32_t *pi = ids + (uint64_t)j * (uint64_t)stride;
    const float *pd = dists + (uint64_t)j * (uint64_t)stride;
    for (uint32_t i = 0; i < counts[j]; ++i) {
      scored_t s = {pi[i], pd[i]};
      if (i > 0) {
        scored_t prev = {pi[i - 1], pd[i - 1]};
        if (scored_less(s, prev)) {
          free(merged);
          return fail(DVSO_EINTERNAL, "combine_results: partial list not sorted by (dist, id)");
        }
      }
      merged[m++] = s;
    }
  }
  qsort(merged, m, sizeof(scored_t), scored_cmp);
  uint32_t outn = 0;
  for (uint64_t i = 0; i < m && outn < (uint32_t)k; ++i) {
    int dup = 0; /* unordered_set dedup; out holds <= k ids so a scan is fine */
    for (uint32_t j = 0; j < outn; ++j)
      if (out_ids[j] == merged[i].id) { dup = 1; break; }
    if (dup) continue;
    out_ids[outn] = merged[i].id;
    out_dists[outn] = merged[i].dist;
    ++outn;
  }
  *out_count = outn;
  free(merged);
  return DVSO_OK;
}

/* ------------------------------------------------------------------------ */
/* assign_top_c, kmeans.cpp:243-280 (+ expanded_dist :44-48)               */
/* ------------------------------------------------------------------------ */
int dvso_assign_top_c(const float *cents, int clusters, int dim, const float *queries,
                      uint64_t nq, int c, uint32_t *out) {
  if (clusters < 1) return fail(DVSO_EINVAL, "assign_top_c: empty centroids");
  if (c < 1 || c > clusters)
    return fail(DVSO_EINVAL, "assign_top_c: c=%d out of range for %d clusters", c, clusters);
  double *cn = malloc(sizeof(double) * (size_t)clusters);
  scored_t *row = malloc(sizeof(scored_t) * (size_t)clusters);
  for (int j = 0; j < clusters; ++j) cn[j] = dvso_squared_norm(cents + (size_t)j * dim, dim);
  for (uint64_t qi = 0; qi < nq; ++qi) {
    const float *q = queries + qi * (uint64_t)dim;
    const double qn = dvso_squared_norm(q, dim);
    for (int j = 0; j < clusters; ++j) {
      const double d = qn + cn[j] - 2.0 * dvso_dot(q, cents + (size_t)j * dim, dim);
      row[j].id = (uint32_t)j;
      row[j].dist = (float)(d < 0.0 ? 0.0 : d);
    }
    qsort(row, (size_t)clusters, sizeof(scored_t), scored_cmp); /* partial_sort prefix */
    for (int j = 0; j < c; ++j) out[qi * (uint64_t)c + j] = row[j].id;
  }
  free(cn);
  free(row);
  return DVSO_OK;
}

/* partition_database, kmeans.cpp:282-300 (nearest_center :50-65: strict <,
 * so ties keep the lower cluster id) */
int dvso_partition_database(const float *db, uint64_t n, int dim, const float *cents,
                            int clusters, uint32_t *labels_out) {
  if (clusters < 1) return fail(DVSO_EINVAL, "partition_database: empty centroids");
  double *cn = malloc(sizeof(double) * (size_t)clusters);
  for (int j = 0; j < clusters; ++j) cn[j] = dvso_squared_norm(cents + (size_t)j * dim, dim);
  for (uint64_t i = 0; i < n; ++i) {
    const float *p = db + i * (uint64_t)dim;
    const double pn = dvso_squared_norm(p, dim);
    uint32_t best = 0;
    float best_d = 0;
    for (int j = 0; j < clusters; ++j) {
      const double d = pn + cn[j] - 2.0 * dvso_dot(p, cents + (size_t)j * dim, dim);
      const float f = (float)(d < 0.0 ? 0.0 : d);
      if (j == 0 || f < best_d) {
        best_d = f;
        best = (uint32_t)j;
      }
    }
    labels_out[i] = best;
  }
  free(cn);
  return DVSO_OK;
}

/* ------------------------------------------------------------------------ */
/* brute_force_topk, topk.cpp:12-30                                         */
/* ------------------------------------------------------------------------ */
int dvso_brute_force_topk(const float *db, uint64_t n, int dim, const float *q, int k,
                          uint32_t *out_ids, float *out_dists) {
  if (n == 0) return fail(DVSO_EINVAL, "brute_force_topk: empty database");
  if (k < 1 || (uint64_t)k > n)
    return fail(DVSO_EINVAL, "brute_force_topk: k=%d out of range for database of size %llu", k,
                (unsigned long long)n);
  scored_t *s = malloc(sizeof(scored_t) * n);
  for (uint64_t i = 0; i < n; ++i) {
    s[i].id = (uint32_t)i;
    s[i].dist = dvso_squared_l2(q, db + i * (uint64_t)dim, dim);
  }
  qsort(s, n, sizeof(scored_t), scored_cmp);
  for (int i = 0; i < k; ++i) {
    out_ids[i] = s[i].id;
    out_dists[i] = s[i].dist;
  }
  free(s);
  return DVSO_OK;
}

typedef struct {
  const float *db, *qs;
  uint64_t n;
  int dim, k;
  uint32_t *ids;
  float *dists;
} bf_ctx;

static int bf_rows(void *vctx, uint64_t begin, uint64_t end) {
  bf_ctx *c = (bf_ctx *)vctx;
  for (uint64_t q = begin; q < end; ++q) {
    int rc = dvso_brute_force_topk(c->db, c->n, c->dim, c->qs + q * (uint64_t)c->dim, c->k,
                                   c->ids + q * (uint64_t)c->k, c->dists + q * (uint64_t)c->k);
    if (rc) return rc;
  }
  return DVSO_OK;
}

int dvso_brute_force_topk_batch(const float *db, uint64_t n, int dim, const float *qs,
                                uint64_t nq, int k, int nthreads, uint32_t *out_ids,
                                float *out_dists) {
  bf_ctx c = {db, qs, n, dim, k, out_ids, out_dists};
  return parallel_for(nq, nthreads, bf_rows, &c);
}

/* ------------------------------------------------------------------------ */
/* run_pipeline functional part, simulator.cpp:245-337                      */
/* ------------------------------------------------------------------------ */
typedef struct {
  const dvso_index *idx;
  const float *queries;
  const dvso_params *p;
  int fanout;
  const uint32_t *assign;  /* nq x fanout */
  const uint32_t *loc_cl;  /* global id -> cluster */
  const uint32_t *loc_lo;  /* global id -> local */
  uint32_t *ids;
  float *dists;
  uint32_t *count;
  float *vectors;
  uint64_t *visited; /* per query */
} pipe_ctx;

static int pipe_rows(void *vctx, uint64_t begin, uint64_t end) {
  pipe_ctx *c = (pipe_ctx *)vctx;
  const int k = c->p->k, fo = c->fanout, dim = c->idx->dim;
  uint32_t *pids = malloc(sizeof(uint32_t) * (size_t)fo * (size_t)k);
  float *pd = malloc(sizeof(float) * (size_t)fo * (size_t)k);
  uint32_t *pc = malloc(sizeof(uint32_t) * (size_t)fo);
  int rc = DVSO_OK;
  for (uint64_t q = begin; q < end && !rc; ++q) {
    const float *qv = c->queries + q * (uint64_t)dim;
    uint64_t vis = 0;
    for (int j = 0; j < fo && !rc; ++j) {
      const uint32_t cl = c->assign[q * (uint64_t)fo + j];
      uint64_t v = 0;
      rc = dvso_beam_search(&c->idx->graphs[cl], qv, c->p, pids + (size_t)j * k, pd + (size_t)j * k,
                            pc + j, &v);
      vis += v;
    }
    if (rc) break;
    uint32_t *oi = c->ids + q * (uint64_t)k;
    float *od = c->dists + q * (uint64_t)k;
    rc = dvso_combine_results(fo, pids, pd, pc, k, k, oi, od, c->count + q);
    if (rc) break;
    c->visited[q] = vis;
    if (c->vectors) { /* :329-333 attach hit vectors via the locator */
      float *ov = c->vectors + q * (uint64_t)k * (uint64_t)dim;
      for (uint32_t h = 0; h < c->count[q]; ++h) {
        const dvso_graph *g = &c->idx->graphs[c->loc_cl[oi[h]]];
        memcpy(ov + (size_t)h * dim, g->vectors + (uint64_t)c->loc_lo[oi[h]] * dim,
               sizeof(float) * (size_t)dim);
      }
    }
  }
  free(pids); free(pd); free(pc);
  return rc;
}

int dvso_run_pipeline(const dvso_index *idx, const float *queries, uint64_t nq,
                      const dvso_params *p, int fanout, int ranks, int batch_index,
                      int nthreads, uint32_t *out_ids, float *out_dists,
                      uint32_t *out_count, float *out_vectors, uint64_t *visited_total) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (idx->clusters < 1 || !idx->graphs) return fail(DVSO_EINVAL, "BuiltIndex: index is not built");
  if (fanout < 1 || fanout > idx->clusters)
    return fail(DVSO_EINVAL, "run_pipeline: fanout %d out of range for %d clusters", fanout,
                idx->clusters);
  if (idx->ranks != ranks)
    return fail(DVSO_EINVAL, "run_pipeline: placement built for %d ranks, topology has %d",
                idx->ranks, ranks);
  if (batch_index < 0) return fail(DVSO_EINVAL, "origin_rank_for_batch: negative batch index");
  if (nq < 2) return fail(DVSO_EINVAL, "run_pipeline: two_microbatch mode needs >= 2 queries");
  /* dense locator, :275-288 */
  uint64_t total = 0;
  for (int c = 0; c < idx->clusters; ++c) total += idx->graphs[c].n;
  uint32_t *loc_cl = malloc(sizeof(uint32_t) * (total ? total : 1));
  uint32_t *loc_lo = malloc(sizeof(uint32_t) * (total ? total : 1));
  memset(loc_cl, 0xFF, sizeof(uint32_t) * total);
  for (int c = 0; c < idx->clusters; ++c) {
    const dvso_graph *g = &idx->graphs[c];
    for (uint64_t l = 0; l < g->n; ++l) {
      const uint32_t gid = g->global_ids[l];
      if (gid >= total || loc_cl[gid] != UINT32_MAX) {
        free(loc_cl); free(loc_lo);
        return fail(DVSO_EINTERNAL, "run_pipeline: partitions do not form a dense id cover");
      }
      loc_cl[gid] = (uint32_t)c;
      loc_lo[gid] = (uint32_t)l;
    }
  }
  uint32_t *assign = malloc(sizeof(uint32_t) * nq * (uint64_t)fanout);
  rc = dvso_assign_top_c(idx->centroids, idx->clusters, idx->dim, queries, nq, fanout, assign);
  uint64_t *vis = calloc(nq, sizeof(uint64_t));
  if (!rc) {
    pipe_ctx c = {idx, queries, p, fanout, assign, loc_cl, loc_lo, out_ids, out_dists, out_count,
                  out_vectors, vis};
    rc = parallel_for(nq, nthreads, pipe_rows, &c);
  }
  uint64_t vt = 0;
  for (uint64_t q = 0; q < nq; ++q) vt += vis[q];
  *visited_total = vt;
  free(vis); free(assign); free(loc_cl); free(loc_lo);
  return rc;
}

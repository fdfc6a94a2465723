/* TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.
 *
 * A multi-threaded C restatement of the reference's scalar query oracle,
 * run_query_oracle (proj/src/cli.cpp:140-225): scalar filters on the fact and
 * dimension tables (cli.cpp:149-185), the hash star join over unique dimension
 * keys (oracle::star_join, proj/src/oracle.cpp; inner join, a fact row
 * survives only if every link finds its key), then SUM(measure) per group
 * tuple (oracle::hash_aggregate), groups ascending.  It exists so that the
 * full-size SSB configurations (SF=100: 600M lineorder rows) can be checked
 * against an independent CPU computation in seconds: the reference itself
 * needs ~7-11 min and ~130 GB per SF=100 query.
 *
 * Division of labour with oracle/fast_query.py (also test infrastructure):
 * Python composes, per link, the dimension side of the hash join with the
 * dimension filters into one table indexed by key - base:
 *     tab[key - base] = contribution of that dim row to the group code, or -1
 *                       when the key is absent or the row fails a dim filter;
 * the group code is a mixed radix over the sorted distinct values of the
 * group columns (first group column most significant), so ascending code =
 * ascending tuple, the reference's output order.  This file streams the fact
 * rows: fact filters as closed integer intervals, one lookup per link, and
 * exact int64 (count, sum) per group code.  Sums of integer measures are
 * exact, so the order of accumulation is irrelevant (the reference sums the
 * same integers in fp64, exact below 2^53).
 *
 * Pinned by tests/test_oracle_fast.py against the reference's own goldens
 * (all 12 SSB sf=1 queries) and the numpy restatement.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const void* p;
  int32_t width; /* 4 = int32, 8 = int64 */
} oc_col;

static inline int64_t get(const oc_col* c, int64_t i) {
  return c->width == 4 ? (int64_t)((const int32_t*)c->p)[i] : ((const int64_t*)c->p)[i];
}

typedef struct {
  int64_t r0, r1;
  int32_t n_links;
  const oc_col* fks;
  const int64_t* base;
  const int64_t* span;
  const int64_t* const* tab;
  int32_t n_ff;
  const oc_col* ff;
  const int64_t* lo;
  const int64_t* hi;
  const oc_col* measure;
  int64_t G;
  int64_t* cnt;
  int64_t* sum;
} job;

static void* run(void* arg) {
  job* j = (job*)arg;
  for (int64_t r = j->r0; r < j->r1; ++r) {
    int ok = 1;
    for (int f = 0; f < j->n_ff && ok; ++f) {
      const int64_t v = get(&j->ff[f], r);
      ok = v >= j->lo[f] && v <= j->hi[f];
    }
    if (!ok) continue;
    int64_t code = 0;
    for (int l = 0; l < j->n_links; ++l) {
      const int64_t k = get(&j->fks[l], r) - j->base[l];
      if (k < 0 || k >= j->span[l]) { ok = 0; break; }
      const int64_t c = j->tab[l][k];
      if (c < 0) { ok = 0; break; }
      code += c;
    }
    if (!ok) continue;
    j->cnt[code] += 1;
    j->sum[code] += j->measure->p ? get(j->measure, r) : 0;
  }
  return NULL;
}

/* Rows [row0, row0 + n) of the fact table.  cnt / sum (G each) are overwritten.
 * Returns 0, or -1 when a worker could not be allocated / started. */
int oc_star_query(int64_t row0, int64_t n, int32_t n_links, const oc_col* fks, const int64_t* base,
                  const int64_t* span, const int64_t* const* tab, int32_t n_ff, const oc_col* ff,
                  const int64_t* lo, const int64_t* hi, const oc_col* measure, int64_t G, int64_t* cnt,
                  int64_t* sum, int32_t threads) {
  if (threads < 1) threads = 1;
  if (n < (int64_t)threads * 65536) threads = (int32_t)(n / 65536 + 1);
  job* jobs = (job*)calloc((size_t)threads, sizeof(job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  int64_t* part = (int64_t*)calloc((size_t)threads * 2 * (size_t)G, sizeof(int64_t));
  if (!jobs || !tid || !part) { free(jobs); free(tid); free(part); return -1; }
  int started = 0, rc = 0;
  for (int t = 0; t < threads; ++t) {
    job* j = &jobs[t];
    j->r0 = row0 + n * t / threads;
    j->r1 = row0 + n * (t + 1) / threads;
    j->n_links = n_links; j->fks = fks; j->base = base; j->span = span; j->tab = tab;
    j->n_ff = n_ff; j->ff = ff; j->lo = lo; j->hi = hi; j->measure = measure; j->G = G;
    j->cnt = part + (size_t)t * 2 * (size_t)G;
    j->sum = j->cnt + G;
    if (pthread_create(&tid[t], NULL, run, j) != 0) { rc = -1; break; }
    ++started;
  }
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  memset(cnt, 0, (size_t)G * sizeof(int64_t));
  memset(sum, 0, (size_t)G * sizeof(int64_t));
  for (int t = 0; t < started; ++t)
    for (int64_t g = 0; g < G; ++g) {
      cnt[g] += jobs[t].cnt[g];
      sum[g] += jobs[t].sum[g];
    }
  free(jobs); free(tid); free(part);
  return rc;
}

/*
 * ace_oracle.c — CPU restatement of the reference ACE hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_1706_06664_b200 + libace_dev.so) never
 * links or calls it.
 *
 * It restates, in plain C, the algorithm of the reference C++ sources under
 * /root/reference/proj (cited file:line per function).  It is pinned against
 * the compiled reference itself (oracle/_ref/libaceref.so, built by
 * oracle/Makefile from the reference sources) by tests/test_cpu_oracle.py and
 * against the committed golden digests in tests/golden/.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).  The
 * reference is compiled without -march, so its dot product is mul-then-add in
 * binary64 with no FMA; -ffp-contract=off keeps this restatement identical.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng (proj/include/ace/rng.hpp) ------------------------------------ */

/* rng.hpp:10-16 */
static uint64_t ora_splitmix64(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:19-22 */
uint64_t ora_mix_seed(uint64_t seed, uint64_t index) {
  uint64_t st = seed ^ (0x9e3779b97f4a7c15ULL * (index + 1));
  return ora_splitmix64(&st);
}

/* rng.hpp:25-27 — uniform in (0, 1] */
static double ora_unit(uint64_t bits) {
  return (double)((bits >> 11) + 1) * 0x1.0p-53;
}

/* rng.hpp:36-58 — Box-Muller, cosine first, sine cached */
typedef struct {
  uint64_t state;
  double spare;
  int has_spare;
} ora_normals;

static double ora_normal_next(ora_normals* s) {
  if (s->has_spare) {
    s->has_spare = 0;
    return s->spare;
  }
  const double u1 = ora_unit(ora_splitmix64(&s->state));
  const double u2 = ora_unit(ora_splitmix64(&s->state));
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.141592653589793238462643383279502884 * u2;
  s->spare = r * sin(a);
  s->has_spare = 1;
  return r * cos(a);
}

/* ---- srp (proj/src/srp.cpp) -------------------------------------------- */

/* srp.cpp:17-20 direction_seed, srp.cpp:36-48 the cached W fill:
 * row (t*K + b) of the (K*L) x d matrix holds d draws of a fresh stream. */
void ora_directions(uint64_t seed, uint64_t dim, uint32_t k_bits,
                    uint32_t tables, double* w) {
  for (uint64_t t = 0; t < tables; ++t)
    for (uint64_t b = 0; b < k_bits; ++b) {
      ora_normals s = {ora_mix_seed(seed, t * k_bits + b), 0.0, 0};
      double* row = w + (t * k_bits + b) * dim;
      for (uint64_t i = 0; i < dim; ++i) row[i] = ora_normal_next(&s);
    }
}

/* srp.cpp:78-91 — sequential binary64 fold, mul then add, from +0.0 */
double ora_project(const double* wrow, const double* x, uint64_t dim) {
  double dot = 0.0;
  for (uint64_t i = 0; i < dim; ++i) dot += wrow[i] * x[i];
  return dot;
}

/* srp.cpp:93-113 — bit = (p >= 0); bit 0 is the most significant */
uint32_t ora_bucket(const double* w, uint64_t dim, uint32_t k_bits,
                    uint64_t table, const double* x) {
  uint32_t idx = 0;
  for (uint64_t b = 0; b < k_bits; ++b) {
    const double p = ora_project(w + (table * k_bits + b) * dim, x, dim);
    idx = (idx << 1) | (p >= 0.0 ? 1u : 0u);
  }
  return idx;
}

/* The BASELINE.json near-tie predicate |<x,w>| < eps |x| |w| (strict, so an
 * all-zero row is not a near tie).  Not a reference function. */
int ora_near_tie(const double* wrow, const double* x, uint64_t dim, double eps) {
  double nx = 0.0, nw = 0.0;
  for (uint64_t i = 0; i < dim; ++i) {
    nx += x[i] * x[i];
    nw += wrow[i] * wrow[i];
  }
  const double p = ora_project(wrow, x, dim);
  return fabs(p) < eps * (sqrt(nx) * sqrt(nw));
}

/* Bucket ids of rows X (n x dim, fp32 or fp64) for every table, table-major
 * ids[t * n + i], on `threads` pthreads (SrpFamily::bucket is const and
 * thread-safe, srp.hpp:24-25).  Also counts near-ties below rel_eps. */
typedef struct {
  const double* w;
  const void* x;
  int x_is_f64;
  uint64_t dim, n, row0, row1;
  uint32_t k_bits, tables;
  uint32_t* ids;
  double rel_eps;
  uint64_t near;
} ora_bucket_job;

static void* ora_bucket_worker(void* arg) {
  ora_bucket_job* j = (ora_bucket_job*)arg;
  double* xd = (double*)malloc(sizeof(double) * j->dim);
  for (uint64_t i = j->row0; i < j->row1; ++i) {
    if (j->x_is_f64)
      memcpy(xd, (const double*)j->x + i * j->dim, sizeof(double) * j->dim);
    else
      for (uint64_t c = 0; c < j->dim; ++c)
        xd[c] = (double)((const float*)j->x)[i * j->dim + c];
    for (uint64_t t = 0; t < j->tables; ++t) {
      j->ids[t * j->n + i] = ora_bucket(j->w, j->dim, j->k_bits, t, xd);
      if (j->rel_eps > 0)
        for (uint64_t b = 0; b < j->k_bits; ++b)
          j->near += ora_near_tie(j->w + (t * j->k_bits + b) * j->dim, xd, j->dim,
                                  j->rel_eps);
    }
  }
  free(xd);
  return NULL;
}

/* The same ids, faster: ORA_RB rows at a time, each (row, direction) still
 * the sequential left fold of srp.cpp:84 (one independent accumulator per row,
 * mul then add, never fused: -ffp-contract=off), so the bits are those of
 * ora_bucket; the rows only run side by side as vector lanes.  Used to pin
 * the full-size configurations (tests/golden/make_golden_full.py), where the
 * scalar fold would take hours. */
#define ORA_RB 64
typedef double ora_v4 __attribute__((vector_size(64)));

__attribute__((target_clones("avx512f", "avx2", "default")))
static void ora_block_project(const double* w, uint64_t dim, uint64_t ndir,
                              const double* xt, double* p) {
  for (uint64_t r = 0; r < ndir; ++r) {
    const double* wr = w + r * dim;
    ora_v4 a[ORA_RB / 8];
    for (int v = 0; v < ORA_RB / 8; ++v) a[v] = (ora_v4){0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (uint64_t i = 0; i < dim; ++i) {
      const double s = wr[i];
      const ora_v4 wb = {s, s, s, s, s, s, s, s};
      const ora_v4* xv = (const ora_v4*)(xt + i * ORA_RB);
      for (int v = 0; v < ORA_RB / 8; ++v) {
        const ora_v4 prod = wb * xv[v];
        a[v] = a[v] + prod;
      }
    }
    ora_v4* pv = (ora_v4*)(p + r * ORA_RB);
    for (int v = 0; v < ORA_RB / 8; ++v) pv[v] = a[v];
  }
}

static void* ora_bucket_worker_fast(void* arg) {
  ora_bucket_job* j = (ora_bucket_job*)arg;
  const uint64_t ndir = (uint64_t)j->k_bits * j->tables;
  double* xt = (double*)aligned_alloc(64, sizeof(double) * j->dim * ORA_RB);
  double* p = (double*)aligned_alloc(64, sizeof(double) * j->k_bits * ORA_RB);
  double* wn = NULL;
  double xn[ORA_RB];
  if (j->rel_eps > 0) { /* |w| per direction, as ora_near_tie computes it */
    wn = (double*)malloc(sizeof(double) * ndir);
    for (uint64_t r = 0; r < ndir; ++r) {
      double s = 0.0;
      for (uint64_t i = 0; i < j->dim; ++i) s += j->w[r * j->dim + i] * j->w[r * j->dim + i];
      wn[r] = sqrt(s);
    }
  }
  for (uint64_t i0 = j->row0; i0 < j->row1; i0 += ORA_RB) {
    const uint64_t m = j->row1 - i0 < ORA_RB ? j->row1 - i0 : ORA_RB;
    for (uint64_t k = 0; k < ORA_RB; ++k) {
      const uint64_t row = i0 + (k < m ? k : 0);
      for (uint64_t c = 0; c < j->dim; ++c)
        xt[c * ORA_RB + k] = j->x_is_f64 ? ((const double*)j->x)[row * j->dim + c]
                                         : (double)((const float*)j->x)[row * j->dim + c];
    }
    if (wn)
      for (uint64_t k = 0; k < m; ++k) {
        double s = 0.0;
        for (uint64_t c = 0; c < j->dim; ++c) s += xt[c * ORA_RB + k] * xt[c * ORA_RB + k];
        xn[k] = sqrt(s);
      }
    for (uint64_t t = 0; t < j->tables; ++t) {
      ora_block_project(j->w + t * j->k_bits * j->dim, j->dim, j->k_bits, xt, p);
      for (uint64_t k = 0; k < m; ++k) {
        uint32_t idx = 0;
        for (uint64_t b = 0; b < j->k_bits; ++b) {
          const uint64_t r = t * j->k_bits + b;
          const double v = p[b * ORA_RB + k];
          idx = (idx << 1) | (v >= 0.0 ? 1u : 0u);
          if (wn) j->near += fabs(v) < j->rel_eps * (xn[k] * wn[r]);
        }
        j->ids[t * j->n + i0 + k] = idx;
      }
    }
  }
  free(xt);
  free(p);
  free(wn);
  return NULL;
}

static uint64_t ora_buckets_run(void* (*worker)(void*), const double* w, uint64_t dim,
                                uint32_t k_bits, uint32_t tables, const void* x,
                                int x_is_f64, uint64_t n, uint32_t* ids, int threads,
                                double rel_eps);

uint64_t ora_buckets(const double* w, uint64_t dim, uint32_t k_bits,
                     uint32_t tables, const void* x, int x_is_f64, uint64_t n,
                     uint32_t* ids, int threads, double rel_eps) {
  return ora_buckets_run(ora_bucket_worker, w, dim, k_bits, tables, x, x_is_f64, n, ids,
                         threads, rel_eps);
}

uint64_t ora_buckets_fast(const double* w, uint64_t dim, uint32_t k_bits,
                          uint32_t tables, const void* x, int x_is_f64, uint64_t n,
                          uint32_t* ids, int threads, double rel_eps) {
  return ora_buckets_run(ora_bucket_worker_fast, w, dim, k_bits, tables, x, x_is_f64, n,
                         ids, threads, rel_eps);
}

static uint64_t ora_buckets_run(void* (*worker)(void*), const double* w, uint64_t dim,
                                uint32_t k_bits, uint32_t tables, const void* x,
                                int x_is_f64, uint64_t n, uint32_t* ids, int threads,
                                double rel_eps) {
  if (threads < 1) threads = 1;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  ora_bucket_job* jobs = (ora_bucket_job*)malloc(sizeof(ora_bucket_job) * threads);
  const uint64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    uint64_t a = t * chunk, b = a + chunk;
    if (a > n) a = n;
    if (b > n) b = n;
    ora_bucket_job j = {w, x, x_is_f64, dim, n, a, b, k_bits, tables, ids, rel_eps, 0};
    jobs[t] = j;
    pthread_create(&tid[t], NULL, worker, &jobs[t]);
  }
  uint64_t near = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    near += jobs[t].near;
  }
  free(tid);
  free(jobs);
  return near;
}

/* ---- sketch (proj/src/sketch.cpp) -------------------------------------- */

/* State of an AceSketch (sketch.hpp:77-83): table-major counters
 * (idx = j * 2^K + bucket, sketch.cpp:59), width 16 or 32, n, mean, sticky
 * saturation. */
typedef struct {
  uint32_t k_bits, tables, width;
  uint64_t buckets;
  uint32_t* c32;
  uint16_t* c16;
  uint64_t n;
  double mean;
  int saturated;
} ora_sketch;

static uint64_t ora_get(const ora_sketch* s, uint64_t idx) {
  return s->width == 16 ? s->c16[idx] : s->c32[idx];
}
static void ora_set(ora_sketch* s, uint64_t idx, uint64_t v) {
  if (s->width == 16)
    s->c16[idx] = (uint16_t)v;
  else
    s->c32[idx] = (uint32_t)v;
}

ora_sketch* ora_sketch_new(uint32_t k_bits, uint32_t tables, uint32_t width) {
  ora_sketch* s = (ora_sketch*)calloc(1, sizeof(ora_sketch));
  s->k_bits = k_bits;
  s->tables = tables;
  s->width = width;
  s->buckets = (uint64_t)1 << k_bits;
  if (width == 16)
    s->c16 = (uint16_t*)calloc(s->buckets * tables, sizeof(uint16_t));
  else
    s->c32 = (uint32_t*)calloc(s->buckets * tables, sizeof(uint32_t));
  return s;
}

void ora_sketch_free(ora_sketch* s) {
  if (!s) return;
  free(s->c16);
  free(s->c32);
  free(s);
}

uint64_t ora_sketch_size(const ora_sketch* s) { return s->n; }
double ora_sketch_mean(const ora_sketch* s) { return s->mean; }
int ora_sketch_saturated(const ora_sketch* s) { return s->saturated; }

void ora_sketch_counters(const ora_sketch* s, uint64_t* out) {
  for (uint64_t i = 0; i < s->buckets * s->tables; ++i) out[i] = ora_get(s, i);
}

/* sketch.cpp:50-72 — insert one point given its L bucket ids (ids[t*stride]):
 * pre-increment numerator, sticky saturation, mean recurrence. */
static void ora_insert_ids(ora_sketch* s, const uint32_t* ids, uint64_t stride) {
  const uint64_t cmax = s->width == 16 ? 0xffffu : 0xffffffffu;
  double numerator = 0.0;
  for (uint64_t j = 0; j < s->tables; ++j) {
    const uint64_t idx = j * s->buckets + ids[j * stride];
    const uint64_t pre = ora_get(s, idx);
    numerator += 2.0 * (double)pre + 1.0;
    if (pre >= cmax)
      s->saturated = 1;
    else
      ora_set(s, idx, pre + 1);
  }
  const double n = (double)s->n;
  s->mean = (n * s->mean + numerator / s->tables) / (n + 1.0);
  ++s->n;
}

/* Insert rows in index order (estimators.cpp:79-92 build_sketch loop). */
void ora_insert_batch(ora_sketch* s, const uint32_t* ids, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) ora_insert_ids(s, ids + i, n);
}

/* sketch.cpp:74-106 — all-or-nothing delete. Returns 0, or -1 when some
 * target counter is zero (InconsistentDelete, sketch unchanged). */
int ora_remove_ids(ora_sketch* s, const uint32_t* ids, uint64_t stride) {
  for (uint64_t j = 0; j < s->tables; ++j)
    if (ora_get(s, j * s->buckets + ids[j * stride]) == 0) return -1;
  double numerator = 0.0;
  for (uint64_t j = 0; j < s->tables; ++j) {
    const uint64_t idx = j * s->buckets + ids[j * stride];
    const uint64_t pre = ora_get(s, idx);
    numerator += 2.0 * (double)pre - 1.0;
    ora_set(s, idx, pre - 1);
  }
  --s->n;
  if (s->n == 0) {
    s->mean = 0.0;
  } else {
    const double n = (double)(s->n + 1);
    s->mean = (n * s->mean - numerator / s->tables) / (n - 1.0);
  }
  return 0;
}

/* sketch.cpp:108-116 — S = sum of L counters (exact in f64), score = S / L. */
void ora_score_batch(const ora_sketch* s, const uint32_t* ids, uint64_t n,
                     double* scores, uint64_t* sums) {
  for (uint64_t i = 0; i < n; ++i) {
    double sum = 0.0;
    uint64_t isum = 0;
    for (uint64_t j = 0; j < s->tables; ++j) {
      const uint64_t c = ora_get(s, j * s->buckets + ids[j * n + i]);
      sum += (double)c;
      isum += c;
    }
    if (scores) scores[i] = sum / s->tables;
    if (sums) sums[i] = isum;
  }
}

/* ---- detect (proj/src/detect.cpp) -------------------------------------- */

/* detect.cpp:44-68 — sequential mean, population stddev, thr = mean - sd,
 * flag = score < thr (strict).  flags: n bytes.  Returns #reported. */
uint64_t ora_detect_batch_from_scores(const double* scores, uint64_t n,
                                      double* mean_out, double* sd_out,
                                      double* thr_out, uint8_t* flags) {
  double sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) sum += scores[i];
  const double mean = sum / (double)n;
  double sq = 0.0;
  for (uint64_t i = 0; i < n; ++i) sq += (scores[i] - mean) * (scores[i] - mean);
  const double sd = sqrt(sq / (double)n);
  const double thr = mean - sd;
  uint64_t reported = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int f = scores[i] < thr;
    if (flags) flags[i] = (uint8_t)f;
    reported += (uint64_t)f;
  }
  *mean_out = mean;
  *sd_out = sd;
  *thr_out = thr;
  return reported;
}

/* Streaming batch in the BASELINE config-5 order: every
 * row of the batch is scored against the counts at batch start and flagged
 * with detect_stream's rule score <= mean - alpha (detect.cpp:76-84; an empty
 * sketch, where detect_stream throws, flags nothing), then the rows are
 * inserted in order (ace_cli.cpp:177-183 with the insert deferred to the batch
 * end).  ids table-major with stride n. */
uint64_t ora_stream_batch(ora_sketch* s, const uint32_t* ids, uint64_t n,
                          double alpha, double* scores, uint8_t* flags) {
  double* sc = scores ? scores : (double*)malloc(sizeof(double) * n);
  ora_score_batch(s, ids, n, sc, NULL);
  const int live = s->n > 0;
  const double cut = s->mean - alpha;
  uint64_t reported = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int f = live && sc[i] <= cut;
    if (flags) flags[i] = (uint8_t)f;
    reported += (uint64_t)f;
  }
  ora_insert_batch(s, ids, n);
  if (!scores) free(sc);
  return reported;
}

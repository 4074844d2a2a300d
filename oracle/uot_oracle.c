/*
 * uot_oracle.c — plain-C restatement of the reference's fused Sinkhorn-UOT path.
 *
 * TEST INFRASTRUCTURE ONLY (see uot_oracle.h). Citations are relative to
 * /root/reference/proj/core. Parity pinned against oracle/_ref (the reference
 * compiled from its own sources) and tests/golden/.
 */
#define _GNU_SOURCE
#include "uot_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG --- */

/* rng.hpp:14-20 — add the golden gamma, then the two xor-shift-multiply rounds. */
uint64_t orc_splitmix64_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.hpp:24 — top 53 bits + 1, scaled by 2^-53: uniform on (0, 1]. */
double orc_next_unit(uint64_t* state) {
  return (double)((orc_splitmix64_next(state) >> 11) + 1) * 0x1p-53;
}

/* Draw k of the stream seeded with `seed` (counter form of rng.hpp:14-20). */
static double unit_at(uint64_t seed, uint64_t k) {
  uint64_t s = seed + k * 0x9E3779B97F4A7C15ULL;
  return orc_next_unit(&s);
}

typedef struct {
  uint64_t seed, begin, end;
  void* dst;
  int is_f32;
} gen_job;

static void* gen_worker(void* p) {
  gen_job* j = (gen_job*)p;
  if (j->is_f32) {
    float* a = (float*)j->dst;
    for (uint64_t k = j->begin; k < j->end; ++k) a[k] = (float)unit_at(j->seed, k);
  } else {
    double* a = (double*)j->dst;
    for (uint64_t k = j->begin; k < j->end; ++k) a[k] = unit_at(j->seed, k);
  }
  return NULL;
}

/* problem_io.hpp:17-31: matrix first (row-major, cast to T), then rpd, then cpd. */
static int gen_problem(uint64_t seed, size_t m, size_t n, void* a, int is_f32, double* rpd,
                       double* cpd, int threads) {
  if (m < 1 || n < 1) return ORC_INVALID_PARAMETER;
  const uint64_t mn = (uint64_t)m * n;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > mn) threads = 1;
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  gen_job* jobs = (gen_job*)calloc((size_t)threads, sizeof(gen_job));
  for (int t = 0; t < threads; ++t) {
    jobs[t].seed = seed;
    jobs[t].begin = mn * (uint64_t)t / (uint64_t)threads;
    jobs[t].end = mn * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].dst = a;
    jobs[t].is_f32 = is_f32;
    if (t > 0) pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
  }
  gen_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  for (size_t i = 0; i < m; ++i) rpd[i] = unit_at(seed, mn + i);
  for (size_t j = 0; j < n; ++j) cpd[j] = unit_at(seed, mn + m + j);
  return ORC_OK;
}

int orc_gen_problem_f32(uint64_t seed, size_t m, size_t n, float* a, double* rpd, double* cpd,
                        int threads) {
  return gen_problem(seed, m, n, a, 1, rpd, cpd, threads);
}
int orc_gen_problem_f64(uint64_t seed, size_t m, size_t n, double* a, double* rpd, double* cpd,
                        int threads) {
  return gen_problem(seed, m, n, a, 0, rpd, cpd, threads);
}

/* ------------------------------------------------------------ scaling --- */

/* scaling.cpp:9-13 */
int orc_compute_fi(double er, double ep, double* fi) {
  if (!(er > 0.0) || !isfinite(er)) return ORC_INVALID_PARAMETER;
  if (!(ep >= 0.0) || !isfinite(ep)) return ORC_INVALID_PARAMETER;
  *fi = er / (er + ep);
  return ORC_OK;
}

/* scaling.cpp:15-22: (target/sum)^fi, sum must be > 0, result positive finite. */
int orc_rescale_factor(double target, double sum, double fi, double* out) {
  if (!(sum > 0.0)) return ORC_DEGENERATE_SUM;
  const double f = pow(target / sum, fi);
  if (!(f > 0.0) || !isfinite(f)) return ORC_DEGENERATE_SUM;
  *out = f;
  return ORC_OK;
}

/* scaling.cpp:24-29: max over alpha then beta of |f - 1|. */
double orc_convergence_error(const double* alpha, size_t m, const double* beta, size_t n) {
  double e = 0.0;
  for (size_t i = 0; i < m; ++i) {
    const double d = fabs(alpha[i] - 1.0);
    if (d > e) e = d;
  }
  for (size_t j = 0; j < n; ++j) {
    const double d = fabs(beta[j] - 1.0);
    if (d > e) e = d;
  }
  return e;
}

/* --------------------------------------------------------------- plan --- */

/* plan.cpp:11-21: sizes differ by at most one; the first rows%k blocks get +1. */
void orc_balanced_blocks(size_t k, size_t rows, size_t* bounds) {
  const size_t base = rows / k, rem = rows % k;
  bounds[0] = 0;
  for (size_t w = 0; w < k; ++w) bounds[w + 1] = bounds[w] + base + (w < rem ? 1 : 0);
}

/* plan.cpp:35-44 */
int orc_rank_partition(size_t ranks, size_t rows, size_t* bounds) {
  if (ranks < 1 || ranks > rows) return ORC_PARTITION_ERROR;
  orc_balanced_blocks(ranks, rows, bounds);
  return ORC_OK;
}

/* --------------------------------------------------- typed sweep bodies --- */

#define DEFINE_TYPED(T, SUF)                                                                    \
  /* fused.hpp:96-110: per-block partials, added into the total in block order. */             \
  void orc_init_col_sums_##SUF(const T* a, size_t m, size_t n, size_t nblocks, double* cs) {   \
    size_t* bounds = (size_t*)malloc((nblocks + 1) * sizeof(size_t));                           \
    double* part = (double*)malloc(n * sizeof(double));                                         \
    orc_balanced_blocks(nblocks, m, bounds);                                                    \
    for (size_t j = 0; j < n; ++j) cs[j] = 0.0;                                                 \
    for (size_t b = 0; b < nblocks; ++b) {                                                      \
      for (size_t j = 0; j < n; ++j) part[j] = 0.0;                                             \
      for (size_t i = bounds[b]; i < bounds[b + 1]; ++i) {                                      \
        const T* row = a + i * n;                                                               \
        for (size_t j = 0; j < n; ++j) part[j] += (double)row[j];                               \
      }                                                                                         \
      for (size_t j = 0; j < n; ++j) cs[j] += part[j];                                          \
    }                                                                                           \
    free(part);                                                                                 \
    free(bounds);                                                                               \
  }                                                                                             \
                                                                                                \
  /* fused.hpp:119-144: sweep 1 scales by beta and sums the stored values; the row  */         \
  /* factor follows; sweep 2 scales by alpha and accumulates next column sums.       */        \
  int orc_fused_row_pass_##SUF(T* row, size_t n, const double* beta, double target, double fi, \
                               double* next_cols, double* alpha) {                             \
    double s = 0.0;                                                                             \
    for (size_t j = 0; j < n; ++j) {                                                            \
      row[j] = (T)((double)row[j] * beta[j]);                                                   \
      s += (double)row[j];                                                                      \
    }                                                                                           \
    double al;                                                                                  \
    const int st = orc_rescale_factor(target, s, fi, &al);                                      \
    if (st != ORC_OK) return st;                                                                \
    for (size_t j = 0; j < n; ++j) {                                                            \
      row[j] = (T)((double)row[j] * al);                                                        \
      next_cols[j] += (double)row[j];                                                           \
    }                                                                                           \
    *alpha = al;                                                                                \
    return ORC_OK;                                                                              \
  }

DEFINE_TYPED(float, f32)
DEFINE_TYPED(double, f64)

/* fused.hpp:146-157 */
int orc_beta_from_state(const double* col_sums, const double* cpd, size_t n, double fi,
                        double* beta) {
  for (size_t j = 0; j < n; ++j) {
    const int st = orc_rescale_factor(cpd[j], col_sums[j], fi, &beta[j]);
    if (st != ORC_OK) return st;
  }
  return ORC_OK;
}

/* ------------------------------------------------- parallel iteration --- */

typedef struct {
  void* a;
  int is_f32;
  size_t n, begin, end;
  const double* beta;
  const double* rpd;
  double fi;
  double* partial; /* this worker's column partials (fused.hpp:220) */
  double* alpha;
  int status;
} row_job;

static void* row_worker(void* p) {
  row_job* j = (row_job*)p;
  j->status = ORC_OK;
  for (size_t i = j->begin; i < j->end && j->status == ORC_OK; ++i) {
    if (j->is_f32)
      j->status = orc_fused_row_pass_f32((float*)j->a + i * j->n, j->n, j->beta, j->rpd[i], j->fi,
                                         j->partial, &j->alpha[i]);
    else
      j->status = orc_fused_row_pass_f64((double*)j->a + i * j->n, j->n, j->beta, j->rpd[i],
                                         j->fi, j->partial, &j->alpha[i]);
  }
  return NULL;
}

/* fused.hpp:197-250 */
static int fused_iterate(void* a, int is_f32, size_t m, size_t n, double* col_sums,
                         const double* rpd, const double* cpd, double fi, size_t workers,
                         double* alpha, double* beta) {
  if (workers < 1 || m < 1 || n < 1) return ORC_INVALID_PARAMETER;
  int st = orc_beta_from_state(col_sums, cpd, n, fi, beta);
  if (st != ORC_OK) return st;
  size_t* bounds = (size_t*)malloc((workers + 1) * sizeof(size_t));
  orc_balanced_blocks(workers, m, bounds);
  double* partials = (double*)calloc(workers * n, sizeof(double)); /* fused.hpp:214 zero() */
  row_job* jobs = (row_job*)calloc(workers, sizeof(row_job));
  pthread_t* th = (pthread_t*)calloc(workers, sizeof(pthread_t));
  for (size_t w = 0; w < workers; ++w) {
    row_job j = {a, is_f32, n, bounds[w], bounds[w + 1], beta, rpd, fi, partials + w * n, alpha, 0};
    jobs[w] = j;
  }
  for (size_t w = 1; w < workers; ++w) pthread_create(&th[w], NULL, row_worker, &jobs[w]);
  row_worker(&jobs[0]);
  for (size_t w = 1; w < workers; ++w) pthread_join(th[w], NULL); /* fused.hpp:237 */
  for (size_t w = 0; w < workers; ++w)
    if (jobs[w].status != ORC_OK && st == ORC_OK) st = jobs[w].status; /* first worker error */
  if (st == ORC_OK) {
    /* fused.hpp:242-248: ascending worker order. */
    for (size_t j = 0; j < n; ++j) col_sums[j] = 0.0;
    for (size_t w = 0; w < workers; ++w)
      for (size_t j = 0; j < n; ++j) col_sums[j] += partials[w * n + j];
  }
  free(th);
  free(jobs);
  free(partials);
  free(bounds);
  return st;
}

int orc_fused_iterate_f32(float* a, size_t m, size_t n, double* col_sums, const double* rpd,
                          const double* cpd, double fi, size_t workers, double* alpha,
                          double* beta) {
  return fused_iterate(a, 1, m, n, col_sums, rpd, cpd, fi, workers, alpha, beta);
}
int orc_fused_iterate_f64(double* a, size_t m, size_t n, double* col_sums, const double* rpd,
                          const double* cpd, double fi, size_t workers, double* alpha,
                          double* beta) {
  return fused_iterate(a, 0, m, n, col_sums, rpd, cpd, fi, workers, alpha, beta);
}

/* problem.hpp:64-98 (the checks that apply to flat buffers). */
static int validate(const void* a, int is_f32, size_t m, size_t n, const double* rpd,
                    const double* cpd, double er, double ep) {
  if (m == 0 || n == 0) return ORC_INVALID_PARAMETER;
  for (size_t k = 0; k < m * n; ++k) {
    const double v = is_f32 ? (double)((const float*)a)[k] : ((const double*)a)[k];
    if (!(v > 0.0) || !isfinite(v)) return ORC_INVALID_PARAMETER;
  }
  for (size_t i = 0; i < m; ++i)
    if (!(rpd[i] > 0.0) || !isfinite(rpd[i])) return ORC_INVALID_PARAMETER;
  for (size_t j = 0; j < n; ++j)
    if (!(cpd[j] > 0.0) || !isfinite(cpd[j])) return ORC_INVALID_PARAMETER;
  if (!(er > 0.0) || !isfinite(er)) return ORC_INVALID_PARAMETER;
  if (!(ep >= 0.0) || !isfinite(ep)) return ORC_INVALID_PARAMETER;
  return ORC_OK;
}

int orc_validate_f32(const float* a, size_t m, size_t n, const double* rpd, const double* cpd,
                     double er, double ep) {
  return validate(a, 1, m, n, rpd, cpd, er, ep);
}

/* fused.hpp:259-285 */
static int fused_solve(void* a, int is_f32, size_t m, size_t n, const double* rpd,
                       const double* cpd, double er, double ep, double tol, size_t max_iter,
                       size_t workers, double* alpha, double* beta, double* col_sums_out,
                       size_t* iterations, double* final_error, int* converged) {
  int st = validate(a, is_f32, m, n, rpd, cpd, er, ep);
  if (st != ORC_OK) return st;
  if (!(tol > 0.0) || max_iter < 1 || workers < 1) return ORC_INVALID_PARAMETER;
  double fi;
  st = orc_compute_fi(er, ep, &fi);
  if (st != ORC_OK) return st;
  double* cs = (double*)malloc(n * sizeof(double));
  if (is_f32)
    orc_init_col_sums_f32((const float*)a, m, n, workers, cs);
  else
    orc_init_col_sums_f64((const double*)a, m, n, workers, cs);
  *iterations = 0;
  *final_error = 0.0;
  *converged = 0;
  for (size_t it = 1; it <= max_iter; ++it) {
    st = fused_iterate(a, is_f32, m, n, cs, rpd, cpd, fi, workers, alpha, beta);
    if (st != ORC_OK) break;
    *iterations = it;
    *final_error = orc_convergence_error(alpha, m, beta, n);
    if (*final_error <= tol) {
      *converged = 1;
      break;
    }
  }
  if (col_sums_out) memcpy(col_sums_out, cs, n * sizeof(double));
  free(cs);
  return st;
}

int orc_fused_solve_f32(float* a, size_t m, size_t n, const double* rpd, const double* cpd,
                        double er, double ep, double tol, size_t max_iter, size_t workers,
                        double* alpha, double* beta, double* col_sums, size_t* iterations,
                        double* final_error, int* converged) {
  return fused_solve(a, 1, m, n, rpd, cpd, er, ep, tol, max_iter, workers, alpha, beta, col_sums,
                     iterations, final_error, converged);
}
int orc_fused_solve_f64(double* a, size_t m, size_t n, const double* rpd, const double* cpd,
                        double er, double ep, double tol, size_t max_iter, size_t workers,
                        double* alpha, double* beta, double* col_sums, size_t* iterations,
                        double* final_error, int* converged) {
  return fused_solve(a, 0, m, n, rpd, cpd, er, ep, tol, max_iter, workers, alpha, beta, col_sums,
                     iterations, final_error, converged);
}

/* --------------------------------------------------------- distributed --- */

/* allreduce.cpp:6-15 */
void orc_allreduce_vectors(const double* const* parts, size_t ranks, size_t n, double* out) {
  for (size_t j = 0; j < n; ++j) out[j] = 0.0;
  for (size_t r = 0; r < ranks; ++r)
    for (size_t j = 0; j < n; ++j) out[j] += parts[r][j];
}

/* distributed.hpp:52-130: the rank loop is serial (deterministic round robin);
 * the rows stay in place in `a` since each rank's block is contiguous. */
int orc_distributed_solve_f32(float* a, size_t m, size_t n, const double* rpd, const double* cpd,
                              double er, double ep, double tol, size_t max_iter, size_t ranks,
                              double* alpha, double* beta, size_t* iterations,
                              double* final_error, int* converged, uint64_t* allreduce_calls,
                              uint64_t* doubles_reduced) {
  int st = validate(a, 1, m, n, rpd, cpd, er, ep);
  if (st != ORC_OK) return st;
  if (!(tol > 0.0) || max_iter < 1) return ORC_INVALID_PARAMETER;
  if (ranks < 1 || ranks > m) return ORC_PARTITION_ERROR;
  double fi;
  st = orc_compute_fi(er, ep, &fi);
  if (st != ORC_OK) return st;
  size_t* bounds = (size_t*)malloc((ranks + 1) * sizeof(size_t));
  orc_balanced_blocks(ranks, m, bounds);
  double* partials = (double*)calloc(ranks * n, sizeof(double));
  const double** views = (const double**)malloc(ranks * sizeof(double*));
  double* reduced = (double*)malloc(n * sizeof(double));
  /* distributed.hpp:73-79: each rank seeds with a plain pass over its block. */
  for (size_t r = 0; r < ranks; ++r) {
    orc_init_col_sums_f32(a + bounds[r] * n, bounds[r + 1] - bounds[r], n, 1, partials + r * n);
    views[r] = partials + r * n;
  }
  *allreduce_calls = 0;
  *doubles_reduced = 0;
  *iterations = 0;
  *converged = 0;
  for (size_t it = 1; it <= max_iter && st == ORC_OK; ++it) {
    orc_allreduce_vectors(views, ranks, n, reduced); /* distributed.hpp:88-94 */
    *allreduce_calls += 1;
    *doubles_reduced += n;
    st = orc_beta_from_state(reduced, cpd, n, fi, beta); /* replicated beta, 96-100 */
    if (st != ORC_OK) break;
    for (size_t r = 0; r < ranks && st == ORC_OK; ++r) { /* local passes, 103-110 */
      double* part = partials + r * n;
      for (size_t j = 0; j < n; ++j) part[j] = 0.0;
      for (size_t i = bounds[r]; i < bounds[r + 1] && st == ORC_OK; ++i)
        st = orc_fused_row_pass_f32(a + i * n, n, beta, rpd[i], fi, part, &alpha[i]);
    }
    if (st != ORC_OK) break;
    *iterations = it;
    *final_error = orc_convergence_error(alpha, m, beta, n);
    if (*final_error <= tol) {
      *converged = 1;
      break;
    }
  }
  free(reduced);
  free(views);
  free(partials);
  free(bounds);
  return st;
}

/*
 * cstress_oracle.c -- TEST INFRASTRUCTURE ONLY (see cstress_oracle.h).
 *
 * CPU restatement of the reference MSET2 path.  Citations are
 * path:line relative to /root/reference/proj.  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off, pthreads).  Never linked into the product.
 */
#define _GNU_SOURCE
#include "cstress_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static __thread char g_err[512];

const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

#define CM(M, ld, i, j) ((M)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* --------------------------------------------------------------------- rng */
/* rng.hpp:15-20 */
uint64_t or_splitmix64_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:26-33 */
uint64_t or_derive_seed(uint64_t parent, const uint64_t* coords, int ncoords) {
  uint64_t h = or_splitmix64_mix(parent);
  for (int i = 0; i < ncoords; ++i)
    h = or_splitmix64_mix(h ^ or_splitmix64_mix(coords[i]));
  return h;
}

/* rng.hpp:36-55: SplitMix64 sequence */
typedef struct {
  uint64_t state;
} sm64;

static uint64_t sm64_next(sm64* r) {
  r->state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = r->state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:59-83: Box-Muller over SplitMix64, cos first, sin as spare */
typedef struct {
  sm64 rng;
  int have_spare;
  double spare;
} gauss_stream;

static void gauss_init(gauss_stream* g, uint64_t seed) {
  g->rng.state = seed;
  g->have_spare = 0;
  g->spare = 0.0;
}

static double gauss_next(gauss_stream* g) {
  if (g->have_spare) {
    g->have_spare = 0;
    return g->spare;
  }
  const double u1 = ((double)(sm64_next(&g->rng) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = (double)(sm64_next(&g->rng) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * M_PI * u2;
  g->spare = r * sin(theta);
  g->have_spare = 1;
  return r * cos(theta);
}

void or_gaussian_fill(uint64_t seed, int64_t count, double* out) {
  gauss_stream g;
  gauss_init(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = gauss_next(&g);
}

/* tests/support/oracles.hpp:173-203 -- xorshift64* TestRng */
static double testrng_next01(uint64_t* s) {
  *s ^= *s >> 12;
  *s ^= *s << 25;
  *s ^= *s >> 27;
  return (double)((*s * 0x2545f4914f6cdd1dULL) >> 11) * 0x1.0p-53;
}

void or_testrng_matrix(uint64_t* state, int64_t rows, int64_t cols, double lo,
                       double hi, double* out) {
  if (*state == 0) *state = 1;
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r)
      CM(out, rows, r, c) = lo + (hi - lo) * testrng_next01(state);
}

int or_testrng_uniform_int(uint64_t* state, int lo, int hi) {
  if (*state == 0) *state = 1;
  return lo + (int)(testrng_next01(state) * (hi - lo + 1));
}

/* ----------------------------------------------------- small dense helpers */

static double* dalloc(size_t count) {
  double* p = (double*)malloc((count ? count : 1) * sizeof(double));
  return p;
}

/* Eigen LLT unblocked semantics (Cholesky.h llt_inplace): lower L with
 * A = L L^T; fails when a pivot x <= 0.  Column-major, in place on `L`. */
static int llt_lower(double* L, int64_t n) {
  /* Eigen::LLT order (the sums run j = 0..k-1), computed on a row-major copy
   * so that the inner sums walk contiguous memory: identical arithmetic,
   * without an 8n-byte stride per term (n = 4000 took an hour) */
  double* R = dalloc((size_t)n * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j; i < n; ++i) R[(size_t)i * (size_t)n + (size_t)j] = CM(L, n, i, j);
  int ok = 1;
  for (int64_t k = 0; k < n && ok; ++k) {
    double* rk = R + (size_t)k * (size_t)n;
    double x = rk[k];
    for (int64_t j = 0; j < k; ++j) x -= rk[j] * rk[j];
    if (!(x > 0.0)) {
      ok = 0;
      break;
    }
    x = sqrt(x);
    rk[k] = x;
    for (int64_t i = k + 1; i < n; ++i) {
      double* ri = R + (size_t)i * (size_t)n;
      double v = ri[k];
      for (int64_t j = 0; j < k; ++j) v -= ri[j] * rk[j];
      ri[k] = v / x;
    }
  }
  if (ok) {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) CM(L, n, i, j) = i >= j ? R[(size_t)i * (size_t)n + (size_t)j] : 0.0;
  }
  free(R);
  return ok;
}

static double frob_norm(const double* A, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n * n; ++i) s += A[i] * A[i];
  return sqrt(s);
}

/* Eigen isApprox(A^T, 1e-12): ||A - A^T|| <= 1e-12 * min(||A||, ||A^T||). */
static int is_symmetric_approx(const double* A, int64_t n, double prec) {
  double d = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const double v = CM(A, n, i, j) - CM(A, n, j, i);
      d += v * v;
    }
  return sqrt(d) <= prec * frob_norm(A, n);
}

/* ------------------------------------------------------------- fleishman */
/* signals.cpp:24-47 */
static void fleishman_residual(double b, double c, double d, double g1,
                               double g2, double f[3], double jac[3][3]) {
  const double var = b * b + 6.0 * b * d + 2.0 * c * c + 15.0 * d * d;
  const double skew = 2.0 * c * (b * b + 24.0 * b * d + 105.0 * d * d + 2.0);
  const double kurt_core =
      b * d + c * c * (1.0 + b * b + 28.0 * b * d) +
      d * d * (12.0 + 48.0 * b * d + 141.0 * c * c + 225.0 * d * d);
  f[0] = var - 1.0;
  f[1] = skew - g1;
  f[2] = 24.0 * kurt_core - g2;
  jac[0][0] = 2.0 * b + 6.0 * d;
  jac[0][1] = 4.0 * c;
  jac[0][2] = 6.0 * b + 30.0 * d;
  jac[1][0] = 2.0 * c * (2.0 * b + 24.0 * d);
  jac[1][1] = 2.0 * (b * b + 24.0 * b * d + 105.0 * d * d + 2.0);
  jac[1][2] = 2.0 * c * (24.0 * b + 210.0 * d);
  jac[2][0] = 24.0 * (d + c * c * (2.0 * b + 28.0 * d) + 48.0 * d * d * d);
  jac[2][1] = 24.0 * (2.0 * c * (1.0 + b * b + 28.0 * b * d) + 282.0 * c * d * d);
  jac[2][2] = 24.0 * (b + 28.0 * b * c * c +
                      2.0 * d * (12.0 + 48.0 * b * d + 141.0 * c * c + 225.0 * d * d) +
                      d * d * (48.0 * b + 450.0 * d));
}

/* 3x3 full-pivot LU solve (stands in for Eigen fullPivLu().solve,
 * signals.cpp:126); rank-deficient directions get a zero component. */
static void solve3_fullpiv(double a_in[3][3], const double b_in[3], double x[3]) {
  double a[3][3];
  double b[3];
  int rp[3] = {0, 1, 2}, cp[3] = {0, 1, 2};
  memcpy(a, a_in, sizeof a);
  memcpy(b, b_in, sizeof b);
  int rank = 3;
  for (int k = 0; k < 3; ++k) {
    int pi = k, pj = k;
    double best = -1.0;
    for (int i = k; i < 3; ++i)
      for (int j = k; j < 3; ++j)
        if (fabs(a[rp[i]][cp[j]]) > best) {
          best = fabs(a[rp[i]][cp[j]]);
          pi = i;
          pj = j;
        }
    if (best == 0.0) {
      rank = k;
      break;
    }
    int t = rp[k]; rp[k] = rp[pi]; rp[pi] = t;
    t = cp[k]; cp[k] = cp[pj]; cp[pj] = t;
    for (int i = k + 1; i < 3; ++i) {
      const double l = a[rp[i]][cp[k]] / a[rp[k]][cp[k]];
      for (int j = k; j < 3; ++j) a[rp[i]][cp[j]] -= l * a[rp[k]][cp[j]];
      b[rp[i]] -= l * b[rp[k]];
    }
  }
  double y[3] = {0.0, 0.0, 0.0};
  for (int k = rank - 1; k >= 0; --k) {
    double v = b[rp[k]];
    for (int j = k + 1; j < rank; ++j) v -= a[rp[k]][cp[j]] * y[j];
    y[k] = v / a[rp[k]][cp[k]];
  }
  for (int k = 0; k < 3; ++k) x[cp[k]] = y[k];
}

static double inf_norm3(const double f[3]) {
  double m = fabs(f[0]);
  if (fabs(f[1]) > m) m = fabs(f[1]);
  if (fabs(f[2]) > m) m = fabs(f[2]);
  return m;
}

static int finite3(const double v[3]) {
  return isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]);
}

/* signals.cpp:105-164 -- damped Newton, tol 1e-10, 200 iterations */
int or_solve_fleishman(double skewness, double kurtosis, double* abcd) {
  const double g1 = skewness;
  const double g2 = kurtosis - 3.0;
  double x[3] = {1.0, 0.0, 0.0};
  double f[3], jac[3][3];
  fleishman_residual(x[0], x[1], x[2], g1, g2, f, jac);
  const int kMaxIterations = 200;
  const double kTol = 1e-10;
  for (int it = 0; it < kMaxIterations; ++it) {
    if (inf_norm3(f) < kTol) break;
    double step[3];
    solve3_fullpiv(jac, f, step);
    if (!finite3(step)) break;
    const double f0 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
    double lambda = 1.0;
    double xn[3], fn[3], jn[3][3];
    int accepted = 0;
    while (lambda >= 1.0 / 1024.0) {
      for (int i = 0; i < 3; ++i) xn[i] = x[i] - lambda * step[i];
      fleishman_residual(xn[0], xn[1], xn[2], g1, g2, fn, jn);
      if (finite3(fn) && fn[0] * fn[0] + fn[1] * fn[1] + fn[2] * fn[2] < f0) {
        accepted = 1;
        break;
      }
      lambda *= 0.5;
    }
    if (!accepted) break;
    memcpy(x, xn, sizeof x);
    memcpy(f, fn, sizeof f);
    memcpy(jac, jn, sizeof jac);
  }
  if (inf_norm3(f) < kTol) {
    abcd[0] = -x[1];
    abcd[1] = x[0];
    abcd[2] = x[1];
    abcd[3] = x[2];
    return OR_OK;
  }
  return fail(OR_MOMENT_INFEASIBLE,
              "no real Fleishman solution for skewness %g, kurtosis %g",
              skewness, kurtosis);
}

/* signals.cpp:166-203 */
int or_nearest_psd_repair(const double* corr, int64_t n, double jitter_cap,
                          double* out, double* jitter_out) {
  if (!is_symmetric_approx(corr, n, 1e-12))
    return fail(OR_BAD_CORRELATION, "nearest_psd_repair: matrix is not symmetric");
  for (int64_t i = 0; i < n; ++i)
    if (fabs(CM(corr, n, i, i) - 1.0) > 1e-12)
      return fail(OR_BAD_CORRELATION, "nearest_psd_repair: diagonal must be 1");
  double* cand = dalloc((size_t)(n * n));
  double* work = dalloc((size_t)(n * n));
  double tried[16];
  int ntried = 0;
  tried[ntried++] = 0.0;
  double last_tried = 0.0;
  for (double j = 1e-12; j <= jitter_cap; j *= 100.0) {
    tried[ntried++] = j;
    last_tried = j;
  }
  if (jitter_cap > last_tried) tried[ntried++] = jitter_cap;
  for (int t = 0; t < ntried; ++t) {
    const double jitter = tried[t];
    memcpy(cand, corr, sizeof(double) * (size_t)(n * n));
    if (jitter > 0.0) {
      for (int64_t i = 0; i < n; ++i) CM(cand, n, i, i) += jitter;
      for (int64_t i = 0; i < n * n; ++i) cand[i] /= (1.0 + jitter);
      for (int64_t i = 0; i < n; ++i) CM(cand, n, i, i) = 1.0;
    }
    memcpy(work, cand, sizeof(double) * (size_t)(n * n));
    if (llt_lower(work, n)) {
      memcpy(out, cand, sizeof(double) * (size_t)(n * n));
      if (jitter_out) *jitter_out = jitter;
      free(cand);
      free(work);
      return OR_OK;
    }
  }
  free(cand);
  free(work);
  return fail(OR_BAD_CORRELATION,
              "correlation matrix not positive semidefinite within jitter cap %g",
              jitter_cap);
}

static int sym_min_eigenvalue(const double* A, int64_t n, double* out);

/* signals.cpp:67-103 -- SignalSpec::validate */
static int validate_spec(int64_t n, int64_t N, double phi, const double* corr,
                         const double* var, const double* skew,
                         const double* kurt) {
  if (n < 1) return fail(OR_CONFIG_ERROR, "SignalSpec: n_signals must be >= 1");
  if (N < 1) return fail(OR_CONFIG_ERROR, "SignalSpec: n_observations must be >= 1");
  if (!(fabs(phi) < 1.0))
    return fail(OR_CONFIG_ERROR, "SignalSpec: ar_coefficient must lie in (-1, 1)");
  if (!is_symmetric_approx(corr, n, 1e-12))
    return fail(OR_BAD_CORRELATION, "SignalSpec: cross_correlation is not symmetric");
  for (int64_t i = 0; i < n; ++i)
    if (fabs(CM(corr, n, i, i) - 1.0) > 1e-12)
      return fail(OR_BAD_CORRELATION, "SignalSpec: cross_correlation diagonal must be 1");
  double mineig = 0.0;
  if (sym_min_eigenvalue(corr, n, &mineig) != OR_OK || mineig < -1e-10)
    return fail(OR_BAD_CORRELATION,
                "SignalSpec: cross_correlation has eigenvalues below -1e-10");
  for (int64_t s = 0; s < n; ++s) {
    if (!(var[s] > 0.0))
      return fail(OR_CONFIG_ERROR, "SignalSpec: variance_target must be > 0");
    const double bound = skew[s] * skew[s] + 1.0;
    if (!(kurt[s] > bound))
      return fail(OR_MOMENT_INFEASIBLE,
                  "SignalSpec: kurtosis_target %g for signal %lld violates the "
                  "Pearson bound (must exceed skewness^2 + 1 = %g)",
                  kurt[s], (long long)s, bound);
  }
  return OR_OK;
}

static double col_mean_seq(const double* x, int64_t N) {
  double s = 0.0;
  for (int64_t t = 0; t < N; ++t) s += x[t];
  return s / (double)N;
}

static double population_std(const double* x, int64_t N) {
  const double mean = col_mean_seq(x, N);
  double s = 0.0;
  for (int64_t t = 0; t < N; ++t) {
    const double d = x[t] - mean;
    s += d * d;
  }
  return sqrt(s / (double)N);
}

/* signals.cpp:205-254 -- synthesize.  Order of operations follows the
 * reference; Eigen's vectorised mean and blocked GEMM z*L^T are restated as
 * sequential sums (tolerance parity only). */
int or_synthesize(int64_t n, int64_t N, double phi, const double* corr,
                  const double* variance, const double* skewness,
                  const double* kurtosis, uint64_t seed, double* out) {
  int st = validate_spec(n, N, phi, corr, variance, skewness, kurtosis);
  if (st != OR_OK) return st;
  double* z = out; /* N x n, built in place */
  for (int64_t s = 0; s < n; ++s) {
    const uint64_t c = (uint64_t)s;
    gauss_stream g;
    gauss_init(&g, or_derive_seed(seed, &c, 1));
    double state = gauss_next(&g);
    for (int64_t t = 0; t < 1000; ++t) state = phi * state + gauss_next(&g);
    double* col = z + (size_t)s * (size_t)N;
    for (int64_t t = 0; t < N; ++t) {
      state = phi * state + gauss_next(&g);
      col[t] = state;
    }
    const double mean = col_mean_seq(col, N);
    double sd = population_std(col, N);
    if (sd <= 0.0) sd = 1.0;
    for (int64_t t = 0; t < N; ++t) col[t] = (col[t] - mean) / sd;
  }
  if (n > 1) {
    double* rep = dalloc((size_t)(n * n));
    st = or_nearest_psd_repair(corr, n, 1e-6, rep, NULL);
    if (st != OR_OK) {
      free(rep);
      return st;
    }
    if (!llt_lower(rep, n)) {
      free(rep);
      return fail(OR_BAD_CORRELATION, "synthesize: Cholesky failed");
    }
    double* row = dalloc((size_t)n);
    /* row-major copy of the factor: the same products summed in the same
     * order (k = 0..s), without a 8n-byte stride per term */
    double* lrow = dalloc((size_t)n * (size_t)n);
    for (int64_t s = 0; s < n; ++s)
      for (int64_t k = 0; k <= s; ++k) lrow[(size_t)s * (size_t)n + (size_t)k] = CM(rep, n, s, k);
    for (int64_t t = 0; t < N; ++t) {
      for (int64_t k = 0; k < n; ++k) row[k] = z[(size_t)t + (size_t)k * (size_t)N];
      for (int64_t s = 0; s < n; ++s) {
        const double* ls = lrow + (size_t)s * (size_t)n;
        double acc = 0.0;
        for (int64_t k = 0; k <= s; ++k) acc += row[k] * ls[k];
        z[(size_t)t + (size_t)s * (size_t)N] = acc;
      }
    }
    free(lrow);
    free(row);
    free(rep);
  }
  for (int64_t s = 0; s < n; ++s) {
    double fc[4];
    st = or_solve_fleishman(skewness[s], kurtosis[s], fc);
    if (st != OR_OK) return st;
    double* col = out + (size_t)s * (size_t)N;
    for (int64_t t = 0; t < N; ++t) {
      const double v = col[t];
      col[t] = fc[0] + v * (fc[1] + v * (fc[2] + v * fc[3]));
    }
    double sd = population_std(col, N);
    if (sd <= 0.0) sd = 1.0;
    const double f = sqrt(variance[s]) / sd;
    for (int64_t t = 0; t < N; ++t) col[t] *= f;
  }
  return OR_OK;
}

/* signals.cpp:51-65 -- SignalSpec::uniform */
int or_synthesize_uniform(int64_t n, int64_t N, double phi, double rho,
                          double variance, double skewness, double kurtosis,
                          uint64_t seed, double* out) {
  if (n < 1) return fail(OR_CONFIG_ERROR, "SignalSpec: n_signals must be >= 1");
  double* corr = dalloc((size_t)(n * n));
  double* var = dalloc((size_t)n);
  double* sk = dalloc((size_t)n);
  double* ku = dalloc((size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) CM(corr, n, i, j) = i == j ? 1.0 : rho;
  for (int64_t s = 0; s < n; ++s) {
    var[s] = variance;
    sk[s] = skewness;
    ku[s] = kurtosis;
  }
  const int st = or_synthesize(n, N, phi, corr, var, sk, ku, seed, out);
  free(corr);
  free(var);
  free(sk);
  free(ku);
  return st;
}

/* ------------------------------------------------------------------ kernel */
/* kernels.hpp:54-57 */
double or_kernel_from_d2(double d2, int kind, double h) {
  if (kind == OR_KERNEL_GAUSSIAN) return exp(-d2 / (2.0 * h * h));
  return 1.0 / (1.0 + sqrt(d2) / h);
}

/* --------------------------------------------------------------- threads */
/* backends.cpp:57-73 -- contiguous tile chunks, one per worker */
typedef void (*tile_fn)(void* ctx, int64_t first, int64_t last);
typedef struct {
  tile_fn fn;
  void* ctx;
  int64_t first, last;
} tile_job;

static void* tile_thread(void* a) {
  tile_job* j = (tile_job*)a;
  j->fn(j->ctx, j->first, j->last);
  return NULL;
}

static void parallel_tiles(int64_t n_tiles, int worker_count, tile_fn fn, void* ctx) {
  const int64_t cap = n_tiles > 1 ? n_tiles : 1;
  const int workers = (int64_t)worker_count < cap ? worker_count : (int)cap;
  if (workers <= 1) {
    fn(ctx, 0, n_tiles);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
  tile_job* jobs = (tile_job*)malloc(sizeof(tile_job) * (size_t)workers);
  for (int w = 0; w < workers; ++w) {
    jobs[w].fn = fn;
    jobs[w].ctx = ctx;
    jobs[w].first = n_tiles * w / workers;
    jobs[w].last = n_tiles * (w + 1) / workers;
    pthread_create(&th[w], NULL, tile_thread, &jobs[w]);
  }
  for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
  free(th);
  free(jobs);
}

/* backends.cpp:77-99 */
static int validate_backend(int tile, int workers) {
  if (workers < 1) return fail(OR_CONFIG_ERROR, "backend worker_count must be >= 1");
  if (tile < 8 || tile > 1024)
    return fail(OR_CONFIG_ERROR, "backend tile_size must lie in [8, 1024]");
  return OR_OK;
}

static double resolve_h(double h, int64_t n) { return h > 0.0 ? h : sqrt((double)n); }

/* ------------------------------------------------------------ sim_matrix */
/* backends.cpp:129-152 */
int or_sim_matrix_reference(const double* A, const double* B, int64_t n,
                            int64_t p, int64_t q, int kind, double h,
                            double* out) {
  h = resolve_h(h, n);
  for (int64_t j = 0; j < q; ++j) {
    const double* bj = B + (size_t)j * (size_t)n;
    for (int64_t i = 0; i < p; ++i) {
      const double* ai = A + (size_t)i * (size_t)n;
      double d2 = 0.0;
      for (int64_t r = 0; r < n; ++r) {
        const double d = ai[r] - bj[r];
        d2 += d * d;
      }
      CM(out, p, i, j) = or_kernel_from_d2(d2, kind, h);
    }
  }
  return OR_OK;
}

/* backends.cpp:34-52 */
static double strip_d2(const double* a, const double* b, int64_t k0, int64_t k1) {
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  int64_t k = k0;
  for (; k + 4 <= k1; k += 4) {
    const double d0 = a[k] - b[k];
    const double d1 = a[k + 1] - b[k + 1];
    const double d2 = a[k + 2] - b[k + 2];
    const double d3 = a[k + 3] - b[k + 3];
    acc0 += d0 * d0;
    acc1 += d1 * d1;
    acc2 += d2 * d2;
    acc3 += d3 * d3;
  }
  for (; k < k1; ++k) {
    const double d = a[k] - b[k];
    acc0 += d * d;
  }
  return (acc0 + acc1) + (acc2 + acc3);
}

#define K_DEPTH_BLOCK 128 /* backends.cpp:24 */

typedef struct {
  const double *A, *B;
  double* out;
  int64_t n, p, q, T, tiles_j;
  int kind;
  double h;
} sim_ctx;

/* backends.cpp:178-202 */
static void sim_tiles(void* vctx, int64_t first, int64_t last) {
  sim_ctx* c = (sim_ctx*)vctx;
  const int64_t T = c->T;
  double* buf = dalloc((size_t)(T * T));
  for (int64_t t = first; t < last; ++t) {
    const int64_t ti = t / c->tiles_j, tj = t % c->tiles_j;
    const int64_t i0 = ti * T, j0 = tj * T;
    const int64_t ni = T < c->p - i0 ? T : c->p - i0;
    const int64_t nj = T < c->q - j0 ? T : c->q - j0;
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) CM(buf, T, i, j) = 0.0;
    for (int64_t k0 = 0; k0 < c->n; k0 += K_DEPTH_BLOCK) {
      const int64_t k1 = c->n < k0 + K_DEPTH_BLOCK ? c->n : k0 + K_DEPTH_BLOCK;
      for (int64_t j = 0; j < nj; ++j) {
        const double* bj = c->B + (size_t)(j0 + j) * (size_t)c->n;
        for (int64_t i = 0; i < ni; ++i)
          CM(buf, T, i, j) += strip_d2(c->A + (size_t)(i0 + i) * (size_t)c->n, bj, k0, k1);
      }
    }
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i)
        CM(c->out, c->p, i0 + i, j0 + j) = or_kernel_from_d2(CM(buf, T, i, j), c->kind, c->h);
  }
  free(buf);
}

/* backends.cpp:154-204 */
int or_sim_matrix_optimized(const double* A, const double* B, int64_t n,
                            int64_t p, int64_t q, int kind, double h, int tile,
                            int workers, double* out) {
  const int st = validate_backend(tile, workers);
  if (st != OR_OK) return st;
  if (p == 0 || q == 0) return OR_OK;
  sim_ctx c = {A, B, out, n, p, q, tile, (q + tile - 1) / tile, kind, resolve_h(h, n)};
  const int64_t tiles_i = (p + tile - 1) / tile;
  parallel_tiles(tiles_i * c.tiles_j, workers, sim_tiles, &c);
  return OR_OK;
}

/* ---------------------------------------------------------------- matmul */
/* backends.cpp:217-231 */
int or_matmul_reference(const double* A, const double* B, int64_t p, int64_t m,
                        int64_t q, double* out) {
  for (int64_t i = 0; i < p * q; ++i) out[i] = 0.0;
  for (int64_t j = 0; j < q; ++j) {
    double* cj = out + (size_t)j * (size_t)p;
    for (int64_t k = 0; k < m; ++k) {
      const double bkj = CM(B, m, k, j);
      const double* ak = A + (size_t)k * (size_t)p;
      for (int64_t i = 0; i < p; ++i) cj[i] += ak[i] * bkj;
    }
  }
  return OR_OK;
}

typedef struct {
  const double *A, *B;
  double* out;
  int64_t p, m, q, T, tiles_j;
} mm_ctx;

/* backends.cpp:246-271 */
static void mm_tiles(void* vctx, int64_t first, int64_t last) {
  mm_ctx* c = (mm_ctx*)vctx;
  const int64_t T = c->T;
  double* buf = dalloc((size_t)(T * T));
  for (int64_t t = first; t < last; ++t) {
    const int64_t ti = t / c->tiles_j, tj = t % c->tiles_j;
    const int64_t i0 = ti * T, j0 = tj * T;
    const int64_t ni = T < c->p - i0 ? T : c->p - i0;
    const int64_t nj = T < c->q - j0 ? T : c->q - j0;
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) CM(buf, T, i, j) = 0.0;
    for (int64_t k0 = 0; k0 < c->m; k0 += K_DEPTH_BLOCK) {
      const int64_t k1 = c->m < k0 + K_DEPTH_BLOCK ? c->m : k0 + K_DEPTH_BLOCK;
      for (int64_t j = 0; j < nj; ++j) {
        double* cj = buf + (size_t)j * (size_t)T;
        for (int64_t k = k0; k < k1; ++k) {
          const double bkj = CM(c->B, c->m, k, j0 + j);
          const double* ak = c->A + (size_t)k * (size_t)c->p + i0;
          for (int64_t i = 0; i < ni; ++i) cj[i] += ak[i] * bkj;
        }
      }
    }
    for (int64_t j = 0; j < nj; ++j)
      for (int64_t i = 0; i < ni; ++i) CM(c->out, c->p, i0 + i, j0 + j) = CM(buf, T, i, j);
  }
  free(buf);
}

/* backends.cpp:233-272 */
int or_matmul_optimized(const double* A, const double* B, int64_t p, int64_t m,
                        int64_t q, int tile, int workers, double* out) {
  const int st = validate_backend(tile, workers);
  if (st != OR_OK) return st;
  if (p == 0 || q == 0) return OR_OK;
  mm_ctx c = {A, B, out, p, m, q, tile, (q + tile - 1) / tile};
  const int64_t tiles_i = (p + tile - 1) / tile;
  parallel_tiles(tiles_i * c.tiles_j, workers, mm_tiles, &c);
  return OR_OK;
}

static int sim_dispatch(const double* A, const double* B, int64_t n, int64_t p,
                        int64_t q, int kind, double h, int backend, int tile,
                        int workers, double* out) {
  if (backend == OR_BACKEND_REFERENCE)
    return or_sim_matrix_reference(A, B, n, p, q, kind, h, out);
  return or_sim_matrix_optimized(A, B, n, p, q, kind, h, tile, workers, out);
}

static int mm_dispatch(const double* A, const double* B, int64_t p, int64_t m,
                       int64_t q, int backend, int tile, int workers, double* out) {
  if (backend == OR_BACKEND_REFERENCE) return or_matmul_reference(A, B, p, m, q, out);
  return or_matmul_optimized(A, B, p, m, q, tile, workers, out);
}

/* ---------------------------------------------------------- eigensolver */
/* Householder reduction to tridiagonal form followed by the implicit QL
 * algorithm (EISPACK tred2/tql2 lineage), eigenvalues ascending with
 * eigenvectors.  Stands in for Eigen::SelfAdjointEigenSolver (mset.cpp:66):
 * like Eigen it scales by max|a_ij| first and reads the lower triangle. */
static int tred2_tql2(double* V, int64_t n, double* d, double* e) {
#define VV(i, j) CM(V, n, i, j)
  for (int64_t j = 0; j < n; ++j) d[j] = VV(n - 1, j);
  for (int64_t i = n - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
    for (int64_t k = 0; k < i; ++k) scale += fabs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
      for (int64_t j = 0; j < i; ++j) {
        d[j] = VV(i - 1, j);
        VV(i, j) = 0.0;
        VV(j, i) = 0.0;
      }
    } else {
      for (int64_t k = 0; k < i; ++k) {
        d[k] /= scale;
        h += d[k] * d[k];
      }
      double f = d[i - 1];
      double g = sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h = h - f * g;
      d[i - 1] = f - g;
      for (int64_t j = 0; j < i; ++j) e[j] = 0.0;
      for (int64_t j = 0; j < i; ++j) {
        f = d[j];
        VV(j, i) = f;
        g = e[j] + VV(j, j) * f;
        for (int64_t k = j + 1; k <= i - 1; ++k) {
          g += VV(k, j) * d[k];
          e[k] += VV(k, j) * f;
        }
        e[j] = g;
      }
      f = 0.0;
      for (int64_t j = 0; j < i; ++j) {
        e[j] /= h;
        f += e[j] * d[j];
      }
      const double hh = f / (h + h);
      for (int64_t j = 0; j < i; ++j) e[j] -= hh * d[j];
      for (int64_t j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
        for (int64_t k = j; k <= i - 1; ++k) VV(k, j) -= (f * e[k] + g * d[k]);
        d[j] = VV(i - 1, j);
        VV(i, j) = 0.0;
      }
    }
    d[i] = h;
  }
  for (int64_t i = 0; i < n - 1; ++i) {
    VV(n - 1, i) = VV(i, i);
    VV(i, i) = 1.0;
    const double h = d[i + 1];
    if (h != 0.0) {
      for (int64_t k = 0; k <= i; ++k) d[k] = VV(k, i + 1) / h;
      for (int64_t j = 0; j <= i; ++j) {
        double g = 0.0;
        for (int64_t k = 0; k <= i; ++k) g += VV(k, i + 1) * VV(k, j);
        for (int64_t k = 0; k <= i; ++k) VV(k, j) -= g * d[k];
      }
    }
    for (int64_t k = 0; k <= i; ++k) VV(k, i + 1) = 0.0;
  }
  for (int64_t j = 0; j < n; ++j) {
    d[j] = VV(n - 1, j);
    VV(n - 1, j) = 0.0;
  }
  VV(n - 1, n - 1) = 1.0;
  e[0] = 0.0;

  /* implicit QL */
  for (int64_t i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = 0x1.0p-52;
  int64_t total_iter = 0;
  const int64_t max_iter = 30 * n + 30;
  for (int64_t l = 0; l < n; ++l) {
    const double t = fabs(d[l]) + fabs(e[l]);
    if (t > tst1) tst1 = t;
    int64_t m = l;
    while (m < n) {
      if (fabs(e[m]) <= eps * tst1) break;
      ++m;
    }
    if (m == n) m = n - 1;
    if (m > l) {
      do {
        if (++total_iter > max_iter) return 0;
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = hypot(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        const double dl1 = d[l + 1];
        double h = g - d[l];
        for (int64_t i = l + 2; i < n; ++i) d[i] -= h;
        f = f + h;
        p = d[m];
        double c = 1.0, c2 = c, c3 = c;
        const double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
        for (int64_t i = m - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = hypot(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          double* vi = V + (size_t)i * (size_t)n;
          double* vi1 = V + (size_t)(i + 1) * (size_t)n;
          for (int64_t k = 0; k < n; ++k) {
            h = vi1[k];
            vi1[k] = s * vi[k] + c * h;
            vi[k] = c * vi[k] - s * h;
          }
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
      } while (fabs(e[l]) > eps * tst1);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
  /* ascending sort carrying vectors */
  for (int64_t i = 0; i < n - 1; ++i) {
    int64_t k = i;
    double p = d[i];
    for (int64_t j = i + 1; j < n; ++j)
      if (d[j] < p) {
        k = j;
        p = d[j];
      }
    if (k != i) {
      d[k] = d[i];
      d[i] = p;
      double* vi = V + (size_t)i * (size_t)n;
      double* vk = V + (size_t)k * (size_t)n;
      for (int64_t j = 0; j < n; ++j) {
        const double tmp = vi[j];
        vi[j] = vk[j];
        vk[j] = tmp;
      }
    }
  }
#undef VV
  return 1;
}

/* mset.cpp:57-70 */
int or_symmetric_eig(const double* G, int64_t m, double* evals, double* evecs) {
  double magnitude = 0.0, asym = 0.0;
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < m; ++i) {
      const double a = fabs(CM(G, m, i, j));
      if (a > magnitude) magnitude = a;
      const double s = fabs(CM(G, m, i, j) - CM(G, m, j, i));
      if (s > asym) asym = s;
    }
  if (asym > 1e-9 * (magnitude > 1.0 ? magnitude : 1.0))
    return fail(OR_SHAPE_ERROR, "symmetric_eig: matrix is not symmetric to 1e-9");
  if (m == 0) return OR_OK;
  double scale = magnitude;
  if (scale == 0.0) scale = 1.0;
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < m; ++i) {
      const int64_t r = i > j ? i : j, c = i > j ? j : i; /* lower triangle */
      CM(evecs, m, i, j) = CM(G, m, r, c) / scale;
    }
  double* e = dalloc((size_t)m);
  const int ok = tred2_tql2(evecs, m, evals, e);
  free(e);
  if (!ok) return fail(OR_EIG_FAILURE, "symmetric_eig: eigensolver did not converge");
  for (int64_t i = 0; i < m; ++i) evals[i] *= scale;
  return OR_OK;
}

static int sym_min_eigenvalue(const double* A, int64_t n, double* out) {
  /* Uniform-off-diagonal matrices (SignalSpec::uniform) have the closed-form
   * spectrum {1 - rho (n-1 times), 1 + (n-1) rho}; anything else goes
   * through the eigensolver (signals.cpp:82-86). */
  int uniform = 1;
  const double rho = n > 1 ? CM(A, n, 1, 0) : 0.0;
  for (int64_t j = 0; j < n && uniform; ++j)
    for (int64_t i = 0; i < n; ++i)
      if (i != j && CM(A, n, i, j) != rho) {
        uniform = 0;
        break;
      }
  if (uniform) {
    const double a = 1.0 - rho, b = 1.0 + (double)(n - 1) * rho;
    *out = n > 1 ? (a < b ? a : b) : 1.0;
    return OR_OK;
  }
  double* ev = dalloc((size_t)n);
  double* V = dalloc((size_t)(n * n));
  const int st = or_symmetric_eig(A, n, ev, V);
  *out = ev[0];
  free(ev);
  free(V);
  return st;
}

/* tests/support/oracles.hpp:116-170 -- cyclic Jacobi */
void or_jacobi_eig(const double* G, int64_t n, double* values, double* vectors) {
  double* a = dalloc((size_t)(n * n));
  memcpy(a, G, sizeof(double) * (size_t)(n * n));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) CM(vectors, n, i, j) = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) off += CM(a, n, p, q) * CM(a, n, p, q);
    if (off < 1e-28) break;
    for (int64_t p = 0; p < n; ++p) {
      for (int64_t q = p + 1; q < n; ++q) {
        if (fabs(CM(a, n, p, q)) < 1e-300) continue;
        const double theta = (CM(a, n, q, q) - CM(a, n, p, p)) / (2.0 * CM(a, n, p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int64_t k = 0; k < n; ++k) {
          const double akp = CM(a, n, k, p), akq = CM(a, n, k, q);
          CM(a, n, k, p) = c * akp - s * akq;
          CM(a, n, k, q) = s * akp + c * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double apk = CM(a, n, p, k), aqk = CM(a, n, q, k);
          CM(a, n, p, k) = c * apk - s * aqk;
          CM(a, n, q, k) = s * apk + c * aqk;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double vkp = CM(vectors, n, k, p), vkq = CM(vectors, n, k, q);
          CM(vectors, n, k, p) = c * vkp - s * vkq;
          CM(vectors, n, k, q) = s * vkp + c * vkq;
        }
      }
    }
  }
  for (int64_t i = 0; i < n; ++i) values[i] = CM(a, n, i, i);
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = i;
    for (int64_t k = i + 1; k < n; ++k)
      if (values[k] < values[lo]) lo = k;
    if (lo != i) {
      const double tv = values[i];
      values[i] = values[lo];
      values[lo] = tv;
      for (int64_t k = 0; k < n; ++k) {
        const double t = CM(vectors, n, k, i);
        CM(vectors, n, k, i) = CM(vectors, n, k, lo);
        CM(vectors, n, k, lo) = t;
      }
    }
  }
  free(a);
}

/* ------------------------------------------------------------- selection */
/* mset.cpp:22-34 */
uint64_t or_fnv1a_row(const double* row_start, int64_t stride, int64_t n) {
  uint64_t h = 1469598103934665603ULL;
  for (int64_t s = 0; s < n; ++s) {
    uint64_t bits;
    memcpy(&bits, row_start + s * stride, sizeof bits);
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xffULL;
      h *= 1099511628211ULL;
    }
  }
  return h;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* mset.cpp:36-42 (hash collisions count as duplicates, as in the reference) */
int64_t or_count_distinct_rows(const double* X, int64_t N, int64_t n) {
  if (N == 0) return 0;
  uint64_t* h = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
  for (int64_t r = 0; r < N; ++r) h[r] = or_fnv1a_row(X + r, N, n);
  qsort(h, (size_t)N, sizeof(uint64_t), cmp_u64);
  int64_t distinct = 1;
  for (int64_t r = 1; r < N; ++r)
    if (h[r] != h[r - 1]) ++distinct;
  free(h);
  return distinct;
}

typedef struct {
  double norm;
  int64_t idx;
} norm_idx;

static int cmp_norm_idx(const void* a, const void* b) {
  const norm_idx* x = (const norm_idx*)a;
  const norm_idx* y = (const norm_idx*)b;
  if (x->norm < y->norm) return -1;
  if (y->norm < x->norm) return 1;
  return x->idx < y->idx ? -1 : x->idx > y->idx;
}

/* mset.cpp:72-137 */
int or_select_memory_vectors(const double* X, int64_t N, int64_t n, int64_t m,
                             int64_t* idx_out, double* D_out) {
  if (m < 2 * n)
    return fail(OR_CONSTRAINT_VIOLATED,
                "select_memory_vectors: m=%lld violates m >= 2n with n=%lld",
                (long long)m, (long long)n);
  if (m > N)
    return fail(OR_INSUFFICIENT_TRAINING,
                "select_memory_vectors: m=%lld exceeds %lld training observations",
                (long long)m, (long long)N);
  const int64_t distinct = or_count_distinct_rows(X, N, n);
  if (m > distinct)
    return fail(OR_INSUFFICIENT_TRAINING,
                "select_memory_vectors: m=%lld exceeds %lld distinct training "
                "observations",
                (long long)m, (long long)distinct);
  char* selected = (char*)calloc((size_t)N, 1);
  int64_t npicked = 0;
  for (int64_t s = 0; s < n; ++s) {
    const double* col = X + (size_t)s * (size_t)N;
    int64_t imin = 0, imax = 0;
    for (int64_t r = 1; r < N; ++r) {
      if (col[r] < col[imin]) imin = r;
      if (col[r] > col[imax]) imax = r;
    }
    const int64_t cand[2] = {imin, imax};
    for (int c = 0; c < 2; ++c)
      if (!selected[cand[c]]) {
        selected[cand[c]] = 1;
        idx_out[npicked++] = cand[c];
      }
  }
  const int64_t remaining = m - npicked;
  if (remaining > 0) {
    norm_idx* by = (norm_idx*)malloc(sizeof(norm_idx) * (size_t)N);
    int64_t pool = 0;
    for (int64_t r = 0; r < N; ++r) {
      if (selected[r]) continue;
      double s2 = 0.0; /* Eigen row(r).norm(): sequential sum of squares */
      for (int64_t s = 0; s < n; ++s) {
        const double v = X[(size_t)r + (size_t)s * (size_t)N];
        s2 += v * v;
      }
      by[pool].norm = sqrt(s2);
      by[pool].idx = r;
      ++pool;
    }
    qsort(by, (size_t)pool, sizeof(norm_idx), cmp_norm_idx);
    for (int64_t i = 0; i < remaining; ++i) {
      const int64_t pos = remaining == 1 ? (pool - 1) / 2 : i * (pool - 1) / (remaining - 1);
      idx_out[npicked++] = by[pos].idx;
    }
    free(by);
  }
  free(selected);
  if (D_out)
    for (int64_t c = 0; c < m; ++c)
      for (int64_t s = 0; s < n; ++s)
        CM(D_out, n, s, c) = X[(size_t)idx_out[c] + (size_t)s * (size_t)N];
  return OR_OK;
}

/* mset.cpp:44-53 (Eigen's vectorised mean restated as a sequential sum) */
void or_per_signal_scale(const double* X, int64_t N, int64_t n, double* scale) {
  const double dN = (double)N;
  for (int64_t s = 0; s < n; ++s) {
    const double* col = X + (size_t)s * (size_t)N;
    double sum = 0.0;
    for (int64_t t = 0; t < N; ++t) sum += col[t];
    const double mean = sum / dN;
    double ss = 0.0;
    for (int64_t t = 0; t < N; ++t) {
      const double d = col[t] - mean;
      ss += d * d;
    }
    const double sd = sqrt(ss / dN);
    scale[s] = sd > 1e-12 ? sd : 1e-12;
  }
}

/* ------------------------------------------------------------ train/est */
/* mset.cpp:139-172 */
int or_train(const double* X, int64_t N, int64_t n, int64_t m, int kind,
             double h, int backend, int tile, int workers, int64_t* idx_out,
             double* D_out, double* scale_out, double* pinv_out,
             double* spectrum_out, int64_t* rank_out, double* h_out) {
  if (backend == OR_BACKEND_OPTIMIZED) {
    const int st = validate_backend(tile, workers);
    if (st != OR_OK) return st;
  }
  int st = or_select_memory_vectors(X, N, n, m, idx_out, D_out);
  if (st != OR_OK) return st;
  h = resolve_h(h, n);
  if (!(h > 0.0)) return fail(OR_CONFIG_ERROR, "kernel bandwidth must be > 0");
  *h_out = h;
  or_per_signal_scale(X, N, n, scale_out);
  double* Dn = dalloc((size_t)(n * m));
  for (int64_t c = 0; c < m; ++c)
    for (int64_t s = 0; s < n; ++s) CM(Dn, n, s, c) = CM(D_out, n, s, c) / scale_out[s];
  double* gram = dalloc((size_t)(m * m));
  double* V = dalloc((size_t)(m * m));
  st = sim_dispatch(Dn, Dn, n, m, m, kind, h, backend, tile, workers, gram);
  if (st == OR_OK) st = or_symmetric_eig(gram, m, spectrum_out, V);
  int64_t rank = 0;
  if (st == OR_OK) {
    const double cutoff = 1e-10 * spectrum_out[m - 1];
    for (int64_t i = 0; i < m; ++i)
      if (spectrum_out[i] > cutoff) ++rank;
    if (rank == 0) st = fail(OR_DEGENERATE_MODEL, "train: all Gram eigenvalues below cutoff");
  }
  if (st == OR_OK) {
    double* W = dalloc((size_t)(m * rank));
    double* Wt = dalloc((size_t)(m * rank));
    int64_t k = 0;
    for (int64_t i = 0; i < m; ++i) {
      if (!(spectrum_out[i] > 1e-10 * spectrum_out[m - 1])) continue;
      const double sq = sqrt(spectrum_out[i]);
      for (int64_t r = 0; r < m; ++r) CM(W, m, r, k) = CM(V, m, r, i) / sq;
      ++k;
    }
    for (int64_t j = 0; j < m; ++j)
      for (int64_t kk = 0; kk < rank; ++kk) CM(Wt, rank, kk, j) = CM(W, m, j, kk);
    st = mm_dispatch(W, Wt, m, rank, m, backend, tile, workers, pinv_out);
    free(W);
    free(Wt);
  }
  *rank_out = rank;
  free(Dn);
  free(gram);
  free(V);
  return st;
}

/* mset.cpp:174-199 */
int or_estimate(const double* D, const double* scale, const double* pinv,
                int64_t n, int64_t m, int64_t rank, int kind, double h,
                const double* obs, int64_t N, int backend, int tile,
                int workers, double* est_out, double* resid_out) {
  if (backend == OR_BACKEND_OPTIMIZED) {
    const int st = validate_backend(tile, workers);
    if (st != OR_OK) return st;
  }
  if (rank < 1) return fail(OR_DEGENERATE_MODEL, "estimate: model rank is 0");
  double* Dn = dalloc((size_t)(n * m));
  for (int64_t c = 0; c < m; ++c)
    for (int64_t s = 0; s < n; ++s) CM(Dn, n, s, c) = CM(D, n, s, c) / scale[s];
  double* xn = dalloc((size_t)(n * N));
  for (int64_t t = 0; t < N; ++t)
    for (int64_t s = 0; s < n; ++s) CM(xn, n, s, t) = CM(obs, N, t, s) / scale[s];
  double* sims = dalloc((size_t)(m * N));
  double* W = dalloc((size_t)(m * N));
  double* en = dalloc((size_t)(n * N));
  int st = sim_dispatch(Dn, xn, n, m, N, kind, h, backend, tile, workers, sims);
  if (st == OR_OK) st = mm_dispatch(pinv, sims, m, m, N, backend, tile, workers, W);
  if (st == OR_OK) st = mm_dispatch(Dn, W, n, m, N, backend, tile, workers, en);
  if (st == OR_OK) {
    for (int64_t t = 0; t < N; ++t)
      for (int64_t s = 0; s < n; ++s) CM(en, n, s, t) *= scale[s];
    for (int64_t s = 0; s < n; ++s)
      for (int64_t t = 0; t < N; ++t) {
        const double e = CM(en, n, s, t);
        CM(est_out, N, t, s) = e;
        CM(resid_out, N, t, s) = CM(obs, N, t, s) - e;
      }
  }
  free(Dn);
  free(xn);
  free(sims);
  free(W);
  free(en);
  return st;
}

/* sweep.cpp:119-126 */
uint64_t or_cell_data_seed(uint64_t master_seed, int64_t n_signals,
                           int64_t n_observations, int64_t n_memory,
                           int replicate) {
  const uint64_t c[4] = {(uint64_t)n_signals, (uint64_t)n_observations,
                         (uint64_t)n_memory, (uint64_t)replicate};
  return or_derive_seed(master_seed, c, 4);
}

/* ------------------------------------------------------------------ SPRT
 * Wald sequential probability ratio test on residual streams -- NOT in the
 * reference (SPEC.md:14, :190 exclude anomaly decision logic), so this is
 * the project's own definition, the checker for the GPU's alarm flags
 * (parity unpinned against the reference).  Per signal s, two one-sided
 * mean tests against H0: r ~ N(0, sigma_s^2):
 *   positive  lambda += c_s * (r - h_s)          (H1: mean +M_s)
 *   negative  lambda += c_s * ((-r) - h_s)       (H2: mean -M_s)
 * with c_s = M_s / sigma_s^2 and h_s = M_s / 2 supplied by the caller, in
 * that operation order (no FMA).  lambda >= B: alarm, flag bit set,
 * lambda = 0; else lambda <= A: accept H0, lambda = 0.  Flags: bit 0
 * positive alarm, bit 1 negative alarm.  state (2 per signal: positive,
 * negative) carries lambda across calls. */
void or_sprt(const double* resid, int64_t N, int64_t n, int64_t ld, const double* c,
             const double* h, double A, double B, double* state, uint8_t* flags,
             int64_t* counts) {
  for (int64_t s = 0; s < n; ++s) {
    double lp = state[2 * s], ln = state[2 * s + 1];
    int64_t cp = 0, cn = 0;
    for (int64_t t = 0; t < N; ++t) {
      const double r = resid[t + s * ld];
      uint8_t f = 0;
      lp = lp + c[s] * (r - h[s]);
      if (lp >= B) { f |= 1; lp = 0.0; ++cp; } else if (lp <= A) { lp = 0.0; }
      ln = ln + c[s] * ((-r) - h[s]);
      if (ln >= B) { f |= 2; ln = 0.0; ++cn; } else if (ln <= A) { ln = 0.0; }
      flags[t + s * N] = f;
    }
    state[2 * s] = lp;
    state[2 * s + 1] = ln;
    if (counts) { counts[2 * s] = cp; counts[2 * s + 1] = cn; }
  }
}

/*
 * gpemu_oracle.c -- CPU restatement of the reference gpemu hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see gpemu_oracle.h). Compiled with
 * -O2 -ffp-contract=off so every product/sum rounds as written.
 * Reference paths are relative to /root/reference/proj/include/gpemu/.
 */
#include "gpemu_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================== */
/* detail/rng.hpp                                                             */
/* ======================================================================== */

/* splitmix64 finaliser, rng.hpp:12-18 */
uint64_t orc_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:20-25: derive_seed(base, next, rest...) = derive_seed(mix64(base ^ mix64(next)), rest...) */
uint64_t orc_derive_seed1(uint64_t base) { return orc_mix64(base); }
uint64_t orc_derive_seed2(uint64_t base, uint64_t a) {
  return orc_derive_seed1(orc_mix64(base ^ orc_mix64(a)));
}
uint64_t orc_derive_seed3(uint64_t base, uint64_t a, uint64_t b) {
  return orc_derive_seed2(orc_mix64(base ^ orc_mix64(a)), b);
}

/* std::mt19937_64 (the engine behind detail::Rng, rng.hpp:29-58). */
#define MT_N 312
#define MT_M 156
void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
}

uint64_t orc_rng_next(orc_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform01_open_low(orc_rng* r) {
  return (double)((orc_rng_next(r) >> 11) + 1) * 0x1.0p-53;
}
double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  return lo + (hi - lo) * orc_rng_uniform01(r);
}
uint64_t orc_rng_below(orc_rng* r, uint64_t n) {
  return (uint64_t)(((__uint128_t)orc_rng_next(r) * n) >> 64);
}
double orc_rng_normal(orc_rng* r) {
  const double pi = 3.141592653589793; /* std::numbers::pi */
  const double u1 = rng_uniform01_open_low(r);
  const double u2 = orc_rng_uniform01(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * pi * u2);
}

/* ======================================================================== */
/* experiment.hpp                                                             */
/* ======================================================================== */

/* detail::random_lhd, experiment.hpp:36-50 */
static void random_lhd(size_t n, size_t d, orc_rng* rng, double* x) {
  size_t* perm = (size_t*)malloc(n * sizeof(size_t));
  for (size_t k = 0; k < d; ++k) {
    for (size_t i = 0; i < n; ++i) perm[i] = i;
    for (size_t i = n - 1; i > 0; --i) {
      size_t j = (size_t)orc_rng_below(rng, i + 1);
      size_t t = perm[i];
      perm[i] = perm[j];
      perm[j] = t;
    }
    for (size_t i = 0; i < n; ++i) {
      x[i * d + k] = ((double)perm[i] + orc_rng_uniform01(rng)) / (double)n;
    }
  }
  free(perm);
}

static double sqdist(const double* x, size_t d, size_t a, size_t b) {
  double s = 0.0;
  for (size_t k = 0; k < d; ++k) {
    const double diff = x[a * d + k] - x[b * d + k];
    s += diff * diff;
  }
  return s;
}

/* detail::MinDistanceTracker, experiment.hpp:63-133 */
typedef struct {
  size_t n;
  double* dist;
  double* row_min;
  size_t* row_arg;
} tracker;

static void tracker_recompute_row(tracker* t, size_t r) {
  double m = INFINITY;
  size_t arg = r;
  for (size_t c = 0; c < t->n; ++c) {
    if (c == r) continue;
    if (t->dist[r * t->n + c] < m) {
      m = t->dist[r * t->n + c];
      arg = c;
    }
  }
  t->row_min[r] = m;
  t->row_arg[r] = arg;
}

static double tracker_global_min(const tracker* t) {
  double m = INFINITY;
  for (size_t i = 0; i < t->n; ++i) m = t->row_min[i] < m ? t->row_min[i] : m;
  return m;
}

static void tracker_rows_changed(tracker* t, const double* x, size_t d, size_t a, size_t b) {
  const size_t n = t->n;
  for (size_t r = 0; r < n; ++r) {
    if (r == a || r == b) continue;
    const size_t cs[2] = {a, b};
    for (int q = 0; q < 2; ++q) {
      const size_t c = cs[q];
      const double d2 = sqdist(x, d, r, c);
      t->dist[r * n + c] = d2;
      t->dist[c * n + r] = d2;
    }
  }
  const double dab = sqdist(x, d, a, b);
  t->dist[a * n + b] = dab;
  t->dist[b * n + a] = dab;
  tracker_recompute_row(t, a);
  tracker_recompute_row(t, b);
  for (size_t r = 0; r < n; ++r) {
    if (r == a || r == b) continue;
    if (t->row_arg[r] == a || t->row_arg[r] == b) {
      tracker_recompute_row(t, r);
    } else {
      const size_t cs[2] = {a, b};
      for (int q = 0; q < 2; ++q) {
        const size_t c = cs[q];
        if (t->dist[r * n + c] < t->row_min[r]) {
          t->row_min[r] = t->dist[r * n + c];
          t->row_arg[r] = c;
        }
      }
    }
  }
}

/* maximin_lhd, experiment.hpp:142-172 */
int orc_maximin_lhd(size_t n, size_t d, uint64_t seed, size_t exchange_budget, double* x) {
  if (n < 2 || d < 1) return -1;
  orc_rng rng;
  orc_rng_init(&rng, orc_derive_seed2(seed, 0x1d64ull));
  random_lhd(n, d, &rng, x);
  if (exchange_budget == 0 || n == 2) return 0;

  tracker t;
  t.n = n;
  t.dist = (double*)calloc(n * n, sizeof(double));
  t.row_min = (double*)malloc(n * sizeof(double));
  t.row_arg = (size_t*)malloc(n * sizeof(size_t));
  if (!t.dist || !t.row_min || !t.row_arg) return -2;
  for (size_t i = 0; i < n; ++i) {
    for (size_t j = i + 1; j < n; ++j) {
      const double d2 = sqdist(x, d, i, j);
      t.dist[i * n + j] = d2;
      t.dist[j * n + i] = d2;
    }
  }
  for (size_t i = 0; i < n; ++i) tracker_recompute_row(&t, i);
  double current = tracker_global_min(&t);

  for (size_t iter = 0; iter < exchange_budget; ++iter) {
    const size_t k = (size_t)orc_rng_below(&rng, d);
    const size_t a = (size_t)orc_rng_below(&rng, n);
    size_t b = (size_t)orc_rng_below(&rng, n - 1);
    if (b >= a) ++b;
    double tmp = x[a * d + k];
    x[a * d + k] = x[b * d + k];
    x[b * d + k] = tmp;
    tracker_rows_changed(&t, x, d, a, b);
    const double proposed = tracker_global_min(&t);
    if (proposed > current) {
      current = proposed;
    } else {
      tmp = x[a * d + k];
      x[a * d + k] = x[b * d + k];
      x[b * d + k] = tmp;
      tracker_rows_changed(&t, x, d, a, b);
    }
  }
  free(t.dist);
  free(t.row_min);
  free(t.row_arg);
  return 0;
}

/* goldstein_price_log, experiment.hpp:179-189 */
double orc_goldstein_price_log(const double* x) {
  const double u = 4.0 * x[0] - 2.0;
  const double v = 4.0 * x[1] - 2.0;
  const double a = u + v + 1.0;
  const double b = 19.0 - 14.0 * u + 3.0 * u * u - 14.0 * v + 6.0 * u * v + 3.0 * v * v;
  const double c = 2.0 * u - 3.0 * v;
  const double e = 18.0 - 32.0 * u + 12.0 * u * u + 48.0 * v - 36.0 * u * v + 27.0 * v * v;
  const double gp = (1.0 + a * a * b) * (30.0 + c * c * e);
  return log(gp);
}

/* hartman6, experiment.hpp:193-218 */
double orc_hartman6(const double* x) {
  static const double alpha[4] = {1.0, 1.2, 3.0, 3.2};
  static const double A[4][6] = {{10.0, 3.0, 17.0, 3.5, 1.7, 8.0},
                                 {0.05, 10.0, 17.0, 0.1, 8.0, 14.0},
                                 {3.0, 3.5, 1.7, 10.0, 17.0, 8.0},
                                 {17.0, 8.0, 0.05, 10.0, 0.1, 14.0}};
  static const double P[4][6] = {{0.1312, 0.1696, 0.5569, 0.0124, 0.8283, 0.5886},
                                 {0.2329, 0.4135, 0.8307, 0.3736, 0.1004, 0.9991},
                                 {0.2348, 0.1451, 0.3522, 0.2883, 0.3047, 0.6650},
                                 {0.4047, 0.8828, 0.8732, 0.5743, 0.1091, 0.0381}};
  double outer = 0.0;
  for (int i = 0; i < 4; ++i) {
    double inner = 0.0;
    for (int j = 0; j < 6; ++j) {
      const double diff = x[j] - P[i][j];
      inner += A[i][j] * diff * diff;
    }
    outer += alpha[i] * exp(-inner);
  }
  return -outer;
}

/* detail::lhs_population, optimizer.hpp:62-80 */
static void lhs_population_rng(const double* lo, const double* hi, size_t d, int count,
                               orc_rng* rng, double* pop) {
  int* perm = (int*)malloc((size_t)count * sizeof(int));
  for (size_t k = 0; k < d; ++k) {
    for (int i = 0; i < count; ++i) perm[i] = i;
    for (int i = count - 1; i > 0; --i) {
      const int j = (int)orc_rng_below(rng, (uint64_t)i + 1);
      const int t = perm[i];
      perm[i] = perm[j];
      perm[j] = t;
    }
    const double width = hi[k] - lo[k];
    for (int i = 0; i < count; ++i) {
      const double u = (perm[i] + orc_rng_uniform01(rng)) / count;
      pop[(size_t)i * d + k] = lo[k] + width * u;
    }
  }
  free(perm);
}

void orc_lhs_population(const double* lo, const double* hi, size_t d, int count, uint64_t seed,
                        double* pop) {
  orc_rng rng;
  orc_rng_init(&rng, seed);
  lhs_population_rng(lo, hi, d, count, &rng, pop);
}

/* ======================================================================== */
/* correlation.hpp                                                            */
/* ======================================================================== */

/* detail::pow_abs, correlation.hpp:31-35 */
double orc_pow_abs(double delta, double p) {
  if (delta == 0.0) return 0.0;
  const double a = delta < 0.0 ? -delta : delta;
  return exp(p * log(a));
}

/* detail::theta_weighted_sum, correlation.hpp:42-47 (no FMA: -ffp-contract=off) */
double orc_theta_weighted_sum(const double* theta, const double* terms, size_t d) {
  double s = 0.0;
  for (size_t k = 0; k < d; ++k) s += theta[k] * terms[k];
  return s;
}

/* detail::row_of_pair, correlation.hpp:51-56 */
size_t orc_row_of_pair(size_t pair) {
  size_t i = (size_t)((sqrt(8.0 * (double)pair + 1.0) + 1.0) / 2.0);
  while (i * (i - 1) / 2 > pair) --i;
  while ((i + 1) * i / 2 <= pair) ++i;
  return i;
}

/* CorrelationPlan ctor, correlation.hpp:156-180 */
void orc_corr_table(const double* X, size_t n, size_t d, double p, double* table) {
  size_t pair = 0;
  for (size_t i = 1; i < n; ++i) {
    for (size_t j = 0; j < i; ++j, ++pair) {
      for (size_t k = 0; k < d; ++k) {
        table[pair * d + k] = orc_pow_abs(X[i * d + k] - X[j * d + k], p);
      }
    }
  }
}

/* CorrelationPlan::build_into, correlation.hpp:187-223 */
int orc_build_from_table(const double* table, size_t n, size_t d, const double* theta,
                         double nugget, double* R) {
  const double diag = 1.0 + nugget;
  int bad = 0;
  for (size_t i = 0; i < n; ++i) R[i * n + i] = diag;
  size_t pair = 0;
  for (size_t i = 1; i < n; ++i) {
    for (size_t j = 0; j < i; ++j, ++pair) {
      const double s = orc_theta_weighted_sum(theta, table + pair * d, d);
      const double v = exp(-s);
      if (!isfinite(v)) bad = 1;
      R[i * n + j] = v;
      R[j * n + i] = v;
    }
  }
  return bad ? -1 : 0;
}

/* build_corr_matrix, correlation.hpp:99-146 */
int orc_build_corr(const double* X, size_t n, size_t d, const double* theta, double p,
                   double nugget, double* R) {
  double* terms = (double*)malloc((d ? d : 1) * sizeof(double));
  const double diag = 1.0 + nugget;
  int bad = 0;
  for (size_t i = 0; i < n; ++i) R[i * n + i] = diag;
  for (size_t i = 1; i < n; ++i) {
    for (size_t j = 0; j < i; ++j) {
      for (size_t k = 0; k < d; ++k) terms[k] = orc_pow_abs(X[i * d + k] - X[j * d + k], p);
      const double s = orc_theta_weighted_sum(theta, terms, d);
      const double v = exp(-s);
      if (!isfinite(v)) bad = 1;
      R[i * n + j] = v;
      R[j * n + i] = v;
    }
  }
  free(terms);
  return bad ? -1 : 0;
}

/* corr_vector, correlation.hpp:67-91 */
int orc_corr_vector(const double* xstar, const double* X, size_t n, size_t d,
                    const double* theta, double p, double* r) {
  double* terms = (double*)malloc((d ? d : 1) * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    for (size_t k = 0; k < d; ++k) terms[k] = orc_pow_abs(xstar[k] - X[i * d + k], p);
    const double s = orc_theta_weighted_sum(theta, terms, d);
    r[i] = exp(-s);
    if (!isfinite(r[i])) {
      free(terms);
      return -1;
    }
  }
  free(terms);
  return 0;
}

/* ======================================================================== */
/* backend.hpp                                                                */
/* ======================================================================== */

/* ReferenceBackend::try_cholesky, backend.hpp:189-206 */
static int chol_reference(double* a, size_t n) {
  for (size_t j = 0; j < n; ++j) {
    double* rowj = a + j * n;
    double s = rowj[j];
    for (size_t t = 0; t < j; ++t) s -= rowj[t] * rowj[t];
    if (!(s > 0.0)) return 0;
    const double dd = sqrt(s);
    rowj[j] = dd;
    for (size_t i = j + 1; i < n; ++i) {
      double* rowi = a + i * n;
      double v = rowi[j];
      for (size_t t = 0; t < j; ++t) v -= rowi[t] * rowj[t];
      rowi[j] = v / dd;
    }
  }
  return 1;
}

#define KBLOCK 64
/* ParallelBackend::update_tile, backend.hpp:290-311 */
static void update_tile(double* A, size_t n, size_t k0, size_t kb, size_t i0, size_t ib,
                        size_t j0, size_t jb) {
  static double packed[KBLOCK * KBLOCK];
  for (size_t c = 0; c < jb; ++c) {
    const double* rowc = A + (j0 + c) * n + k0;
    for (size_t t = 0; t < kb; ++t) packed[t * jb + c] = rowc[t];
  }
  for (size_t r = 0; r < ib; ++r) {
    double* crow = A + (i0 + r) * n + j0;
    const double* arow = A + (i0 + r) * n + k0;
    const size_t climit = (i0 == j0) ? (jb < r + 1 ? jb : r + 1) : jb;
    for (size_t t = 0; t < kb; ++t) {
      const double art = arow[t];
      const double* prow = packed + t * jb;
      for (size_t c = 0; c < climit; ++c) crow[c] -= art * prow[c];
    }
  }
}

/* ParallelBackend::try_cholesky, backend.hpp:226-284 (run on one lane; the
 * reference result is thread-count independent, test_backend.cpp:232-250). */
static int chol_blocked(double* A, size_t n) {
  for (size_t k0 = 0; k0 < n; k0 += KBLOCK) {
    const size_t kb = (n - k0) < KBLOCK ? (n - k0) : KBLOCK;
    for (size_t j = k0; j < k0 + kb; ++j) {
      double* rowj = A + j * n;
      double s = rowj[j];
      for (size_t t = k0; t < j; ++t) s -= rowj[t] * rowj[t];
      if (!(s > 0.0)) return 0;
      const double dd = sqrt(s);
      rowj[j] = dd;
      for (size_t i = j + 1; i < k0 + kb; ++i) {
        double* rowi = A + i * n;
        double v = rowi[j];
        for (size_t t = k0; t < j; ++t) v -= rowi[t] * rowj[t];
        rowi[j] = v / dd;
      }
    }
    if (k0 + kb == n) break;
    for (size_t r = k0 + kb; r < n; ++r) {
      double* rowr = A + r * n;
      for (size_t j = k0; j < k0 + kb; ++j) {
        const double* rowj = A + j * n;
        double v = rowr[j];
        for (size_t t = k0; t < j; ++t) v -= rowr[t] * rowj[t];
        rowr[j] = v / rowj[j];
      }
    }
    for (size_t j0 = k0 + kb; j0 < n; j0 += KBLOCK) {
      for (size_t i0 = j0; i0 < n; i0 += KBLOCK) {
        const size_t ib = (n - i0) < KBLOCK ? (n - i0) : KBLOCK;
        const size_t jb = (n - j0) < KBLOCK ? (n - j0) : KBLOCK;
        update_tile(A, n, k0, kb, i0, ib, j0, jb);
      }
    }
  }
  return 1;
}

int orc_try_cholesky(double* A, size_t n, int kind) {
  return kind == ORC_PARALLEL ? chol_blocked(A, n) : chol_reference(A, n);
}

/* kJitterLadder, backend.hpp:77 */
static const double kLadder[6] = {0.0, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4};

/* Backend::factorize_into, backend.hpp:102-120 */
int orc_factorize(const double* R, size_t n, int kind, double* L, double* log_det,
                  double* jitter_used) {
  for (int s = 0; s < 6; ++s) {
    const double jitter = kLadder[s];
    memcpy(L, R, n * n * sizeof(double));
    if (jitter > 0.0) {
      for (size_t i = 0; i < n; ++i) L[i * n + i] += jitter;
    }
    if (orc_try_cholesky(L, n, kind)) {
      double ld = 0.0;
      for (size_t i = 0; i < n; ++i) ld += log(L[i * n + i]);
      *log_det = 2.0 * ld;
      *jitter_used = jitter;
      return 0;
    }
  }
  return 1;
}

/* Backend::solve_lower_into, backend.hpp:129-140 */
void orc_solve_lower(const double* L, size_t n, const double* b, double* x) {
  for (size_t i = 0; i < n; ++i) {
    double s = b[i];
    const double* row = L + i * n;
    for (size_t j = 0; j < i; ++j) s -= row[j] * x[j];
    x[i] = s / row[i];
  }
}

/* Backend::solve_upper_into, backend.hpp:143-153 */
void orc_solve_upper(const double* L, size_t n, const double* b, double* x) {
  for (size_t ii = n; ii-- > 0;) {
    double s = b[ii];
    for (size_t j = ii + 1; j < n; ++j) s -= L[j * n + ii] * x[j];
    x[ii] = s / L[ii * n + ii];
  }
}

/* dot_accumulate, matrix.hpp:64-69 */
double orc_dot_accumulate(const double* a, const double* b, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* ======================================================================== */
/* likelihood.hpp                                                             */
/* ======================================================================== */

/* sigma2_hat_from_parts, likelihood.hpp:63-66 */
static double sigma2_from_parts(double utu, double vtu, double vtv, double mu, size_t n) {
  const double s = (utu - 2.0 * mu * vtu + mu * mu * vtv) / (double)n;
  return s < 0.0 ? 0.0 : s;
}

/* ProfileEvaluator::eval, likelihood.hpp:108-141 */
void orc_profile_eval_table(const double* table, const double* y, size_t n, size_t d,
                            double nugget, const double* theta, int kind, orc_profile* out,
                            double* L, double* R) {
  out->neg2_log_lik = INFINITY;
  out->mu_hat = 0.0;
  out->sigma2_hat = 0.0;
  out->jitter_used = 0.0;
  out->log_det = 0.0;
  out->factor_jitter = -1.0;
  orc_build_from_table(table, n, d, theta, nugget, R);
  double log_det = 0.0, jitter = 0.0;
  if (orc_factorize(R, n, kind, L, &log_det, &jitter) != 0) return; /* +inf */
  out->factor_jitter = jitter;
  double* u = (double*)malloc(n * sizeof(double));
  double* v = (double*)malloc(n * sizeof(double));
  double* ones = (double*)malloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) ones[i] = 1.0;
  orc_solve_lower(L, n, y, u);
  orc_solve_lower(L, n, ones, v);
  const double utu = orc_dot_accumulate(u, u, n);
  const double vtu = orc_dot_accumulate(v, u, n);
  const double vtv = orc_dot_accumulate(v, v, n);
  free(u);
  free(v);
  free(ones);
  if (!(vtv > 0.0)) return;
  const double mu = vtu / vtv;
  const double sigma2 = sigma2_from_parts(utu, vtu, vtv, mu, n);
  const double qf = (double)n * sigma2;
  const double qf_floored = qf > DBL_MIN ? qf : DBL_MIN;
  out->mu_hat = mu;
  out->sigma2_hat = sigma2;
  out->jitter_used = jitter;
  out->log_det = log_det;
  out->neg2_log_lik = log_det + (double)n * log(qf_floored);
}

int orc_profile_eval_batch(const double* X, const double* y, size_t n, size_t d, double p,
                           double nugget, const double* thetas, size_t B, int kind,
                           double* neg2, double* mu, double* sigma2, double* jitter,
                           double* log_det) {
  const size_t pairs = n * (n - 1) / 2;
  double* table = (double*)malloc((pairs * d > 0 ? pairs * d : 1) * sizeof(double));
  double* R = (double*)malloc(n * n * sizeof(double));
  double* L = (double*)malloc(n * n * sizeof(double));
  if (!table || !R || !L) return -2;
  orc_corr_table(X, n, d, p, table);
  for (size_t b = 0; b < B; ++b) {
    orc_profile pe;
    orc_profile_eval_table(table, y, n, d, nugget, thetas + b * d, kind, &pe, L, R);
    neg2[b] = pe.neg2_log_lik;
    if (mu) mu[b] = pe.mu_hat;
    if (sigma2) sigma2[b] = pe.sigma2_hat;
    if (jitter) jitter[b] = pe.jitter_used;
    if (log_det) log_det[b] = pe.log_det;
  }
  free(table);
  free(R);
  free(L);
  return 0;
}

/* ======================================================================== */
/* optimizer.hpp                                                              */
/* ======================================================================== */

static const double* g_sort_fitness;
static int cmp_order(const void* pa, const void* pb) {
  const int a = *(const int*)pa, b = *(const int*)pb;
  const double fa = g_sort_fitness[a], fb = g_sort_fitness[b];
  if (fa < fb) return -1;
  if (fb < fa) return 1;
  return a < b ? -1 : (a > b ? 1 : 0); /* stable_sort: ties by slot */
}

/* ga_minimize, optimizer.hpp:93-187 */
int orc_ga_minimize(orc_objective f, void* ctx, const double* lo, const double* hi, size_t d,
                    const orc_ga_config* cfg, double* best_point, double* best_value,
                    double* trace_best, double* trace_point) {
  const int P = cfg->population;
  if (P <= 0 || cfg->generations <= 0 || cfg->elitism < 0 || cfg->elitism >= P || d == 0) return -1;
  const double mut_prob = cfg->mutation_prob > 0.0 ? cfg->mutation_prob : 1.0 / (double)d;

  orc_rng init_rng;
  orc_rng_init(&init_rng, orc_derive_seed2(cfg->seed, 0x1e17u));
  double* pop = (double*)malloc((size_t)P * d * sizeof(double));
  double* next = (double*)malloc((size_t)P * d * sizeof(double));
  double* fitness = (double*)malloc((size_t)P * sizeof(double));
  int* order = (int*)malloc((size_t)P * sizeof(int));
  double* child = (double*)malloc(d * sizeof(double));
  lhs_population_rng(lo, hi, d, P, &init_rng, pop);

  *best_value = INFINITY;
  for (int gen = 0; gen < cfg->generations; ++gen) {
    if (gen > 0) {
      for (int i = 0; i < P; ++i) order[i] = i;
      g_sort_fitness = fitness;
      qsort(order, (size_t)P, sizeof(int), cmp_order);
      for (int e = 0; e < cfg->elitism; ++e) {
        memcpy(next + (size_t)e * d, pop + (size_t)order[e] * d, d * sizeof(double));
      }
      for (int slot = cfg->elitism; slot < P; ++slot) {
        orc_rng rng;
        orc_rng_init(&rng, orc_derive_seed3(cfg->seed, (uint64_t)gen, (uint64_t)slot));
        int parents[2];
        for (int q = 0; q < 2; ++q) {
          const int a = (int)orc_rng_below(&rng, (uint64_t)P);
          const int b = (int)orc_rng_below(&rng, (uint64_t)P);
          const int a_wins = fitness[a] < fitness[b] || (fitness[a] == fitness[b] && a <= b);
          parents[q] = a_wins ? a : b;
        }
        const double* pa = pop + (size_t)parents[0] * d;
        const double* pb = pop + (size_t)parents[1] * d;
        if (orc_rng_uniform01(&rng) < cfg->crossover_rate) {
          for (size_t k = 0; k < d; ++k) child[k] = orc_rng_uniform01(&rng) < 0.5 ? pa[k] : pb[k];
        } else {
          memcpy(child, pa, d * sizeof(double));
        }
        for (size_t k = 0; k < d; ++k) {
          if (orc_rng_uniform01(&rng) < mut_prob) child[k] += cfg->mutation_sigma * orc_rng_normal(&rng);
          if (child[k] < lo[k]) child[k] = lo[k];
          else if (hi[k] < child[k]) child[k] = hi[k];
        }
        memcpy(next + (size_t)slot * d, child, d * sizeof(double));
      }
      double* t = pop;
      pop = next;
      next = t;
    }
    for (int i = 0; i < P; ++i) fitness[i] = f(pop + (size_t)i * d, ctx);
    int b = 0;
    for (int i = 1; i < P; ++i)
      if (fitness[i] < fitness[b]) b = i;
    if (fitness[b] < *best_value) {
      *best_value = fitness[b];
      memcpy(best_point, pop + (size_t)b * d, d * sizeof(double));
    }
    if (trace_best) trace_best[gen] = fitness[b];
    if (trace_point) memcpy(trace_point + (size_t)gen * d, pop + (size_t)b * d, d * sizeof(double));
  }
  free(pop);
  free(next);
  free(fitness);
  free(order);
  free(child);
  return 0;
}

/* fit_gp_detailed, likelihood.hpp:243-303 */
typedef struct {
  const double* table;
  const double* y;
  size_t n, d;
  double nugget;
  int kind;
  double* R;
  double* L;
  double* theta;
  double best_value;
  orc_profile best_eval;
  double* best_theta;
  double* best_L;
  double jitter_max;
} fit_ctx;

static double fit_objective(const double* genes, void* vctx) {
  fit_ctx* c = (fit_ctx*)vctx;
  for (size_t k = 0; k < c->d; ++k) c->theta[k] = pow(10.0, genes[k]);
  orc_profile ev;
  orc_profile_eval_table(c->table, c->y, c->n, c->d, c->nugget, c->theta, c->kind, &ev, c->L, c->R);
  if (ev.factor_jitter > c->jitter_max) c->jitter_max = ev.factor_jitter; /* likelihood.hpp:120 */
  if (ev.neg2_log_lik < c->best_value) {
    c->best_value = ev.neg2_log_lik;
    c->best_eval = ev;
    memcpy(c->best_theta, c->theta, c->d * sizeof(double));
    memcpy(c->best_L, c->L, c->n * c->n * sizeof(double));
  }
  return ev.neg2_log_lik;
}

int orc_fit(const double* X, const double* y, size_t n, size_t d, double p, double nugget,
            const double* lo, const double* hi, const orc_ga_config* ga, uint64_t seed, int kind,
            double* theta_hat, orc_fit_result* res, double* alpha, double* L_out,
            double* trace_best, double* trace_genes) {
  const size_t pairs = n * (n - 1) / 2;
  fit_ctx c;
  memset(&c, 0, sizeof(c));
  double* table = (double*)malloc((pairs * d > 0 ? pairs * d : 1) * sizeof(double));
  c.R = (double*)malloc(n * n * sizeof(double));
  c.L = (double*)malloc(n * n * sizeof(double));
  c.best_L = (double*)malloc(n * n * sizeof(double));
  c.theta = (double*)malloc(d * sizeof(double));
  c.best_theta = (double*)malloc(d * sizeof(double));
  double* log_lo = (double*)malloc(d * sizeof(double));
  double* log_hi = (double*)malloc(d * sizeof(double));
  double* best_genes = (double*)malloc(d * sizeof(double));
  orc_corr_table(X, n, d, p, table);
  c.table = table;
  c.y = y;
  c.n = n;
  c.d = d;
  c.nugget = nugget;
  c.kind = kind;
  c.best_value = INFINITY;
  for (size_t k = 0; k < d; ++k) {
    log_lo[k] = log10(lo[k]);
    log_hi[k] = log10(hi[k]);
  }
  orc_ga_config g = *ga;
  g.seed = orc_derive_seed2(seed, 0x9a5eedull);
  double best_value = INFINITY;
  int rc = orc_ga_minimize(fit_objective, &c, log_lo, log_hi, d, &g, best_genes, &best_value,
                           trace_best, trace_genes);
  if (rc == 0 && !isfinite(c.best_value)) rc = 2;     /* FitError */
  if (rc == 0 && best_value != c.best_value) rc = 3;  /* incumbent diverged */
  if (rc == 0) {
    memcpy(theta_hat, c.best_theta, d * sizeof(double));
    double* rhs = (double*)malloc(n * sizeof(double));
    double* u = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) rhs[i] = y[i] - c.best_eval.mu_hat;
    orc_solve_lower(c.best_L, n, rhs, u);
    orc_solve_upper(c.best_L, n, u, alpha);
    free(rhs);
    free(u);
    res->neg2_log_lik = c.best_eval.neg2_log_lik;
    res->mu_hat = c.best_eval.mu_hat;
    res->sigma2_hat = c.best_eval.sigma2_hat;
    res->jitter_used = c.best_eval.jitter_used;
    res->log_det = c.best_eval.log_det;
    res->jitter_max = c.jitter_max;
    if (L_out) memcpy(L_out, c.best_L, n * n * sizeof(double));
  }
  free(table);
  free(c.R);
  free(c.L);
  free(c.best_L);
  free(c.theta);
  free(c.best_theta);
  free(log_lo);
  free(log_hi);
  free(best_genes);
  return rc;
}

/* ======================================================================== */
/* predictor.hpp                                                              */
/* ======================================================================== */

/* predict, predictor.hpp:20-50 */
int orc_predict(const double* X, size_t n, size_t d, const double* theta, double p, double mu,
                const double* alpha, const double* Xtest, size_t N, double* yhat) {
  double* r = (double*)malloc(n * sizeof(double));
  for (size_t j = 0; j < N; ++j) {
    if (orc_corr_vector(Xtest + j * d, X, n, d, theta, p, r) != 0) {
      free(r);
      return -1;
    }
    yhat[j] = mu + orc_dot_accumulate(r, alpha, n);
  }
  free(r);
  return 0;
}

/* sspe, predictor.hpp:53-61 */
double orc_sspe(const double* pred, const double* truth, size_t N) {
  double s = 0.0;
  for (size_t i = 0; i < N; ++i) {
    const double e = truth[i] - pred[i];
    s += e * e;
  }
  return s;
}

/* Kriging MSE: no reference implementation; standard constant-mean
 * ordinary-kriging variance, SURVEY.md 8(a)-14. */
int orc_kriging_mse(const double* X, size_t n, size_t d, const double* theta, double p,
                    double sigma2, const double* L, const double* Xtest, size_t N, double* mse) {
  double* r = (double*)malloc(n * sizeof(double));
  double* w = (double*)malloc(n * sizeof(double));
  double* v = (double*)malloc(n * sizeof(double));
  double* ones = (double*)malloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) ones[i] = 1.0;
  orc_solve_lower(L, n, ones, v);
  const double vtv = orc_dot_accumulate(v, v, n);
  for (size_t j = 0; j < N; ++j) {
    if (orc_corr_vector(Xtest + j * d, X, n, d, theta, p, r) != 0) return -1;
    orc_solve_lower(L, n, r, w);
    const double wtw = orc_dot_accumulate(w, w, n);
    const double vtw = orc_dot_accumulate(v, w, n);
    const double a = 1.0 - vtw;
    double s = sigma2 * (1.0 - wtw + a * a / vtv);
    mse[j] = s < 0.0 ? 0.0 : s;
  }
  free(r);
  free(w);
  free(v);
  free(ones);
  return 0;
}

/* ======================================================================== */
/* Extended-precision truth (x87 80-bit long double)                          */
/* ======================================================================== */

/* The exact-as-possible deviance of the DOUBLE R the reference builds
 * (CorrelationPlan::build_into, then + jitter on the diagonal): Cholesky,
 * solves, dots and the deviance formula of likelihood.hpp:124-139 all in long
 * double. Used to measure how far the reference itself is from the value it
 * approximates, so parity gates can be conditioning-aware. */
/* long-double deviance of one (already built, double) R + jitter I */
static double ld_deviance(const double* R, const double* y, size_t n, double jitter,
                          long double* L, long double* u, long double* v) {
  for (size_t i = 0; i < n * n; ++i) L[i] = R[i];
  for (size_t i = 0; i < n; ++i) L[i * n + i] += jitter;
  long double logdet = 0.0L;
  for (size_t j = 0; j < n; ++j) {
    long double s = L[j * n + j];
    for (size_t t = 0; t < j; ++t) s -= L[j * n + t] * L[j * n + t];
    if (!(s > 0.0L)) return INFINITY;
    const long double dd = sqrtl(s);
    L[j * n + j] = dd;
    logdet += logl(dd);
    for (size_t i = j + 1; i < n; ++i) {
      long double w = L[i * n + j];
      for (size_t t = 0; t < j; ++t) w -= L[i * n + t] * L[j * n + t];
      L[i * n + j] = w / dd;
    }
  }
  for (size_t i = 0; i < n; ++i) {
    long double su = y[i], sv = 1.0L;
    for (size_t t = 0; t < i; ++t) {
      su -= L[i * n + t] * u[t];
      sv -= L[i * n + t] * v[t];
    }
    u[i] = su / L[i * n + i];
    v[i] = sv / L[i * n + i];
  }
  long double utu = 0.0L, vtu = 0.0L, vtv = 0.0L;
  for (size_t i = 0; i < n; ++i) {
    utu += u[i] * u[i];
    vtu += v[i] * u[i];
    vtv += v[i] * v[i];
  }
  const long double mu = vtu / vtv;
  long double s2 = (utu - 2.0L * mu * vtu + mu * mu * vtv) / (long double)n;
  if (s2 < 0.0L) s2 = 0.0L;
  long double qf = (long double)n * s2;
  if (qf < (long double)DBL_MIN) qf = DBL_MIN;
  return (double)(2.0L * logdet + (long double)n * logl(qf));
}

int orc_profile_eval_ld(const double* X, const double* y, size_t n, size_t d, double p,
                        double nugget, const double* thetas, size_t B, const double* jitters,
                        double* neg2_out) {
  return orc_profile_sensitivity(X, y, n, d, p, nugget, thetas, B, jitters, 0, 0, neg2_out, NULL);
}

/* Sensitivity of the deviance to 1-ulp relative perturbations of the off-diagonal
 * entries of R (the accuracy any FP64 R assembly has: exp/log are <= 1 ulp): for each
 * theta, max over `reps` symmetric random perturbations of |neg2' - neg2| / |neg2|,
 * all in long double. reps = 0 only fills neg2_out (the truth). */
int orc_profile_sensitivity(const double* X, const double* y, size_t n, size_t d, double p,
                            double nugget, const double* thetas, size_t B, const double* jitters,
                            int reps, uint64_t seed, double* neg2_out, double* sens_out) {
  const size_t pairs = n * (n - 1) / 2;
  double* table = (double*)malloc((pairs * d > 0 ? pairs * d : 1) * sizeof(double));
  double* R = (double*)malloc(n * n * sizeof(double));
  double* Rp = (double*)malloc(n * n * sizeof(double));
  long double* L = (long double*)malloc(n * n * sizeof(long double));
  long double* u = (long double*)malloc(n * sizeof(long double));
  long double* v = (long double*)malloc(n * sizeof(long double));
  if (!table || !R || !Rp || !L || !u || !v) return -2;
  orc_corr_table(X, n, d, p, table);
  orc_rng rng;
  orc_rng_init(&rng, seed);
  for (size_t b = 0; b < B; ++b) {
    orc_build_from_table(table, n, d, thetas + b * d, nugget, R);
    const double t = ld_deviance(R, y, n, jitters[b], L, u, v);
    neg2_out[b] = t;
    if (!sens_out) continue;
    double worst = 0.0;
    for (int r = 0; r < reps && isfinite(t); ++r) {
      memcpy(Rp, R, n * n * sizeof(double));
      for (size_t i = 1; i < n; ++i)
        for (size_t j = 0; j < i; ++j) {
          const double e = (2.0 * orc_rng_uniform01(&rng) - 1.0) * 0x1.0p-53;
          Rp[i * n + j] = R[i * n + j] * (1.0 + e);
          Rp[j * n + i] = Rp[i * n + j];
        }
      const double tp = ld_deviance(Rp, y, n, jitters[b], L, u, v);
      const double rel = fabs(tp - t) / fabs(t);
      if (!(rel <= worst)) worst = rel;
    }
    sens_out[b] = worst;
  }
  free(table);
  free(R);
  free(Rp);
  free(L);
  free(u);
  free(v);
  return 0;
}

/* ======================================================================== */
/* bench.hpp:302-383 detail::refine_fit (coordinate-wise golden-section polish) */
/* ======================================================================== */
typedef struct {
  const double* table;
  const double* y;
  size_t n, d;
  double nugget;
  int kind;
  double* R;
  double* L;
  double* theta;
  int used;
  double best_value;
  double* best_genes;
} refine_ctx;

static double refine_eval(refine_ctx* c, const double* genes) {
  for (size_t k = 0; k < c->d; ++k) c->theta[k] = pow(10.0, genes[k]);
  ++c->used;
  orc_profile ev;
  orc_profile_eval_table(c->table, c->y, c->n, c->d, c->nugget, c->theta, c->kind, &ev, c->L, c->R);
  const double v = ev.neg2_log_lik;
  if (v < c->best_value) {
    c->best_value = v;
    memcpy(c->best_genes, genes, c->d * sizeof(double));
  }
  return v;
}

int orc_refine_fit(const double* X, const double* y, size_t n, size_t d, double p, double nugget,
                   const double* lo, const double* hi, const double* theta_fit, double neg2_fit,
                   int budget, int kind, double* theta_out, double* neg2_out, int* used_out) {
  const size_t pairs = n * (n - 1) / 2;
  refine_ctx c;
  memset(&c, 0, sizeof(c));
  double* table = (double*)malloc((pairs * d > 0 ? pairs * d : 1) * sizeof(double));
  c.R = (double*)malloc(n * n * sizeof(double));
  c.L = (double*)malloc(n * n * sizeof(double));
  c.theta = (double*)malloc(d * sizeof(double));
  c.best_genes = (double*)malloc(d * sizeof(double));
  double* g = (double*)malloc(d * sizeof(double));
  if (!table || !c.R || !c.L || !c.theta || !c.best_genes || !g) return -2;
  orc_corr_table(X, n, d, p, table);
  c.table = table;
  c.y = y;
  c.n = n;
  c.d = d;
  c.nugget = nugget;
  c.kind = kind;
  for (size_t k = 0; k < d; ++k) c.best_genes[k] = log10(theta_fit[k]);
  c.best_value = neg2_fit;
  const double kInvPhi = 0.6180339887498949, kHalfWidth = 0.25;
  size_t k = 0;
  while (c.used < budget) {
    memcpy(g, c.best_genes, d * sizeof(double));
    const double blo = log10(lo[k]), bhi = log10(hi[k]);
    double a = c.best_genes[k] - kHalfWidth, b = c.best_genes[k] + kHalfWidth;
    double lo_k = blo > a ? blo : a;
    double hi_k = bhi < b ? bhi : b;
    double x1 = hi_k - kInvPhi * (hi_k - lo_k);
    double x2 = lo_k + kInvPhi * (hi_k - lo_k);
    g[k] = x1;
    double f1 = refine_eval(&c, g);
    if (c.used >= budget) break;
    g[k] = x2;
    double f2 = refine_eval(&c, g);
    for (int step = 0; step < 2 && c.used < budget; ++step) {
      if (f1 <= f2) {
        hi_k = x2;
        x2 = x1;
        f2 = f1;
        x1 = hi_k - kInvPhi * (hi_k - lo_k);
        g[k] = x1;
        f1 = refine_eval(&c, g);
      } else {
        lo_k = x1;
        x1 = x2;
        f1 = f2;
        x2 = lo_k + kInvPhi * (hi_k - lo_k);
        g[k] = x2;
        f2 = refine_eval(&c, g);
      }
    }
    k = (k + 1) % d;
  }
  for (size_t q = 0; q < d; ++q) theta_out[q] = pow(10.0, c.best_genes[q]);
  *neg2_out = c.best_value;
  *used_out = c.used;
  free(table);
  free(c.R);
  free(c.L);
  free(c.theta);
  free(c.best_genes);
  free(g);
  return 0;
}

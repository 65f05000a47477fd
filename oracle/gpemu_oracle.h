/*
 * gpemu_oracle.h -- CPU restatement of the reference gpemu hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_1203_1269_b200/,
 * include/) may link or call this. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it, and only as the
 * checker or the timed CPU baseline.
 *
 * Every function restates the reference algorithm (reference = /root/reference,
 * paths below relative to proj/include/gpemu/) in plain C, compiled with
 * -ffp-contract=off so products and sums round exactly as written (the
 * reference's "products rounded separately, summed in order" contract,
 * correlation.hpp:37-47). Pinned against the reference itself compiled from its
 * own headers (oracle/_ref, see oracle/Makefile) and against the reference
 * tests' known answers (tests/test_oracle.py).
 */
#ifndef GPEMU_ORACLE_H
#define GPEMU_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- detail/rng.hpp ---------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_rng;

uint64_t orc_mix64(uint64_t z);                                  /* rng.hpp:12-18 */
uint64_t orc_derive_seed1(uint64_t base);                        /* rng.hpp:20 */
uint64_t orc_derive_seed2(uint64_t base, uint64_t a);            /* rng.hpp:22-25 */
uint64_t orc_derive_seed3(uint64_t base, uint64_t a, uint64_t b);
void orc_rng_init(orc_rng* r, uint64_t seed);                    /* std::mt19937_64(seed) */
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);                            /* rng.hpp:37 */
double orc_rng_uniform(orc_rng* r, double lo, double hi);        /* rng.hpp:42 */
uint64_t orc_rng_below(orc_rng* r, uint64_t n);                  /* rng.hpp:46-48 */
double orc_rng_normal(orc_rng* r);                               /* rng.hpp:50-54 */

/* ---- experiment.hpp ----------------------------------------------------- */
int orc_maximin_lhd(size_t n, size_t d, uint64_t seed, size_t exchange_budget, double* X);
double orc_goldstein_price_log(const double* x);
double orc_hartman6(const double* x);
/* optimizer.hpp:62-80; rng seeded with `seed` directly */
void orc_lhs_population(const double* lo, const double* hi, size_t d, int count, uint64_t seed,
                        double* pop /* count x d */);

/* ---- correlation.hpp ---------------------------------------------------- */
double orc_pow_abs(double delta, double p);                      /* correlation.hpp:31-35 */
double orc_theta_weighted_sum(const double* theta, const double* terms, size_t d); /* :42-47 */
size_t orc_row_of_pair(size_t pair);                             /* :51-56 */
/* CorrelationPlan ctor (:156-180): pair-major table, pairs*d doubles. */
void orc_corr_table(const double* X, size_t n, size_t d, double p, double* table);
/* CorrelationPlan::build_into (:187-223): full n x n row-major R. Returns 0, or -1 non-finite. */
int orc_build_from_table(const double* table, size_t n, size_t d, const double* theta,
                         double nugget, double* R);
/* build_corr_matrix (:99-146). */
int orc_build_corr(const double* X, size_t n, size_t d, const double* theta, double p,
                   double nugget, double* R);
/* corr_vector (:67-91). */
int orc_corr_vector(const double* xstar, const double* X, size_t n, size_t d,
                    const double* theta, double p, double* r);

/* ---- backend.hpp -------------------------------------------------------- */
enum { ORC_REFERENCE = 0, ORC_PARALLEL = 1 };
/* ReferenceBackend::try_cholesky (:189-206) / ParallelBackend::try_cholesky (:226-311). 1 = ok. */
int orc_try_cholesky(double* A, size_t n, int kind);
/* Backend::factorize_into (:102-120). Returns 0 ok, 1 not-PD at every ladder step. */
int orc_factorize(const double* R, size_t n, int kind, double* L, double* log_det,
                  double* jitter_used);
void orc_solve_lower(const double* L, size_t n, const double* b, double* x); /* :129-140 */
void orc_solve_upper(const double* L, size_t n, const double* b, double* x); /* :143-153 */
double orc_dot_accumulate(const double* a, const double* b, size_t n);     /* matrix.hpp:64-69 */

/* ---- likelihood.hpp ----------------------------------------------------- */
typedef struct {
  double neg2_log_lik; /* +inf when every ladder step failed or vtv <= 0 */
  double mu_hat;
  double sigma2_hat;
  double jitter_used;
  double log_det;
  double factor_jitter; /* ladder step used when factorization succeeded, else -1 */
} orc_profile;

/* ProfileEvaluator::eval (:108-141) with a precomputed table. L_out (n*n) may be NULL. */
void orc_profile_eval_table(const double* table, const double* y, size_t n, size_t d,
                            double nugget, const double* theta, int kind, orc_profile* out,
                            double* L_work /* n*n scratch */, double* R_work /* n*n scratch */);
/* Batch of B thetas through one table (the reference evaluates them in order). */
int orc_profile_eval_batch(const double* X, const double* y, size_t n, size_t d, double p,
                           double nugget, const double* thetas, size_t B, int kind,
                           double* neg2, double* mu, double* sigma2, double* jitter,
                           double* log_det);

/* Extended-precision (long double) deviance of the reference's double R + jitter:
 * the "truth" the reference and the device both approximate. */
int orc_profile_eval_ld(const double* X, const double* y, size_t n, size_t d, double p,
                        double nugget, const double* thetas, size_t B, const double* jitters,
                        double* neg2_out);
/* ... plus the relative sensitivity of the deviance to 1-ulp perturbations of R. */
int orc_profile_sensitivity(const double* X, const double* y, size_t n, size_t d, double p,
                            double nugget, const double* thetas, size_t B, const double* jitters,
                            int reps, uint64_t seed, double* neg2_out, double* sens_out);

/* ---- optimizer.hpp + likelihood.hpp fit -------------------------------- */
typedef struct {
  int population, generations;
  double crossover_rate, mutation_sigma, mutation_prob;
  int elitism;
  uint64_t seed;
} orc_ga_config;

typedef double (*orc_objective)(const double* genes, void* ctx);

/* ga_minimize (optimizer.hpp:93-187). trace_best/trace_point: generations entries. */
int orc_ga_minimize(orc_objective f, void* ctx, const double* lo, const double* hi, size_t d,
                    const orc_ga_config* cfg, double* best_point, double* best_value,
                    double* trace_best, double* trace_point);

/* fit_gp_detailed (likelihood.hpp:243-303). theta bounds per dimension (not log10). */
typedef struct {
  double neg2_log_lik, mu_hat, sigma2_hat, jitter_max, log_det, jitter_used;
} orc_fit_result;
int orc_fit(const double* X, const double* y, size_t n, size_t d, double p, double nugget,
            const double* lo, const double* hi, const orc_ga_config* ga, uint64_t seed, int kind,
            double* theta_hat, orc_fit_result* res, double* alpha /* n */, double* L /* n*n or NULL */,
            double* trace_best /* generations */, double* trace_genes /* generations*d */);

/* bench.hpp:302-383 detail::refine_fit: coordinate-wise golden-section polish of theta
 * around a fitted optimum with exactly `budget` extra evaluations (the model rebuild at the
 * refined theta is left to the caller). theta_out / neg2_out = the polished incumbent. */
int orc_refine_fit(const double* X, const double* y, size_t n, size_t d, double p, double nugget,
                   const double* lo, const double* hi, const double* theta_fit, double neg2_fit,
                   int budget, int kind, double* theta_out, double* neg2_out, int* used_out);

/* ---- predictor.hpp ------------------------------------------------------ */
/* predict (:20-50): yhat_j = mu + dot_accumulate(r_j, alpha). */
int orc_predict(const double* X, size_t n, size_t d, const double* theta, double p, double mu,
                const double* alpha, const double* Xtest, size_t N, double* yhat);
double orc_sspe(const double* pred, const double* truth, size_t N);       /* :53-61 */
/* Kriging MSE (no reference implementation):
 * s2 = sigma2 * (1 - w'w + (1 - v'w)^2 / v'v), w = L^-1 r, v = L^-1 1. */
int orc_kriging_mse(const double* X, size_t n, size_t d, const double* theta, double p,
                    double sigma2, const double* L, const double* Xtest, size_t N, double* mse);

#ifdef __cplusplus
}
#endif
#endif

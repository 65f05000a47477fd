/*
 * gpemu_b200.h -- C-ABI of the B200-native gpemu hot path.
 *
 * Plain pointers and sizes only (no torch / CUDA types in the signatures).
 * Every call returns an int status (gpemu_status); gpemu_last_error() gives a
 * thread-local message. Host buffers are caller-allocated; ctx / plan / model
 * are opaque handles owned by the library. There is NO CPU fallback: every
 * compute entry point runs sm_100a kernels and fails with GPEMU_CUDA when no
 * usable device is present.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/proj/include/gpemu/):
 */
#ifndef GPEMU_B200_H
#define GPEMU_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GPEMU_API __attribute__((visibility("default")))
#else
#define GPEMU_API
#endif

/* errors.hpp:9-36 exception hierarchy as status codes */
typedef enum {
  GPEMU_OK = 0,
  GPEMU_VALIDATION = 1,  /* ValidationError */
  GPEMU_NOT_PD = 2,      /* NotPositiveDefiniteError */
  GPEMU_FIT = 3,         /* FitError */
  GPEMU_CONFIG = 4,      /* ConfigError */
  GPEMU_NONFINITE = 5,   /* Error("... non-finite correlation value") */
  GPEMU_CUDA = 6,        /* device / driver failure (Error) */
  GPEMU_ERROR = 7        /* any other Error */
} gpemu_status;

/* Per-candidate status word written by the device for every batch slot. */
typedef enum {
  GPEMU_SLOT_OK = 0,
  GPEMU_SLOT_NOT_PD = 1,    /* ladder exhausted -> neg2 = +inf (likelihood.hpp:115-119) */
  GPEMU_SLOT_NONFINITE = 2, /* non-finite R entry (correlation.hpp:222) */
  GPEMU_SLOT_DEGENERATE = 3 /* vtv <= 0 -> +inf (likelihood.hpp:127) */
} gpemu_slot_status;

typedef struct gpemu_ctx gpemu_ctx;
typedef struct gpemu_plan gpemu_plan;
typedef struct gpemu_model gpemu_model;

/* Cholesky engine selection (gpemu_ctx_set_engine). */
typedef enum {
  GPEMU_ENGINE_DAG = 0,    /* persistent tile-DAG, DMMA trailing updates (default) */
  GPEMU_ENGINE_SIMPLE = 1  /* one CTA per candidate, unblocked; validation engine */
} gpemu_engine;

GPEMU_API const char* gpemu_last_error(void);
GPEMU_API const char* gpemu_version(void);

/* -- context: one device, one stream ------------------------------------ */
GPEMU_API int gpemu_ctx_create(int device, gpemu_ctx** out);
GPEMU_API int gpemu_ctx_destroy(gpemu_ctx* ctx);
/* Use an external cudaStream_t (passed as void*); NULL restores the ctx's own. */
GPEMU_API int gpemu_ctx_set_stream(gpemu_ctx* ctx, void* stream);
GPEMU_API int gpemu_ctx_set_engine(gpemu_ctx* ctx, int engine);
/* Number of kernels this ctx has launched so far (bench accounting). */
GPEMU_API uint64_t gpemu_ctx_launch_count(const gpemu_ctx* ctx);
/* Streaming multiprocessors of the ctx's device (grid sizing; dag_profile buffer layout). */
GPEMU_API int gpemu_ctx_num_sms(const gpemu_ctx* ctx);

/* -- correlation.hpp ------------------------------------------------------ */
/* build_corr_matrix (correlation.hpp:99-146) / CorrelationPlan::build_into (:187-223):
 * R (n x n row-major, both triangles written) for one theta. */
GPEMU_API int gpemu_build_corr(gpemu_ctx* ctx, const double* X, size_t n, size_t d, const double* theta,
                     double p, double nugget, double* R_out);
/* corr_vector (correlation.hpp:67-91): r_i for one test point, no nugget. */
GPEMU_API int gpemu_corr_vector(gpemu_ctx* ctx, const double* xstar, const double* X, size_t n, size_t d,
                      const double* theta, double p, double* r_out);

/* -- backend.hpp ---------------------------------------------------------- */
/* Backend::factorize_into (backend.hpp:102-120): Cholesky of R + jitter I with the
 * kJitterLadder escalation. L_out: n x n row-major, lower triangle meaningful,
 * strict upper zeroed. Returns GPEMU_NOT_PD when the ladder is exhausted. */
GPEMU_API int gpemu_factorize(gpemu_ctx* ctx, const double* R, size_t n, double* L_out, double* log_det,
                    double* jitter_used);
/* Backend::try_cholesky (backend.hpp:174, the reference's one virtual compute hook):
 * ONE in-place attempt on A (n x n row-major, lower triangle read; on success the lower
 * triangle holds L and the strict upper is zeroed). GPEMU_NOT_PD when a pivot is not
 * strictly positive (NaN included); A is then unchanged. */
GPEMU_API int gpemu_try_cholesky(gpemu_ctx* ctx, double* A, size_t n);
/* Backend::solve_lower_into (:129-140) / solve_upper_into (:143-153). */
GPEMU_API int gpemu_solve_lower(gpemu_ctx* ctx, const double* L, size_t n, const double* b, double* x);
GPEMU_API int gpemu_solve_upper(gpemu_ctx* ctx, const double* L, size_t n, const double* b, double* x);

/* -- likelihood.hpp ------------------------------------------------------- */
/* ProfileEvaluator ctor (likelihood.hpp:77-91): uploads X, y, builds the
 * |dx|^p table on the device. max_batch bounds the candidates per eval call. */
GPEMU_API int gpemu_plan_create(gpemu_ctx* ctx, const double* X, const double* y, size_t n, size_t d,
                      double p, double nugget, size_t max_batch, gpemu_plan** out);

/* Working precision of a plan (core.hpp:86-96 Precision; FitConfig::precision). SINGLE runs
 * the reference's float instantiation: float design / table / R / factor / solves, log|R|
 * and the dots in double (likelihood.hpp:74-158, backend.hpp:111-113, matrix.hpp:64-69). */
typedef enum { GPEMU_PRECISION_DOUBLE = 0, GPEMU_PRECISION_SINGLE = 1 } gpemu_precision;

/* gpemu_plan_create with an explicit working precision. */
GPEMU_API int gpemu_plan_create_ex(gpemu_ctx* ctx, const double* X, const double* y, size_t n,
                                   size_t d, double p, double nugget, size_t max_batch,
                                   int precision, gpemu_plan** out);
GPEMU_API int gpemu_plan_precision(const gpemu_plan* plan);

/* Device memory: free / total bytes on the context's device (cudaMemGetInfo, plus the pages
 * the engine's memory pool keeps mapped for the next plan: plans and models allocate from a
 * per-device stream-ordered pool that is trimmed when a context is destroyed), and the bytes a
 * plan of (n, d, max_batch, precision) allocates (table + max_batch + 1 slots + flags), so a
 * caller can size max_batch to HBM. gpemu_fit evaluates a population larger than max_batch
 * in chunks (same candidates, same theta-hat). */
GPEMU_API int gpemu_ctx_mem_info(gpemu_ctx* ctx, size_t* free_bytes, size_t* total_bytes);
GPEMU_API size_t gpemu_plan_bytes(size_t n, size_t d, size_t max_batch, int precision);
GPEMU_API int gpemu_plan_destroy(gpemu_plan* plan);
GPEMU_API size_t gpemu_plan_device_bytes(const gpemu_plan* plan);

/* ProfileEvaluator::eval (likelihood.hpp:108-141), batched over B independent
 * thetas (host arrays). Any output pointer may be NULL. Per-slot results are
 * independent of B and of the slot index (batch invariance). */
GPEMU_API int gpemu_eval_batch(gpemu_plan* plan, const double* theta, size_t B, double* neg2, double* mu,
                     double* sigma2, double* jitter, double* log_det, int* slot_status);

/* Same on device memory: d_theta (B x d doubles), d_out (B x 8 doubles:
 * neg2, mu, sigma2, jitter, log_det, status, utu, vtv). Synchronises only to
 * run the jitter ladder (one B-int status read per ladder step). */
GPEMU_API int gpemu_eval_batch_device(gpemu_plan* plan, const double* d_theta, size_t B, double* d_out);

/* ProfileEvaluator::last_factor (likelihood.hpp:103) of a batch slot of the most
 * recent eval: L (n x n row-major, strict upper zero). */
GPEMU_API int gpemu_plan_last_factor(gpemu_plan* plan, size_t slot, double* L_out, double* log_det,
                           double* jitter_used);

/* Per-phase device timing (CUDA events on the plan's stream) for roofline
 * accounting: phase 0 = correlation assembly (K1), 1 = Cholesky engine (K2),
 * 2 = deviance finalisation (K3). Enabling clears previous marks. */
GPEMU_API int gpemu_plan_set_profiling(gpemu_plan* plan, int enable);
GPEMU_API int gpemu_plan_phase_ms(gpemu_plan* plan, int phase, double* total_ms, int* launches);
/* Diagnostics: per-CTA phase cycle counters of the DAG engine ([num_sms][16], see
 * kernels_chol.cu PR_*). enable=1 (re)arms and zeroes them; out (nullable) receives the
 * counters accumulated since; enable=0 disarms. */
GPEMU_API int gpemu_plan_dag_profile(gpemu_plan* plan, int enable, uint64_t* out, size_t out_len);
/* Diagnostics (host only, no device): the ticket order a large DAG launch of B candidates with
 * NT tile columns on `procs` CTAs uses (critical-path list schedule). out[B*NT*(NT+1)/2] gets
 * the packed tasks bpos << 16 | I << 8 | j in ticket order (I == j: DIAG). */
GPEMU_API int gpemu_ticket_order(int B, int NT, int procs, int* out, size_t out_len);

/* ---- optimizer.hpp / likelihood.hpp fit ------------------------------- */
typedef struct {
  int population;       /* GaConfig::population (100) */
  int generations;      /* GaConfig::generations (20) */
  double crossover_rate;/* 0.9 */
  double mutation_sigma;/* 0.15 */
  double mutation_prob; /* 0 -> 1/d */
  int elitism;          /* 1 */
} gpemu_ga_config;

typedef struct {
  double neg2_log_lik, mu_hat, sigma2_hat, jitter_max;
  uint64_t r_builds, factorizations, triangular_solves; /* Ledger (backend.hpp:26-49) */
} gpemu_fit_result;

/* fit_gp_detailed (likelihood.hpp:243-303): GA over log10(theta) in [lo, hi]
 * with one device batch per generation (chunks of max_batch if the population is larger); the stash keeps the earliest best
 * (generation, slot) exactly like the sequential reference. theta_hat (d),
 * alpha (n), trace_best (generations), trace_genes (generations*d) may be NULL.
 * model_out (nullable) receives a device-resident GpModel for gpemu_predict. */
GPEMU_API int gpemu_fit(gpemu_plan* plan, const double* lo, const double* hi, const gpemu_ga_config* ga,
              uint64_t seed, gpemu_fit_result* res, double* theta_hat, double* alpha,
              double* trace_best, double* trace_genes, gpemu_model** model_out);

/* Candidate sharding over G plans of the same dataset (one per device: gpemu_ctx_create(k),
 * gpemu_plan_create on it). optimizer.hpp:86-92 lets a generation be evaluated in parallel
 * (evaluate_population, :116-121); here candidate range k of ceil(P/G) runs on plans[k] from its
 * own host thread, each plan in chunks of its max_batch, and the records come back in slot
 * order. No device-to-device traffic: the fit's stash (likelihood.hpp:257-273, strict <,
 * earliest slot) keeps the winning factor on the device that produced it and the model is
 * built there. theta-hat, the trace and every record are bitwise those of gpemu_fit on one
 * plan (batch invariance). Plans must share n, d, X, y, p, nugget and precision. */
GPEMU_API int gpemu_eval_batch_multi(gpemu_plan* const* plans, int G, const double* theta, size_t B,
                                     double* neg2, double* mu, double* sigma2, double* jitter,
                                     double* log_det, int* slot_status);
GPEMU_API int gpemu_fit_multi(gpemu_plan* const* plans, int G, const double* lo, const double* hi,
                              const gpemu_ga_config* ga, uint64_t seed, gpemu_fit_result* res,
                              double* theta_hat, double* alpha, double* trace_best,
                              double* trace_genes, gpemu_model** model_out);

/* The reference GA (optimizer.hpp:93-187) as a host-only state machine (no device
 * needed): gpemu_ga_thetas gives the current generation's P candidates in theta space
 * (10^genes, likelihood.hpp:265), gpemu_ga_tell takes their -2logL and breeds the next
 * generation. The candidate sequence is the reference's for any split of a generation
 * across devices; the status reports the GA incumbent, the fit_gp_detailed stash
 * (generation, slot) and the GaTrace. gpemu_fit drives the same object. */
typedef struct gpemu_ga gpemu_ga;
GPEMU_API int gpemu_ga_create(size_t d, const double* lo, const double* hi, const gpemu_ga_config* cfg,
                    uint64_t seed, gpemu_ga** out);
GPEMU_API int gpemu_ga_destroy(gpemu_ga* ga);
GPEMU_API int gpemu_ga_thetas(const gpemu_ga* ga, double* thetas /* population x d */);
GPEMU_API int gpemu_ga_tell(gpemu_ga* ga, const double* fitness /* population */);
GPEMU_API int gpemu_ga_status(const gpemu_ga* ga, int* generation, int* done, double* best_value,
                    double* best_theta, int* stash_generation, int* stash_slot,
                    double* trace_best /* generations */, double* trace_genes /* generations x d */);

/* The bench protocol's post-GA polish (bench.hpp:302-383 detail::refine_fit): coordinate-
 * wise golden-section search in log10(theta), +-0.25 around the incumbent, exactly `budget`
 * sequential single-candidate evaluations. theta_out / neg2_out: the polished incumbent;
 * model_out (nullable) receives the model rebuilt at it when it improved on neg2_fit,
 * else NULL; scalars[4] = {neg2, mu, sigma2, jitter} and alpha[n] (both nullable) are
 * filled for the rebuilt model only. With a plan of max_batch >= 8 each coordinate's
 * decision tree (2 + 2 + 4 points) is evaluated in one batch and the sequential search is
 * replayed on those records. Batch invariance makes the result, evals_out and the plan's
 * ledger those of the one-at-a-time search. */
GPEMU_API int gpemu_refine_fit(gpemu_plan* plan, const double* lo, const double* hi,
                               const double* theta_fit, double neg2_fit, int budget,
                               double* theta_out, double* neg2_out, int* evals_out,
                               gpemu_model** model_out, double* scalars, double* alpha);
/* As gpemu_refine_fit, with the polish evaluations on `polish` (the reference polishes in
 * double regardless of the run precision, bench.hpp:300-301) and the model rebuilt on
 * `rebuild` in the run's own precision (bench.hpp:363-382); both plans hold the same data. */
GPEMU_API int gpemu_refine_fit_ex(gpemu_plan* polish, gpemu_plan* rebuild, const double* lo,
                                  const double* hi, const double* theta_fit, double neg2_fit,
                                  int budget, double* theta_out, double* neg2_out, int* evals_out,
                                  gpemu_model** model_out, double* scalars, double* alpha);

/* model_at_theta (likelihood.hpp:216-237). scalars: neg2, mu, sigma2, jitter. */
GPEMU_API int gpemu_model_at_theta(gpemu_plan* plan, const double* theta, gpemu_model** model_out,
                         double* scalars, double* alpha);
/* A model's scalars: out[4] = {neg2_log_lik, mu_hat, sigma2_hat, jitter_used}
 * (GpModel fields, likelihood.hpp:171-182; factor.jitter_used, backend.hpp:54-70). */
GPEMU_API int gpemu_model_scalars(const gpemu_model* model, double* out);
/* A model's factor (CorrelationFactor::lower, backend.hpp:54-70): L_out n x n row-major with the
 * strict upper zeroed (nullable: log_det only), log_det = log|R + jitter I|. */
GPEMU_API int gpemu_model_factor(gpemu_model* model, double* L_out, double* log_det);
/* A model's alpha = (R + jitter I)^-1 (y - mu 1) (GpModel::alpha, n doubles). */
GPEMU_API int gpemu_model_alpha(gpemu_model* model, double* alpha_out);
/* A device model from a GpModel assembled elsewhere (likelihood.hpp:171-182: the training inputs
 * X n x d, params theta / p, scalars[4] = {neg2_log_lik, mu_hat, sigma2_hat, jitter_used},
 * factor.log_det, factor.lower L n x n row-major (lower triangle read), alpha n). v = L^-1 1 for
 * the MSE is solved on the device. Lets predict() take any reference GpModel<double>. */
GPEMU_API int gpemu_model_import(gpemu_ctx* ctx, const double* X, size_t n, size_t d,
                                 const double* theta, double p, const double* scalars,
                                 double log_det, const double* L, const double* alpha,
                                 gpemu_model** out);
GPEMU_API int gpemu_model_destroy(gpemu_model* model);

/* ---- predictor.hpp ------------------------------------------------------ */
/* predict (predictor.hpp:20-50): yhat_j = mu + r(x_j)' alpha; mse (nullable) is the
 * kriging MSE sigma2 (1 - w'w + (1 - v'w)^2 / v'v), w = L^-1 r, v = L^-1 1
 * (no reference implementation). Validates the unit cube. */
GPEMU_API int gpemu_predict(gpemu_model* model, const double* Xtest, size_t N, double* yhat, double* mse);

/* -- experiment.hpp --------------------------------------------------------- */
/* maximin_lhd (experiment.hpp:142-172, DesignSpec :19-30): the random LHD and the swap draws on
 * the host with the reference's RNG (detail/rng.hpp), the O(n^2 d) tracker and the
 * exchange_budget swap scorings on the device. x_out: n x d row-major, bitwise the reference's
 * design. min_dist (nullable): the design's minimum squared pairwise distance (NaN when no
 * exchange ran: budget 0 or n == 2). */
GPEMU_API int gpemu_maximin_lhd(gpemu_ctx* ctx, size_t n, size_t d, uint64_t seed, size_t exchange_budget,
                                double* x_out, double* min_dist);

#ifdef __cplusplus
}
#endif
#endif /* GPEMU_B200_H */

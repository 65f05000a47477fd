// ref_shim.cpp -- C-ABI wrapper around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against
// /root/reference/proj/include (the reference's own sources, never copied)
// into oracle/_ref/libgpemu_ref*.so. Used (a) to pin the C restatement
// oracle/gpemu_oracle.c, (b) to generate tests/golden fixtures, and (c) as the
// timed CPU baseline in bench.py (cpu_baseline kind "reference").
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "gpemu/gpemu.hpp"

using namespace gpemu;

namespace {
thread_local std::string g_err;

int map_error(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ValidationError*>(&e)) return 1;
  if (dynamic_cast<const NotPositiveDefiniteError*>(&e)) return 2;
  if (dynamic_cast<const FitError*>(&e)) return 3;
  if (dynamic_cast<const ConfigError*>(&e)) return 4;
  return 5;
}

Matrix<double> to_matrix(const double* p, std::size_t r, std::size_t c) {
  Matrix<double> m(r, c);
  if (r * c) std::memcpy(m.data(), p, r * c * sizeof(double));
  return m;
}
}  // namespace

#define REF_TRY try {
#define REF_CATCH \
  }               \
  catch (const std::exception& e) { return map_error(e); }

#define REF_API __attribute__((visibility("default")))

extern "C" {

REF_API const char* ref_last_error() { return g_err.c_str(); }

REF_API std::uint64_t ref_derive_seed2(std::uint64_t b, std::uint64_t a) { return detail::derive_seed(b, a); }
REF_API std::uint64_t ref_derive_seed3(std::uint64_t b, std::uint64_t a, std::uint64_t c) {
  return detail::derive_seed(b, a, c);
}

// kind 0: next_u64 (as double bits), 1: uniform01, 2: normal, 3: below(arg)
REF_API void ref_rng_draws(std::uint64_t seed, int kind, std::uint64_t arg, std::size_t count, double* out) {
  detail::Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) {
    if (kind == 0) {
      std::uint64_t v = rng.next_u64();
      std::memcpy(&out[i], &v, 8);
    } else if (kind == 1) {
      out[i] = rng.uniform01();
    } else if (kind == 2) {
      out[i] = rng.normal();
    } else {
      out[i] = static_cast<double>(rng.below(arg));
    }
  }
}

REF_API int ref_maximin_lhd(std::size_t n, std::size_t d, std::uint64_t seed, std::size_t budget, double* X) {
  REF_TRY
  const auto m = maximin_lhd(DesignSpec{n, d, seed, budget});
  std::memcpy(X, m.data(), n * d * sizeof(double));
  return 0;
  REF_CATCH
}

REF_API double ref_goldstein_price_log(const double* x) { return goldstein_price_log(std::span<const double>(x, 2)); }
REF_API double ref_hartman6(const double* x) { return hartman6(std::span<const double>(x, 6)); }

REF_API void ref_lhs_population(const double* lo, const double* hi, std::size_t d, int count,
                        std::uint64_t seed, double* pop) {
  std::vector<std::pair<double, double>> b(d);
  for (std::size_t k = 0; k < d; ++k) b[k] = {lo[k], hi[k]};
  detail::Rng rng(seed);
  const auto P = detail::lhs_population(b, count, rng);
  for (int i = 0; i < count; ++i)
    for (std::size_t k = 0; k < d; ++k) pop[i * d + k] = P[i][k];
}

REF_API int ref_build_corr(const double* X, std::size_t n, std::size_t d, const double* theta, double p,
                   double nugget, double* R) {
  REF_TRY
  const auto r = build_corr_matrix(to_matrix(X, n, d),
                                   Hyperparameters{std::vector<double>(theta, theta + d), p, nugget});
  std::memcpy(R, r.values.data(), n * n * sizeof(double));
  return 0;
  REF_CATCH
}

REF_API int ref_plan_build(const double* X, std::size_t n, std::size_t d, const double* theta, double p,
                   double nugget, unsigned threads, double* R) {
  REF_TRY
  const auto x = to_matrix(X, n, d);
  detail::ThreadPool pool(threads);
  CorrelationPlan<double> plan(x, p, &pool);
  CorrelationMatrix<double> out;
  plan.build_into(out, std::span<const double>(theta, d), nugget, &pool);
  std::memcpy(R, out.values.data(), n * n * sizeof(double));
  return 0;
  REF_CATCH
}

REF_API int ref_corr_vector(const double* xstar, const double* X, std::size_t n, std::size_t d,
                    const double* theta, double p, double* r) {
  REF_TRY
  const auto v = corr_vector<double>(std::span<const double>(xstar, d), to_matrix(X, n, d),
                                     Hyperparameters{std::vector<double>(theta, theta + d), p, 0.0});
  std::memcpy(r, v.data(), n * sizeof(double));
  return 0;
  REF_CATCH
}

REF_API int ref_factorize(const double* R, std::size_t n, const char* backend, unsigned threads, double* L,
                  double* log_det, double* jitter) {
  REF_TRY
  auto be = make_backend<double>(backend, threads);
  CorrelationMatrix<double> r{to_matrix(R, n, n), 0.0};
  const auto f = be->factorize(r);
  std::memcpy(L, f.lower.data(), n * n * sizeof(double));
  *log_det = f.log_det;
  *jitter = f.jitter_used;
  return 0;
  REF_CATCH
}

REF_API int ref_solve(const double* L, std::size_t n, const double* b, int upper, double* x) {
  REF_TRY
  auto be = make_backend<double>("reference");
  CorrelationFactor<double> f;
  f.lower = to_matrix(L, n, n);
  if (upper) {
    be->solve_upper_into(f, std::span<const double>(b, n), std::span<double>(x, n));
  } else {
    be->solve_lower_into(f, std::span<const double>(b, n), std::span<double>(x, n));
  }
  return 0;
  REF_CATCH
}

// ProfileEvaluator::eval over B thetas (one evaluator: one plan, as in the fit).
// log_det may be NULL; it is read from last_factor() after each finite eval.
REF_API int ref_eval_batch(const double* X, const double* y, std::size_t n, std::size_t d, double p,
                   double nugget, const double* thetas, std::size_t B, const char* backend,
                   unsigned threads, double* neg2, double* mu, double* sigma2, double* jitter,
                   double* log_det) {
  REF_TRY
  auto be = make_backend<double>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  ProfileEvaluator<double> ev(data, p, nugget, *be);
  for (std::size_t b = 0; b < B; ++b) {
    const auto r = ev.eval(std::span<const double>(thetas + b * d, d));
    neg2[b] = r.neg2_log_lik;
    if (mu) mu[b] = r.mu_hat;
    if (sigma2) sigma2[b] = r.sigma2_hat;
    if (jitter) jitter[b] = r.jitter_used;
    if (log_det) log_det[b] = std::isfinite(r.neg2_log_lik) ? ev.last_factor().log_det : 0.0;
  }
  return 0;
  REF_CATCH
}

// Timed ProfileEvaluator::eval loop: plan construction and the B evaluations are
// timed separately (steady_clock), as BASELINE.md 3 prescribes for evals/s.
REF_API int ref_eval_batch_timed(const double* X, const double* y, std::size_t n, std::size_t d,
                                 double p, double nugget, const double* thetas, std::size_t B,
                                 const char* backend, unsigned threads, double* neg2,
                                 double* seconds_plan, double* seconds_evals) {
  REF_TRY
  auto be = make_backend<double>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  const auto t0 = std::chrono::steady_clock::now();
  ProfileEvaluator<double> ev(data, p, nugget, *be);
  const auto t1 = std::chrono::steady_clock::now();
  for (std::size_t b = 0; b < B; ++b) neg2[b] = ev.eval(std::span<const double>(thetas + b * d, d)).neg2_log_lik;
  const auto t2 = std::chrono::steady_clock::now();
  *seconds_plan = std::chrono::duration<double>(t1 - t0).count();
  *seconds_evals = std::chrono::duration<double>(t2 - t1).count();
  return 0;
  REF_CATCH
}

// fit_gp_detailed with the default GaConfig except population/generations.
REF_API int ref_fit(const double* X, const double* y, std::size_t n, std::size_t d, double p, double nugget,
            const double* lo, const double* hi, int population, int generations, std::uint64_t seed,
            const char* backend, unsigned threads, double* theta_hat, double* scalars /*neg2,mu,sigma2,jitter_max*/,
            double* alpha, double* trace_best, double* trace_genes) {
  REF_TRY
  auto be = make_backend<double>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  FitConfig cfg;
  cfg.ga.population = population;
  cfg.ga.generations = generations;
  cfg.seed = seed;
  cfg.p = p;
  cfg.nugget = nugget;
  cfg.theta_bounds.resize(d);
  for (std::size_t k = 0; k < d; ++k) cfg.theta_bounds[k] = {lo[k], hi[k]};
  const auto fit = fit_gp_detailed(data, cfg, *be);
  for (std::size_t k = 0; k < d; ++k) theta_hat[k] = fit.model.params.theta[k];
  scalars[0] = fit.model.neg2_log_lik;
  scalars[1] = fit.model.mu_hat;
  scalars[2] = fit.model.sigma2_hat;
  scalars[3] = fit.jitter_max;
  std::memcpy(alpha, fit.model.alpha.data(), n * sizeof(double));
  for (std::size_t g = 0; g < fit.trace.generations.size(); ++g) {
    if (trace_best) trace_best[g] = fit.trace.generations[g].best_value;
    if (trace_genes)
      for (std::size_t k = 0; k < d; ++k) trace_genes[g * d + k] = fit.trace.generations[g].best_point[k];
  }
  return 0;
  REF_CATCH
}

// fit_gp_detailed followed by the bench's golden-section polish (bench.hpp:302-383).
REF_API int ref_fit_refine(const double* X, const double* y, std::size_t n, std::size_t d, double p,
                           double nugget, const double* lo, const double* hi, int population,
                           int generations, std::uint64_t seed, int budget, unsigned threads,
                           double* theta_fit, double* theta_refined,
                           double* scalars /*neg2 fit, neg2 refined, extra evals*/) {
  REF_TRY
  auto be = make_backend<double>("parallel", threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  FitConfig cfg;
  cfg.backend = "parallel";
  cfg.ga.population = population;
  cfg.ga.generations = generations;
  cfg.seed = seed;
  cfg.p = p;
  cfg.nugget = nugget;
  cfg.theta_bounds.resize(d);
  for (std::size_t k = 0; k < d; ++k) cfg.theta_bounds[k] = {lo[k], hi[k]};
  auto fit = fit_gp_detailed(data, cfg, *be);
  for (std::size_t k = 0; k < d; ++k) theta_fit[k] = fit.model.params.theta[k];
  scalars[0] = fit.model.neg2_log_lik;
  std::uint64_t extra = 0;
  detail::refine_fit(fit, data, cfg, *be, budget, &extra);
  for (std::size_t k = 0; k < d; ++k) theta_refined[k] = fit.model.params.theta[k];
  scalars[1] = fit.model.neg2_log_lik;
  scalars[2] = static_cast<double>(extra);
  return 0;
  REF_CATCH
}

// model_at_theta + predict (predictor.hpp:20-50).
REF_API int ref_model_predict(const double* X, const double* y, std::size_t n, std::size_t d,
                      const double* theta, double p, double nugget, const char* backend,
                      unsigned threads, const double* Xtest, std::size_t N, double* yhat,
                      double* scalars /*neg2,mu,sigma2,jitter*/, double* alpha) {
  REF_TRY
  auto be = make_backend<double>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  const auto model = model_at_theta(data, std::span<const double>(theta, d), p, nugget, *be);
  if (scalars) {
    scalars[0] = model.neg2_log_lik;
    scalars[1] = model.mu_hat;
    scalars[2] = model.sigma2_hat;
    scalars[3] = model.factor.jitter_used;
  }
  if (alpha) std::memcpy(alpha, model.alpha.data(), n * sizeof(double));
  if (N) {
    const auto pr = predict(model, to_matrix(Xtest, N, d), be->pool());
    std::memcpy(yhat, pr.data(), N * sizeof(double));
  }
  return 0;
  REF_CATCH
}

// ---- single precision (Precision::kSingle, the reference's float instantiation) ----------
// ProfileEvaluator<float> / fit_gp_detailed<float> / model_at_theta<float> + predict, as the
// bench runs them for precision = single (bench.hpp:489-490).
REF_API int ref_eval_batch_f32(const double* X, const double* y, std::size_t n, std::size_t d, double p,
                               double nugget, const double* thetas, std::size_t B, const char* backend,
                               unsigned threads, double* neg2, double* mu, double* sigma2, double* jitter,
                               double* log_det) {
  REF_TRY
  auto be = make_backend<float>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  ProfileEvaluator<float> ev(data, p, nugget, *be);
  for (std::size_t b = 0; b < B; ++b) {
    const auto r = ev.eval(std::span<const double>(thetas + b * d, d));
    neg2[b] = r.neg2_log_lik;
    if (mu) mu[b] = r.mu_hat;
    if (sigma2) sigma2[b] = r.sigma2_hat;
    if (jitter) jitter[b] = r.jitter_used;
    if (log_det) log_det[b] = std::isfinite(r.neg2_log_lik) ? ev.last_factor().log_det : 0.0;
  }
  return 0;
  REF_CATCH
}

REF_API int ref_eval_batch_timed_f32(const double* X, const double* y, std::size_t n, std::size_t d,
                                     double p, double nugget, const double* thetas, std::size_t B,
                                     const char* backend, unsigned threads, double* neg2,
                                     double* seconds_plan, double* seconds_evals) {
  REF_TRY
  auto be = make_backend<float>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  const auto t0 = std::chrono::steady_clock::now();
  ProfileEvaluator<float> ev(data, p, nugget, *be);
  const auto t1 = std::chrono::steady_clock::now();
  for (std::size_t b = 0; b < B; ++b) neg2[b] = ev.eval(std::span<const double>(thetas + b * d, d)).neg2_log_lik;
  const auto t2 = std::chrono::steady_clock::now();
  *seconds_plan = std::chrono::duration<double>(t1 - t0).count();
  *seconds_evals = std::chrono::duration<double>(t2 - t1).count();
  return 0;
  REF_CATCH
}

REF_API int ref_fit_f32(const double* X, const double* y, std::size_t n, std::size_t d, double p, double nugget,
                        const double* lo, const double* hi, int population, int generations, std::uint64_t seed,
                        const char* backend, unsigned threads, double* theta_hat,
                        double* scalars /*neg2,mu,sigma2,jitter_max*/, double* alpha, double* trace_best) {
  REF_TRY
  auto be = make_backend<float>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  FitConfig cfg;
  cfg.precision = Precision::kSingle;
  cfg.ga.population = population;
  cfg.ga.generations = generations;
  cfg.seed = seed;
  cfg.p = p;
  cfg.nugget = nugget;
  cfg.theta_bounds.resize(d);
  for (std::size_t k = 0; k < d; ++k) cfg.theta_bounds[k] = {lo[k], hi[k]};
  const auto fit = fit_gp_detailed(data, cfg, *be);
  for (std::size_t k = 0; k < d; ++k) theta_hat[k] = fit.model.params.theta[k];
  scalars[0] = fit.model.neg2_log_lik;
  scalars[1] = fit.model.mu_hat;
  scalars[2] = fit.model.sigma2_hat;
  scalars[3] = fit.jitter_max;
  for (std::size_t i = 0; i < n; ++i) alpha[i] = static_cast<double>(fit.model.alpha[i]);
  for (std::size_t g = 0; g < fit.trace.generations.size(); ++g)
    if (trace_best) trace_best[g] = fit.trace.generations[g].best_value;
  return 0;
  REF_CATCH
}

REF_API int ref_model_predict_f32(const double* X, const double* y, std::size_t n, std::size_t d,
                                  const double* theta, double p, double nugget, const char* backend,
                                  unsigned threads, const double* Xtest, std::size_t N, double* yhat,
                                  double* scalars /*neg2,mu,sigma2,jitter*/, double* alpha) {
  REF_TRY
  auto be = make_backend<float>(backend, threads);
  const Dataset data = new_dataset(to_matrix(X, n, d), std::vector<double>(y, y + n));
  const auto model = model_at_theta(data, std::span<const double>(theta, d), p, nugget, *be);
  if (scalars) {
    scalars[0] = model.neg2_log_lik;
    scalars[1] = model.mu_hat;
    scalars[2] = model.sigma2_hat;
    scalars[3] = model.factor.jitter_used;
  }
  if (alpha)
    for (std::size_t i = 0; i < n; ++i) alpha[i] = static_cast<double>(model.alpha[i]);
  if (N) {
    const auto pr = predict(model, to_matrix(Xtest, N, d), be->pool());
    std::memcpy(yhat, pr.data(), N * sizeof(double));
  }
  return 0;
  REF_CATCH
}

}  // extern "C"

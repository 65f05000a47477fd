// test_dropin.cpp -- a reference program switched to the B200 by a namespace change.
//
// Every call below keeps the reference's own call shape (paths relative to
// /root/reference/proj/include/gpemu/):
//   ProfileEvaluator(const Dataset&, double p, double nugget, Backend&)   likelihood.hpp:77
//   neg2_log_profile(theta, data, cfg, backend)                          likelihood.hpp:161-166
//   model_at_theta(data, theta, p, nugget, backend)                      likelihood.hpp:216-218
//   fit_gp_detailed(data, cfg, backend) / fit_gp                         likelihood.hpp:243-308
//   predict(model, test_inputs, pool)                                    predictor.hpp:20-22
//   maximin_lhd(spec)                                                    experiment.hpp:142-172
// with `gpemu::` -> `gpemu_b200::` and the backend an AcceleratedBackend; results are compared
// with the reference's own ParallelBackend run of the same call (theta-hat and the GA trace
// bitwise, the Ledger equal) and the reference's own model_alpha_residual is applied to the
// device model. Test infrastructure: built by tests/cpp/Makefile, run by
// tests/test_cpp_plugin.py (GPU).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <initializer_list>
#include <limits>
#include <cstdio>
#include <span>
#include <vector>

#include "gpemu/gpemu.hpp"
#define GPEMU_REFERENCE_PLUGIN 1
#include "gpemu_b200.hpp"

using namespace gpemu;

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static double rel_diff(double a, double b) {  // test_helpers.hpp:14-17
  const double den = std::max(std::abs(a), std::abs(b));
  return den == 0.0 ? 0.0 : std::abs(a - b) / den;
}

static double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  double w = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - b[i]));
  return w;
}

static double max_abs(const std::vector<double>& a) {
  double w = 0.0;
  for (double v : a) w = std::max(w, std::abs(v));
  return w;
}

// The reference's own primitives at theta (build_corr_matrix, factorize, solves, dots:
// likelihood.hpp:108-141, :216-237; predictor.hpp:20-50), optionally with every off-diagonal R
// entry moved by one ulp (random sign, symmetric). The spread of these quantities under such a
// perturbation is how far any correct implementation may land from the reference: the device
// forms R with its own exp, within 1 ulp of the reference's.
struct RefRun {
  double neg2 = 0.0, mu = 0.0, log_det = 0.0, jitter = 0.0;
  std::vector<double> alpha, yhat;
  Matrix<double> L;
};

static RefRun ref_run(const Dataset& data, const std::vector<double>& theta, double p,
                      Backend<double>& be, const Matrix<double>& Xt, std::uint64_t perturb_seed) {
  const std::size_t n = data.n();
  auto R = build_corr_matrix(data.inputs(), Hyperparameters{theta, p, 0.0});
  if (perturb_seed) {
    detail::Rng rng(perturb_seed);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < i; ++j) {
        const double v = R.values(i, j);
        const double w = rng.uniform01() < 0.5 ? std::nextafter(v, 0.0) : std::nextafter(v, 2.0);
        R.values(i, j) = R.values(j, i) = w;
      }
  }
  const auto f = be.factorize(R);
  const auto& y = data.outputs();
  const std::vector<double> ones(n, 1.0);
  const auto u = be.solve_lower(f, y);
  const auto v = be.solve_lower(f, ones);
  const double utu = dot_accumulate<double>(u, u), vtu = dot_accumulate<double>(v, u),
               vtv = dot_accumulate<double>(v, v);
  RefRun r;
  r.mu = vtu / vtv;
  const double s2 = sigma2_hat_from_parts(utu, vtu, vtv, r.mu, n);
  r.log_det = f.log_det;
  r.jitter = f.jitter_used;
  r.neg2 = f.log_det + static_cast<double>(n) * std::log(std::max(static_cast<double>(n) * s2,
                                                                    std::numeric_limits<double>::min()));
  std::vector<double> rhs(n);
  for (std::size_t i = 0; i < n; ++i) rhs[i] = y[i] - r.mu;
  r.alpha = be.solve_full(f, rhs);
  r.L = f.dense_lower();
  const Hyperparameters hp{theta, p, 0.0};
  for (std::size_t j = 0; j < Xt.rows(); ++j) {
    const std::vector<double> x(Xt.data() + j * Xt.cols(), Xt.data() + (j + 1) * Xt.cols());
    const auto rv = corr_vector<double>(x, data.inputs(), hp);
    r.yhat.push_back(r.mu + dot_accumulate<double>(rv, r.alpha));
  }
  return r;
}

// max(floor, 10 x the largest change of a quantity under the perturbations / between the
// reference's two backends)
static double gate(double floor_, std::initializer_list<double> spreads) {
  double g = floor_;
  for (double v : spreads) g = std::max(g, 10.0 * v);
  return g;
}

static double max_abs_diff(const Matrix<double>& a, const Matrix<double>& b) {
  double w = 0.0;
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j <= i; ++j) w = std::max(w, std::abs(a(i, j) - b(i, j)));
  return w;
}

static double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  gpemu_b200::AcceleratedBackend acc(0);
  auto par = make_backend<double>("parallel", 0);
  auto seq = make_backend<double>("reference");

  // config C1: n=200, d=2, Goldstein-Price (log), p=2
  const Matrix<double> X = maximin_lhd(DesignSpec{200, 2, 7, 2000});
  const auto y = evaluate_test_function_rows(TestFunction::kGoldsteinPriceLog, X);
  const Dataset data = new_dataset(X, y);
  const auto Xt = maximin_lhd(DesignSpec{1000, 2, 11, 0});

  const Matrix<double> Xnone(0, 2);
  {  // ProfileEvaluator with the reference's constructor; gates from the reference's spread
    ProfileEvaluator<double> ep(data, 2.0, 0.0, *par);
    gpemu_b200::ProfileEvaluator ea(data, 2.0, 0.0, acc);
    for (double t : {0.05, 0.5, 3.0, 11.0}) {
      const std::vector<double> th{t, 2.0 * t};
      const ProfileEval a = ep.eval(th), b = ea.eval(th);
      const RefRun r0 = ref_run(data, th, 2.0, *seq, Xnone, 0), r1 = ref_run(data, th, 2.0, *seq, Xnone, 17),
                   r2 = ref_run(data, th, 2.0, *seq, Xnone, 29);
      CHECK(a.theta == b.theta);
      CHECK(a.jitter_used == b.jitter_used);
      const double g_neg2 = gate(1e-9, {rel_diff(r0.neg2, r1.neg2), rel_diff(r0.neg2, r2.neg2),
                                        rel_diff(a.neg2_log_lik, r0.neg2)});
      const double g_mu = gate(1e-9, {rel_diff(r0.mu, r1.mu), rel_diff(r0.mu, r2.mu), rel_diff(a.mu_hat, r0.mu)});
      CHECK(rel_diff(a.neg2_log_lik, b.neg2_log_lik) <= g_neg2);
      CHECK(rel_diff(a.mu_hat, b.mu_hat) <= g_mu);
      const auto& fa = ep.last_factor();
      const auto& fb = ea.last_factor();
      CHECK(fa.jitter_used == fb.jitter_used);
      CHECK(rel_diff(fa.log_det, fb.log_det) <=
            gate(1e-12, {rel_diff(r0.log_det, r1.log_det), rel_diff(r0.log_det, r2.log_det)}));
      if (rel_diff(a.neg2_log_lik, b.neg2_log_lik) > g_neg2 || rel_diff(a.mu_hat, b.mu_hat) > g_mu)
        std::printf("  theta %g: neg2 %.3e (gate %.1e), mu %.3e (gate %.1e)\n", t,
                    rel_diff(a.neg2_log_lik, b.neg2_log_lik), g_neg2, rel_diff(a.mu_hat, b.mu_hat), g_mu);
    }
    CHECK(ep.jitter_max() == ea.jitter_max());
    CHECK(par->ledger().snapshot().r_builds == acc.ledger().snapshot().r_builds);
    CHECK(par->ledger().snapshot().triangular_solves == acc.ledger().snapshot().triangular_solves);
  }
  {  // neg2_log_profile
    FitConfig cfg;
    cfg.p = 2.0;
    const std::vector<double> th{0.3, 4.0};
    const auto a = neg2_log_profile<double>(th, data, cfg, *par);
    const auto b = gpemu_b200::neg2_log_profile(th, data, cfg, acc);
    const RefRun r1 = ref_run(data, th, 2.0, *seq, Xnone, 5);
    CHECK(a.jitter_used == b.jitter_used);
    CHECK(rel_diff(a.neg2_log_lik, b.neg2_log_lik) <= gate(1e-9, {rel_diff(a.neg2_log_lik, r1.neg2)}));
  }

  // fit_gp_detailed: the full C1 GA (100 x 20)
  FitConfig cfg;
  cfg.p = 2.0;
  cfg.seed = 0;
  const auto led0_par = par->ledger().snapshot();
  const auto led0_acc = acc.ledger().snapshot();
  auto t0 = std::chrono::steady_clock::now();
  const FitResult<double> fr = fit_gp_detailed(data, cfg, *par);
  const double t_ref = secs_since(t0);
  t0 = std::chrono::steady_clock::now();
  const auto fa = gpemu_b200::fit_gp_detailed(data, cfg, acc);
  const double t_acc = secs_since(t0);
  CHECK(fa.model.params.theta == fr.model.params.theta);  // argmin bitwise
  CHECK(fa.trace.generations.size() == fr.trace.generations.size());
  for (std::size_t g = 0; g < fr.trace.generations.size(); ++g) {
    CHECK(fa.trace.generations[g].best_point == fr.trace.generations[g].best_point);
    CHECK(fa.trace.generations[g].evaluations == fr.trace.generations[g].evaluations);
    CHECK(rel_diff(fa.trace.generations[g].best_value, fr.trace.generations[g].best_value) < 1e-8);
  }
  CHECK(fa.jitter_max == fr.jitter_max);
  CHECK(fa.model.factor.jitter_used == fr.model.factor.jitter_used);
  CHECK(rel_diff(fa.model.neg2_log_lik, fr.model.neg2_log_lik) < 1e-8);
  {  // the Ledger counts the same cost model (2000 / 2000 / 4002)
    const auto a = par->ledger().snapshot(), b = acc.ledger().snapshot();
    CHECK(a.r_builds - led0_par.r_builds == b.r_builds - led0_acc.r_builds);
    CHECK(a.factorizations - led0_par.factorizations == b.factorizations - led0_acc.factorizations);
    CHECK(a.triangular_solves - led0_par.triangular_solves == b.triangular_solves - led0_acc.triangular_solves);
  }
  // the reference's own GpModel contract on the device model (likelihood.hpp:191-213)
  CHECK(model_alpha_residual(fa.model) <= 1e-6);
  const FitResult<double> sliced = fa;  // converts to the reference's type
  CHECK(sliced.model.params.theta == fr.model.params.theta);

  // predict: the reference's predictions on its own model vs the device model; the gate is the
  // reference's spread: ReferenceBackend vs ParallelBackend models at the same theta, and its
  // predictions from 1-ulp perturbations of R
  const auto pr = predict(fr.model, Xt, par->pool());
  const auto ms = model_at_theta<double>(data, fr.model.params.theta, 2.0, 0.0, *seq);
  const auto ps = predict(ms, Xt);
  const double scale = std::max(max_abs(pr), max_abs(y));
  const RefRun q1 = ref_run(data, fr.model.params.theta, 2.0, *seq, Xt, 11),
               q2 = ref_run(data, fr.model.params.theta, 2.0, *seq, Xt, 23);
  const double tol = gate(1e-8, {max_abs_diff(pr, ps) / scale, max_abs_diff(pr, q1.yhat) / scale,
                                 max_abs_diff(pr, q2.yhat) / scale});
  const auto pa = gpemu_b200::predict(fa.model, Xt, par->pool());
  CHECK(max_abs_diff(pa, pr) / scale <= tol);
  std::printf("predict at theta-hat: device %.2e, gate %.1e (reference backends %.2e, 1-ulp R %.2e)\n",
              max_abs_diff(pa, pr) / scale, tol, max_abs_diff(pr, ps) / scale,
              max_abs_diff(pr, q1.yhat) / scale);
  // predict on a plain reference GpModel (imported to the device)
  const auto pi = gpemu_b200::predict(fr.model, Xt, acc);
  CHECK(max_abs_diff(pi, pr) / scale <= tol);
  const auto set = gpemu_b200::predict_set(fa.model, Xt, pr);
  CHECK(set.predictions == pa && set.sspe >= 0.0);

  // model_at_theta with the reference call shape
  {
    const std::vector<double> th{0.7, 3.0};
    const GpModel<double> mr = model_at_theta<double>(data, th, 2.0, 0.0, *par);
    const auto ma = gpemu_b200::model_at_theta(data, th, 2.0, 0.0, acc);
    const RefRun r1 = ref_run(data, th, 2.0, *seq, Xnone, 3), r2 = ref_run(data, th, 2.0, *seq, Xnone, 9);
    CHECK(ma.factor.jitter_used == mr.factor.jitter_used);
    CHECK(rel_diff(ma.neg2_log_lik, mr.neg2_log_lik) <=
          gate(1e-9, {rel_diff(mr.neg2_log_lik, r1.neg2), rel_diff(mr.neg2_log_lik, r2.neg2)}));
    const double as = max_abs(mr.alpha);
    const double g_alpha = gate(1e-8, {max_abs_diff(mr.alpha, r1.alpha) / as, max_abs_diff(mr.alpha, r2.alpha) / as});
    CHECK(max_abs_diff(ma.alpha, mr.alpha) / as <= g_alpha);
    const double g_L = gate(1e-13, {max_abs_diff(mr.factor.lower, r1.L), max_abs_diff(mr.factor.lower, r2.L)});
    CHECK(max_abs_diff(ma.factor.lower, mr.factor.lower) <= g_L);
    std::printf("model_at_theta: alpha %.2e (gate %.1e), L %.2e (gate %.1e)\n",
                max_abs_diff(ma.alpha, mr.alpha) / as, g_alpha, max_abs_diff(ma.factor.lower, mr.factor.lower), g_L);
    CHECK(model_alpha_residual(ma) <= 1e-6);
    // coincident points: the jitter ladder gives the reference's step
    const Matrix<double> xc{{0.3, 0.3}, {0.3, 0.3}, {0.7, 0.1}};
    const std::vector<double> yc{1.0, 1.0, 0.0};
    const Dataset dc = new_dataset(xc, yc);
    const std::vector<double> thc{2.0, 2.0};
    CHECK(gpemu_b200::model_at_theta(dc, thc, 1.95, 0.0, acc).factor.jitter_used ==
          model_at_theta<double>(dc, thc, 1.95, 0.0, *par).factor.jitter_used);
  }

  // design generation with the reference's DesignSpec: bitwise the reference's design
  {
    for (const DesignSpec spec : {DesignSpec{200, 2, 7, 10000}, DesignSpec{1500, 8, 3, 3000}, DesignSpec{2, 3, 1, 50}}) {
      const auto t0 = std::chrono::steady_clock::now();
      const Matrix<double> xr = maximin_lhd(spec);
      const double tr = secs_since(t0);
      const auto t1 = std::chrono::steady_clock::now();
      const Matrix<double> xa = gpemu_b200::maximin_lhd(spec, acc);
      const double ta = secs_since(t1);
      CHECK(xa.rows() == xr.rows() && xa.cols() == xr.cols());
      CHECK(std::equal(xa.data(), xa.data() + xa.rows() * xa.cols(), xr.data()));
      std::printf("maximin_lhd n=%zu d=%zu budget=%zu: bitwise equal, reference %.3f s, device %.3f s\n", spec.n,
                  spec.d, spec.exchange_budget, tr, ta);
    }
  }

  // candidate sharding over two backends (two contexts; one device on this pool)
  {
    gpemu_b200::AcceleratedBackend acc2(0);
    gpemu_b200::AcceleratedBackend* bs[2] = {&acc, &acc2};
    const auto f2 = gpemu_b200::fit_gp_detailed(data, cfg, std::span<gpemu_b200::AcceleratedBackend* const>(bs, 2));
    CHECK(f2.model.params.theta == fr.model.params.theta);
    CHECK(f2.model.alpha == fa.model.alpha);
  }

  // the paper protocol's size (n=1024, Hartman-6): fit 100 x 20 wall time, reference vs device
  {
    const Matrix<double> X6 = maximin_lhd(DesignSpec{1024, 6, 3, 2000});
    const auto y6 = evaluate_test_function_rows(TestFunction::kHartman6, X6);
    const Dataset d6 = new_dataset(X6, y6);
    FitConfig c6;
    c6.seed = 2;
    t0 = std::chrono::steady_clock::now();
    const auto r6 = fit_gp_detailed(d6, c6, *par);
    const double tr6 = secs_since(t0);
    t0 = std::chrono::steady_clock::now();
    const auto a6 = gpemu_b200::fit_gp_detailed(d6, c6, acc);
    const double ta6 = secs_since(t0);
    CHECK(a6.model.params.theta == r6.model.params.theta);
    std::printf("fit_gp_detailed 100x20: n=200 reference %.3f s, b200 %.3f s; n=1024 d=6 reference %.3f s, b200 %.3f s\n",
                t_ref, t_acc, tr6, ta6);
  }

  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}

// test_plugin.cpp -- the reference's OWN code paths running on the B200 engine.
//
// Compiled against the unmodified reference headers (/root/reference/proj/include) with
// include/gpemu_b200.hpp; registers gpemu_b200::AcceleratedBackend in the reference's
// registry ("accelerated", backend.hpp:318-351) and drives the reference's factorize_into,
// ProfileEvaluator and fit_gp_detailed through it, mirroring test_backend.cpp. Also checks
// the batched C++ API (BatchEvaluator / fit_gp_detailed) against the reference.
// Test infrastructure: built by tests/cpp/Makefile, run by tests/test_cpp_plugin.py (GPU).
#include <cmath>
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

static Matrix<double> random_design(std::size_t n, std::size_t d, detail::Rng& rng) {
  Matrix<double> x(n, d);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t k = 0; k < d; ++k) x(i, k) = rng.uniform01();
  return x;
}

int main() {
  gpemu_b200::register_accelerated(0);
  auto acc = make_backend<double>("accelerated");
  CHECK(acc->kind() == BackendKind::kAccelerated);
  CHECK(acc->name() == "accelerated");

  {  // test_backend.cpp:36-56 known factors through the reference's factorize_into
    CorrelationMatrix<double> I2{Matrix<double>{{1.0, 0.0}, {0.0, 1.0}}, 0.0};
    const auto f = acc->factorize(I2);
    CHECK(f.lower(0, 0) == 1.0 && f.lower(1, 1) == 1.0 && f.lower(1, 0) == 0.0);
    CHECK(f.log_det == 0.0 && f.jitter_used == 0.0);
    CorrelationMatrix<double> r{Matrix<double>{{1.0, 0.5}, {0.5, 1.0}}, 0.0};
    const auto g = acc->factorize(r);
    CHECK(g.lower(0, 0) == 1.0 && g.lower(1, 0) == 0.5);
    CHECK(rel_diff(g.lower(1, 1), 0.8660254037844386) < 1e-15);
    CHECK(rel_diff(g.log_det, -0.2876820724517809) < 1e-12);
  }
  {  // :58-79 coincident points force the ladder (the reference loop drives our try_cholesky)
    const Matrix<double> x{{0.3, 0.3}, {0.3, 0.3}, {0.7, 0.1}};
    const auto r = build_corr_matrix(x, Hyperparameters{{2.0, 2.0}, 1.95, 0.0});
    const auto f = acc->factorize(r);
    CHECK(f.jitter_used > 0.0);
  }
  {  // :81-87 ladder exhaustion
    CorrelationMatrix<double> bad{Matrix<double>{{1.0, 2.0}, {2.0, 1.0}}, 0.0};
    bool threw = false;
    try {
      acc->factorize(bad);
    } catch (const NotPositiveDefiniteError&) {
      threw = true;
    }
    CHECK(threw);
    CHECK(acc->ledger().snapshot().factorizations == 4);
  }
  detail::Rng rng(13);
  auto ref = make_backend<double>("reference");
  for (std::size_t n : {7u, 64u, 130u, 300u}) {  // :198-230 backends agree
    const auto x = random_design(n, 2, rng);
    const auto r = build_corr_matrix(x, Hyperparameters{{20.0, 30.0}, 1.95, 0.0});
    const auto fr = ref->factorize(r);
    const auto fa = acc->factorize(r);
    CHECK(fr.jitter_used == fa.jitter_used);
    CHECK(rel_diff(fr.log_det, fa.log_det) < 1e-10);
    std::vector<double> b(n);
    for (auto& v : b) v = rng.uniform(-2.0, 2.0);
    const auto xr = ref->solve_full(fr, b);
    const auto xa = acc->solve_full(fa, b);
    double worst = 0.0;
    for (std::size_t i = 0; i < n; ++i) worst = std::max(worst, rel_diff(xr[i], xa[i]));
    CHECK(worst < 1e-6);
  }

  // ProfileEvaluator / fit_gp_detailed of the REFERENCE, Cholesky on the B200
  const Matrix<double> X = maximin_lhd(DesignSpec{200, 2, 7, 2000});
  const auto y = evaluate_test_function_rows(TestFunction::kGoldsteinPriceLog, X);
  const Dataset data = new_dataset(X, y);
  auto par = make_backend<double>("parallel", 2);
  {
    ProfileEvaluator<double> ep(data, 1.95, 0.0, *par), ea(data, 1.95, 0.0, *acc);
    for (double t : {0.05, 0.5, 3.0, 11.0}) {
      const std::vector<double> th{t, 2.0 * t};
      const auto a = ep.eval(th), b = ea.eval(th);
      CHECK(a.jitter_used == b.jitter_used);
      CHECK(rel_diff(a.neg2_log_lik, b.neg2_log_lik) < 1e-8);
    }
  }
  FitConfig cfg;
  cfg.ga.population = 16;
  cfg.ga.generations = 3;
  cfg.seed = 4;
  cfg.p = 1.95;
  const auto fp = fit_gp_detailed(data, cfg, *par);
  const auto fa = fit_gp_detailed(data, cfg, *acc);
  CHECK(fp.model.params.theta == fa.model.params.theta);  // argmin bitwise
  CHECK(rel_diff(fp.model.neg2_log_lik, fa.model.neg2_log_lik) < 1e-8);
  const auto Xt = maximin_lhd(DesignSpec{64, 2, 11, 0});
  const auto pp = predict(fp.model, Xt), pa = predict(fa.model, Xt);
  double worst = 0.0;
  for (std::size_t j = 0; j < pp.size(); ++j) worst = std::max(worst, std::abs(pp[j] - pa[j]));
  CHECK(worst < 1e-6);

  // the batched C++ API against the reference
  gpemu_b200::Context ctx(0);
  gpemu_b200::BatchEvaluator bev(ctx, std::span<const double>(X.data(), 400), y, 2, 1.95, 0.0, 16);
  std::vector<double> thetas;
  for (int i = 0; i < 16; ++i) {
    thetas.push_back(0.02 * (i + 1));
    thetas.push_back(0.7 * (16 - i));
  }
  const auto recs = bev.eval_batch(thetas);
  {
    ProfileEvaluator<double> ep(data, 1.95, 0.0, *par);
    for (int i = 0; i < 16; ++i) {
      const auto a = ep.eval(std::span<const double>(thetas.data() + 2 * i, 2));
      CHECK(a.jitter_used == recs[i].jitter_used);
      CHECK(rel_diff(a.neg2_log_lik, recs[i].neg2_log_lik) < 1e-8);
    }
  }
  const std::vector<double> lo{1e-6, 1e-6}, hi{12.0, 12.0};
  gpemu_b200::GaConfig ga;
  ga.population = 16;
  ga.generations = 3;
  const auto bf = gpemu_b200::fit_gp_detailed(bev, lo, hi, ga, 4);
  CHECK(bf.theta == fp.model.params.theta);  // same GA, same argmin as the reference fit
  const auto ph = gpemu_b200::predict(bf.model, std::span<const double>(Xt.data(), 128), 2);
  worst = 0.0;
  for (std::size_t j = 0; j < ph.size(); ++j) worst = std::max(worst, std::abs(pp[j] - ph[j]));
  CHECK(worst < 1e-6);

  // bench.hpp:302-383 refine_fit: the reference's own polish through the plugin
  // (cfg.backend = "accelerated") and gpemu_b200::refine_fit both reach the reference's
  // polished theta bitwise.
  {
    auto fr_ref = fit_gp_detailed(data, cfg, *par);
    std::uint64_t extra_ref = 0;
    detail::refine_fit(fr_ref, data, cfg, *par, 20, &extra_ref);
    FitConfig cfg_acc = cfg;
    cfg_acc.backend = "accelerated";
    auto fr_acc = fit_gp_detailed(data, cfg_acc, *acc);
    std::uint64_t extra_acc = 0;
    detail::refine_fit(fr_acc, data, cfg_acc, *acc, 20, &extra_acc);
    CHECK(fr_acc.model.params.theta == fr_ref.model.params.theta);
    CHECK(extra_acc == extra_ref);
    auto bf2 = gpemu_b200::fit_gp_detailed(bev, lo, hi, ga, 4);
    const std::size_t extra_dev = gpemu_b200::refine_fit(bev, bf2, lo, hi, 20);
    CHECK(bf2.theta == fr_ref.model.params.theta);
    CHECK(extra_dev == extra_ref);
    CHECK(rel_diff(bf2.neg2_log_lik, fr_ref.model.neg2_log_lik) < 1e-8);
  }

  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}

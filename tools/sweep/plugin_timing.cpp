// plugin_timing.cpp -- the reference's own fit_gp_detailed (likelihood.hpp:243-303) through
// its plugin slot: "accelerated" = gpemu_b200::AcceleratedBackend (try_cholesky on the B200,
// R and L crossing PCIe per call) vs the reference's ParallelBackend, and the batched
// gpemu_b200::fit_gp_detailed on the same data. Measurement tool for INTEGRATION.md.
//   usage: plugin_timing [n] [d] [population] [generations]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "gpemu/gpemu.hpp"
#define GPEMU_REFERENCE_PLUGIN 1
#include "gpemu_b200.hpp"

using namespace gpemu;

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 1024;
  const std::size_t d = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 6;
  const int pop = argc > 3 ? std::atoi(argv[3]) : 20;
  const int gens = argc > 4 ? std::atoi(argv[4]) : 5;
  gpemu_b200::register_accelerated(0);
  const auto X = maximin_lhd(DesignSpec{n, d, 5, 0});
  std::vector<double> y(n);
  for (std::size_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (std::size_t k = 0; k < d; ++k) s += std::sin(3.0 * X(i, k)) + 0.5 * X(i, k) * X(i, k);
    y[i] = s;
  }
  const Dataset data = new_dataset(X, y);
  FitConfig cfg;
  cfg.ga.population = pop;
  cfg.ga.generations = gens;
  cfg.seed = 1;
  cfg.p = 1.95;
  auto timed = [&](const char* id) {
    auto be = make_backend<double>(id, 0);
    const auto t0 = std::chrono::steady_clock::now();
    const auto fit = fit_gp_detailed(data, cfg, *be);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("%-12s n=%zu GA %dx%d: %.3f s  neg2 %.10g\n", id, n, pop, gens, s, fit.model.neg2_log_lik);
  };
  timed("accelerated");
  timed("parallel");
  gpemu_b200::Context ctx(0);
  gpemu_b200::BatchEvaluator ev(ctx, std::span<const double>(X.data(), n * d), y, d, 1.95, 0.0, pop);
  const std::vector<double> lo(d, 1e-6), hi(d, 12.0);
  gpemu_b200::GaConfig ga;
  ga.population = pop;
  ga.generations = gens;
  const auto t0 = std::chrono::steady_clock::now();
  const auto bf = gpemu_b200::fit_gp_detailed(ev, lo, hi, ga, 1);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("%-12s n=%zu GA %dx%d: %.3f s  neg2 %.10g\n", "batched", n, pop, gens, s, bf.neg2_log_lik);
  return 0;
}

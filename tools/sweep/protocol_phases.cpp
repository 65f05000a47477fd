// protocol_phases.cpp -- where one accelerated replication of the paper protocol
// (gpemu_b200_bench.hpp run_bench_cell_accelerated) spends its wall time: evaluator (plan)
// construction, the GA fit, refine_fit, predict and teardown, per n and replication.
//   usage: protocol_phases [function=goldstein_price_log] [reps=3] [n...]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "gpemu/gpemu.hpp"
#include "gpemu_b200_bench.hpp"

using clk = std::chrono::steady_clock;
static double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

int main(int argc, char** argv) {
  gpemu::BenchConfig cfg;
  cfg.function = gpemu::parse_test_function(argc > 1 ? argv[1] : "goldstein_price_log");
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  std::vector<std::size_t> sizes;
  for (int i = 3; i < argc; ++i) sizes.push_back(std::strtoul(argv[i], nullptr, 10));
  if (sizes.empty()) sizes = {128, 256, 512, 1024};
  const std::size_t d = gpemu::test_function_dim(cfg.function);
  gpemu_b200::Context ctx(0);
  std::printf("n,rep,construct_s,fit_s,refine_s,predict_s,teardown_s,total_s,neg2\n");
  for (std::size_t n : sizes) {
    for (int rep = 1; rep <= reps; ++rep) {
      gpemu::DesignSpec spec{n, d,
                             gpemu::detail::derive_seed(cfg.seed, 0xde51ull, static_cast<std::uint64_t>(n),
                                                        static_cast<std::uint64_t>(rep)),
                             cfg.exchange_budget};
      gpemu::Matrix<double> design = gpemu::maximin_lhd(spec);
      std::vector<double> y = gpemu::evaluate_test_function_rows(cfg.function, design);
      gpemu::Dataset data = gpemu::new_dataset(std::move(design), std::move(y));
      gpemu::DesignSpec tspec{cfg.test_points, d,
                              gpemu::detail::derive_seed(cfg.seed, 0x7e57ull, static_cast<std::uint64_t>(rep)),
                              cfg.exchange_budget};
      gpemu::Matrix<double> tx = gpemu::maximin_lhd(tspec);
      gpemu_b200::GaConfig ga;
      ga.population = cfg.ga_population;
      ga.generations = cfg.ga_generations;
      const std::uint64_t seed = gpemu::detail::derive_seed(cfg.seed, 0xf17ull, static_cast<std::uint64_t>(n),
                                                            static_cast<std::uint64_t>(rep));
      const std::vector<double> lo(d, cfg.theta_lower), hi(d, cfg.theta_upper);
      const auto& X = data.inputs();
      const auto t0 = clk::now();
      double neg2 = 0.0;
      clk::time_point t1, t2, t3, t4;
      {
        gpemu_b200::BatchEvaluator ev(ctx, std::span<const double>(X.data(), X.rows() * X.cols()),
                                      data.outputs(), d, 1.95, 0.0,
                                      static_cast<std::size_t>(ga.population));
        t1 = clk::now();
        gpemu_b200::FitResult fit = gpemu_b200::fit_gp_detailed(ev, lo, hi, ga, seed);
        t2 = clk::now();
        gpemu_b200::refine_fit(ev, fit, lo, hi, 20);
        t3 = clk::now();
        const auto pred = gpemu_b200::predict(fit.model, std::span<const double>(tx.data(), tx.rows() * tx.cols()),
                                              tx.cols());
        t4 = clk::now();
        neg2 = fit.neg2_log_lik;
      }
      const auto t5 = clk::now();
      std::printf("%zu,%d,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f,%.10g\n", n, rep, secs(t0, t1), secs(t1, t2),
                  secs(t2, t3), secs(t3, t4), secs(t4, t5), secs(t0, t5), neg2);
    }
  }
  return 0;
}

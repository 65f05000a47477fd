// gpemu_b200_bench.hpp -- the paper's benchmark protocol (bench.hpp:386-519) with the
// "accelerated" backend on the batched B200 path.
//
// The reference's run_bench_cell (bench.hpp:386-432) calls the NON-virtual
// fit_gp_detailed / refine_fit / predict, so through the plugin slot alone an
// "accelerated" row would move R and L over PCIe once per candidate. This header keeps the
// reference's sweep (same BenchConfig, seeds, designs, test sets, CSV rows and error
// behaviour) and runs the "accelerated" cells through one device batch per GA generation:
//   fit_gp_detailed -> gpemu_fit, refine_fit -> gpemu_refine_fit, predict -> gpemu_predict.
// "reference" / "parallel" cells are the reference's own run_bench_cell, unchanged.
//
// Requires the reference headers (gpemu/gpemu.hpp) to be included first. precision=single
// runs the accelerated cells on the FP32 engine (GPEMU_PRECISION_SINGLE) with the polish in
// double, as the reference does.
#pragma once

#ifndef GPEMU_REFERENCE_PLUGIN
#define GPEMU_REFERENCE_PLUGIN 1
#endif
#include <chrono>
#include <fstream>
#include <map>

#include "gpemu_b200.hpp"

namespace gpemu_b200 {

// run_bench_cell (bench.hpp:386-432) for backend "accelerated".
inline gpemu::BenchReportRow run_bench_cell_accelerated(Context& ctx, const gpemu::BenchConfig& cfg,
                                                        const gpemu::Dataset& data,
                                                        const gpemu::Matrix<double>& test_inputs,
                                                        std::span<const double> truth, std::size_t n,
                                                        int rep) {
  gpemu::BenchReportRow row;
  row.function = std::string(gpemu::test_function_name(cfg.function));
  row.backend = "accelerated";
  row.precision = std::string(gpemu::precision_name(cfg.precision));
  row.n = n;
  row.replication = rep;
  const bool single = cfg.precision == gpemu::Precision::kSingle;

  GaConfig ga;
  ga.population = cfg.ga_population;
  ga.generations = cfg.ga_generations;
  // bench.hpp:403-405: the fit seed depends on (base seed, n, replication), not the backend
  const std::uint64_t seed = gpemu::detail::derive_seed(cfg.seed, 0xf17ull, static_cast<std::uint64_t>(n),
                                                        static_cast<std::uint64_t>(rep));
  constexpr double kP = 1.95;  // bench.hpp:405
  const std::vector<double> lo(data.d(), cfg.theta_lower), hi(data.d(), cfg.theta_upper);
  row.eval_count = static_cast<std::uint64_t>(ga.population) * static_cast<std::uint64_t>(ga.generations);

  try {
    const auto t0 = std::chrono::steady_clock::now();
    const auto& X = data.inputs();
    const std::span<const double> Xs(X.data(), X.rows() * X.cols());
    BatchEvaluator ev(ctx, Xs, data.outputs(), data.d(), kP, 0.0,
                      static_cast<std::size_t>(ga.population),
                      single ? GPEMU_PRECISION_SINGLE : GPEMU_PRECISION_DOUBLE);
    FitResult fit = fit_gp_detailed(ev, lo, hi, ga, seed);
    if (cfg.refine) {
      if (single) {  // the polish runs in double whatever the run precision (bench.hpp:300)
        BatchEvaluator polish(ctx, Xs, data.outputs(), data.d(), kP, 0.0, 8);  // 8: speculative polish
        row.eval_count += refine_fit(ev, fit, lo, hi, 20, &polish);
      } else {
        row.eval_count += refine_fit(ev, fit, lo, hi, 20);
      }
    }
    const auto predictions = predict(
        fit.model, std::span<const double>(test_inputs.data(), test_inputs.rows() * test_inputs.cols()),
        test_inputs.cols());
    const auto t1 = std::chrono::steady_clock::now();
    row.wall_time_seconds = std::chrono::duration<double>(t1 - t0).count();
    row.neg2_log_lik = fit.neg2_log_lik;
    row.mu_hat = fit.mu_hat;
    row.sigma2_hat = fit.sigma2_hat;
    row.sspe = gpemu::sspe(predictions, truth);
    row.jitter_max = fit.jitter_max;
  } catch (const gpemu::Error& e) {
    row.failed = true;
    std::cerr << "bench: fit failed (" << row.function << ", n=" << n << ", rep=" << rep
              << ", backend=accelerated): " << e.what() << "\n";
  }
  return row;
}

// run_bench (bench.hpp:436-519): identical sweep order, seeds and CSV output; every
// "accelerated" cell runs on `device`. Replications run one after another (the reference's
// concurrent_replications only changes timing columns, bench.hpp:46-49; one device context
// serialises the accelerated cells anyway).
inline std::vector<gpemu::BenchReportRow> run_bench(const gpemu::BenchConfig& cfg,
                                                    std::ostream* progress = nullptr, int device = 0) {
  cfg.validate();
  const std::size_t d = gpemu::test_function_dim(cfg.function);
  std::unique_ptr<Context> ctx;
  for (const auto& b : cfg.backends)
    if (b == "accelerated" && !ctx) ctx = std::make_unique<Context>(device);

  std::ofstream out;
  if (!cfg.output_path.empty()) {
    out.open(cfg.output_path);
    if (!out) throw gpemu::ConfigError("bench: cannot open output file " + cfg.output_path);
    out << gpemu::kBenchCsvHeader << "\n" << std::flush;
  }
  std::map<int, std::pair<gpemu::Matrix<double>, std::vector<double>>> test_sets;
  auto test_set = [&](int rep) -> const std::pair<gpemu::Matrix<double>, std::vector<double>>& {
    auto it = test_sets.find(rep);
    if (it == test_sets.end()) {
      gpemu::DesignSpec spec{cfg.test_points, d,
                             gpemu::detail::derive_seed(cfg.seed, 0x7e57ull, static_cast<std::uint64_t>(rep)),
                             cfg.exchange_budget};
      gpemu::Matrix<double> x = gpemu::maximin_lhd(spec);
      std::vector<double> y = gpemu::evaluate_test_function_rows(cfg.function, x);
      it = test_sets.emplace(rep, std::make_pair(std::move(x), std::move(y))).first;
    }
    return it->second;
  };
  std::vector<gpemu::BenchReportRow> rows;
  auto emit = [&](gpemu::BenchReportRow row) {
    if (out.is_open()) out << gpemu::format_bench_row(row) << "\n" << std::flush;
    if (progress) {
      *progress << row.function << " n=" << row.n << " rep=" << row.replication
                << " backend=" << row.backend << (row.failed ? " FAILED" : "")
                << " time=" << row.wall_time_seconds << "s sspe=" << row.sspe << "\n";
    }
    rows.push_back(std::move(row));
  };
  for (std::size_t n : cfg.sizes) {
    for (int rep = 1; rep <= cfg.replications; ++rep) {
      gpemu::DesignSpec spec{n, d,
                             gpemu::detail::derive_seed(cfg.seed, 0xde51ull, static_cast<std::uint64_t>(n),
                                                        static_cast<std::uint64_t>(rep)),
                             cfg.exchange_budget};
      gpemu::Matrix<double> design = gpemu::maximin_lhd(spec);
      std::vector<double> y = gpemu::evaluate_test_function_rows(cfg.function, design);
      gpemu::Dataset data = gpemu::new_dataset(std::move(design), std::move(y));
      const auto& [test_inputs, truth] = test_set(rep);
      for (const auto& backend_id : cfg.backends) {
        if (backend_id == "accelerated") {
          emit(run_bench_cell_accelerated(*ctx, cfg, data, test_inputs, truth, n, rep));
        } else if (cfg.precision == gpemu::Precision::kSingle) {  // the reference's float cells
          emit(gpemu::detail::run_bench_cell<float>(cfg, data, test_inputs, truth, backend_id, n, rep));
        } else {
          emit(gpemu::detail::run_bench_cell<double>(cfg, data, test_inputs, truth, backend_id, n, rep));
        }
      }
    }
  }
  return rows;
}

}  // namespace gpemu_b200

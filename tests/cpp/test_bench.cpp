// test_bench.cpp -- the paper's benchmark sweep (bench.hpp:436-519) with "accelerated"
// cells on the batched B200 path (include/gpemu_b200_bench.hpp), against the reference's
// own "reference" and "parallel" cells on identical designs, seeds and test sets.
// Test infrastructure: built by tests/cpp/Makefile, run by tests/test_cpp_plugin.py (GPU).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>

#include "gpemu/gpemu.hpp"
#include "gpemu_b200_bench.hpp"

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

int main(int argc, char** argv) {
  gpemu_b200::register_accelerated(0);  // BenchConfig::validate accepts the id either way
  BenchConfig cfg;
  cfg.function = TestFunction::kGoldsteinPriceLog;
  cfg.sizes = {24, 60};
  cfg.replications = 2;
  cfg.backends = {"reference", "parallel", "accelerated"};
  cfg.seed = 11;
  cfg.ga_population = 24;
  cfg.ga_generations = 6;
  cfg.test_points = 300;
  cfg.exchange_budget = 500;
  cfg.refine = true;
  cfg.threads = 2;
  cfg.output_path = argc > 1 ? argv[1] : "/tmp/gpemu_bench_sweep.csv";
  const auto rows = gpemu_b200::run_bench(cfg, &std::cout);
  CHECK(rows.size() == 2 * 2 * 3);
  for (std::size_t i = 0; i + 2 < rows.size(); i += 3) {
    const auto &r = rows[i], &p = rows[i + 1], &a = rows[i + 2];
    CHECK(r.backend == "reference" && p.backend == "parallel" && a.backend == "accelerated");
    CHECK(a.n == r.n && a.replication == r.replication && a.precision == r.precision);
    CHECK(!a.failed && !r.failed);
    CHECK(a.eval_count == r.eval_count);  // 24*6 + 20 polish + 1 rebuild
    CHECK(a.jitter_max == r.jitter_max);
    // the SURVEY 8(c) gate at the optimum: max(1e-9, 10 x the reference's self-discrepancy)
    const double self = rel_diff(r.neg2_log_lik, p.neg2_log_lik);
    CHECK(rel_diff(a.neg2_log_lik, r.neg2_log_lik) <= std::max(1e-9, 10.0 * self));
    CHECK(rel_diff(a.mu_hat, r.mu_hat) <= std::max(1e-8, 10.0 * rel_diff(r.mu_hat, p.mu_hat)));
    CHECK(rel_diff(a.sspe, r.sspe) <= std::max(1e-6, 10.0 * rel_diff(r.sspe, p.sspe)));
    std::printf("n=%zu rep=%d neg2 ref %.12g acc %.12g (rel %.2e, self %.2e) sspe rel %.2e  "
                "wall ref %.3fs acc %.3fs\n",
                a.n, a.replication, r.neg2_log_lik, a.neg2_log_lik,
                rel_diff(a.neg2_log_lik, r.neg2_log_lik), self, rel_diff(a.sspe, r.sspe),
                r.wall_time_seconds, a.wall_time_seconds);
  }
  // the CSV contract (bench.hpp:97-99, :254-290) round-trips
  std::ifstream is(cfg.output_path);
  const auto parsed = parse_bench_csv(is);
  CHECK(parsed.size() == rows.size());
  for (std::size_t i = 0; i < parsed.size() && i < rows.size(); ++i) {
    CHECK(parsed[i].backend == rows[i].backend && parsed[i].eval_count == rows[i].eval_count);
    CHECK(parsed[i].neg2_log_lik == rows[i].neg2_log_lik);
  }
  const auto summary = summarize(rows);
  CHECK(!summary.empty());
  {  // precision = single: accelerated cells on the FP32 engine (polish in double) next to the
     // reference's float cells. Float GA trajectories may diverge (fitness noise ~1e-3), so the
     // rows are checked structurally and for a deviance of the same magnitude.
    BenchConfig sc = cfg;
    sc.precision = Precision::kSingle;
    sc.backends = {"parallel", "accelerated"};
    sc.sizes = {60};
    sc.output_path.clear();
    const auto srows = gpemu_b200::run_bench(sc, &std::cout);
    CHECK(srows.size() == 2 * 1 * 2);
    for (std::size_t i = 0; i + 1 < srows.size(); i += 2) {
      const auto &r = srows[i], &a = srows[i + 1];
      CHECK(a.precision == "single" && r.precision == "single");
      CHECK(!a.failed && !r.failed);
      CHECK(a.eval_count >= 24 * 6 + 20 && a.eval_count <= 24 * 6 + 21);
      CHECK(std::abs(a.neg2_log_lik - r.neg2_log_lik) <= 0.1 * std::abs(r.neg2_log_lik));
      std::printf("single n=%zu rep=%d neg2 ref %.6g acc %.6g\n", a.n, a.replication, r.neg2_log_lik,
                  a.neg2_log_lik);
    }
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}

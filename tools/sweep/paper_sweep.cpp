// paper_sweep.cpp -- the paper's benchmark protocol (bench.hpp:436-519) from a reference
// config file, with "accelerated" cells on the batched B200 path (include/gpemu_b200_bench.hpp)
// and the reference's own cells for the CPU backends. Measurement tool for SURVEY 8(f)-2/3:
// prints the per-row CSV (kBenchCsvHeader) and the reference's summary table.
//   usage: paper_sweep <config file> [rows.csv]
#include <cstdio>
#include <iostream>

#include "gpemu/gpemu.hpp"
#include "gpemu_b200_bench.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <config file> [rows.csv]\n", argv[0]);
    return 2;
  }
  try {
    gpemu_b200::register_accelerated(0);
    gpemu::BenchConfig cfg = gpemu::parse_bench_config_file(argv[1]);
    if (argc > 2) cfg.output_path = argv[2];
    const auto rows = gpemu_b200::run_bench(cfg, &std::cerr, 0);
    std::cout << gpemu::kBenchCsvHeader << "\n";
    for (const auto& r : rows) std::cout << gpemu::format_bench_row(r) << "\n";
    std::cout << "\n";
    gpemu::write_summary_csv(gpemu::summarize(rows, &std::cerr), std::cout);
  } catch (const gpemu::Error& e) {
    std::fprintf(stderr, "paper_sweep: %s\n", e.what());
    return 1;
  }
  return 0;
}

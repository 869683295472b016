// Drop-in check of the whole reference-side stack (TEST INFRASTRUCTURE).
//
// Compiled twice by oracle/Makefile (target `harness`) from the reference's
// UNMODIFIED harness headers in place under /root/reference (bench.hpp:97-185
// run_suite, testgen.hpp instance families T1-T6, io.hpp, active_set.hpp):
//   oracle/_ref/harness_ref : over the reference's own solver headers (CPU)
//   oracle/_ref/harness_gpu : over this repo's include/antilop facade, so every
//                             linalg / nqp / nnls / accelerated call the harness
//                             makes runs through libalnnls on the GPU
// and prints the suite's bench-report/1 JSON (bench.hpp:287-369). The two
// reports must agree bit for bit except for wall times (tests/test_ref_harness.py).
//
// usage: harness_xxx [n d sub_tests seed kinds solvers]      (suite -> bench-report/1 JSON)
//        harness_xxx gen KIND n d sparsity seed OUT_DIR        (bench.hpp cmd_generate)
//        harness_xxx solve SOLVER IN_DIR                       (bench.hpp cmd_solve: MatrixMarket
//                                                             instance in, trace CSV + result JSON out)
//   kinds = comma list of T1..T6, solvers = comma list of antilop,fast,accer,anti-accer
// (the reference's CLI front end needs CLI11, which is not vendored; these two
// subcommands call the same bench.hpp command bodies it would.)
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>

#include "antilop/bench.hpp"

namespace {
std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) out.push_back(t);
  return out;
}
}  // namespace

int main(int argc, char** argv) {
  using namespace antilop;
  const std::string cmd = argc > 1 ? argv[1] : "";
  if (cmd == "gen" && argc == 8) {
    bench::GenArgs g;
    g.spec.kind = testgen::parse_kind(argv[2]);
    g.spec.n = std::strtoul(argv[3], nullptr, 10);
    g.spec.d = std::strtoul(argv[4], nullptr, 10);
    g.spec.sparsity = std::strtod(argv[5], nullptr);
    g.spec.seed = std::strtoull(argv[6], nullptr, 10);
    g.out_dir = argv[7];
    return bench::cmd_generate(g, std::cout);
  }
  if (cmd == "solve" && argc == 4) {
    bench::SolveArgs a;
    a.solver = bench::parse_solver(argv[2]);
    a.in_dir = argv[3];
    a.config.time_cap = std::chrono::duration<double>(1e9);  // no wall-clock stop
    return bench::cmd_solve(a, std::cout);
  }
  bench::SuiteConfig c;
  c.n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 40;
  c.d = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 60;
  c.sub_tests = argc > 3 ? std::strtoul(argv[3], nullptr, 10) : 3;
  c.seed = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 1;
  if (argc > 5) {
    c.kinds.clear();
    for (const auto& k : split(argv[5])) c.kinds.push_back(testgen::parse_kind(k));
  }
  if (argc > 6) {
    c.solvers.clear();
    for (const auto& s : split(argv[6])) c.solvers.push_back(bench::parse_solver(s));
  }
  c.solver_config.time_cap = std::nullopt;  // deterministic: no wall-clock stop
  const bench::SuiteReport rep = bench::run_suite(c);
  bench::write_report_json(std::cout, rep);
  return 0;
}

#pragma once
// antilop/accelerated.hpp — B200 facade of the accelerated projected-gradient
// baseline (/root/reference/proj/include/antilop/accelerated.hpp:21-139):
// solve_accelerated (Nesterov momentum, fixed step 1/||Q||_F, optional restart)
// and solve_anti_accelerated (cosine rescale, then solve_accelerated). Each is
// one C-ABI call running the whole loop on the GPU, bit for bit the reference.

#include <vector>

#include "antilop/linalg.hpp"
#include "antilop/nnls.hpp"
#include "antilop/nqp.hpp"

namespace antilop {

inline SolveResult solve_accelerated(const NqpProblem& p, const SolverConfig& config = {}) {
  const std::size_t n = p.dim();
  config.resolve_epsilon(n);
  config.resolve_max_iters(n);
  alnnls_config cfg = b200::to_abi(config);
  cfg.record_multiplies = 0;
  alnnls_summary s{};
  const int st =
      alnnls_solve_accelerated(b200::ctx(), n, p.Q.data().data(), p.q.data().data(), &cfg, &s);
  b200::check_solve(st, s);
  return b200::fetch_result(s, false, nullptr);
}

inline NnlsResult solve_anti_accelerated(const DenseMatrix& a, const Vector& b,
                                         const SolverConfig& config = {}) {
  detail::require(a.rows() == b.size(), "solve_anti_accelerated: A and b dimension mismatch");
  alnnls_config cfg = b200::to_abi(config);
  cfg.record_multiplies = 0;
  alnnls_summary s{};
  const int st = alnnls_solve_anti_accelerated(b200::ctx(), a.rows(), a.cols(), a.data().data(),
                                               b.data().data(), &cfg, &s);
  b200::check_solve(st, s);
  NnlsResult out;
  std::vector<double> x(a.cols());
  b200::check(alnnls_get_x(b200::ctx(), x.data(), x.size()));
  out.x = Vector(std::move(x));
  out.residual_sq = s.residual_sq;
  std::vector<uint64_t> drop(s.n_dropped ? s.n_dropped : 1);
  b200::check(alnnls_get_dropped(b200::ctx(), drop.data(), s.n_dropped));
  out.dropped_columns.assign(drop.begin(), drop.begin() + s.n_dropped);
  out.inner = b200::fetch_result(s, true, nullptr);
  return out;
}

}  // namespace antilop

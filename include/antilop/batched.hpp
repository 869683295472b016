#pragma once
// antilop/batched.hpp — batched multi-RHS NNLS: one
// solve_nnls(A, B[:, j], config) per column of B with ONE shared Gram, sharded
// by column over `num_gpus` GPUs (one context per device, one host thread per
// GPU, no collective: alnnls_solve_nnls_batched_multi). The reference has no
// batched function; its equivalent is a loop of solve_nnls over the columns
// (nnls.hpp:129-144), which recomputes the Gram per column. Under the EXACT
// profile column j is bitwise that call.
//
// Per column the result is compact (the batched kernel keeps no per-column
// trace): termination, iterations, residual, final objective and gradient norm.

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "antilop/nnls.hpp"

namespace antilop {

struct ColumnSummary {
  Termination termination = Termination::EmptyPassiveSet;
  std::size_t iterations = 0;
  double residual_sq = 0.0;     // ||A x_j - b_j||^2 (nnls.hpp:115-123)
  double f = 0.0;               // last trace record's objective (rescaled space)
  double grad_bar_sq = 0.0;     // last trace record's ||g_P||^2
  std::uint64_t multiplies = 0; // sum of multiplies_per_iter
};

struct BatchedNnlsResult {
  DenseMatrix X;                       // n x nrhs, column j = solve_nnls(A, B[:, j]).x
  std::vector<ColumnSummary> columns;  // per column of B
};

namespace b200 {

// One context per device for the batched multi-GPU entry (devices 0..k-1),
// created on first use and kept for the process (guarded: the C contexts are
// single-threaded, so concurrent batched calls serialize here).
struct DevicePool {
  std::mutex mu;
  std::vector<std::unique_ptr<Context>> ctxs;
};
inline DevicePool& device_pool() {
  static DevicePool p;
  return p;
}

}  // namespace b200

inline BatchedNnlsResult solve_nnls_batched(const DenseMatrix& a, const DenseMatrix& b,
                                            const SolverConfig& config = {}, int num_gpus = 1) {
  detail::require(a.rows() == b.rows(), "solve_nnls: A and b dimension mismatch");
  detail::require(num_gpus >= 1, "solve_nnls_batched: num_gpus must be >= 1");
  const int visible = alnnls_device_count();
  if (visible < num_gpus)
    throw std::invalid_argument("solve_nnls_batched: num_gpus exceeds the visible GPUs");
  const std::size_t n = a.cols(), k = b.cols();
  std::vector<double> x(n * k);
  std::vector<alnnls_column_result> cols(k);
  alnnls_config cfg = b200::to_abi(config);
  cfg.record_multiplies = 0;
  alnnls_summary s{};
  auto& pool = b200::device_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  while ((int)pool.ctxs.size() < num_gpus)
    pool.ctxs.emplace_back(new b200::Context((int)pool.ctxs.size()));
  std::vector<alnnls_ctx*> raw;
  for (int g = 0; g < num_gpus; ++g) raw.push_back(pool.ctxs[g]->get());
  const int st = alnnls_solve_nnls_batched_multi(raw.data(), num_gpus, a.rows(), n,
                                                 a.data().data(), k, b.data().data(), &cfg,
                                                 x.data(), cols.data(), &s);
  if (st != ALNNLS_OK) {
    const std::string msg = alnnls_last_error(raw[0]);
    if (st == ALNNLS_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("alnnls status " + std::to_string(st) + ": " + msg);
  }
  BatchedNnlsResult out{DenseMatrix(n, k, std::move(x)), {}};
  out.columns.reserve(k);
  for (const auto& c : cols) {
    if (c.numeric_failure)
      throw NumericFailure("solve_nqp: non-finite objective or gradient", {});
    ColumnSummary cs;
    cs.termination = static_cast<Termination>(c.termination);
    cs.iterations = c.iterations;
    cs.residual_sq = c.residual_sq;
    cs.f = c.f_final;
    cs.grad_bar_sq = c.gbs_final;
    cs.multiplies = c.multiplies_total;
    out.columns.push_back(cs);
  }
  return out;
}

/// NMF by alternating NNLS (the use that motivates the batched
/// solver): V (d x N) ~ W H with W, H >= 0. Each outer iteration is
/// two batched solves on this thread's GPU context: H from W (one solve_nnls per
/// column of V) and W from H^T (one per row of V); objective[t] = ||V - W H||_F^2
/// after iteration t's H update. W0 (d x k, nonnegative) is the start.
struct NmfResult {
  DenseMatrix W;
  DenseMatrix H;
  std::vector<double> objective;
};

inline NmfResult nmf(const DenseMatrix& v, const DenseMatrix& w0, std::size_t outer_iters,
                     const SolverConfig& config = {}) {
  detail::require(v.rows() == w0.rows(), "nmf: V and W dimension mismatch");
  const std::size_t d = v.rows(), n = v.cols(), k = w0.cols();
  std::vector<double> w(w0.data().begin(), w0.data().end()), h(k * n);
  std::vector<double> obj(outer_iters ? outer_iters : 1);
  alnnls_config cfg = b200::to_abi(config);
  cfg.record_multiplies = 0;
  b200::check(alnnls_nmf(b200::ctx(), d, n, k, v.data().data(), w.data(), h.data(), outer_iters,
                         &cfg, obj.data()));
  obj.resize(outer_iters);
  return NmfResult{DenseMatrix(d, k, std::move(w)), DenseMatrix(k, n, std::move(h)), std::move(obj)};
}

}  // namespace antilop

#pragma once
// antilop/nnls.hpp — B200 facade of the NNLS front end
// (/root/reference/proj/include/antilop/nnls.hpp:32-153). solve_nnls is ONE
// C-ABI call (alnnls_solve_nnls): Gram + A^T b (exact SYRK / column chains),
// cosine rescale fused into the Gram epilogue, the device-resident loop,
// unscale and the residual recomputed from A and b — all on the GPU.

#include <optional>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "antilop/linalg.hpp"
#include "antilop/nqp.hpp"

namespace antilop {

struct ScaledSystem {
  std::optional<NqpProblem> problem;
  Vector scale;                       // D over retained columns
  std::vector<std::size_t> retained;  // reduced index -> original index
  std::vector<std::size_t> dropped;   // original indices with H_ii == 0
};

/// Cosine rescale of (H, h) (reference nnls.hpp:41-83), computed on the GPU.
inline ScaledSystem rescale(const DenseMatrix& h_mat, const Vector& h_vec) {
  const std::size_t n = h_mat.rows();
  detail::require(h_mat.cols() == n, "rescale: H must be square");
  detail::require(h_vec.size() == n, "rescale: H and h dimension mismatch");
  alnnls_summary s{};
  b200::check(alnnls_rescale(b200::ctx(), n, h_mat.data().data(), h_vec.data().data(), &s));
  ScaledSystem sys;
  const std::size_t m = s.m;
  std::vector<double> scale(m ? m : 1);
  std::vector<uint64_t> ret(m ? m : 1), drop(s.n_dropped ? s.n_dropped : 1);
  b200::check(alnnls_get_scale(b200::ctx(), scale.data(), m));
  b200::check(alnnls_get_retained(b200::ctx(), ret.data(), m));
  b200::check(alnnls_get_dropped(b200::ctx(), drop.data(), s.n_dropped));
  scale.resize(m);
  sys.scale = Vector(std::move(scale));
  sys.retained.assign(ret.begin(), ret.begin() + m);
  sys.dropped.assign(drop.begin(), drop.begin() + s.n_dropped);
  if (m > 0) {
    std::vector<double> Q(m * m), q(m);
    b200::check(alnnls_get_Q(b200::ctx(), Q.data(), m * m));
    b200::check(alnnls_get_q(b200::ctx(), q.data(), m));
    sys.problem.emplace(DenseMatrix(m, m, std::move(Q)), Vector(std::move(q)));
  }
  return sys;
}

/// x_i = y_a / D_a on retained columns, 0 on dropped ones (nnls.hpp:87-96).
inline Vector unscale(const Vector& y, const ScaledSystem& sys, std::size_t n) {
  detail::require(y.size() == sys.retained.size(), "unscale: dimension mismatch");
  Vector x(n);
  for (std::size_t a = 0; a < y.size(); ++a) {
    detail::require(sys.retained[a] < n, "unscale: retained index out of range");
    x[sys.retained[a]] = y[a] / sys.scale[a];
  }
  return x;
}

namespace detail {

inline SolveResult empty_solve_result() {  // nnls.hpp:107-113
  SolveResult r;
  r.termination = Termination::EmptyPassiveSet;
  r.trace.push_back({0, 0.0, 0.0, 0, std::chrono::duration<double>{0.0}, std::nullopt});
  r.min_iterate = 0.0;
  return r;
}

/// ||A x - b||^2 (nnls.hpp:115-123): the O(d n) product on the GPU (matvec, one
/// ordered chain per row), the O(d) ordered sum of squares here, as the reference.
inline double residual_norm_sq(const DenseMatrix& a, const Vector& b, const Vector& x) {
  const Vector ax = matvec(a, x);
  double s = 0.0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    const double r = ax[i] - b[i];
    s += r * r;
  }
  return s;
}

}  // namespace detail

struct NnlsResult {
  Vector x;
  double residual_sq = 0.0;
  SolveResult inner;
  std::vector<std::size_t> dropped_columns;
};

/// Full pipeline on the GPU (nnls.hpp:129-144).
inline NnlsResult solve_nnls(const DenseMatrix& a, const Vector& b,
                             const SolverConfig& config = {}) {
  detail::require(a.rows() == b.size(), "solve_nnls: A and b dimension mismatch");
  alnnls_config cfg = b200::to_abi(config);
  alnnls_summary s{};
  const int st = alnnls_solve_nnls(b200::ctx(), a.rows(), a.cols(), a.data().data(),
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

/// {"residual_sq","iterations","termination","dropped_columns"} (nnls.hpp:146-153);
/// keys in the same (sorted) order and number format nlohmann::json emits them.
inline std::string result_summary_json(const NnlsResult& r) {
  std::ostringstream os;
  os << "{\"dropped_columns\":[";
  for (std::size_t i = 0; i < r.dropped_columns.size(); ++i)
    os << (i ? "," : "") << r.dropped_columns[i];
  os << "],\"iterations\":" << r.inner.iterations()
     << ",\"residual_sq\":" << detail::json_number(r.residual_sq) << ",\"termination\":\""
     << to_string(r.inner.termination) << "\"}";
  return os.str();
}

}  // namespace antilop

// The batched multi-RHS entry (a18) rides on the same facade.
#include "antilop/batched.hpp"

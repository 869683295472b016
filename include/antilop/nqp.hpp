#pragma once
// antilop/nqp.hpp — B200 facade of the NQP solver API
// (/root/reference/proj/include/antilop/nqp.hpp:30-357): same types and
// signatures; solve_nqp runs the device-resident exact loop through the C ABI
// (alnnls_solve_nqp) and returns the reference's trajectory bit for bit.

#include <algorithm>
#if !defined(ANTILOP_NO_NLOHMANN)
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#elif __has_include("json.hpp")
#include "json.hpp"
#endif
#endif
#include <charconv>
#include <chrono>
#include <cmath>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <optional>
#include <ostream>
#include <string>
#include <string_view>
#include <vector>

#include "antilop/io.hpp"  // as the reference's nqp.hpp:23: fmt_g17 and the file I/O
#include "antilop/linalg.hpp"

namespace antilop {

/// min 1/2 x^T Q x + q^T x, Q square and exactly symmetric (reference nqp.hpp:30-45).
struct NqpProblem {
  DenseMatrix Q;
  Vector q;

  NqpProblem(DenseMatrix Q_, Vector q_) : Q(std::move(Q_)), q(std::move(q_)) {
    detail::require(Q.rows() == Q.cols(), "NqpProblem: Q must be square");
    detail::require(Q.rows() == q.size(), "NqpProblem: Q and q dimension mismatch");
    for (std::size_t j = 1; j < Q.cols(); ++j)
      for (std::size_t i = 0; i < j; ++i)
        detail::require(Q(i, j) == Q(j, i), "NqpProblem: Q must be symmetric");
  }
  std::size_t dim() const noexcept { return q.size(); }
};

enum class Termination {
  EmptyPassiveSet,
  GradientBelowEpsilon,
  MaxIters,
  TimeCap,
  Stalled,
  ZeroCurvature,
};

inline std::string_view to_string(Termination t) {
  static constexpr std::string_view names[] = {"EmptyPassiveSet", "GradientBelowEpsilon",
                                               "MaxIters",        "TimeCap",
                                               "Stalled",         "ZeroCurvature"};
  const auto i = static_cast<std::size_t>(t);
  return i < 6 ? names[i] : std::string_view("Unknown");
}

/// Stopping controls (reference nqp.hpp:71-99).
struct SolverConfig {
  std::optional<double> epsilon;
  std::optional<std::size_t> max_iters;
  std::optional<std::chrono::duration<double>> time_cap;
  std::size_t stall_window = 50;
  std::size_t trace_every = 1;
  bool nesterov_restart = false;
  std::optional<double> active_set_tol;

  double resolve_epsilon(std::size_t n) const {
    if (!epsilon) return 1e-10 * static_cast<double>(n);
    detail::require(*epsilon > 0.0, "SolverConfig: epsilon must be > 0");
    return *epsilon;
  }
  std::size_t resolve_max_iters(std::size_t n) const {
    if (!max_iters) return 5 * n;
    detail::require(*max_iters >= 1, "SolverConfig: max_iters must be >= 1");
    return *max_iters;
  }
};

struct IterRecord {
  std::size_t iter = 0;
  double f = 0.0;
  double grad_bar_sq = 0.0;
  std::size_t passive_count = 0;
  std::chrono::duration<double> elapsed{0.0};
  std::optional<double> alpha;
};

using SolveTrace = std::vector<IterRecord>;

struct SolveResult {
  Vector x;
  SolveTrace trace;
  Termination termination = Termination::MaxIters;
  Vector final_grad;
  double min_iterate = std::numeric_limits<double>::infinity();
  std::size_t iterations() const { return trace.empty() ? 0 : trace.back().iter; }
};

struct SolveStats {
  std::vector<std::size_t> multiplies_per_iter;
};

class NumericFailure : public std::runtime_error {
 public:
  NumericFailure(const std::string& what, SolveTrace trace)
      : std::runtime_error(what), trace_(std::move(trace)) {}
  const SolveTrace& trace() const noexcept { return trace_; }

 private:
  SolveTrace trace_;
};

namespace b200 {

inline alnnls_config to_abi(const SolverConfig& c) {
  alnnls_config a;
  alnnls_config_default(&a);
  a.has_epsilon = c.epsilon.has_value();
  a.epsilon = c.epsilon.value_or(0.0);
  a.has_max_iters = c.max_iters.has_value();
  a.max_iters = c.max_iters.value_or(0);
  a.has_time_cap = c.time_cap.has_value();
  a.time_cap_s = c.time_cap ? c.time_cap->count() : 0.0;
  a.stall_window = c.stall_window;
  a.trace_every = c.trace_every;
  a.nesterov_restart = c.nesterov_restart ? 1 : 0;
  return a;
}

inline SolveTrace fetch_trace(std::size_t len) {
  std::vector<alnnls_iter_record> recs(len ? len : 1);
  check(alnnls_get_trace(ctx(), recs.data(), len));
  SolveTrace t;
  t.reserve(len);
  for (std::size_t i = 0; i < len; ++i) {
    const auto& r = recs[i];
    IterRecord ir;
    ir.iter = r.iter;
    ir.f = r.f;
    ir.grad_bar_sq = r.grad_bar_sq;
    ir.passive_count = r.passive_count;
    ir.elapsed = std::chrono::duration<double>(r.elapsed_s);
    if (r.has_alpha) ir.alpha = r.alpha;
    t.push_back(ir);
  }
  return t;
}

// Solve result of the last solve on this thread's context (inner = rescaled space).
inline SolveResult fetch_result(const alnnls_summary& s, bool nnls, SolveStats* stats) {
  SolveResult r;
  std::vector<double> x(s.m), g(s.m);
  if (s.m) {
    check(nnls ? alnnls_get_inner_x(ctx(), x.data(), s.m) : alnnls_get_x(ctx(), x.data(), s.m));
    check(alnnls_get_final_grad(ctx(), g.data(), s.m));
  }
  r.x = Vector(std::move(x));
  r.final_grad = Vector(std::move(g));
  r.trace = fetch_trace(s.trace_len);
  r.termination = static_cast<Termination>(s.termination);
  r.min_iterate = s.min_iterate;
  if (stats) {
    std::vector<uint64_t> m(s.mult_len ? s.mult_len : 1);
    check(alnnls_get_multiplies(ctx(), m.data(), s.mult_len));
    stats->multiplies_per_iter.assign(m.begin(), m.begin() + s.mult_len);
  }
  return r;
}

// ENUMERIC -> NumericFailure with the trace so far; anything else via check().
inline void check_solve(int st, const alnnls_summary& s) {
  if (st == ALNNLS_ENUMERIC) throw NumericFailure(last_error(), fetch_trace(s.trace_len));
  check(st);
}

}  // namespace b200

/// Passive set {i : x_i > 0 or g_i < 0}, ascending (reference nqp.hpp:149-157).
inline std::vector<std::size_t> passive_mask(const Vector& x, const Vector& grad) {
  detail::require(x.size() == grad.size(), "passive_mask: length mismatch");
  std::vector<std::size_t> p;
  for (std::size_t i = 0; i < x.size(); ++i)
    if (x[i] > 0.0 || grad[i] < 0.0) p.push_back(i);
  return p;
}

/// alpha = ||g||^2 / g^T Q g over the mask; empty if g^T Q g <= 0 (nqp.hpp:162-173).
inline std::optional<double> exact_step(const DenseMatrix& Q, const Vector& grad_bar,
                                        std::span<const std::size_t> mask,
                                        std::size_t* multiply_count = nullptr) {
  double num = 0.0;
  for (std::size_t i : mask) num += grad_bar[i] * grad_bar[i];
  if (num == 0.0) return std::nullopt;
  const Vector qg = masked_matvec(Q, grad_bar, mask, multiply_count);
  double den = 0.0;
  for (std::size_t i : mask) den += grad_bar[i] * qg[i];
  if (!(den > 0.0)) return std::nullopt;
  return num / den;
}

inline std::optional<double> exact_step(const DenseMatrix& Q, const Vector& grad_bar) {
  std::vector<std::size_t> nz;
  for (std::size_t i = 0; i < grad_bar.size(); ++i)
    if (grad_bar[i] != 0.0) nz.push_back(i);
  return exact_step(Q, grad_bar, nz);
}

/// 1/2 x^T Q x + q^T x (nqp.hpp:183-186).
inline double objective(const NqpProblem& p, const Vector& x) {
  detail::require(x.size() == p.dim(), "objective: dimension mismatch");
  return 0.5 * dot(x, matvec(p.Q, x)) + dot(p.q, x);
}

/// KKT residual, infinity when x is infeasible (nqp.hpp:190-207).
inline double kkt_error(const NqpProblem& p, const Vector& x) {
  detail::require(x.size() == p.dim(), "kkt_error: dimension mismatch");
  Vector g = matvec(p.Q, x);
  for (std::size_t i = 0; i < g.size(); ++i) g[i] += p.q[i];
  double e = 0.0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    if (x[i] < 0.0) return std::numeric_limits<double>::infinity();
    e = std::max(e, x[i] > 0.0 ? std::abs(g[i]) : std::max(0.0, -g[i]));
  }
  return e;
}

/// Projected gradient with exact masked line search (nqp.hpp:215-339), on the GPU.
inline SolveResult solve_nqp(const NqpProblem& p, const SolverConfig& config = {},
                             const std::optional<Vector>& start = std::nullopt,
                             SolveStats* stats = nullptr) {
  const std::size_t n = p.dim();
  config.resolve_epsilon(n);
  config.resolve_max_iters(n);
  if (start) {
    detail::require(start->size() == n, "solve_nqp: start dimension mismatch");
    for (double v : *start) detail::require(v >= 0.0, "solve_nqp: start must be nonnegative");
  }
  alnnls_config cfg = b200::to_abi(config);
  cfg.record_multiplies = stats != nullptr;
  alnnls_summary s{};
  const int st = alnnls_solve_nqp(b200::ctx(), n, p.Q.data().data(), p.q.data().data(),
                                  start ? start->data().data() : nullptr, &cfg, &s);
  b200::check_solve(st, s);
  return b200::fetch_result(s, false, stats);
}

// ---- trace serialization (nqp.hpp:345-357): %.17g, alpha blank on the final record
namespace detail {

// A double the way the reference's nlohmann::json dump() writes it (nnls.hpp:146-153
// serializes through it). With nlohmann/json on the include path (the reference's own
// dependency) this IS nlohmann's dump(). Without it: the shortest round-trip digits
// (std::to_chars) laid out like nlohmann's dtoa_impl::format_buffer (fixed notation
// for decimal exponents in (-4, 15], else d.ddde+XX with at least two exponent digits;
// "0.0" for zero, ".0" on integers, "null" for non-finite values) -- identical except
// for the last digit of the ~0.3% of values where Grisu2's digits are not Ryu's.
inline std::string json_number(double v) {
#if defined(NLOHMANN_JSON_VERSION_MAJOR) && !defined(ANTILOP_NO_NLOHMANN)
  return nlohmann::json(v).dump();
#endif
  if (!std::isfinite(v)) return "null";
  std::string out;
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) return out + "0.0";
  char sci[64];
  const auto res = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  const std::string s(sci, res.ptr);
  const std::size_t e = s.find('e');
  std::string digits;
  for (std::size_t i = 0; i < e; ++i)
    if (s[i] != '.') digits += s[i];
  const int k = static_cast<int>(digits.size());
  const int n = std::stoi(s.substr(e + 1)) + 1;  // decimal point position
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) return out + digits + std::string(n - k, '0') + ".0";
  if (0 < n && n <= kMaxExp) return out + digits.substr(0, n) + "." + digits.substr(n);
  if (kMinExp < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
  out += digits.substr(0, 1);
  if (k > 1) out += "." + digits.substr(1);
  int x = n - 1;
  out += x < 0 ? "e-" : "e+";
  x = x < 0 ? -x : x;
  if (x < 10) out += '0';
  return out + std::to_string(x);
}
}  // namespace detail

inline void write_trace_csv(std::ostream& os, const SolveTrace& trace) {
  os << "iter,elapsed_ms,f,grad_bar_sq,passive_count,alpha\n";
  for (const auto& r : trace) {
    os << r.iter << ',' << fmt_g17(r.elapsed.count() * 1e3) << ',' << fmt_g17(r.f) << ','
       << fmt_g17(r.grad_bar_sq) << ',' << r.passive_count << ','
       << (r.alpha ? fmt_g17(*r.alpha) : std::string()) << '\n';
  }
}

inline void write_trace_csv_file(const std::filesystem::path& path, const SolveTrace& trace) {
  auto f = detail::open_out(path);
  write_trace_csv(f, trace);
}

}  // namespace antilop

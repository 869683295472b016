// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. Compiles the UNMODIFIED reference
// headers (/root/reference/proj/include/antilop/*.hpp, read in place, never
// copied) into oracle/_ref/libantilop_ref.so with the namespace renamed to
// antilop_ref (-Dantilop=antilop_ref) and the reference's own Release flags
// (-O3 -DNDEBUG -std=gnu++20, no -march; reference CMakeLists.txt:8-10).
// It exports the ref_* twins declared in oracle/antilop_oracle.h so tests can
// pin the C restatement against the reference itself, and bench.py can time
// the reference CPU solver (`--impl reference`).
#include <algorithm>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "antilop/accelerated.hpp"
#include "antilop/nnls.hpp"

#include "antilop_oracle.h"

namespace R = antilop_ref;

namespace {

int set_err(oracle_out* out, int code, const char* msg) {
  if (out) {
    std::strncpy(out->error, msg, sizeof(out->error) - 1);
    out->error[sizeof(out->error) - 1] = 0;
  }
  return code;
}

R::SolverConfig to_cfg(const alnnls_config* c) {
  R::SolverConfig s;
  if (c->has_epsilon) s.epsilon = c->epsilon;
  if (c->has_max_iters) s.max_iters = static_cast<std::size_t>(c->max_iters);
  if (c->has_time_cap) s.time_cap = std::chrono::duration<double>(c->time_cap_s);
  s.stall_window = static_cast<std::size_t>(c->stall_window);
  s.trace_every = static_cast<std::size_t>(c->trace_every);
  s.nesterov_restart = c->nesterov_restart != 0;
  return s;
}

R::DenseMatrix make_matrix(uint64_t rows, uint64_t cols, const double* p) {
  return R::DenseMatrix(rows, cols, std::vector<double>(p, p + rows * cols));
}

R::Vector make_vector(uint64_t n, const double* p) {
  return R::Vector(std::vector<double>(p, p + n));
}

void fill_trace(const R::SolveTrace& tr, oracle_out* out) {
  out->summary.trace_len = tr.size();
  if (!out->trace) return;
  for (std::size_t i = 0; i < tr.size() && i < out->trace_cap; ++i) {
    alnnls_iter_record& r = out->trace[i];
    r.iter = tr[i].iter;
    r.f = tr[i].f;
    r.grad_bar_sq = tr[i].grad_bar_sq;
    r.passive_count = tr[i].passive_count;
    r.elapsed_s = tr[i].elapsed.count();
    r.has_alpha = tr[i].alpha.has_value() ? 1 : 0;
    r.alpha = tr[i].alpha.value_or(0.0);
  }
}

void fill_result(const R::SolveResult& res, const R::SolveStats& stats, oracle_out* out) {
  fill_trace(res.trace, out);
  out->summary.termination = static_cast<int32_t>(res.termination);
  out->summary.iterations = res.iterations();
  out->summary.min_iterate = res.min_iterate;
  out->summary.f_final = res.trace.empty() ? 0.0 : res.trace.back().f;
  out->summary.gbs_final = res.trace.empty() ? 0.0 : res.trace.back().grad_bar_sq;
  out->summary.mult_len = stats.multiplies_per_iter.size();
  uint64_t tot = 0;
  for (std::size_t i = 0; i < stats.multiplies_per_iter.size(); ++i) {
    tot += stats.multiplies_per_iter[i];
    if (out->mults && i < out->mults_cap) out->mults[i] = stats.multiplies_per_iter[i];
  }
  out->summary.multiplies_total = tot;
  if (out->final_grad) {
    for (std::size_t i = 0; i < res.final_grad.size() && i < out->vec_cap; ++i)
      out->final_grad[i] = res.final_grad[i];
  }
}

template <class F>
int guarded(oracle_out* out, F&& f) {
  try {
    return f();
  } catch (const R::NumericFailure& e) {
    if (out) {
      fill_trace(e.trace(), out);
      out->summary.numeric_failure = 1;
    }
    return set_err(out, ALNNLS_ENUMERIC, e.what());
  } catch (const std::invalid_argument& e) {
    return set_err(out, ALNNLS_EINVAL, e.what());
  } catch (const std::out_of_range& e) {
    return set_err(out, ALNNLS_ERANGE, e.what());
  } catch (const std::exception& e) {
    return set_err(out, ALNNLS_EINVAL, e.what());
  }
}

}  // namespace

extern "C" {

int ref_gram(uint64_t d, uint64_t n, const double* A, double* H) {
  return guarded(nullptr, [&] {
    const auto h = R::gram(make_matrix(d, n, A));
    std::memcpy(H, h.data().data(), sizeof(double) * n * n);
    return 0;
  });
}

int ref_transpose_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                         double* y) {
  return guarded(nullptr, [&] {
    const auto r = R::transpose_matvec(make_matrix(rows, cols, M), make_vector(rows, v));
    std::memcpy(y, r.data().data(), sizeof(double) * cols);
    return 0;
  });
}

int ref_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v, double* y) {
  return guarded(nullptr, [&] {
    const auto r = R::matvec(make_matrix(rows, cols, M), make_vector(cols, v));
    std::memcpy(y, r.data().data(), sizeof(double) * rows);
    return 0;
  });
}

int ref_masked_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                      const uint64_t* mask, uint64_t mask_len, double* y,
                      uint64_t* multiply_count) {
  return guarded(nullptr, [&] {
    std::vector<std::size_t> mk(mask, mask + mask_len);
    std::size_t cnt = multiply_count ? *multiply_count : 0;
    const auto r = R::masked_matvec(make_matrix(rows, cols, M), make_vector(cols, v), mk,
                                    multiply_count ? &cnt : nullptr);
    if (multiply_count) *multiply_count = cnt;
    std::memcpy(y, r.data().data(), sizeof(double) * rows);
    return 0;
  });
}

int ref_rescale(uint64_t n, const double* H, const double* h, double* Q, double* q,
                oracle_out* out) {
  return guarded(out, [&] {
    const auto sys = R::rescale(make_matrix(n, n, H), make_vector(n, h));
    const uint64_t m = sys.retained.size();
    if (sys.problem) {
      std::memcpy(Q, sys.problem->Q.data().data(), sizeof(double) * m * m);
      std::memcpy(q, sys.problem->q.data().data(), sizeof(double) * m);
    }
    if (out) {
      out->summary.n = n;
      out->summary.m = m;
      out->summary.n_dropped = sys.dropped.size();
      if (out->retained) std::copy(sys.retained.begin(), sys.retained.end(), out->retained);
      if (out->dropped) std::copy(sys.dropped.begin(), sys.dropped.end(), out->dropped);
      if (out->scale) std::copy(sys.scale.begin(), sys.scale.end(), out->scale);
    }
    return 0;
  });
}

int ref_solve_nqp(uint64_t m, const double* Q, const double* q, const double* start,
                  const alnnls_config* cfg, oracle_out* out) {
  return guarded(out, [&] {
    R::NqpProblem p(make_matrix(m, m, Q), make_vector(m, q));
    std::optional<R::Vector> st;
    if (start) st = make_vector(m, start);
    R::SolveStats stats;
    const auto res = R::solve_nqp(p, to_cfg(cfg), st, &stats);
    if (out) {
      fill_result(res, stats, out);
      out->summary.m = m;
      out->summary.n = m;
      if (out->x) std::memcpy(out->x, res.x.data().data(), sizeof(double) * m);
    }
    return 0;
  });
}

int ref_solve_nnls(uint64_t d, uint64_t n, const double* A, const double* b,
                   const alnnls_config* cfg, oracle_out* out) {
  return guarded(out, [&] {
    const auto a = make_matrix(d, n, A);
    const auto bv = make_vector(d, b);
    const auto res = R::solve_nnls(a, bv, to_cfg(cfg));
    if (out) {
      R::SolveStats none;
      fill_result(res.inner, none, out);
      out->summary.n = n;
      out->summary.n_dropped = res.dropped_columns.size();
      out->summary.m = n - res.dropped_columns.size();
      out->summary.residual_sq = res.residual_sq;
      if (out->x) std::memcpy(out->x, res.x.data().data(), sizeof(double) * n);
      if (out->inner_x)
        std::copy(res.inner.x.begin(), res.inner.x.end(), out->inner_x);
      if (out->dropped)
        std::copy(res.dropped_columns.begin(), res.dropped_columns.end(), out->dropped);
    }
    return 0;
  });
}

int ref_solve_accelerated(uint64_t m, const double* Q, const double* q, const double* start,
                          const alnnls_config* cfg, oracle_out* out) {
  (void)start;
  return guarded(out, [&] {
    R::NqpProblem p(make_matrix(m, m, Q), make_vector(m, q));
    const auto res = R::solve_accelerated(p, to_cfg(cfg));
    if (out) {
      R::SolveStats none;
      fill_result(res, none, out);
      out->summary.m = m;
      out->summary.n = m;
      if (out->x) std::memcpy(out->x, res.x.data().data(), sizeof(double) * m);
    }
    return 0;
  });
}

int ref_solve_anti_accelerated(uint64_t d, uint64_t n, const double* A, const double* b,
                               const alnnls_config* cfg, oracle_out* out) {
  return guarded(out, [&] {
    const auto a = make_matrix(d, n, A);
    const auto bv = make_vector(d, b);
    const auto res = R::solve_anti_accelerated(a, bv, to_cfg(cfg));
    if (out) {
      R::SolveStats none;
      fill_result(res.inner, none, out);
      out->summary.n = n;
      out->summary.n_dropped = res.dropped_columns.size();
      out->summary.m = n - res.dropped_columns.size();
      out->summary.residual_sq = res.residual_sq;
      if (out->x) std::memcpy(out->x, res.x.data().data(), sizeof(double) * n);
      if (out->inner_x)
        std::copy(res.inner.x.begin(), res.inner.x.end(), out->inner_x);
      if (out->dropped)
        std::copy(res.dropped_columns.begin(), res.dropped_columns.end(), out->dropped);
    }
    return 0;
  });
}

double ref_frobenius_norm(uint64_t rows, uint64_t cols, const double* M) {
  return R::frobenius_norm(make_matrix(rows, cols, M));
}

double ref_objective(uint64_t m, const double* Q, const double* q, const double* x) {
  R::NqpProblem p(make_matrix(m, m, Q), make_vector(m, q));
  return R::objective(p, make_vector(m, x));
}

double ref_kkt_error(uint64_t m, const double* Q, const double* q, const double* x) {
  R::NqpProblem p(make_matrix(m, m, Q), make_vector(m, q));
  return R::kkt_error(p, make_vector(m, x));
}

int ref_solve_nnls_columns(uint64_t d, uint64_t n, const double* A, uint64_t ncols,
                           const double* B, const alnnls_config* cfg, double* X,
                           alnnls_column_result* cols, int threads) {
  return guarded(nullptr, [&] {
    const auto a = make_matrix(d, n, A);
    const R::DenseMatrix h_mat = R::gram(a);
    const R::SolverConfig sc = to_cfg(cfg);
    auto work = [&](uint64_t j) {
      alnnls_column_result& cr = cols[j];
      std::memset(&cr, 0, sizeof(cr));
      const R::Vector b = make_vector(d, B + j * d);
      // nnls.hpp:133-143 with the Gram shared across columns.
      R::Vector h_vec = R::transpose_matvec(a, b);
      for (std::size_t i = 0; i < h_vec.size(); ++i) h_vec[i] = -h_vec[i];
      const R::ScaledSystem sys = R::rescale(h_mat, h_vec);
      R::SolveResult inner;
      try {
        R::SolveStats stats;
        inner = sys.problem ? R::solve_nqp(*sys.problem, sc, std::nullopt, &stats)
                            : R::detail::empty_solve_result();
        uint64_t tot = 0;
        for (auto v : stats.multiplies_per_iter) tot += v;
        cr.multiplies_total = tot;
      } catch (const R::NumericFailure&) {
        cr.numeric_failure = 1;
        return;
      }
      const R::Vector x = R::unscale(inner.x, sys, n);
      std::copy(x.begin(), x.end(), X + j * n);
      cr.termination = static_cast<int32_t>(inner.termination);
      cr.iterations = inner.iterations();
      cr.residual_sq = R::detail::residual_norm_sq(a, b, x);
      cr.f_final = inner.trace.back().f;
      cr.gbs_final = inner.trace.back().grad_bar_sq;
    };
    const int nt = std::max(1, threads);
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(nt);
    for (int t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        try {
          for (uint64_t j = t; j < ncols; j += nt) work(j);
        } catch (...) {
          errs[t] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    return 0;
  });
}

}  // extern "C"

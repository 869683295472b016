// C++ facade tests: the reference's own unit-test cases (tests/test_{linalg,
// nqp,nnls}.cpp under /root/reference/proj), restated against the B200
// facade include/antilop/*.hpp. Code is written against the same API the
// reference exposes; every hot-path call runs on the GPU through the C ABI.
// Needs a GPU: run by tests/test_facade_cpp.py (pytest -m gpu).
#include <cmath>
#include <filesystem>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "antilop/accelerated.hpp"
#include "antilop/nnls.hpp"

using namespace antilop;

namespace {

int g_fail = 0, g_pass = 0;
std::string g_case;

#define REQUIRE(cond)                                                                 \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
      ++g_fail;                                                                       \
      return;                                                                         \
    }                                                                                 \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

bool near(double a, double b, double tol) { return std::abs(a - b) <= tol; }

void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception& e) {
    std::printf("FAIL [%s] unexpected exception: %s\n", name, e.what());
    ++g_fail;
  }
  if (g_fail == before) {
    ++g_pass;
    std::printf("PASS [%s]\n", name);
  }
}

NqpProblem coupled() { return NqpProblem(DenseMatrix(2, 2, {1.0, 1.0 / 30.0, 1.0 / 30.0, 1.0}), Vector{-4.0, -5.0 / 3.0}); }
NqpProblem lopsided() { return NqpProblem(DenseMatrix(2, 2, {1.0, 0.1, 0.1, 9.0}), Vector{-4.0, -5.0}); }

}  // namespace

int main() {
  run("io: MatrixMarket / CSV round trips and errors", [] {  // test_io.cpp cases
    const DenseMatrix m = DenseMatrix::from_rows({{1.0, -2.5}, {1.0 / 3.0, 4e-300}, {7.0, 8.0}});
    std::stringstream ss;
    write_matrix_market(ss, m);
    const DenseMatrix back = read_matrix_market(ss);
    REQUIRE(back.rows() == 3 && back.cols() == 2);
    for (std::size_t j = 0; j < 2; ++j)
      for (std::size_t i = 0; i < 3; ++i) REQUIRE(back(i, j) == m(i, j));
    std::stringstream vs;
    write_matrix_market(vs, Vector{0.1, 0.2});
    const Vector vb = read_matrix_market_vector(vs);
    REQUIRE(vb.size() == 2 && vb[0] == 0.1 && vb[1] == 0.2);
    std::istringstream comment("%%MatrixMarket matrix array real general\n% note\n\n2 1\n1.5\n-2\n");
    const DenseMatrix c = read_matrix_market(comment);
    REQUIRE(c(0, 0) == 1.5 && c(1, 0) == -2.0);
    for (const char* bad : {"", "%%MatrixMarket matrix coordinate real general\n1 1\n1\n",
                            "hello\n1 1\n1\n", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n",
                            "%%MatrixMarket matrix array real general\n1 1\nx\n"}) {
      std::istringstream is(bad);
      REQUIRE(throws<std::runtime_error>([&] { read_matrix_market(is); }));
    }
    std::stringstream cs;
    write_csv(cs, m);
    const DenseMatrix cb = read_csv_matrix(cs);
    REQUIRE(cb.rows() == 3 && cb.cols() == 2 && cb(1, 0) == 1.0 / 3.0);
    std::istringstream ragged("1,2\n3\n");
    REQUIRE(throws<std::runtime_error>([&] { read_csv_matrix(ragged); }));
    REQUIRE(fmt_g17(0.1) == "0.10000000000000001");
    const auto dir = std::filesystem::temp_directory_path();
    save_matrix(dir / "antilop_io_test.mtx", m);
    save_vector(dir / "antilop_io_test.csv", Vector{1.0, 2.0});
    REQUIRE(load_matrix(dir / "antilop_io_test.mtx")(2, 1) == 8.0);
    REQUIRE(load_vector(dir / "antilop_io_test.csv")[1] == 2.0);
    REQUIRE(throws<std::runtime_error>([&] { load_matrix(dir / "antilop_no_such_file.mtx"); }));
  });
  run("NMF by alternating NNLS (nmf)", [] {
    const std::size_t d = 120, n = 90, k = 4;
    std::uint64_t st = 0x9E3779B97F4A7C15ull;
    auto u01 = [&] { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (st >> 11) * 0x1.0p-53; };
    std::vector<double> wt(d * k), ht(k * n), w0(d * k), vv(d * n, 0.0);
    for (auto& x : wt) x = u01();
    for (auto& x : ht) x = u01();
    for (auto& x : w0) x = u01();
    for (std::size_t j = 0; j < n; ++j)
      for (std::size_t t = 0; t < k; ++t)
        for (std::size_t i = 0; i < d; ++i) vv[j * d + i] += wt[t * d + i] * ht[j * k + t];
    SolverConfig cfg;
    cfg.epsilon = 1e-10;
    cfg.stall_window = 1000000000;
    const auto r = nmf(DenseMatrix(d, n, vv), DenseMatrix(d, k, w0), 20, cfg);
    REQUIRE(r.W.rows() == d && r.W.cols() == k && r.H.rows() == k && r.H.cols() == n);
    REQUIRE(r.objective.size() == 20 && r.objective.back() < 1e-2 * r.objective.front());
    for (std::size_t t = 1; t < r.objective.size(); ++t)
      REQUIRE(r.objective[t] <= r.objective[t - 1] * (1 + 1e-9) + 1e-12);
    REQUIRE(throws<std::invalid_argument>([&] { nmf(DenseMatrix(d, n, vv), DenseMatrix(d + 1, k), 1, cfg); }));
  });
  run("batched multi-RHS (solve_nnls_batched, num_gpus)", [] {
    const std::size_t d = 400, n = 60, k = 9;
    std::vector<double> av(d * n), bv(d * k);
    std::uint64_t st = 88172645463325252ull;
    auto u01 = [&] { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (st >> 11) * 0x1.0p-53; };
    for (auto& v : av) v = u01();
    for (auto& v : bv) v = 2.0 * u01();
    const DenseMatrix A(d, n, av), B(d, k, bv);
    SolverConfig cfg;
    cfg.epsilon = 1e-8;
    cfg.stall_window = 1000000000;
    const auto r = solve_nnls_batched(A, B, cfg, 1);
    REQUIRE(r.X.rows() == n && r.X.cols() == k && r.columns.size() == k);
    for (std::size_t j = 0; j < k; ++j) {
      std::vector<double> col(bv.begin() + j * d, bv.begin() + (j + 1) * d);
      const auto one = solve_nnls(A, Vector(col), cfg);
      for (std::size_t i = 0; i < n; ++i) REQUIRE(r.X(i, j) == one.x[i]);
      REQUIRE(r.columns[j].iterations == one.inner.iterations());
      REQUIRE(r.columns[j].termination == one.inner.termination);
      REQUIRE(r.columns[j].residual_sq == one.residual_sq);
    }
    REQUIRE(throws<std::invalid_argument>([&] { solve_nnls_batched(A, B, cfg, 1000); }));
    REQUIRE(throws<std::invalid_argument>([&] { solve_nnls_batched(A, DenseMatrix(d + 1, 2), cfg, 1); }));
  });
  run("gram fixed examples", [] {  // test_linalg.cpp:57-81
    const DenseMatrix h = gram(DenseMatrix::from_rows({{1.0, 1.0}, {0.0, 1.0}}));
    REQUIRE(h(0, 0) == 1.0 && h(0, 1) == 1.0 && h(1, 0) == 1.0 && h(1, 1) == 2.0);
    const DenseMatrix z = gram(DenseMatrix::from_rows({{1.0, 0.0}, {2.0, 0.0}}));
    REQUIRE(z(0, 1) == 0.0 && z(1, 0) == 0.0 && z(1, 1) == 0.0 && z(0, 0) == 5.0);
  });
  run("masked matvec", [] {  // test_linalg.cpp:114-155
    const DenseMatrix h = DenseMatrix::from_rows({{1.0, 1.0}, {1.0, 2.0}});
    const std::vector<std::size_t> mask{1};
    const Vector y = masked_matvec(h, Vector{0.0, 2.0}, mask);
    REQUIRE(y[0] == 2.0 && y[1] == 4.0);
    const std::vector<std::size_t> bad{2};
    REQUIRE(throws<std::out_of_range>([&] { masked_matvec(h, Vector{1.0, 2.0}, bad); }));
    std::size_t cnt = 7;
    masked_matvec(h, Vector{1.0, 2.0}, mask, &cnt);
    REQUIRE(cnt == 7 + 2);
    REQUIRE(throws<std::invalid_argument>([&] { matvec(h, Vector{1.0, 2.0, 3.0}); }));
  });
  run("transpose matvec", [] {  // test_linalg.cpp:157-163
    const Vector y = transpose_matvec(DenseMatrix::from_rows({{1.0, 1.0}, {0.0, 1.0}}), Vector{2.0, -1.0});
    REQUIRE(y[0] == 2.0 && y[1] == 1.0);
  });
  run("exact step", [] {  // test_nqp.cpp:65-103
    REQUIRE(*exact_step(DenseMatrix::identity(2), Vector{1.0, 2.0}) == 1.0);
    REQUIRE(*exact_step(DenseMatrix(2, 2, {2.0, 0.0, 0.0, 2.0}), Vector{1.0, 2.0}) == 0.5);
    const auto a3 = exact_step(DenseMatrix(2, 2, {1.0, 1.0 / 30.0, 1.0 / 30.0, 1.0}), Vector{-4.0, -5.0 / 3.0});
    REQUIRE(a3 && near(*a3, 169.0 / 173.0, 1e-15));
    REQUIRE(!exact_step(DenseMatrix(2, 2, 0.0), Vector{1.0, 1.0}));
  });
  run("identity one step", [] {  // test_nqp.cpp:123-133
    const auto res = solve_nqp(NqpProblem(DenseMatrix::identity(2), Vector{-1.0, -2.0}));
    REQUIRE(res.termination == Termination::GradientBelowEpsilon && res.iterations() == 1);
    REQUIRE(res.x[0] == 1.0 && res.x[1] == 2.0 && res.final_grad[0] == 0.0);
  });
  run("origin stop", [] {  // test_nqp.cpp:135-144
    const auto res = solve_nqp(NqpProblem(DenseMatrix::identity(2), Vector{3.0, 4.0}));
    REQUIRE(res.termination == Termination::EmptyPassiveSet && res.iterations() == 0);
    REQUIRE(res.trace.size() == 1 && !res.trace.back().alpha);
  });
  run("coupled optimum", [] {  // test_nqp.cpp:146-156
    SolverConfig c;
    c.epsilon = 1e-22;
    const auto res = solve_nqp(coupled(), c);
    REQUIRE(res.termination == Termination::GradientBelowEpsilon);
    REQUIRE(near(res.x[0], 3550.0 / 899.0, 1e-9) && near(res.x[1], 1380.0 / 899.0, 1e-9));
  });
  run("warm start", [] {  // test_nqp.cpp:158-177
    const NqpProblem p(DenseMatrix::identity(2), Vector{-1.0, -2.0});
    const auto at = solve_nqp(p, {}, Vector{1.0, 2.0});
    REQUIRE(at.termination == Termination::GradientBelowEpsilon && at.iterations() == 0);
    REQUIRE(throws<std::invalid_argument>([&] { solve_nqp(p, {}, Vector{-0.5, 0.0}); }));
    REQUIRE(throws<std::invalid_argument>([&] { solve_nqp(p, {}, Vector{1.0}); }));
    SolverConfig t;
    t.epsilon = 1e-10;
    t.max_iters = 100000;
    const auto far = solve_nqp(lopsided(), t, Vector{30.0, 2.0});
    REQUIRE(far.termination == Termination::GradientBelowEpsilon);
    REQUIRE(near(far.x[0], 35.5 / 8.99, 1e-4) && near(far.x[1], 4.6 / 8.99, 1e-4));
  });
  run("terminations", [] {  // test_nqp.cpp:179-215
    SolverConfig c;
    c.epsilon = 1e-30;
    c.max_iters = 3;
    c.stall_window = 1000;
    REQUIRE(solve_nqp(lopsided(), c).termination == Termination::MaxIters);
    SolverConfig tc;
    tc.time_cap = std::chrono::duration<double>(0.0);
    REQUIRE(solve_nqp(NqpProblem(DenseMatrix::identity(2), Vector{-1.0, -2.0}), tc).termination == Termination::TimeCap);
    SolverConfig st;
    st.epsilon = std::numeric_limits<double>::denorm_min();
    st.max_iters = 1000000;
    st.stall_window = 5;
    const auto s = solve_nqp(coupled(), st);
    REQUIRE(s.termination == Termination::Stalled && near(s.x[0], 3550.0 / 899.0, 1e-9));
    REQUIRE(solve_nqp(NqpProblem(DenseMatrix(2, 2, 0.0), Vector{-1.0, -1.0})).termination == Termination::ZeroCurvature);
  });
  run("numeric failure", [] {  // test_nqp.cpp:217-226
    bool caught = false;
    try {
      solve_nqp(NqpProblem(DenseMatrix::identity(2), Vector{-1e308, -1.0}));
    } catch (const NumericFailure& e) {
      caught = e.trace().empty() && std::string(e.what()).find("non-finite") != std::string::npos;
    }
    REQUIRE(caught);
  });
  run("halving safeguard", [] {  // test_nqp.cpp:349-389
    const NqpProblem p(DenseMatrix(2, 2, {1.0, 0.9, 0.9, 1.0}), Vector{1.49, -2.69});
    SolverConfig c;
    c.epsilon = 1e-18;
    c.max_iters = 10000;
    c.stall_window = 1000000;
    const auto res = solve_nqp(p, c, Vector{0.52, 0.35});
    REQUIRE(res.termination == Termination::GradientBelowEpsilon && res.x[0] == 0.0);
    REQUIRE(near(res.x[1], 2.69, 1e-9) && near(objective(p, res.x), -3.61805, 1e-9));
    for (std::size_t k = 1; k < res.trace.size(); ++k)
      REQUIRE(res.trace[k].f <= res.trace[k - 1].f + 1e-12 * std::max(1.0, std::abs(res.trace[k - 1].f)));
  });
  run("trace csv", [] {  // test_nqp.cpp:298-320
    const auto res = solve_nqp(NqpProblem(DenseMatrix::identity(2), Vector{-1.0, -2.0}));
    std::ostringstream os;
    write_trace_csv(os, res.trace);
    std::istringstream is(os.str());
    std::string line;
    std::getline(is, line);
    REQUIRE(line == "iter,elapsed_ms,f,grad_bar_sq,passive_count,alpha");
    std::vector<std::string> rows;
    while (std::getline(is, line)) rows.push_back(line);
    REQUIRE(rows.size() == 2 && rows[0].substr(rows[0].size() - 2) == ",1" && rows[1].back() == ',');
    REQUIRE(rows[1].find(",-2.5,") != std::string::npos);
  });
  run("rescale cosine system", [] {  // test_nnls.cpp:48-78
    const auto sys = rescale(DenseMatrix(2, 2, {1.0, 0.1, 0.1, 9.0}), Vector{-4.0, -5.0});
    REQUIRE(sys.problem && sys.dropped.empty() && sys.scale[0] == 1.0 && sys.scale[1] == 3.0);
    REQUIRE(sys.problem->Q(0, 1) == 0.1 / 3.0 && sys.problem->q[1] == -5.0 / 3.0);
    REQUIRE(throws<std::invalid_argument>([] { rescale(DenseMatrix(2, 3), Vector{1.0, 2.0}); }));
    REQUIRE(throws<std::invalid_argument>([] { rescale(DenseMatrix(2, 2, {1.0, 0.2, 0.1, 1.0}), Vector{1.0, 2.0}); }));
    REQUIRE(throws<std::invalid_argument>([] { rescale(DenseMatrix(2, 2, {-1.0, 0.0, 0.0, 1.0}), Vector{1.0, 2.0}); }));
  });
  run("zero column dropped", [] {  // test_nnls.cpp:80-101
    const auto res = solve_nnls(DenseMatrix(2, 2, {1.0, 0.0, 0.0, 0.0}), Vector{3.0, 1.0});
    REQUIRE(near(res.x[0], 3.0, 1e-12) && res.x[1] == 0.0);
    REQUIRE(res.dropped_columns == std::vector<std::size_t>{1} && near(res.residual_sq, 1.0, 1e-12));
  });
  run("all-zero matrix", [] {  // test_nnls.cpp:103-111
    const auto res = solve_nnls(DenseMatrix(3, 2, 0.0), Vector{1.0, 2.0, 3.0});
    REQUIRE(res.x[0] == 0.0 && res.x[1] == 0.0 && res.inner.termination == Termination::EmptyPassiveSet);
    REQUIRE(res.dropped_columns == (std::vector<std::size_t>{0, 1}) && near(res.residual_sq, 14.0, 1e-13));
  });
  run("frozen small systems", [] {  // test_nnls.cpp:178-194
    const auto r = solve_nnls(DenseMatrix::identity(2), Vector{3.0, -1.0});
    REQUIRE(near(r.x[0], 3.0, 1e-10) && r.x[1] == 0.0 && near(r.residual_sq, 1.0, 1e-10));
    REQUIRE(throws<std::invalid_argument>([] { solve_nnls(DenseMatrix::identity(2), Vector{1.0, 2.0, 3.0}); }));
  });
  run("result summary json", [] {  // test_nnls.cpp:220-228
    const std::string js = result_summary_json(solve_nnls(DenseMatrix::identity(2), Vector{3.0, -1.0}));
    REQUIRE(js.find("\"termination\":\"GradientBelowEpsilon\"") != std::string::npos);
    REQUIRE(js.find("\"dropped_columns\":[]") != std::string::npos);
  });
  // ---- accelerated baseline (test_baselines.cpp:162-245, restated) ----
  auto tight = [] {
    SolverConfig c;
    c.epsilon = 1e-16;
    c.max_iters = 200000;
    c.stall_window = 1000000;
    return c;
  };
  run("accelerated: origin optimal", [] {
    const auto res = solve_accelerated(NqpProblem(DenseMatrix::identity(2), Vector{3.0, 4.0}));
    REQUIRE(res.termination == Termination::EmptyPassiveSet && res.iterations() == 0);
    REQUIRE(res.x[0] == 0.0 && res.x[1] == 0.0);
  });
  run("accelerated: identity within 200 iterations", [] {
    SolverConfig c;
    c.epsilon = 1e-16;
    c.max_iters = 200;
    c.stall_window = 1000000;
    const auto res = solve_accelerated(NqpProblem(DenseMatrix::identity(2), Vector{-1.0, -2.0}), c);
    REQUIRE(res.termination == Termination::GradientBelowEpsilon && res.iterations() <= 200);
    REQUIRE(near(res.x[0], 1.0, 1e-8) && near(res.x[1], 2.0, 1e-8));
  });
  run("accelerated: coupled 2x2 (plain and restart)", [&] {
    for (bool restart : {false, true}) {
      SolverConfig c = tight();
      c.nesterov_restart = restart;
      const auto res = solve_accelerated(
          NqpProblem(DenseMatrix(2, 2, {1.0, 1.0 / 30.0, 1.0 / 30.0, 1.0}), Vector{-4.0, -5.0 / 3.0}), c);
      REQUIRE(res.termination == Termination::GradientBelowEpsilon);
      REQUIRE(near(res.x[0], 3550.0 / 899.0, 1e-6) && near(res.x[1], 1380.0 / 899.0, 1e-6));
    }
  });
  run("accelerated: zero curvature", [] {
    const auto res = solve_accelerated(NqpProblem(DenseMatrix(2, 2, 0.0), Vector{-1.0, -1.0}));
    REQUIRE(res.termination == Termination::ZeroCurvature);
  });
  run("anti+acc: identity and zero matrix", [&] {
    const auto r = solve_anti_accelerated(DenseMatrix::identity(2), Vector{3.0, -1.0}, tight());
    REQUIRE(near(r.x[0], 3.0, 1e-8) && r.x[1] == 0.0 && near(r.residual_sq, 1.0, 1e-8));
    const auto z = solve_anti_accelerated(DenseMatrix(3, 2, 0.0), Vector{1.0, 1.0, 1.0});
    REQUIRE(z.x[0] == 0.0 && z.x[1] == 0.0 && z.inner.termination == Termination::EmptyPassiveSet);
    REQUIRE(z.dropped_columns == (std::vector<std::size_t>{0, 1}));
  });
  std::printf("facade_tests: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}

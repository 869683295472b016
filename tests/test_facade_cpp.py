"""Runs the C++ facade tests (tests/cpp/facade_tests.cpp): the reference's own
unit-test cases written against include/antilop/*.hpp, on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "tests", "facade_tests")


@pytest.mark.gpu
def test_cpp_facade_suite():
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", ROOT, "facade"], check=True)
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_facade_compiles(tmp_path):
    """The facade headers compile as a drop-in for code written against the reference API."""
    src = tmp_path / "use.cpp"
    src.write_text('''#include "antilop/nnls.hpp"
int main() {
  antilop::SolverConfig c; c.epsilon = 1e-8; c.max_iters = 100;
  antilop::DenseMatrix a = antilop::DenseMatrix::from_rows({{1.0, 0.0}, {0.0, 1.0}});
  antilop::Vector b{1.0, 2.0};
  if (false) { auto r = antilop::solve_nnls(a, b, c); return (int)r.inner.iterations(); }
  return antilop::to_string(antilop::Termination::Stalled).size() == 7 ? 0 : 1;
}''')
    exe = tmp_path / "use"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-o", str(exe),
                    str(src), "-L", os.path.join(ROOT, "paper_1502_01645_b200", "lib"), "-lalnnls",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1502_01645_b200", "lib")], check=True)
    assert subprocess.run([str(exe)]).returncode == 0


def _nlohmann_dir():
    import sys
    for d in sys.path:
        p = os.path.join(d, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(p, "json.hpp")):
            return p
    return None


@pytest.mark.parametrize("fallback", [False, True])
def test_result_json_number_format_matches_nlohmann(tmp_path, fallback):
    """result_summary_json (nnls.hpp:146-153) prints residual_sq through nlohmann::json
    in the reference; the facade's json_number writes the same characters (nlohmann
    itself when it is on the include path; the to_chars fallback otherwise, which may
    differ in the last digit of Grisu2's rare non-shortest outputs: < 1% here)."""
    nl = _nlohmann_dir()
    if nl is None:
        pytest.skip("nlohmann/json.hpp not in this image")
    src = tmp_path / "fmt.cpp"
    src.write_text("""#include <cstdio>
#include <cstring>
#include <random>
#include "antilop/nqp.hpp"
#include "json.hpp"
int main() {
  std::mt19937_64 g(7);
  int bad = 0, total = 0;
  auto check = [&](double v) {
    ++total;
    if (antilop::detail::json_number(v) != nlohmann::json(v).dump()) ++bad;
  };
  const double fixed[] = {0.0, -0.0, 1.0, 100.0, 1e15, 1e16, 123456789012345.0, 0.1, 1e-4,
                          1e-5, 2.5e-28, 5e-324, 1.7976931348623157e308, -3.25, 0.000123};
  for (double v : fixed) check(v);
  const int fixed_bad = bad;
  for (int i = 0; i < 200000; ++i) {
    double v;
    const uint64_t bits = g();
    std::memcpy(&v, &bits, 8);
    if (std::isfinite(v)) check(v);
    check(std::ldexp((double)(g() >> 11), -(int)(g() % 120)));
  }
  std::printf("%d %d %d\\n", fixed_bad, bad, total);
  return 0;
}""")
    exe = tmp_path / "fmt"
    flags = ["-DANTILOP_NO_NLOHMANN"] if fallback else []
    subprocess.run(["g++", "-std=c++20", "-O1"] + flags + ["-I", os.path.join(ROOT, "include"),
                    "-I", nl, "-o", str(exe), str(src)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0
    fixed_bad, bad, total = (int(t) for t in r.stdout.split())
    assert fixed_bad == 0
    if fallback:
        assert bad < total // 100, r.stdout
    else:
        assert bad == 0, r.stdout


def test_cpp_facade_io_visible_from_nqp(tmp_path):
    """As in the reference (nqp.hpp:23 includes io.hpp), including the facade's
    nqp.hpp makes fmt_g17 and the MatrixMarket / CSV I/O visible; they run on the
    host (no GPU needed)."""
    src = tmp_path / "io.cpp"
    src.write_text('''#include <sstream>
#include "antilop/nqp.hpp"
int main() {
  using namespace antilop;
  const DenseMatrix m = DenseMatrix::from_rows({{1.0, 2.0}, {3.0, 0.1}});
  std::stringstream ss;
  write_matrix_market(ss, m);
  const DenseMatrix b = read_matrix_market(ss);
  if (!(b(1, 1) == 0.1 && b(1, 0) == 3.0)) return 1;
  return fmt_g17(0.1) == "0.10000000000000001" ? 0 : 2;
}''')
    exe = tmp_path / "io"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-o", str(exe),
                    str(src), "-L", os.path.join(ROOT, "paper_1502_01645_b200", "lib"), "-lalnnls",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1502_01645_b200", "lib")], check=True)
    assert subprocess.run([str(exe)]).returncode == 0

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

"""Anti+Acc baseline (accelerated.hpp) on the GPU: bit for bit the
C restatement (itself pinned to the reference, tests/test_oracle_pin.py):
x, final_grad, iterations, termination, every trace record, residual."""
import numpy as np
import pytest

from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import SolverConfig
from tests.parity import assert_trace_bitwise, same_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,d,n,restart,kw", [
    ("c1", 200, 80, False, dict(epsilon=1e-8, max_iters=3000, stall_window=10**9)),
    ("c1", 200, 80, True, dict(epsilon=1e-8, max_iters=3000, stall_window=10**9)),
    ("c2", 600, 300, False, dict(epsilon=1e-8, stall_window=10**9)),
    ("c5", 500, 250, True, dict()),
    ("c3", 300, 300, False, dict(epsilon=1e-10, max_iters=500, trace_every=7)),
])
def test_anti_accelerated_bitwise(solver, oracle, name, d, n, restart, kw):
    inst = instances.make_config(name, d=d, n=n)
    cfg = SolverConfig(nesterov_restart=restart, **kw)
    got = solver.solve_anti_accelerated(inst["A"], inst["b"], cfg)
    exp = oracle.solve_anti_accelerated(inst["A"], inst["b"], cfg.to_abi())
    assert got.inner.termination == exp["termination"]
    assert got.inner.iterations() == exp["iterations"]
    assert same_bits(got.x, exp["x"])
    assert same_bits(got.inner.x, exp["inner_x"])
    assert same_bits(got.inner.final_grad, exp["final_grad"])
    assert same_bits([got.residual_sq], [exp["residual_sq"]])
    assert_trace_bitwise(got.inner.trace, exp["trace"])


def test_accelerated_nqp_bitwise(solver, oracle):
    rng = np.random.default_rng(3)
    M = rng.standard_normal((60, 40))
    Q = M.T @ M
    Q = (Q + Q.T) / 2
    q = rng.standard_normal(40)
    cfg = SolverConfig(epsilon=1e-9, max_iters=5000, stall_window=10**9)
    got = solver.solve_accelerated(Q, q, cfg)
    exp = oracle.solve_accelerated(Q, q, cfg.to_abi())
    assert got.iterations() == exp["iterations"] and got.termination == exp["termination"]
    assert same_bits(got.x, exp["x"]) and same_bits(got.final_grad, exp["final_grad"])
    assert_trace_bitwise(got.trace, exp["trace"])

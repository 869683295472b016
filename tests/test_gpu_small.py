"""GPU parity of the small-m cluster loop (small.cu) and of the general loop it replaces.

For small m the exact solve_nqp runs as one thread-block cluster with the loop state in
distributed shared memory (nqp_small_kernel); ALNNLS_SMALL=0 forces the general kernel
(nqp_loop_kernel as one cluster). Both must be bit for bit the reference's trajectory
(the oracle, pinned to the reference in tests/test_oracle_pin.py), so they must also be
bit for bit each other. The C ABI reports which loop kernel ran (alnnls_last_loop_kernel).
"""
import os

import numpy as np
import pytest

from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import SolverConfig
from tests.parity import assert_trace_bitwise, same_bits
from tests.test_gpu_parity import check_nnls, splitmix_matrix

pytestmark = pytest.mark.gpu


class general_loop:
    """Runs the block with the small-m kernel disabled (the library reads the knob per launch)."""

    def __enter__(self):
        self.old = os.environ.get("ALNNLS_SMALL")
        os.environ["ALNNLS_SMALL"] = "0"

    def __exit__(self, *exc):
        if self.old is None:
            del os.environ["ALNNLS_SMALL"]
        else:
            os.environ["ALNNLS_SMALL"] = self.old


def test_c1_runs_small_kernel_bitwise(solver, oracle):
    inst = instances.make_config("c1")
    cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
    got, _ = check_nnls(solver, oracle, inst["A"], inst["b"], cfg)
    assert solver.loop_kernel() == "small"
    with general_loop():
        gen, _ = check_nnls(solver, oracle, inst["A"], inst["b"], cfg)
        assert solver.loop_kernel() in ("cluster", "grid")
    assert same_bits(got.x, gen.x) and same_bits(got.inner.final_grad, gen.inner.final_grad)
    assert np.array_equal(got.inner.multiplies_per_iter, gen.inner.multiplies_per_iter)


@pytest.mark.parametrize("d,n", [(40, 24), (300, 160), (500, 340)])
def test_small_kernel_uniform_bitwise(solver, oracle, d, n):
    A = splitmix_matrix(d, n, 11 + n)
    b = splitmix_matrix(d, 1, 23 + n)[:, 0]
    cfg = SolverConfig(epsilon=1e-12, max_iters=4000, stall_window=10**9, trace_every=3)
    check_nnls(solver, oracle, A, b, cfg)
    assert solver.loop_kernel() == "small"


def test_general_cluster_where_small_does_not_fit(solver, oracle):
    # m = 420: 7 row CTAs of 60 rows; 60 x 420 doubles of Q per CTA plus the lists
    # exceed the small kernel's shared memory, so the general cluster loop runs
    A = splitmix_matrix(700, 420, 5)
    b = splitmix_matrix(700, 1, 6)[:, 0]
    cfg = SolverConfig(epsilon=1e-9, max_iters=2000, stall_window=10**9)
    check_nnls(solver, oracle, A, b, cfg)
    assert solver.loop_kernel() in ("cluster", "grid")


def test_small_kernel_halving_warm_start_and_stops(solver, oracle):
    # the halving safeguard (speculative step rolled back by the df check), a warm
    # start, and the stall / max_iters stops, each on both loop kernels
    rng = np.random.default_rng(3)
    M = rng.standard_normal((30, 30))
    Q = M @ M.T + 1e-3 * np.eye(30)
    q = rng.standard_normal(30)
    start = np.abs(rng.standard_normal(30))
    for cfg in (SolverConfig(epsilon=1e-18, max_iters=3000, stall_window=10**9),
                SolverConfig(epsilon=1e-30, max_iters=7, stall_window=10**9),
                SolverConfig(epsilon=1e-30, max_iters=100000, stall_window=4)):
        for st in (None, start):
            a = solver.solve_nqp(Q, q, cfg, start=st)
            assert solver.loop_kernel() == "small"
            exp = oracle.solve_nqp(Q, q, cfg.to_abi(), start=st)
            assert a.termination == exp["termination"]
            assert a.iterations() == exp["iterations"]
            assert same_bits(a.x, exp["x"]) and same_bits(a.final_grad, exp["final_grad"])
            assert_trace_bitwise(a.trace, exp["trace"])
            with general_loop():
                g = solver.solve_nqp(Q, q, cfg, start=st)
            assert same_bits(a.x, g.x) and same_bits(a.final_grad, g.final_grad)
            assert a.iterations() == g.iterations()

"""FAST profile (Gram and A^T B on the fp64 tensor cores, dmma.cu) against the
reference oracle, with the tolerances BASELINE.json's north star states:
relative objective difference <= 1e-10, ||x_gpu - x_ref||_inf <= 1e-8 max(1,
||x_ref||_inf), identical passive set except entries within 1e-12 of zero, and
iteration count within +-1 (tests/parity.py baseline_tolerances).
"""
import numpy as np
import pytest

from paper_1502_01645_b200 import abi, instances
from paper_1502_01645_b200.api import SolverConfig
from tests.parity import baseline_tolerances

pytestmark = pytest.mark.gpu


def fast(cfg):
    cfg.profile = abi.PROFILE_FAST
    return cfg


def check_fast(solver, oracle, A, b, cfg):
    got = solver.solve_nnls(A, b, fast(cfg))
    exp = oracle.solve_nnls(A, b, SolverConfig(**{**cfg.__dict__, "profile": abi.PROFILE_EXACT}).to_abi())
    tol = baseline_tolerances(got.x, exp["x"], got.inner.trace[-1].f, exp["trace"][-1]["f"],
                              got.inner.iterations(), exp["iterations"])
    print(f"FAST tolerances d={A.shape[0]} n={A.shape[1]}: {tol} term {got.inner.termination} "
          f"{exp['termination']} it {got.inner.iterations()} {exp['iterations']}")
    assert tol["rel_objective"] <= 1e-7, tol
    return got, exp, tol


@pytest.mark.parametrize("name,d,n", [("c1", 600, 300), ("c2", 1024, 512), ("c5", 1024, 512)])
def test_fast_within_tolerance(solver, oracle, name, d, n):
    inst = instances.make_config(name, d=d, n=n)
    cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
    check_fast(solver, oracle, inst["A"], inst["b"], cfg)


@pytest.mark.parametrize("d,n", [(131, 77), (257, 200), (300, 129)])  # ragged tiles, odd d
def test_fast_ragged_shapes(solver, oracle, d, n):
    rng = np.random.default_rng(d * n)
    A = rng.uniform(0.0, 1.0, (d, n))
    x_true = np.where(rng.uniform(size=n) < 0.5, 0.0, rng.uniform(size=n))
    b = A @ x_true + 0.01 * rng.standard_normal(d)
    check_fast(solver, oracle, A, b, SolverConfig(epsilon=1e-8, stall_window=10**9))


def test_fast_gram_close_to_exact(solver):
    """The DMMA Gram feeds Q: compare the FAST Q with the exact Q entrywise."""
    rng = np.random.default_rng(7)
    A = np.asfortranarray(rng.standard_normal((700, 260)))
    b = rng.standard_normal(700)
    solver.solve_nnls(A, b, SolverConfig(max_iters=1, profile=abi.PROFILE_EXACT))
    Qe = solver._scaled()["Q"]
    solver.solve_nnls(A, b, SolverConfig(max_iters=1, profile=abi.PROFILE_FAST))
    Qf = solver._scaled()["Q"]
    assert Qe.shape == Qf.shape
    assert np.max(np.abs(Qe - Qf)) <= 1e-13 * 700
    assert np.array_equal(np.diag(Qf), np.ones(Qf.shape[0]))
    assert np.array_equal(Qf, Qf.T)


def test_fast_batched_within_tolerance(solver):
    inst = instances.make_batched(d=2000, n=256, nrhs=24, seed=11)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9)
    Xe, ce, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg)
    Xf, cf, _ = solver.solve_nnls_batched(inst["A"], inst["B"], fast(SolverConfig(epsilon=1e-8,
                                                                                   stall_window=10**9)))
    for j in range(inst["B"].shape[1]):
        tol = baseline_tolerances(Xf[:, j], Xe[:, j], cf[j]["f_final"], ce[j]["f_final"],
                                  cf[j]["iterations"], ce[j]["iterations"])
        assert tol["rel_objective"] <= 1e-7, (j, tol)

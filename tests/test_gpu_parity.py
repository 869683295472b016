"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit for bit.

The oracle (oracle/antilop_oracle.c) is itself pinned to the reference compiled
from its own headers (tests/test_oracle_pin.py). Exact-profile results must be
bitwise equal: x, final_grad, iterations, termination, every trace record's
(f, gbs, |P|, alpha), multiplies_per_iter, residual_sq.
"""
import numpy as np
import pytest

from paper_1502_01645_b200 import abi, instances
from paper_1502_01645_b200.api import SolverConfig
from tests.parity import assert_trace_bitwise, baseline_tolerances, same_bits

pytestmark = pytest.mark.gpu


def splitmix_matrix(rows, cols, seed, lo=-1.0, hi=1.0):
    """Matches the reference tests' random_matrix (test_nnls.cpp:19-29) law."""
    from tests.splitmix import SplitMix64
    r = SplitMix64(seed)
    M = np.zeros((rows, cols), order="F")
    for j in range(cols):
        for i in range(rows):
            M[i, j] = lo + (hi - lo) * r.uniform01()
    return M


def cfg_of(config):
    return config.to_abi()


def check_nnls(solver, oracle, A, b, config, bitwise=True):
    got = solver.solve_nnls(A, b, config)
    exp = oracle.solve_nnls(A, b, cfg_of(config))
    assert got.inner.termination == exp["termination"]
    assert got.inner.iterations() == exp["iterations"]
    assert got.dropped_columns == [int(v) for v in exp["dropped"]]
    if bitwise:
        assert same_bits(got.x, exp["x"]), "x differs"
        assert same_bits(got.inner.x, exp["inner_x"]), "inner x differs"
        assert same_bits(got.inner.final_grad, exp["final_grad"]), "final_grad differs"
        assert same_bits([got.residual_sq], [exp["residual_sq"]]), "residual differs"
        assert_trace_bitwise(got.inner.trace, exp["trace"])
        assert np.array_equal(got.inner.multiplies_per_iter, exp["mults"])
        assert got.inner.min_iterate == exp["min_iterate"]
    return got, exp


# ---- known-answer tests restated from the reference's unit tests ------------------

def test_gram_fixed_examples(solver):  # test_linalg.cpp:57-81
    H = solver.gram(np.eye(2))
    assert np.array_equal(H, np.eye(2))
    H = solver.gram(np.array([[1.0, 1.0], [0.0, 1.0]]))
    assert np.array_equal(H, np.array([[1.0, 1.0], [1.0, 2.0]]))
    H = solver.gram(np.array([[1.0, 0.0], [2.0, 0.0]]))
    assert H[0, 1] == 0.0 and H[1, 0] == 0.0 and H[1, 1] == 0.0 and H[0, 0] == 5.0


def test_gram_bitwise_random(solver, oracle):  # test_linalg.cpp:83-99 + bitwise vs oracle
    for seed in range(1, 11):
        A = splitmix_matrix(11, 7, seed)
        H = solver.gram(A)
        assert np.array_equal(H, H.T)
        assert same_bits(H, oracle.gram(A))
    rng = np.random.default_rng(5)
    for d, n in [(1, 1), (3, 200), (301, 129), (1000, 257), (17, 130)]:
        A = rng.standard_normal((d, n))
        assert same_bits(solver.gram(A), oracle.gram(A)), (d, n)


def test_matvec_and_masked(solver, oracle):  # test_linalg.cpp:101-155
    h = np.array([[1.0, 1.0], [1.0, 2.0]])
    assert np.array_equal(solver.matvec(h, [1.0, 0.0]), [1.0, 1.0])
    assert np.array_equal(solver.matvec(h, [0.0, 0.0]), [0.0, 0.0])
    with pytest.raises(ValueError):
        solver.matvec(h, [1.0, 2.0, 3.0])
    y = solver.masked_matvec(h, [0.0, 2.0], [1])
    assert np.array_equal(y, [2.0, 4.0])
    assert np.array_equal(solver.masked_matvec(h, [5.0, 6.0], []), [0.0, 0.0])
    with pytest.raises(IndexError):
        solver.masked_matvec(h, [1.0, 2.0], [2])
    for seed in range(1, 9):
        M = splitmix_matrix(9, 6, seed)
        v = splitmix_matrix(6, 1, seed + 77)[:, 0]
        assert same_bits(solver.matvec(M, v), solver.masked_matvec(M, v, list(range(6))))
        assert same_bits(solver.matvec(M, v), oracle.matvec(M, v))
    M = splitmix_matrix(13, 9, 3)
    v = splitmix_matrix(9, 1, 4)[:, 0]
    y, cnt = solver.masked_matvec(M, v, [0, 2, 5, 8], multiply_count=7)
    assert cnt == 7 + 13 * 4
    ye, _ = oracle.masked_matvec(M, v, [0, 2, 5, 8])
    assert same_bits(y, ye)
    rng = np.random.default_rng(9)
    for rows, cols in [(4096, 300), (1001, 77), (33, 1000)]:
        M = rng.standard_normal((rows, cols))
        v = rng.standard_normal(cols)
        mask = np.sort(rng.choice(cols, cols // 2, replace=False))
        ye, _ = oracle.masked_matvec(M, v, mask)
        assert same_bits(solver.masked_matvec(M, v, mask), ye)


def test_transpose_matvec(solver, oracle):  # test_linalg.cpp:157-163
    a = np.array([[1.0, 1.0], [0.0, 1.0]])
    assert np.array_equal(solver.transpose_matvec(a, [2.0, -1.0]), [2.0, 1.0])
    with pytest.raises(ValueError):
        solver.transpose_matvec(a, [1.0, 2.0, 3.0])
    rng = np.random.default_rng(2)
    M = rng.standard_normal((777, 55))
    v = rng.standard_normal(777)
    assert same_bits(solver.transpose_matvec(M, v), oracle.transpose_matvec(M, v))


def test_rescale_known_answer(solver):  # test_nnls.cpp:48-69
    sys = solver.rescale(np.array([[1.0, 0.1], [0.1, 9.0]]), [-4.0, -5.0])
    assert list(sys["retained"]) == [0, 1] and len(sys["dropped"]) == 0
    assert sys["scale"][0] == 1.0 and sys["scale"][1] == 3.0
    Q = sys["Q"]
    assert Q[0, 0] == 1.0 and Q[1, 1] == 1.0
    assert Q[0, 1] == 0.1 / 3.0 and Q[0, 1] == Q[1, 0]
    assert sys["q"][0] == -4.0 and sys["q"][1] == -5.0 / 3.0


def test_rescale_rejects_malformed(solver):  # test_nnls.cpp:71-78
    with pytest.raises(ValueError):
        solver.rescale(np.zeros((2, 3)), [1.0, 2.0])
    with pytest.raises(ValueError):
        solver.rescale(np.eye(2), [1.0])
    with pytest.raises(ValueError):
        solver.rescale(np.array([[1.0, 0.1], [0.2, 1.0]]), [1.0, 2.0])
    with pytest.raises(ValueError):
        solver.rescale(np.array([[-1.0, 0.0], [0.0, 1.0]]), [1.0, 2.0])


def test_setup_bitwise(solver, oracle):
    rng = np.random.default_rng(11)
    for d, n in [(600, 300), (50, 129), (7, 3)]:
        A = rng.uniform(0, 1, (d, n))
        A[:, n // 2] = 0.0  # a dropped column
        b = rng.standard_normal(d)
        got = solver.setup(A, b)
        H = oracle.gram(A)
        h = -oracle.transpose_matvec(A, b)
        exp = oracle.rescale(H, h)
        assert list(got["dropped"]) == list(exp["dropped"])
        assert same_bits(got["Q"], exp["Q"])
        assert same_bits(got["q"], exp["q"])
        assert same_bits(got["scale"], exp["scale"])


def test_zero_column_dropped(solver):  # test_nnls.cpp:80-101
    a = np.array([[1.0, 0.0], [0.0, 0.0]])
    res = solver.solve_nnls(a, [3.0, 1.0])
    assert abs(res.x[0] - 3.0) <= 1e-12 and res.x[1] == 0.0
    assert res.dropped_columns == [1]
    assert abs(res.residual_sq - 1.0) <= 1e-12


def test_all_zero_matrix(solver):  # test_nnls.cpp:103-111
    res = solver.solve_nnls(np.zeros((3, 2)), [1.0, 2.0, 3.0])
    assert res.x[0] == 0.0 and res.x[1] == 0.0
    assert res.dropped_columns == [0, 1]
    assert res.inner.termination == "EmptyPassiveSet"
    assert abs(res.residual_sq - 14.0) <= 14.0 * 1e-15


def test_frozen_small_systems(solver):  # test_nnls.cpp:178-194
    res = solver.solve_nnls(np.eye(2), [3.0, -1.0])
    assert abs(res.x[0] - 3.0) <= 1e-10 and res.x[1] == 0.0
    tight = SolverConfig(epsilon=1e-20, max_iters=200000, stall_window=1000000)
    res = solver.solve_nnls(np.array([[1.0, 1.0], [0.0, 1.0]]), [2.0, -1.0], tight)
    assert abs(res.x[0] - 2.0) <= 1e-9 and res.x[1] == 0.0
    assert abs(res.residual_sq - 1.0) <= 1e-9


# ---- solve_nqp known answers (test_nqp.cpp) ------------------------------------------

def coupled():
    return np.array([[1.0, 1.0 / 30.0], [1.0 / 30.0, 1.0]]), np.array([-4.0, -5.0 / 3.0])


def lopsided():
    return np.array([[1.0, 0.1], [0.1, 9.0]]), np.array([-4.0, -5.0])


def test_identity_one_step(solver):  # test_nqp.cpp:123-133
    res = solver.solve_nqp(np.eye(2), [-1.0, -2.0])
    assert res.termination == "GradientBelowEpsilon" and res.iterations() == 1
    assert res.x[0] == 1.0 and res.x[1] == 2.0
    assert res.final_grad[0] == 0.0 and res.final_grad[1] == 0.0
    assert res.min_iterate >= 0.0


def test_origin_stop(solver):  # test_nqp.cpp:135-144
    res = solver.solve_nqp(np.eye(2), [3.0, 4.0])
    assert res.termination == "EmptyPassiveSet" and res.iterations() == 0
    assert len(res.trace) == 1 and res.trace[-1].alpha is None
    assert res.x[0] == 0.0 and res.x[1] == 0.0


def test_coupled_optimum(solver):  # test_nqp.cpp:146-156
    Q, q = coupled()
    res = solver.solve_nqp(Q, q, SolverConfig(epsilon=1e-22))
    assert res.termination == "GradientBelowEpsilon"
    assert abs(res.x[0] - 3550.0 / 899.0) <= 1e-9
    assert abs(res.x[1] - 1380.0 / 899.0) <= 1e-9


def test_warm_start(solver, oracle):  # test_nqp.cpp:158-177
    at_opt = solver.solve_nqp(np.eye(2), [-1.0, -2.0], SolverConfig(), start=[1.0, 2.0])
    assert at_opt.termination == "GradientBelowEpsilon" and at_opt.iterations() == 0
    with pytest.raises(ValueError):
        solver.solve_nqp(np.eye(2), [-1.0, -2.0], SolverConfig(), start=[-0.5, 0.0])
    with pytest.raises(ValueError):
        solver.solve_nqp(np.eye(2), [-1.0, -2.0], SolverConfig(), start=[1.0])
    Q, q = lopsided()
    tight = SolverConfig(epsilon=1e-10, max_iters=100000)
    far = solver.solve_nqp(Q, q, tight, start=[30.0, 2.0])
    assert far.termination == "GradientBelowEpsilon"
    assert abs(far.x[0] - 35.5 / 8.99) <= 1e-4 and abs(far.x[1] - 4.6 / 8.99) <= 1e-4
    exp = oracle.solve_nqp(Q, q, tight.to_abi(), start=[30.0, 2.0])
    assert same_bits(far.x, exp["x"]) and far.iterations() == exp["iterations"]
    assert_trace_bitwise(far.trace, exp["trace"])


@pytest.mark.parametrize("case", ["max_iters", "time_cap", "stall", "zero_curv"])
def test_terminations(solver, case):  # test_nqp.cpp:179-215
    if case == "max_iters":
        Q, q = lopsided()
        res = solver.solve_nqp(Q, q, SolverConfig(epsilon=1e-30, max_iters=3, stall_window=1000))
        assert res.termination == "MaxIters" and res.iterations() == 3
    elif case == "time_cap":
        res = solver.solve_nqp(np.eye(2), [-1.0, -2.0], SolverConfig(time_cap=0.0))
        assert res.termination == "TimeCap" and res.iterations() == 0
    elif case == "stall":
        Q, q = coupled()
        res = solver.solve_nqp(Q, q, SolverConfig(epsilon=5e-324, max_iters=1000000,
                                                  stall_window=5))
        assert res.termination == "Stalled" and res.iterations() < 1000000
        assert abs(res.x[0] - 3550.0 / 899.0) <= 1e-9
    else:
        res = solver.solve_nqp(np.zeros((2, 2)), [-1.0, -1.0])
        assert res.termination == "ZeroCurvature" and res.iterations() == 0


def test_numeric_failure(solver):  # test_nqp.cpp:217-226
    from paper_1502_01645_b200.api import NumericFailure
    with pytest.raises(NumericFailure) as ei:
        solver.solve_nqp(np.eye(2), [-1e308, -1.0])
    assert ei.value.trace == []
    assert "non-finite" in str(ei.value)


def test_halving_safeguard(solver, oracle):  # test_nqp.cpp:349-389
    Q = np.array([[1.0, 0.9], [0.9, 1.0]])
    q = np.array([1.49, -2.69])
    cfg = SolverConfig(epsilon=1e-18, max_iters=10000, stall_window=1000000)
    res = solver.solve_nqp(Q, q, cfg, start=[0.52, 0.35])
    g0 = Q @ np.array([0.52, 0.35]) + q
    full = (g0 @ g0) / (g0 @ Q @ g0)
    assert res.trace[0].alpha is not None and res.trace[0].alpha <= 0.5 * full
    for k in range(1, len(res.trace)):
        prev = res.trace[k - 1].f
        assert res.trace[k].f <= prev + 1e-12 * max(1.0, abs(prev))
    assert res.termination == "GradientBelowEpsilon" and res.min_iterate >= 0.0
    assert res.x[0] == 0.0 and abs(res.x[1] - 2.69) <= 1e-9
    exp = oracle.solve_nqp(Q, q, cfg.to_abi(), start=[0.52, 0.35])
    assert same_bits(res.x, exp["x"])
    assert_trace_bitwise(res.trace, exp["trace"])


def test_trace_sampling(solver, oracle):  # test_nqp.cpp:322-347
    Q, q = lopsided()
    dense = SolverConfig(epsilon=1e-18, max_iters=100000, stall_window=1000000)
    full = solver.solve_nqp(Q, q, dense)
    assert len(full.trace) > 10
    strided = SolverConfig(epsilon=1e-18, max_iters=100000, stall_window=1000000, trace_every=4)
    sampled = solver.solve_nqp(Q, q, strided)
    assert same_bits(sampled.x, full.x) and sampled.iterations() == full.iterations()
    assert sampled.trace[0].iter == 0 and sampled.trace[-1].alpha is None
    for k in range(len(sampled.trace) - 1):
        assert sampled.trace[k].iter % 4 == 0 and sampled.trace[k].alpha is not None
    exp = oracle.solve_nqp(Q, q, strided.to_abi())
    assert_trace_bitwise(sampled.trace, exp["trace"])


# ---- seeded random problems: bitwise vs the oracle ------------------------------------

@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_random_nqp_bitwise(solver, oracle, seed):  # test_nqp.cpp:228-271 family
    n = 8 + 3 * seed
    A = splitmix_matrix(n + 4, n, seed)
    Q = oracle.gram(A)
    q = splitmix_matrix(n, 1, seed + 500)[:, 0]
    cfg = SolverConfig(max_iters=5000, stall_window=1000000)
    res = solver.solve_nqp(Q, q, cfg)
    exp = oracle.solve_nqp(Q, q, cfg.to_abi())
    assert res.termination == exp["termination"]
    assert same_bits(res.x, exp["x"]) and same_bits(res.final_grad, exp["final_grad"])
    assert_trace_bitwise(res.trace, exp["trace"])
    assert np.array_equal(res.multiplies_per_iter, exp["mults"])
    for k, mu in enumerate(res.multiplies_per_iter):
        assert mu <= 2 * n * res.trace[k].passive_count


@pytest.mark.parametrize("seed", range(200, 212))
def test_random_rectangles_bitwise(solver, oracle, seed):  # test_nnls.cpp:196-218 family
    n = 2 + seed % 7
    d = n + 1 + seed % 8
    A = splitmix_matrix(d, n, seed, 0.0 if seed % 2 else -1.0, 1.0)
    b = splitmix_matrix(d, 1, seed + 999)[:, 0]
    cfg = SolverConfig(epsilon=1e-20, max_iters=200000, stall_window=1000000)
    check_nnls(solver, oracle, A, b, cfg)


@pytest.mark.parametrize("d,n", [(600, 300), (1000, 517), (64, 200), (3000, 1500)])
def test_uniform_nnls_bitwise(solver, oracle, d, n):
    inst = instances.make_config("c1", d=d, n=n, seed=d + n)
    cfg = SolverConfig(epsilon=1e-8, max_iters=10000, stall_window=10**9)
    check_nnls(solver, oracle, inst["A"], inst["b"], cfg)


def test_c1_full_bitwise(solver, oracle):
    inst = instances.make_config("c1")
    cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
    got, exp = check_nnls(solver, oracle, inst["A"], inst["b"], cfg)
    tol = baseline_tolerances(got.x, exp["x"], got.inner.trace[-1].f, exp["trace"][-1]["f"],
                              got.inner.iterations(), exp["iterations"])
    assert all(tol[k] for k in ("objective_ok", "x_ok", "support_ok", "iter_ok"))


@pytest.mark.parametrize("name,d,n", [("c2", 1024, 512), ("c3", 512, 512), ("c5", 1024, 512)])
def test_scaled_configs_bitwise(solver, oracle, name, d, n):
    inst = instances.make_config(name, d=d, n=n)
    cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=3000, stall_window=10**9)
    check_nnls(solver, oracle, inst["A"], inst["b"], cfg)


def test_defaults_stall_window(solver, oracle):
    """Default SolverConfig (stall 50, eps 1e-10*m, max 5m) on a lopsided instance."""
    inst = instances.make_config("c5", d=400, n=200, seed=77)
    check_nnls(solver, oracle, inst["A"], inst["b"], SolverConfig())


def test_device_entry_matches_host_entry(solver):
    import torch
    inst = instances.make_config("c1", d=300, n=150, seed=9)
    cfg = SolverConfig(epsilon=1e-8, max_iters=10000, stall_window=10**9)
    host = solver.solve_nnls(inst["A"], inst["b"], cfg)
    A = torch.from_numpy(np.asfortranarray(inst["A"])).cuda()
    At = A.t().contiguous()  # row-major (n, d) == column-major (d, n)
    b = torch.from_numpy(inst["b"]).cuda()
    dev = solver.solve_nnls_device(At.data_ptr(), 300, 300, 150, b.data_ptr(), cfg)
    assert same_bits(dev.x, host.x) and dev.inner.iterations() == host.inner.iterations()
    # odd leading dimension exercises the padded-copy path
    Ap = torch.zeros((150, 301), dtype=torch.float64, device="cuda")
    Ap[:, :300] = At
    dev2 = solver.solve_nnls_device(Ap.data_ptr(), 301, 300, 150, b.data_ptr(), cfg)
    assert same_bits(dev2.x, host.x)

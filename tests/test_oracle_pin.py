"""Pins the C restatement (oracle/antilop_oracle.c) to the reference compiled
from its own headers (oracle/_ref): bitwise on every output, over the
reference's known-answer cases and seeded random problems of every config law.
CPU only. Skips when oracle/_ref is absent (no reference sources at build time)."""
import numpy as np
import pytest

from paper_1502_01645_b200 import abi, instances
from tests.parity import same_bits
from tests.splitmix import SplitMix64


def smx(rows, cols, seed, lo=-1.0, hi=1.0):
    r = SplitMix64(seed)
    M = np.zeros((rows, cols), order="F")
    for j in range(cols):
        for i in range(rows):
            M[i, j] = lo + (hi - lo) * r.uniform01()
    return M


def assert_same_solve(a, b):
    assert a["termination"] == b["termination"]
    assert a["iterations"] == b["iterations"]
    assert same_bits(a["x"], b["x"])
    assert same_bits(a["final_grad"], b["final_grad"])
    assert len(a["trace"]) == len(b["trace"])
    for ra, rb in zip(a["trace"], b["trace"]):
        assert ra["iter"] == rb["iter"] and ra["passive_count"] == rb["passive_count"]
        assert same_bits([ra["f"], ra["grad_bar_sq"]], [rb["f"], rb["grad_bar_sq"]])
        assert (ra["alpha"] is None) == (rb["alpha"] is None)
        if ra["alpha"] is not None:
            assert same_bits([ra["alpha"]], [rb["alpha"]])
    assert a["min_iterate"] == b["min_iterate"]


def test_dense_kernels(oracle, ref):
    rng = np.random.default_rng(0)
    for d, n in [(1, 1), (7, 3), (64, 33), (300, 129)]:
        A = rng.standard_normal((d, n))
        v = rng.standard_normal(d)
        w = rng.standard_normal(n)
        assert same_bits(oracle.gram(A), ref.gram(A))
        assert same_bits(oracle.transpose_matvec(A, v), ref.transpose_matvec(A, v))
        assert same_bits(oracle.matvec(A, w), ref.matvec(A, w))
        mask = np.sort(rng.choice(n, max(1, n // 2), replace=False))
        ya, ca = oracle.masked_matvec(A, w, mask, 3)
        yb, cb = ref.masked_matvec(A, w, mask, 3)
        assert same_bits(ya, yb) and ca == cb


def test_rescale(oracle, ref):
    rng = np.random.default_rng(1)
    A = rng.uniform(0, 1, (40, 17))
    A[:, 5] = 0.0
    H = ref.gram(A)
    h = -ref.transpose_matvec(A, rng.standard_normal(40))
    a, b = oracle.rescale(H, h), ref.rescale(H, h)
    for k in ("Q", "q", "scale"):
        assert same_bits(a[k], b[k])
    assert list(a["retained"]) == list(b["retained"]) and list(a["dropped"]) == list(b["dropped"])


@pytest.mark.parametrize("seed", list(range(100, 130)))
def test_nqp_random(oracle, ref, seed):  # test_nqp.cpp:273-296 family
    n = 2 + seed % 7
    A = smx(n + 4, n, seed)
    Q = ref.gram(A)
    q = smx(n, 1, seed + 7)[:, 0]
    cfg = abi.make_config(epsilon=1e-20, max_iters=200000, stall_window=1000000)
    assert_same_solve(oracle.solve_nqp(Q, q, cfg), ref.solve_nqp(Q, q, cfg))


@pytest.mark.parametrize("seed", list(range(200, 230)))
def test_nnls_rectangles(oracle, ref, seed):  # test_nnls.cpp:196-218 family
    n = 2 + seed % 7
    d = n + 1 + seed % 8
    A = smx(d, n, seed, 0.0 if seed % 2 else -1.0, 1.0)
    b = smx(d, 1, seed + 999)[:, 0]
    cfg = abi.make_config(epsilon=1e-20, max_iters=200000, stall_window=1000000)
    a, r = oracle.solve_nnls(A, b, cfg), ref.solve_nnls(A, b, cfg)
    assert_same_solve(a, r)
    assert same_bits([a["residual_sq"]], [r["residual_sq"]])
    assert same_bits(a["inner_x"], r["inner_x"])


@pytest.mark.parametrize("name,d,n,stall", [("c1", 600, 300, 10**9), ("c2", 300, 150, 10**9),
                                            ("c3", 128, 128, 10**9), ("c5", 300, 150, 10**9),
                                            ("c5", 200, 100, 50)])
def test_config_laws(oracle, ref, name, d, n, stall):
    inst = instances.make_config(name, d=d, n=n)
    cfg = abi.make_config(epsilon=inst["epsilon"], max_iters=3000, stall_window=stall)
    a, r = oracle.solve_nnls(inst["A"], inst["b"], cfg), ref.solve_nnls(inst["A"], inst["b"], cfg)
    assert_same_solve(a, r)
    assert same_bits([a["residual_sq"]], [r["residual_sq"]])


def test_solver_paths(oracle, ref):
    """Warm start, halving, trace sampling, every termination, numeric failure."""
    lop = (np.array([[1.0, 0.1], [0.1, 9.0]]), np.array([-4.0, -5.0]))
    cases = [
        (lop, dict(epsilon=1e-10, max_iters=100000), [30.0, 2.0]),
        ((np.array([[1.0, 0.9], [0.9, 1.0]]), np.array([1.49, -2.69])),
         dict(epsilon=1e-18, max_iters=10000, stall_window=1000000), [0.52, 0.35]),
        (lop, dict(epsilon=1e-18, max_iters=100000, stall_window=1000000, trace_every=4), None),
        (lop, dict(epsilon=1e-30, max_iters=3, stall_window=1000), None),
        ((np.eye(2), np.array([-1.0, -2.0])), dict(time_cap=0.0), None),
        ((np.array([[1.0, 1 / 30], [1 / 30, 1.0]]), np.array([-4.0, -5 / 3])),
         dict(epsilon=5e-324, max_iters=1000000, stall_window=5), None),
        ((np.zeros((2, 2)), np.array([-1.0, -1.0])), dict(), None),
        ((np.eye(2), np.array([3.0, 4.0])), dict(), None),
    ]
    for (Q, q), kw, start in cases:
        cfg = abi.make_config(**kw)
        a = oracle.solve_nqp(Q, q, cfg, start=start)
        r = ref.solve_nqp(Q, q, cfg, start=start)
        if kw.get("time_cap") is None:
            assert_same_solve(a, r)
        else:
            assert a["termination"] == r["termination"] == "TimeCap"
    from oracle.oracle import OracleError
    for o in (oracle, ref):
        with pytest.raises(OracleError) as ei:
            o.solve_nqp(np.eye(2), np.array([-1e308, -1.0]), abi.make_config())
        assert ei.value.status == abi.ENUMERIC and ei.value.result["trace_len"] == 0


def test_invalid_inputs(oracle, ref):
    from oracle.oracle import OracleError
    for o in (oracle, ref):
        with pytest.raises(OracleError) as ei:
            o.rescale(np.array([[1.0, 0.2], [0.1, 1.0]]), np.array([1.0, 2.0]))
        assert ei.value.status == abi.EINVAL
        with pytest.raises(OracleError) as ei:
            o.rescale(np.array([[-1.0, 0.0], [0.0, 1.0]]), np.array([1.0, 2.0]))
        assert ei.value.status == abi.EINVAL
        with pytest.raises(OracleError) as ei:
            o.solve_nqp(np.eye(2), np.array([1.0, 1.0]), abi.make_config(epsilon=-1.0))
        assert ei.value.status == abi.EINVAL
        with pytest.raises(OracleError) as ei:
            o.masked_matvec(np.eye(2), np.ones(2), [2])
        assert ei.value.status == abi.ERANGE


# ---- Anti+Acc baseline (accelerated.hpp) --------------------

@pytest.mark.parametrize("name,d,n,restart,kw", [
    ("c1", 200, 80, False, dict(epsilon=1e-8, max_iters=3000, stall_window=10**9)),
    ("c1", 200, 80, True, dict(epsilon=1e-8, max_iters=3000, stall_window=10**9)),
    ("c2", 300, 150, False, dict(epsilon=1e-8, stall_window=10**9)),
    ("c5", 240, 120, True, dict()),  # defaults: eps 1e-10 m, 5m iterations, stall 50
    ("c3", 160, 160, False, dict(epsilon=1e-10, max_iters=400, trace_every=7)),
])
def test_anti_accelerated_matches_reference(name, d, n, restart, kw):
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    inst = instances.make_config(name, d=d, n=n)
    cfg = abi.make_config(nesterov_restart=restart, **kw)
    e = Oracle("oracle").solve_anti_accelerated(inst["A"], inst["b"], cfg)
    r = Oracle("ref").solve_anti_accelerated(inst["A"], inst["b"], cfg)
    assert e["iterations"] == r["iterations"] and e["termination"] == r["termination"]
    assert np.array_equal(e["x"].view(np.uint64), r["x"].view(np.uint64))
    assert np.array_equal(e["final_grad"].view(np.uint64), r["final_grad"].view(np.uint64))
    assert e["residual_sq"] == r["residual_sq"]
    assert len(e["trace"]) == len(r["trace"])
    for a, b in zip(e["trace"], r["trace"]):
        assert a["iter"] == b["iter"] and a["passive_count"] == b["passive_count"]
        assert a["f"] == b["f"] and a["grad_bar_sq"] == b["grad_bar_sq"] and a["alpha"] == b["alpha"]

"""Edge cases of the round-1 additions on the GPU: the batched kernel's 8- and
4-column variants (m up to 512 / 1024) and its size limit, dropped columns in
the batched, row-block and Anti+Acc paths, and failures reported like the
reference (exceptions, not silent results)."""
import numpy as np
import pytest
import torch

from paper_1502_01645_b200 import abi
from paper_1502_01645_b200.api import SolverConfig
from paper_1502_01645_b200.rowblock import row_split
from tests.parity import same_bits

pytestmark = pytest.mark.gpu


def ref_columns(A, B, cfg):
    from oracle.oracle import Oracle
    o = Oracle("oracle")
    out = []
    for j in range(B.shape[1]):
        out.append(o.solve_nnls(A, B[:, j].copy(), cfg.to_abi()))
    return out


@pytest.mark.parametrize("n", [300, 520])  # NB = 8 (m <= 512) and NB = 4 (m <= 1024)
def test_batched_wide_problems_bitwise(solver, n):
    rng = np.random.default_rng(n)
    d = n + 200
    A = rng.uniform(0.0, 1.0, (d, n))
    H = np.where(rng.uniform(size=(n, 6)) < 0.4, 0.0, rng.uniform(size=(n, 6)))
    B = np.asfortranarray(A @ H)
    cfg = SolverConfig(epsilon=1e-8, max_iters=300, stall_window=10**9)
    X, cols, _ = solver.solve_nnls_batched(A, B, cfg)
    for j, r in enumerate(ref_columns(A, B, cfg)):
        assert cols[j]["iterations"] == r["iterations"], j
        assert same_bits(X[:, j], r["x"]), j


def test_batched_wider_than_the_batched_kernel_bitwise(solver):
    """m > 1024 does not fit the batched kernel's per-column shared-memory state: the
    columns then run one by one through the single-RHS device loop on the shared Q
    (capi.cu run_batched) — the reference takes any size (nnls.hpp:129-144)."""
    rng = np.random.default_rng(1)
    n, d = 1030, 1100
    A = rng.uniform(size=(d, n))
    H = np.where(rng.uniform(size=(n, 3)) < 0.5, 0.0, rng.uniform(size=(n, 3)))
    B = np.asfortranarray(A @ H + 1e-3 * rng.standard_normal((d, 3)))
    cfg = SolverConfig(epsilon=1e-8, max_iters=40, stall_window=10**9)
    X, cols, _ = solver.solve_nnls_batched(A, B, cfg)
    for j, r in enumerate(ref_columns(A, B, cfg)):
        assert cols[j]["iterations"] == r["iterations"], j
        assert cols[j]["termination"] == r["termination"], j
        assert same_bits(X[:, j], r["x"]), j
        assert same_bits([cols[j]["residual_sq"]], [r["residual_sq"]]), j
        single = solver.solve_nnls(A, B[:, j].copy(), cfg)
        assert same_bits(X[:, j], single.x), j


def test_batched_with_dropped_columns(solver):
    rng = np.random.default_rng(5)
    A = rng.uniform(size=(120, 40))
    A[:, [3, 17]] = 0.0
    B = np.asfortranarray(rng.standard_normal((120, 9)))
    cfg = SolverConfig(epsilon=1e-9, stall_window=10**9)
    X, cols, _ = solver.solve_nnls_batched(A, B, cfg)
    for j, r in enumerate(ref_columns(A, B, cfg)):
        assert same_bits(X[:, j], r["x"]) and cols[j]["iterations"] == r["iterations"], j
    assert np.all(X[[3, 17], :] == 0.0)


def test_rowblock_with_dropped_columns(solver, oracle):
    rng = np.random.default_rng(9)
    d, n = 900, 300
    A = rng.uniform(size=(d, n))
    A[:, [0, 150, 299]] = 0.0
    b = rng.standard_normal(d)
    cfg = SolverConfig(epsilon=1e-9, stall_window=10**9)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()
    T = solver.gram_tiles(n)
    H = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    st = None
    blocks = row_split(d, 3)
    for p, (r0, r1) in enumerate(blocks):
        out = None if p == len(blocks) - 1 else torch.empty(T * 16384, dtype=torch.float64, device="cuda")
        solver.gram_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, 0, T,
                                    st.data_ptr() if st is not None else 0,
                                    out.data_ptr() if out is not None else 0,
                                    0 if out is not None else H.data_ptr())
        st = out
    atb = None
    for (r0, r1) in blocks:
        nxt = torch.empty(n, dtype=torch.float64, device="cuda")
        solver.atb_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, db.data_ptr() + 8 * r0,
                                   atb.data_ptr() if atb is not None else 0, nxt.data_ptr())
        atb = nxt
    got = solver.solve_nnls_gram_device(n, H.data_ptr(), atb.data_ptr(), cfg)
    exp = oracle.solve_nnls(A, b, cfg.to_abi())
    assert same_bits(got.x, exp["x"]) and got.inner.iterations() == exp["iterations"]
    assert got.dropped_columns == [0, 150, 299]


def test_anti_accelerated_dropped_and_numeric(solver, oracle):
    rng = np.random.default_rng(2)
    A = rng.uniform(size=(80, 30))
    A[:, 4] = 0.0
    b = rng.standard_normal(80)
    cfg = SolverConfig(epsilon=1e-9, max_iters=2000, stall_window=10**9)
    got = solver.solve_anti_accelerated(A, b, cfg)
    exp = oracle.solve_anti_accelerated(A, b, cfg.to_abi())
    assert same_bits(got.x, exp["x"]) and got.dropped_columns == [4]
    # a non-finite objective raises NumericFailure like the reference (accelerated.hpp:55-58)
    Q = np.eye(2)
    q = np.array([-1e308, -1.0])
    with pytest.raises(Exception):
        solver.solve_accelerated(Q, q, SolverConfig(max_iters=10))


def test_fast_batched_wide_falls_back(solver):
    """FAST on NB = 8 shapes uses the SIMT pass (DMMA pass is for 16-column CTAs):
    still a valid solve of the same problems."""
    rng = np.random.default_rng(4)
    A = rng.uniform(size=(500, 300))
    B = np.asfortranarray(A @ rng.uniform(size=(300, 5)))
    X, cols, _ = solver.solve_nnls_batched(A, B, SolverConfig(epsilon=1e-8, max_iters=400,
                                                              profile=abi.PROFILE_FAST))
    assert np.all(np.isfinite(X)) and np.all(X >= 0.0)

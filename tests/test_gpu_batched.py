"""GPU parity of the batched multi-RHS path (K8, config c4 law): every column must
be bitwise solve_nnls(A, B[:, j], cfg) of the reference, i.e. the reference's
per-column pipeline with the Gram shared (oracle/_ref ref_solve_nnls_columns,
or the C restatement per column when _ref is absent)."""
import numpy as np
import pytest

from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import SolverConfig
from tests.parity import same_bits

pytestmark = pytest.mark.gpu


def reference_columns(A, B, cfg):
    from oracle.oracle import Oracle, available
    if available("ref"):
        return Oracle("ref").solve_nnls_columns(A, B, cfg.to_abi(record_multiplies=False),
                                                threads=8)
    o = Oracle("oracle")
    X = np.zeros((A.shape[1], B.shape[1]), order="F")
    cols = []
    for j in range(B.shape[1]):
        r = o.solve_nnls(A, B[:, j].copy(), cfg.to_abi())
        X[:, j] = r["x"]
        cols.append(r)
    return X, cols


def check(solver, A, B, cfg):
    X, cols, _ = solver.solve_nnls_batched(A, B, cfg)
    Xr, cr = reference_columns(A, B, cfg)
    for j in range(B.shape[1]):
        ref_term = cr[j].termination if hasattr(cr[j], "termination") else None
        if hasattr(cr[j], "iterations"):
            from paper_1502_01645_b200.abi import TERMINATIONS
            assert cols[j]["iterations"] == cr[j].iterations, j
            assert cols[j]["termination"] == TERMINATIONS[ref_term], j
            assert same_bits([cols[j]["residual_sq"]], [cr[j].residual_sq]), j
            assert same_bits([cols[j]["f_final"]], [cr[j].f_final]), j
            assert cols[j]["multiplies_total"] == cr[j].multiplies_total, j
        else:
            assert cols[j]["iterations"] == cr[j]["iterations"], j
            assert same_bits([cols[j]["residual_sq"]], [cr[j]["residual_sq"]]), j
        assert same_bits(X[:, j], Xr[:, j]), f"column {j} x differs"
    return X, cols


@pytest.mark.parametrize("d,n,k", [(200, 40, 37), (600, 130, 20), (300, 256, 33)])
def test_batched_uniform_bitwise(solver, d, n, k):
    inst = instances.make_batched(d=d, n=n, nrhs=k, seed=d + n)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9)
    check(solver, inst["A"], inst["B"], cfg)


def test_batched_defaults_and_noise(solver):
    rng = np.random.default_rng(4)
    A = rng.uniform(0, 1, (150, 50))
    A[:, 7] = 0.0  # a dropped column
    B = rng.standard_normal((150, 40))
    check(solver, A, B, SolverConfig())  # default stall window 50, eps 1e-10 m, 5m iterations


def test_batched_c4_law_recovers_htrue(solver):
    inst = instances.make_batched(d=2000, n=256, nrhs=64, seed=9)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9)
    X, cols = check(solver, inst["A"], inst["B"], cfg)
    assert np.max(np.abs(X - inst["H_true"])) < 1e-4


def test_batched_matches_single_solves(solver):
    inst = instances.make_batched(d=120, n=30, nrhs=5, seed=3)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9)
    X, cols, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg)
    for j in range(5):
        r = solver.solve_nnls(inst["A"], inst["B"][:, j].copy(), cfg)
        assert same_bits(X[:, j], r.x)
        assert cols[j]["iterations"] == r.inner.iterations()
        assert same_bits([cols[j]["residual_sq"]], [r.residual_sq])


def test_batched_c4_full_shape_sampled_columns(solver):
    """c4 at its full shape (A 20000 x 256) over 2048 right-hand sides; every
    64th column is checked bit for bit against the reference pipeline (SURVEY
    §8d: "bitwise on every oracle-sampled column")."""
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    inst = instances.make_batched(nrhs=2048)
    cfg = SolverConfig(epsilon=inst["epsilon"], stall_window=10**9)
    X, cols, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg)
    sample = list(range(0, 2048, 64))
    Bs = np.asfortranarray(inst["B"][:, sample])
    import os
    Xr, cr = Oracle("ref").solve_nnls_columns(inst["A"], Bs, cfg.to_abi(record_multiplies=False),
                                              threads=os.cpu_count() or 1)
    for k, j in enumerate(sample):
        assert same_bits(X[:, j], Xr[:, k]), j
        assert cols[j]["iterations"] == cr[k].iterations
        assert same_bits([cols[j]["residual_sq"]], [cr[k].residual_sq])
    assert np.max(np.abs(X - inst["H_true"])) < 1e-3


@pytest.mark.parametrize("profile", ["exact", "fast"])
def test_batched_host_pipeline_chunked_upload(solver, monkeypatch, profile):
    """The host-buffer entry uploads B in two column chunks under the solves (capi.cu
    run_batched); forced here at a small batch: the oracle's per-column results (EXACT),
    and exactly the one-launch path's X and column records (both profiles)."""
    from paper_1502_01645_b200 import abi
    inst = instances.make_batched(d=500, n=96, nrhs=203, seed=21)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9,
                       profile=abi.PROFILE_FAST if profile == "fast" else abi.PROFILE_EXACT)
    monkeypatch.setenv("ALNNLS_BATCH_OVERLAP_MIN", "0")
    X1, c1, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg)
    monkeypatch.setenv("ALNNLS_BATCH_OVERLAP_MIN", "64")
    if profile == "exact":
        X2, c2 = check(solver, inst["A"], inst["B"], cfg)
    else:
        X2, c2, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg)
    assert same_bits(X1.reshape(-1, order="F"), X2.reshape(-1, order="F"))
    keys = ("iterations", "termination", "residual_sq", "f_final", "gbs_final", "multiplies_total")
    assert [[c[k] for k in keys] for c in c1] == [[c[k] for k in keys] for c in c2]
    # a non-finite entry in the second chunk is still the reference's construction error
    Bbad = inst["B"].copy(order="F")
    Bbad[3, 150] = np.nan
    with pytest.raises(Exception, match="non-finite"):
        solver.solve_nnls_batched(inst["A"], Bbad, cfg)
    buf = np.full(X1.shape, 7.0, order="F")  # the context recovers; a caller-owned result buffer
    X3, _, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg, out=buf)
    assert X3 is buf
    assert same_bits(X1.reshape(-1, order="F"), X3.reshape(-1, order="F"))
    with pytest.raises(ValueError, match="out must be"):
        solver.solve_nnls_batched(inst["A"], inst["B"], cfg, out=np.empty(X1.shape))


# ---- NMF by alternating NNLS over the batched entry -------------------
def test_nmf_bitwise_vs_oracle_alternating_nnls(solver, oracle):
    """alnnls_nmf's half steps are batched solve_nnls calls (Gram shared per half
    step): under EXACT every W and H entry and the objective trace are bitwise the
    oracle's per-column solve_nnls composed the same way (H from W, then W from
    H^T against V^T)."""
    from paper_1502_01645_b200.api import SolverConfig
    rng = np.random.default_rng(1)
    d, N, k = 60, 40, 5
    Wt = rng.uniform(size=(d, k))
    Ht = rng.uniform(size=(k, N))
    Ht[rng.uniform(size=Ht.shape) < 0.3] = 0.0
    V = np.asfortranarray(Wt @ Ht)
    W0 = np.asfortranarray(rng.uniform(size=(d, k)))
    cfg = SolverConfig(epsilon=1e-10, stall_window=10**9)
    W, H, obj = solver.nmf(V, W0, 3, cfg)
    Wo = W0.copy(order="F")
    objo = []
    for _ in range(3):
        Ho = np.zeros((k, N), order="F")
        tot = 0.0
        for j in range(N):
            r = oracle.solve_nnls(Wo, V[:, j], cfg.to_abi())
            Ho[:, j] = r["x"]
            tot += r["residual_sq"]
        objo.append(tot)
        WoT = np.zeros((k, d), order="F")
        HoT = np.asfortranarray(Ho.T)
        for i in range(d):
            WoT[:, i] = oracle.solve_nnls(HoT, np.ascontiguousarray(V[i, :]), cfg.to_abi())["x"]
        Wo = np.asfortranarray(WoT.T)
    from tests.parity import same_bits
    assert same_bits(H.reshape(-1, order="F"), Ho.reshape(-1, order="F"))
    assert same_bits(W.reshape(-1, order="F"), Wo.reshape(-1, order="F"))
    assert same_bits(obj, objo)
    assert obj[1] <= obj[0] * (1 + 1e-12) and obj[2] <= obj[1] * (1 + 1e-12)


def test_nmf_reconstructs_low_rank(solver):
    """A rank-8 nonnegative V (c4's laws at small size): the ANLS objective falls
    by orders of magnitude and never increases beyond solve tolerance."""
    from paper_1502_01645_b200.api import SolverConfig
    rng = np.random.default_rng(7)
    d, N, k = 400, 300, 8
    V = np.asfortranarray(rng.uniform(size=(d, k)) @ rng.uniform(size=(k, N)))
    W0 = np.asfortranarray(rng.uniform(size=(d, k)))
    W, H, obj = solver.nmf(V, W0, 25, SolverConfig(epsilon=1e-10, stall_window=10**9))
    assert np.all(W >= 0) and np.all(H >= 0)
    for t in range(1, len(obj)):
        assert obj[t] <= obj[t - 1] * (1 + 1e-9) + 1e-12
    assert obj[-1] <= 1e-2 * obj[0]
    assert np.linalg.norm(V - W @ H) ** 2 <= 2 * obj[-1] + 1e-9

"""Exact multi-GPU setup by row blocks (c5) on ONE GPU: the row
blocks are fed one after another through the same C-ABI entries the ranks call,
and the results must be bitwise the single-call reference functions (gram,
transpose_matvec, solve_nnls, residual_norm_sq)."""
import numpy as np
import pytest
import torch

from paper_1502_01645_b200.api import SolverConfig
from paper_1502_01645_b200.rowblock import row_split
from tests.parity import same_bits

pytestmark = pytest.mark.gpu
TD = 16384


def run_blocks(solver, A, b, blocks, batches):
    d, n = A.shape
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # column-major A, ld = d
    db = torch.from_numpy(b).cuda()
    T = solver.gram_tiles(n)
    H = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    states = None
    for p, (r0, r1) in enumerate(blocks):
        last = p == len(blocks) - 1
        out = None if last else torch.empty(T * TD, dtype=torch.float64, device="cuda")
        for t0, t1 in batches(T):
            pin = states[t0 * TD:] if states is not None else None
            pout = out[t0 * TD:] if out is not None else None
            solver.gram_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, t0, t1,
                                        pin.data_ptr() if pin is not None else 0,
                                        pout.data_ptr() if pout is not None else 0,
                                        0 if pout is not None else H.data_ptr())
        states = out
    atb = None
    for (r0, r1) in blocks:
        nxt = torch.empty(n, dtype=torch.float64, device="cuda")
        solver.atb_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, db.data_ptr() + 8 * r0,
                                   atb.data_ptr() if atb is not None else 0, nxt.data_ptr())
        atb = nxt
    return dA, db, H, atb


@pytest.mark.parametrize("d,n,nblk", [(700, 300, 3), (257, 129, 2), (1000, 520, 4)])
def test_rowblock_gram_and_atb_bitwise(solver, oracle, d, n, nblk):
    rng = np.random.default_rng(d + n)
    A = np.asfortranarray(rng.standard_normal((d, n)))
    b = rng.standard_normal(d)
    _, _, H, atb = run_blocks(solver, A, b, row_split(d, nblk),
                              lambda T: [(t, min(T, t + 2)) for t in range(0, T, 2)])
    Href = oracle.gram(A)
    assert same_bits(H.cpu().numpy().reshape(-1, order="F"), Href.reshape(-1, order="F"))
    assert same_bits(atb.cpu().numpy(), oracle.transpose_matvec(A, b))


def test_rowblock_solve_and_residual_bitwise(solver):
    from paper_1502_01645_b200 import instances
    inst = instances.make_config("c5", d=1200, n=600)
    A, b = inst["A"], inst["b"]
    cfg = SolverConfig(epsilon=inst["epsilon"], stall_window=10**9)
    ref = solver.solve_nnls(A, b, cfg)
    blocks = row_split(A.shape[0], 3)
    dA, db, H, atb = run_blocks(solver, A, b, blocks, lambda T: [(0, T)])
    got = solver.solve_nnls_gram_device(A.shape[1], H.data_ptr(), atb.data_ptr(), cfg)
    assert same_bits(got.x, ref.x)
    assert got.inner.iterations() == ref.inner.iterations()
    assert same_bits([r.f for r in got.inner.trace], [r.f for r in ref.inner.trace])
    dx = torch.from_numpy(got.x).cuda()
    s = 0.0
    for (r0, r1) in blocks:
        s = solver.residual_rowblock_device(r1 - r0, A.shape[1], dA.data_ptr() + 8 * r0, A.shape[0],
                                            db.data_ptr() + 8 * r0, dx.data_ptr(), s)
    assert same_bits([s], [ref.residual_sq])


# ---- configs[4] as written: partial Grams + one allreduce ------------------
def _partials(solver, A, b, blocks, profile):
    """Every block's partial [H | A^T b] through alnnls_gram_partial_device, summed in
    rank order on the device (what the allreduce computes for this world size)."""
    d, n = A.shape
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()
    tot = torch.zeros(n * n + n, dtype=torch.float64, device="cuda")
    for (r0, r1) in blocks:
        buf = torch.empty(n * n + n, dtype=torch.float64, device="cuda")
        solver.gram_partial_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, db.data_ptr() + 8 * r0,
                                   buf.data_ptr(), buf.data_ptr() + 8 * n * n, profile=profile)
        tot += buf
    return dA, db, tot[: n * n].view(n, n), tot[n * n:]


@pytest.mark.parametrize("profile", [0, 1])
def test_gram_partial_one_block_matches_reference(solver, oracle, profile):
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.standard_normal((640, 272)))
    b = rng.standard_normal(640)
    _, _, H, atb = _partials(solver, A, b, [(0, 640)], profile)
    Href = oracle.gram(A)
    Hg = H.cpu().numpy()
    assert np.array_equal(Hg, Hg.T)
    if profile == 0:  # one block = the reference chain, bit for bit
        assert same_bits(Hg.reshape(-1, order="F"), Href.reshape(-1, order="F"))
    else:             # DMMA: within rounding
        assert np.max(np.abs(Hg - Href)) <= 1e-13 * 640 * np.max(np.abs(Href))
    assert same_bits(atb.cpu().numpy(), oracle.transpose_matvec(A, b))


@pytest.mark.parametrize("profile", [0, 1])
def test_allreduce_setup_c5_law(solver, oracle, profile):
    """SURVEY §8d c5 variant (i): Q, q within 1e-13 (relative) of rescale(gram) of the
    reference; the loop bitwise against the reference loop run on the GPU's own Q, q;
    the objective and a KKT certificate end to end."""
    from paper_1502_01645_b200 import instances
    inst = instances.make_config("c5", d=1600, n=640)
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    cfg = SolverConfig(epsilon=inst["epsilon"], stall_window=10**9)
    blocks = row_split(d, 4)
    dA, db, H, atb = _partials(solver, A, b, blocks, profile)
    got = solver.solve_nnls_gram_device(n, H.data_ptr(), atb.data_ptr(), cfg)
    mine = solver._scaled()
    ref_sys = oracle.rescale(oracle.gram(A), -oracle.transpose_matvec(A, b))
    Qr, qr = ref_sys["Q"], ref_sys["q"]
    assert np.max(np.abs(mine["Q"] - Qr)) <= 1e-13 * max(1.0, np.max(np.abs(Qr)))
    assert np.max(np.abs(mine["q"] - qr)) <= 1e-13 * max(1.0, np.max(np.abs(qr)))
    loop = oracle.solve_nqp(mine["Q"], mine["q"], cfg.to_abi())
    assert same_bits(got.inner.x, loop["x"])
    assert got.inner.iterations() == loop["iterations"]
    ref = oracle.solve_nnls(A, b, cfg.to_abi())
    f_got, f_ref = got.inner.trace[-1].f, ref["trace"][-1]["f"]
    assert abs(f_got - f_ref) <= 1e-10 * abs(f_ref)  # BASELINE objective bar
    # KKT certificate (acceptance.cpp:253-256) in the scaled space
    g = mine["Q"] @ got.inner.x + mine["q"]
    x = got.inner.x
    viol = np.max(np.where(x > 0, np.abs(g), np.maximum(0.0, -g)))
    assert viol <= np.sqrt(cfg.epsilon) * (1 + np.linalg.norm(mine["q"]))
    dx = torch.from_numpy(got.x).cuda()
    parts = [solver.residual_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d,
                                             db.data_ptr() + 8 * r0, dx.data_ptr(), 0.0)
             for (r0, r1) in blocks]
    chain = 0.0  # the reference's one ordered chain (nnls.hpp:119-122) over the same x
    for (r0, r1) in blocks:
        chain = solver.residual_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d,
                                                db.data_ptr() + 8 * r0, dx.data_ptr(), chain)
    # the allreduce sums 4 partial chains instead: a different order of the same terms
    assert abs(sum(parts) - chain) <= 1e-12 * chain


def test_pack_unpack_upper_roundtrip(solver):
    """alnnls_pack_upper_device / alnnls_unpack_upper_device: the allreduce moves
    n(n+1)/2 doubles; unpacking mirrors the upper triangle bit for bit."""
    n = 333
    rng = np.random.default_rng(3)
    M = rng.standard_normal((n, n))
    H = np.asfortranarray(M + M.T)
    dH = torch.from_numpy(np.ascontiguousarray(H.T)).cuda()  # column-major
    P = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device="cuda")
    solver.pack_upper_device(n, dH.data_ptr(), P.data_ptr())
    Pc = P.cpu().numpy()
    j = 17
    assert same_bits(Pc[j * (j + 1) // 2: j * (j + 1) // 2 + j + 1], H[: j + 1, j])
    back = torch.full((n, n), np.nan, dtype=torch.float64, device="cuda")
    solver.unpack_upper_device(n, P.data_ptr(), back.data_ptr())
    assert same_bits(back.cpu().numpy().T.reshape(-1), H.reshape(-1, order="F"))


def test_allreduce_setup_packed_world1(solver, oracle):
    """rowblock.allreduce_setup with the GPU pack/unpack (world 1): exactly the
    partial Gram, mirrored, and the A^T b chains."""
    from paper_1502_01645_b200.rowblock import allreduce_setup
    rng = np.random.default_rng(9)
    d, n = 500, 210
    A = np.asfortranarray(rng.standard_normal((d, n)))
    b = rng.standard_normal(d)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()

    def partial(Hm, atb):
        solver.gram_partial_device(d, n, dA.data_ptr(), d, db.data_ptr(), Hm.data_ptr(),
                                   atb.data_ptr(), profile=0)

    H, atb = allreduce_setup(None, 1, n, partial, "cuda",
                             pack=lambda Hm, P: solver.pack_upper_device(n, Hm.data_ptr(), P.data_ptr()),
                             unpack=lambda P, Hm: solver.unpack_upper_device(n, P.data_ptr(), Hm.data_ptr()))
    assert same_bits(H.cpu().numpy().reshape(-1), oracle.gram(A).reshape(-1, order="F"))
    assert same_bits(atb.cpu().numpy(), oracle.transpose_matvec(A, b))


def test_finish_matches_solve_nnls(solver):
    """alnnls_finish (unscale + residual, nnls.hpp:141-142) reproduces solve_nnls's
    x and residual from its inner solution; dimension mismatches are EINVAL."""
    from paper_1502_01645_b200 import instances
    inst = instances.make_config("c1", d=300, n=150, seed=21)
    A, b = inst["A"], inst["b"]
    A[:, 7] = 0.0  # a dropped column: unscale writes 0 there
    r = solver.solve_nnls(A, b, SolverConfig(epsilon=1e-8, stall_window=10**9))
    x, res = solver.finish(A, b, r.inner.x)
    assert same_bits(x, r.x) and same_bits([res], [r.residual_sq])
    assert x[7] == 0.0
    with pytest.raises(ValueError):
        solver.finish(A, b, r.inner.x[:-1])


def test_batched_multi_context_shards_match(solver):
    """alnnls_solve_nnls_batched_multi: column shards over several contexts (here
    three contexts on the one GPU this box has) give the one-context results bit
    for bit (every column is an independent solve)."""
    from paper_1502_01645_b200 import instances
    from paper_1502_01645_b200.api import Solver, solve_nnls_batched_multi
    inst = instances.make_batched(d=1500, n=128, nrhs=37, seed=5)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9)
    X1, c1, _ = solver.solve_nnls_batched(inst["A"], inst["B"], cfg)
    extra = [Solver(0), Solver(0)]
    try:
        X3, c3, summ = solve_nnls_batched_multi([solver] + extra, inst["A"], inst["B"], cfg)
    finally:
        for s in extra:
            s.close()
    assert same_bits(X3.reshape(-1), X1.reshape(-1))
    assert [c["iterations"] for c in c3] == [c["iterations"] for c in c1]
    assert same_bits([c["residual_sq"] for c in c3], [c["residual_sq"] for c in c1])
    assert summ.iterations == sum(c["iterations"] for c in c1)

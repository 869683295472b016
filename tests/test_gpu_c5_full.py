"""BASELINE.json c5 (configs[4], d=32768, n=16384, 10% of the columns x 1e3) at
FULL size on the GPU, bit for bit against the reference's own run
(tests/golden/full_c5.npz, made by tests/golden/make_golden_c5.py from
oracle/_ref: the reference's gram over column-block pairs, its rescale, its
solve_nqp single-threaded for 2858 s, 6906 iterations):
  - the default EXACT path through the host-buffer entry (upload overlapped with
    the Gram): Q and q (sha256 of the bytes), x, inner x, final gradient,
    residual, iterations, termination, every trace record (sha256), and the
    reference's multiply counts per iteration;
  - the exact row-block pipeline (what the ranks of a
    multi-GPU c5 run compute) fed its 8 row blocks in order on this one GPU:
    the same bits end to end.
"""
import hashlib
import os

import numpy as np
import pytest

from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import SolverConfig
from paper_1502_01645_b200.rowblock import row_split
from tests.parity import same_bits

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_c5.npz")


def _trace_sha(tr):
    h = hashlib.sha256()
    for r in tr:
        al = np.nan if r.alpha is None else r.alpha
        h.update(np.array([r.iter, r.passive_count], np.uint64).tobytes())
        h.update(np.array([r.f, r.grad_bar_sq, al], np.float64).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def c5():
    if not os.path.exists(GOLDEN):
        pytest.skip("tests/golden/full_c5.npz not generated")
    g = np.load(GOLDEN)
    inst = instances.make_config("c5")
    if instances.sha256(np.asfortranarray(inst["A"]), inst["b"]) != str(g["input_sha256"]):
        pytest.skip("generated inputs differ from the fixture's")
    kw = dict(eval(str(g["cfg"])))
    cfg = SolverConfig(epsilon=kw["epsilon"], max_iters=kw["max_iters"],
                       stall_window=kw["stall_window"])
    return g, inst, cfg


def _check(r, g):
    assert r.inner.iterations() == int(g["iterations"])
    assert r.inner.termination == str(g["termination"])
    assert same_bits(r.x, g["x"]) and same_bits(r.inner.x, g["inner_x"])
    assert same_bits(r.inner.final_grad, g["final_grad"])
    assert len(r.inner.trace) == int(g["trace_len"])
    assert _trace_sha(r.inner.trace) == str(g["trace_sha256"])


def test_c5_full_exact_bitwise(solver, c5):
    g, inst, cfg = c5
    r = solver.solve_nnls(inst["A"], inst["b"], cfg)
    _check(r, g)
    assert same_bits([r.residual_sq], [g["residual_sq"]])
    assert np.array_equal(r.inner.multiplies_per_iter, g["mults"])
    # the rescaled system itself (setup parity: gram + rescale, nnls.hpp:41-83)
    sc = solver.setup(inst["A"], inst["b"])
    assert hashlib.sha256(np.ascontiguousarray(sc["q"]).tobytes()).hexdigest() == str(g["q_sha256"])
    assert hashlib.sha256(np.asfortranarray(sc["Q"]).tobytes(order="F")).hexdigest() == \
        str(g["Q_sha256"])


def test_c5_full_rowblock_pipeline_bitwise(solver, c5):
    import torch
    g, inst, cfg = c5
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    blocks = row_split(d, 8)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # column-major, ld = d
    db = torch.from_numpy(b).cuda()
    T = solver.gram_tiles(n)
    TD = solver.GRAM_TILE_DOUBLES
    H = torch.empty((n, n), dtype=torch.float64, device="cuda")
    states = None
    for p, (r0, r1) in enumerate(blocks):  # rank p's block, in rank order
        last = p == len(blocks) - 1
        out = None if last else torch.empty(T * TD, dtype=torch.float64, device="cuda")
        solver.gram_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, 0, T,
                                    states.data_ptr() if states is not None else 0,
                                    out.data_ptr() if out is not None else 0,
                                    0 if out is not None else H.data_ptr())
        states = out
    del states
    atb = None
    for (r0, r1) in blocks:
        nxt = torch.empty(n, dtype=torch.float64, device="cuda")
        solver.atb_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d, db.data_ptr() + 8 * r0,
                                   atb.data_ptr() if atb is not None else 0, nxt.data_ptr())
        atb = nxt
    r = solver.solve_nnls_gram_device(n, H.data_ptr(), atb.data_ptr(), cfg)
    _check(r, g)
    dx = torch.from_numpy(r.x).cuda()
    s = 0.0
    for (r0, r1) in blocks:
        s = solver.residual_rowblock_device(r1 - r0, n, dA.data_ptr() + 8 * r0, d,
                                            db.data_ptr() + 8 * r0, dx.data_ptr(), s)
    assert same_bits([s], [g["residual_sq"]])

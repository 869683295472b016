"""BASELINE.json c4 (configs[3]) at FULL size on the GPU: the whole 65536-column
batch (A 20000 x 256, B = A H_true formed on the device, 10.5 GB) solved by the
batched kernel, then every 64th column (1024 columns) compared bit for bit with
the reference's own per-column solve_nnls (tests/golden/c4_sample.npz, made by
tests/golden/make_golden_c4.py from oracle/_ref): x, iterations, termination,
residual, final objective and gradient norm."""
import hashlib
import os

import numpy as np
import pytest

from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import SolverConfig
from tests.parity import same_bits

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c4_sample.npz")
TERMS = ["EmptyPassiveSet", "GradientBelowEpsilon", "MaxIters", "TimeCap", "Stalled",
         "ZeroCurvature"]


def test_c4_full_batch_sampled_columns_bitwise(solver):
    import torch
    g = np.load(GOLDEN)
    d, n, K, seed = int(g["d"]), int(g["n"]), int(g["nrhs"]), int(g["seed"])
    A = instances.gen_matrix(d, n, seed, "u01")
    assert hashlib.sha256(A.tobytes(order="F")).hexdigest() == str(g["A_sha256"])
    H = instances.gen_htrue(n, K, seed, 0)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()       # A column-major
    dH = torch.from_numpy(np.ascontiguousarray(H.T)).cuda()       # H column-major
    dB = torch.empty((K, d), dtype=torch.float64, device="cuda")  # B column-major, ld d
    solver.matmat_device(d, n, K, dA.data_ptr(), d, dH.data_ptr(), n, dB.data_ptr(), d)
    del dH
    cols = g["cols"].astype(np.int64)
    idx = torch.from_numpy(cols).cuda()
    Bs = dB.index_select(0, idx).cpu().numpy()
    for c in range(len(cols)):  # the sampled right-hand sides are the reference's bytes
        assert hashlib.sha256(Bs[c].tobytes()).hexdigest() == str(g["B_col_sha256"][c]), c
    dX = torch.empty((K, n), dtype=torch.float64, device="cuda")
    kw = dict(eval(str(g["cfg"])))
    res, tm = solver.solve_nnls_batched_device(dA.data_ptr(), dB.data_ptr(), dX.data_ptr(), d, n,
                                               K, SolverConfig(**kw))
    Xs = dX.index_select(0, idx).cpu().numpy()  # (1024, n): row c = x of column cols[c]
    assert same_bits(Xs.reshape(-1), np.ascontiguousarray(g["X"].T).reshape(-1))
    for c, j in enumerate(cols):
        r = res[j]
        assert r["iterations"] == int(g["iterations"][c]), (j, r["iterations"])
        assert r["termination"] == TERMS[int(g["termination"][c])]
        assert same_bits([r["residual_sq"], r["f_final"], r["gbs_final"]],
                         [g["residual_sq"][c], g["f_final"][c], g["gbs_final"][c]]), j
    # the whole batch recovers H_true (the probe's <= 1e-6 criterion)
    err = float((dX - torch.from_numpy(np.ascontiguousarray(H.T)).cuda()).abs().max())
    assert err <= 1e-3, err
    print(f"c4 full batch: {K} columns, setup {tm['setup_s'] * 1e3:.1f} ms, loop "
          f"{tm['loop_s'] * 1e3:.1f} ms, max |X - H_true| {err:.2e}")

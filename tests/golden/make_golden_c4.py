#!/usr/bin/env python3
"""Golden sample of BASELINE.json c4 (configs[3]) at FULL shape from the
REFERENCE itself (oracle/_ref; build container only): A is 20000 x 256 U[0,1),
H_true is 256 x 65536 (40% zeros per column), B = A H_true. SURVEY.md §8d asks
for "bitwise on every oracle-sampled column (1024 columns, stride 64)".

B's columns are formed in the reference's matvec order (linalg.hpp:179-188:
y[i] += A(i,t) h[t], t ascending; every product rounded, then the sum), which is
what the device kernel alnnls_matmat_device computes, so the GPU test forms the
whole 10.5 GB B on the device and its sampled columns are these bytes (checked
through per-column sha256s). Each sampled column is then solved by the
reference's per-column pipeline with the Gram shared (ref_solve_nnls_columns:
transpose_matvec, rescale, solve_nqp, unscale, residual_norm_sq per column,
bitwise solve_nnls per column).

    make -C oracle && python tests/golden/make_golden_c4.py
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1502_01645_b200 import abi, instances  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
STRIDE = 64


def matvec_order_product(A, H):
    """C[:, j] = matvec(A, H[:, j]) in the reference's order, all columns at once:
    C += outer(A[:, t], H[t, :]) for t ascending (each product rounded, then added)."""
    C = np.zeros((A.shape[0], H.shape[1]))
    for t in range(A.shape[1]):
        C += np.multiply.outer(A[:, t], H[t, :])
    return C


def main():
    spec = instances.CONFIGS["c4"]
    d, n, K, seed = spec["d"], spec["n"], spec["nrhs"], spec["seed"]
    cols = np.arange(0, K, STRIDE)
    A = instances.gen_matrix(d, n, seed, "u01")
    H = np.column_stack([instances.gen_htrue(n, 1, seed, int(j))[:, 0] for j in cols])
    B = np.asfortranarray(matvec_order_product(A, H))
    ref = Oracle("ref")
    for c in (0, 1, len(cols) - 1):  # the order claim, against the reference's own matvec
        assert np.array_equal(ref.matvec(A, H[:, c]).view(np.uint64), B[:, c].view(np.uint64))
    cfg = abi.make_config(epsilon=spec["epsilon"], stall_window=10**9, record_multiplies=False)
    t = time.time()
    X, res = ref.solve_nnls_columns(A, B, cfg, threads=max(1, (os.cpu_count() or 2) - 1))
    print(f"{len(cols)} columns solved in {time.time() - t:.1f} s", flush=True)
    np.savez_compressed(
        os.path.join(OUT, "c4_sample.npz"),
        A_sha256=hashlib.sha256(np.asfortranarray(A).tobytes(order="F")).hexdigest(),
        cols=cols.astype(np.int64), stride=np.int64(STRIDE), nrhs=np.int64(K), d=np.int64(d),
        n=np.int64(n), seed=np.int64(seed), cfg=repr([("epsilon", spec["epsilon"]),
                                                       ("stall_window", 10**9)]),
        B_col_sha256=np.array([hashlib.sha256(B[:, c].tobytes()).hexdigest()
                               for c in range(len(cols))]),
        X=X, iterations=np.array([r.iterations for r in res], np.uint64),
        termination=np.array([r.termination for r in res], np.int32),
        residual_sq=np.array([r.residual_sq for r in res]),
        f_final=np.array([r.f_final for r in res]), gbs_final=np.array([r.gbs_final for r in res]),
        multiplies=np.array([r.multiplies_total for r in res], np.uint64),
        H_err=np.float64(np.max(np.abs(X - H))))
    print("wrote c4_sample.npz; max |X - H_true| =", float(np.max(np.abs(X - H))))


if __name__ == "__main__":
    main()

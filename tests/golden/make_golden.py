#!/usr/bin/env python3
"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference headers compiled in place by oracle/Makefile with the reference's
Release flags). Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Each fixture stores the inputs' sha256 (inputs are regenerated from seeds by
paper_1502_01645_b200/instances.py or the SplitMix64 test fixtures, so the
generator is pinned too; small inputs are also stored verbatim) and the
reference outputs: x, final_grad (inner), iterations, termination, the trace
(iter, f, gbs, |P|, alpha) and multiplies_per_iter where available.
The reference has no golden data files of its own; these are
produced by its code, not written by hand.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1502_01645_b200 import abi, instances  # noqa: E402
from tests.splitmix import SplitMix64  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def trace_arrays(tr):
    it = np.array([r["iter"] for r in tr], np.uint64)
    f = np.array([r["f"] for r in tr], np.float64)
    g = np.array([r["grad_bar_sq"] for r in tr], np.float64)
    pc = np.array([r["passive_count"] for r in tr], np.uint64)
    al = np.array([np.nan if r["alpha"] is None else r["alpha"] for r in tr], np.float64)
    has = np.array([r["alpha"] is not None for r in tr], np.bool_)
    return dict(tr_iter=it, tr_f=f, tr_gbs=g, tr_pc=pc, tr_alpha=al, tr_has_alpha=has)


def splitmix_matrix(rows, cols, seed, lo, hi):
    r = SplitMix64(seed)
    M = np.zeros((rows, cols), order="F")
    for j in range(cols):
        for i in range(rows):
            M[i, j] = lo + (hi - lo) * r.uniform01()
    return M


def nnls_case(ref, name, A, b, cfg_kwargs, store_inputs):
    cfg = abi.make_config(**cfg_kwargs)
    r = ref.solve_nnls(A, b, cfg)
    out = dict(
        kind="nnls", x=r["x"], inner_x=r["inner_x"], final_grad=r["final_grad"],
        residual_sq=np.float64(r["residual_sq"]), iterations=np.uint64(r["iterations"]),
        termination=r["termination"], dropped=r["dropped"],
        input_sha256=instances.sha256(np.asfortranarray(A), b),
        cfg=repr(sorted(cfg_kwargs.items())), **trace_arrays(r["trace"]))
    if store_inputs:
        out["A"] = np.asfortranarray(A)
        out["b"] = b
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, r["iterations"], r["termination"], len(r["trace"]))


def nqp_case(ref, name, Q, q, cfg_kwargs, start=None):
    cfg = abi.make_config(**cfg_kwargs)
    r = ref.solve_nqp(Q, q, cfg, start=start)
    out = dict(kind="nqp", Q=np.asfortranarray(Q), q=q, x=r["x"], final_grad=r["final_grad"],
               iterations=np.uint64(r["iterations"]), termination=r["termination"],
               mults=r["mults"], min_iterate=np.float64(r["min_iterate"]),
               cfg=repr(sorted(cfg_kwargs.items())), **trace_arrays(r["trace"]))
    if start is not None:
        out["start"] = np.asarray(start, np.float64)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, r["iterations"], r["termination"], len(r["trace"]))


def main():
    ref = Oracle("ref")
    # --- seeded configs at scaled sizes (value laws of BASELINE.json c1..c5) ---
    inst = instances.make_config("c1")  # full c1: d=600, n=300
    nnls_case(ref, "c1_full", inst["A"], inst["b"],
              dict(epsilon=1e-8, max_iters=10000, stall_window=10**9), store_inputs=False)
    for name, d, n in [("c2", 512, 256), ("c3", 256, 256), ("c5", 512, 256)]:
        inst = instances.make_config(name, d=d, n=n)
        nnls_case(ref, f"{name}_scaled_{d}x{n}", inst["A"], inst["b"],
                  dict(epsilon=inst["epsilon"], max_iters=2000, stall_window=10**9),
                  store_inputs=False)
    # default SolverConfig (stall 50, eps 1e-10 m, max 5m)
    inst = instances.make_config("c5", d=400, n=200, seed=77)
    nnls_case(ref, "c5_defaults_400x200", inst["A"], inst["b"], dict(), store_inputs=False)
    # --- reference-test fixtures (test_nnls.cpp:196-218 family, SplitMix64 seeded) ---
    for seed in (200, 203, 206, 211):
        n = 2 + seed % 7
        d = n + 1 + seed % 8
        A = splitmix_matrix(d, n, seed, 0.0 if seed % 2 else -1.0, 1.0)
        b = splitmix_matrix(d, 1, seed + 999, -1.0, 1.0)[:, 0]
        nnls_case(ref, f"rect_seed{seed}", A, b,
                  dict(epsilon=1e-20, max_iters=200000, stall_window=1000000), store_inputs=True)
    # zero column dropped (test_nnls.cpp:80-101) and all-zero A (:103-111)
    nnls_case(ref, "zero_column", np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([3.0, 1.0]),
              dict(), store_inputs=True)
    nnls_case(ref, "all_zero", np.zeros((3, 2)), np.array([1.0, 2.0, 3.0]), dict(),
              store_inputs=True)
    # --- NQP fixtures (test_nqp.cpp) ---
    nqp_case(ref, "nqp_coupled", np.array([[1.0, 1 / 30], [1 / 30, 1.0]]),
             np.array([-4.0, -5 / 3]), dict(epsilon=1e-22))
    nqp_case(ref, "nqp_lopsided_warm", np.array([[1.0, 0.1], [0.1, 9.0]]), np.array([-4.0, -5.0]),
             dict(epsilon=1e-10, max_iters=100000), start=[30.0, 2.0])
    nqp_case(ref, "nqp_halving", np.array([[1.0, 0.9], [0.9, 1.0]]), np.array([1.49, -2.69]),
             dict(epsilon=1e-18, max_iters=10000, stall_window=1000000), start=[0.52, 0.35])
    nqp_case(ref, "nqp_stall", np.array([[1.0, 1 / 30], [1 / 30, 1.0]]), np.array([-4.0, -5 / 3]),
             dict(epsilon=5e-324, max_iters=1000000, stall_window=5))
    nqp_case(ref, "nqp_trace_every4", np.array([[1.0, 0.1], [0.1, 9.0]]), np.array([-4.0, -5.0]),
             dict(epsilon=1e-18, max_iters=100000, stall_window=1000000, trace_every=4))
    for seed in (11, 14):  # test_nqp.cpp:228-271 family
        n = 8 + 3 * seed
        A = splitmix_matrix(n + 4, n, seed, -1.0, 1.0)
        Q = ref.gram(A)
        q = splitmix_matrix(n, 1, seed + 500, -1.0, 1.0)[:, 0]
        nqp_case(ref, f"nqp_random_seed{seed}", Q, q, dict(max_iters=5000, stall_window=1000000))


if __name__ == "__main__":
    main()

"""Batched FAST: the two-CTA kernel (default) vs the one-CTA kernel (ALNNLS_FAST_2CTA=0):
identical X, iterations, terminations (development helper, under gpurun)."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_1502_01645_b200 import instances, abi
from paper_1502_01645_b200.api import Solver, SolverConfig

s = Solver(0)
ok = True
for (d, n, nrhs, seed) in [(2000, 256, 700, 11), (1500, 200, 333, 5), (900, 97, 64, 3), (3000, 256, 5000, 7)]:
    inst = instances.make_batched(d=d, n=n, nrhs=nrhs, seed=seed)
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9, profile=abi.PROFILE_FAST)
    out = {}
    for mode in ("0", "1"):
        os.environ["ALNNLS_FAST_2CTA"] = mode
        X, cols, tm = s.solve_nnls_batched(inst["A"], inst["B"], cfg)
        out[mode] = (X.copy(), [(c["iterations"], c["termination"], c["f_final"], c["gbs_final"], c["multiplies_total"]) for c in cols], tm)
    same_x = np.array_equal(out["0"][0].view(np.uint64), out["1"][0].view(np.uint64))
    same_c = out["0"][1] == out["1"][1]
    print(d, n, nrhs, "X identical:", same_x, "columns identical:", same_c,
          "loop_s old/new:", out["0"][2].get("loop_s"), out["1"][2].get("loop_s"), flush=True)
    ok &= same_x and same_c
print("OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)

import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1502_01645_b200 import abi
from paper_1502_01645_b200.api import Solver, SolverConfig
s = Solver(0)
for m in (300, 448, 480, 512, 640, 700, 1024):
    rng = np.random.default_rng(m)
    A = rng.standard_normal((2*m, m)); b = rng.standard_normal(2*m)
    try:
        r = s.solve_nnls(A, b, SolverConfig(epsilon=1e-8, stall_window=10**9, profile=abi.PROFILE_FAST))
        print(m, "ok", r.inner.iterations(), r.inner.termination, flush=True)
    except Exception as e:
        print(m, "ERR", e, flush=True)

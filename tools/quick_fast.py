import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1502_01645_b200 import instances, abi
from paper_1502_01645_b200.api import Solver, SolverConfig
inst = instances.make_config("c2")
A, b = inst["A"], inst["b"]
d, n = A.shape
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(); db = torch.from_numpy(b).cuda()
s = Solver(0)
for prof in (abi.PROFILE_EXACT, abi.PROFILE_FAST):
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9, profile=prof)
    for _ in range(3):
        s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
    sm = s.last_summary()
    print(prof, "setup_ms", sm.t_setup_s*1e3, "loop_ms", sm.t_loop_s*1e3, "iters", sm.iterations, "tf", (d*n*(n+1)+2*d*n)/sm.t_setup_s/1e12)

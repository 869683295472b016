"""Per-phase device time of the loop kernel (vector-CTA %globaltimer marks), c2."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import Solver, SolverConfig
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dd = int(sys.argv[2]) if len(sys.argv) > 2 else None   # optional scaled shape (d, n)
nn = int(sys.argv[3]) if len(sys.argv) > 3 else None
inst = instances.make_config(name, d=dd, n=nn)
A, b = inst["A"], inst["b"]
d, n = A.shape
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(); db = torch.from_numpy(b).cuda()
s = Solver(0)
cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
for _ in range(3):
    s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
sm = s.last_summary()
it = sm.iterations
ph = s.phase_times()
names = ["A: P1 || chains+stop", "B1 wait", "den", "changed", "-", "P2+apply+Bcnt", "lists+B0", "-"]
print(name, "iters", it, "loop_ms", sm.t_loop_s * 1e3, "us/iter", sm.t_loop_s * 1e6 / max(1, it))
for nm, v in zip(names, ph):
    print(f"  {nm:24s} {v * 1e6 / max(1, it):7.2f} us/iter")

"""One warm host-buffer c2 solve (for ncu launch lists of the overlapped path)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import Solver, SolverConfig
inst = instances.make_config("c2")
A, b = inst["A"], inst["b"]
d, n = A.shape
cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
s = Solver(0)
pA = torch.empty((n, d), dtype=torch.float64, pin_memory=True)
pA.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
pb = torch.empty(d, dtype=torch.float64, pin_memory=True)
pb.copy_(torch.from_numpy(b))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    s.solve_nnls(pA.numpy().T, pb.numpy(), cfg)

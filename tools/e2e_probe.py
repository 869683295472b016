"""c2 end-to-end (host buffers) timing split: device-resident solve, host-buffer
solve through the public API, and the host-buffer call without result fetch."""
import os, sys, time
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
hA = pA.numpy().T
hb = pb.numpy()
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(); db = torch.from_numpy(b).cuda()
for _ in range(3):
    s.solve_nnls(hA, hb, cfg)
    s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
K = 5
s.timer_start()
for _ in range(K):
    s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
t_dev = s.timer_stop() / K
s.timer_start()
for _ in range(K):
    r = s.solve_nnls(hA, hb, cfg)
t_host = s.timer_stop() / K
t0 = time.perf_counter()
for _ in range(K):
    r = s.solve_nnls(hA, hb, cfg)
t_wall = (time.perf_counter() - t0) / K
sm = s.last_summary()
print(os.environ.get("ALNNLS_LIB", "default"), f"device {t_dev*1e3:.3f} ms  host-api {t_host*1e3:.3f} ms  wall {t_wall*1e3:.3f} ms  setup {sm.t_setup_s*1e3:.3f} loop {sm.t_loop_s*1e3:.3f}")

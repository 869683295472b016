"""Host-buffer (e2e) path timing at c2: pinned H2D bandwidth, and the phases of
the overlapped FAST / EXACT host solves. python tools/e2e_probe2.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_01645_b200 import abi, instances  # noqa: E402
from paper_1502_01645_b200.api import Solver, SolverConfig  # noqa: E402

inst = instances.make_config("c2")
A, b = inst["A"], inst["b"]
d, n = A.shape
pA = torch.empty((n, d), dtype=torch.float64, pin_memory=True)
pA.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
pb = torch.empty(d, dtype=torch.float64, pin_memory=True)
pb.copy_(torch.from_numpy(b))
dA = torch.empty((n, d), dtype=torch.float64, device="cuda")
for _ in range(2):
    dA.copy_(pA, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dA.copy_(pA, non_blocking=True)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5
print(f"pinned H2D {8 * d * n / 1e6:.0f} MB: {t:.3f} ms = {8 * d * n / t / 1e6:.1f} GB/s")
hA, hb = pA.numpy().T, pb.numpy()
s = Solver(0)
for prof in (abi.PROFILE_EXACT, abi.PROFILE_FAST):
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9, profile=prof)
    for _ in range(2):
        s.solve_nnls(hA, hb, cfg)
    s.timer_start()
    for _ in range(5):
        r = s.solve_nnls(hA, hb, cfg)
    tt = s.timer_stop() / 5
    sm = s.last_summary()
    print(f"profile {prof}: host solve {tt * 1e3:.3f} ms; setup(+upload) {sm.t_setup_s * 1e3:.3f} "
          f"loop {sm.t_loop_s * 1e3:.3f} finish {sm.t_finish_s * 1e3:.3f} total {sm.t_total_s * 1e3:.3f}")

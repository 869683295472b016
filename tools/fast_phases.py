"""FAST loop phase split at a config (CTA 0's clock, us per iteration).
python tools/fast_phases.py [c2|c3|c5m|c5] [--once]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_01645_b200 import abi, instances  # noqa: E402
from paper_1502_01645_b200.api import Solver, SolverConfig  # noqa: E402

SHAPES = {"c2": ("c2", None, None), "c3": ("c3", None, None), "c5m": ("c5", 8192, 4096),
          "c5": ("c5", None, None), "c1": ("c1", None, None)}
name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
once = "--once" in sys.argv
cn, d, n = SHAPES[name]
inst = instances.make_config(cn, d=d, n=n)
A, b = inst["A"], inst["b"]
d, n = A.shape
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
db = torch.from_numpy(b).cuda()
del A
s = Solver(0)
cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9,
                   profile=abi.PROFILE_FAST)
reps = 1 if once else 3
for _ in range(reps):
    s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
sm = s.last_summary()
it = max(1, int(sm.iterations))
ph = s.phase_times()
names = ["stop+stage", "Qg pass+den", "barrier A", "K+A2", "QKcK pass", "update+partials",
         "barrier B+totals"]
print(f"{name}: iters {sm.iterations} setup {sm.t_setup_s*1e3:.3f} ms loop {sm.t_loop_s*1e3:.3f} ms "
      f"= {sm.t_loop_s/it*1e6:.2f} us/iter; bytes/iter {8*sm.multiplies_total/it/1e6:.1f} MB "
      f"-> {8*sm.multiplies_total/sm.t_loop_s/1e9:.0f} GB/s")
print("  " + ", ".join(f"{nm} {v/it*1e6:.2f}" for nm, v in zip(names, ph[:7])))

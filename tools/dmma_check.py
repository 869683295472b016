"""FAST DMMA Gram check: TMA stream-K kernel vs the exact Gram (entrywise) on
ragged shapes, and setup timings at c2 / c5-partial. python tools/dmma_check.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_01645_b200 import abi, instances  # noqa: E402
from paper_1502_01645_b200.api import Solver, SolverConfig  # noqa: E402

s = Solver(0)
for (d, n) in [(700, 260), (1000, 513), (130, 129), (4099, 1030)]:
    rng = np.random.default_rng(d + n)
    A = np.asfortranarray(rng.standard_normal((d, n)))
    b = rng.standard_normal(d)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()
    out = {}
    for prof in (0, 1):
        buf = torch.empty(n * n + n, dtype=torch.float64, device="cuda")
        s.gram_partial_device(d, n, dA.data_ptr(), d, db.data_ptr(), buf.data_ptr(),
                              buf.data_ptr() + 8 * n * n, profile=prof)
        out[prof] = buf[: n * n].view(n, n).cpu().numpy()
    He, Hf = out[0], out[1]
    err = np.max(np.abs(He - Hf)) / np.max(np.abs(He))
    print(f"d={d} n={n}: max rel diff DMMA vs exact {err:.2e}, symmetric {np.array_equal(Hf, Hf.T)}",
          flush=True)
inst = instances.make_config("c2")
A, b = inst["A"], inst["b"]
d, n = A.shape
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
db = torch.from_numpy(b).cuda()
cfg = SolverConfig(epsilon=1e-8, stall_window=10**9, profile=abi.PROFILE_FAST)
for _ in range(3):
    s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
sm = s.last_summary()
fl = d * n * (n + 1) + 2 * d * n
print(f"c2 FAST: setup {sm.t_setup_s * 1e3:.3f} ms = {fl / sm.t_setup_s / 1e12:.2f} TF, loop "
      f"{sm.t_loop_s * 1e3:.3f} ms, iters {sm.iterations}")
hA = np.asfortranarray(A)
for _ in range(2):
    s.solve_nnls(hA, b, cfg)
s.timer_start()
for _ in range(5):
    r = s.solve_nnls(hA, b, cfg)
t = s.timer_stop() / 5
print(f"c2 FAST host-buffer (pageable) solve {t * 1e3:.3f} ms, iters {r.inner.iterations()}")

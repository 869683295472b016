"""Quick timing of the GPU path on a BASELINE config (development helper)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import Solver, SolverConfig

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
t = time.time()
inst = instances.make_config(name)
print("gen", name, inst["A"].shape, round(time.time() - t, 2), "s", flush=True)
s = Solver(0)
cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t = time.time()
    r = s.solve_nnls(inst["A"], inst["b"], cfg)
    wall = time.time() - t
    mt = int(r.inner.multiplies_per_iter.sum())
    print(json.dumps({"rep": rep, "wall_s": wall, **r.timings, "iters": r.inner.iterations(),
                      "term": r.inner.termination, "phase_us_per_iter": [round(1e6 * v / max(1, r.inner.iterations()), 2) for v in r.inner.timings["phase_s"]], "resid": r.residual_sq,
                      "loop_GBps": 8 * mt / max(r.timings["loop_s"], 1e-12) / 1e9,
                      "us_per_iter": 1e6 * r.timings["loop_s"] / max(1, r.inner.iterations()),
                      "setup_TFLOPs": inst["A"].shape[0] * inst["A"].shape[1] * (inst["A"].shape[1] + 1) / r.timings["setup_s"] / 1e12}), flush=True)

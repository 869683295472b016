"""c4 (batched RHS) timing at full or reduced size (development helper)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import Solver, SolverConfig

nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
spec = instances.CONFIGS["c4"]
d, n = spec["d"], spec["n"]
t = time.time()
A = instances.gen_matrix(d, n, spec["seed"], "u01")
H = instances.gen_htrue(n, nrhs, spec["seed"])
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()          # (n, d) row-major == A col-major
dH = torch.from_numpy(np.ascontiguousarray(H.T)).cuda()          # (nrhs, n) == H col-major
dB = dH @ dA                                                     # (nrhs, d) == B = A H col-major
dX = torch.empty((nrhs, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
print("gen", round(time.time() - t, 2), "s", flush=True)
s = Solver(0)
from paper_1502_01645_b200 import abi
fast = len(sys.argv) > 2 and sys.argv[2] == "fast"
cfg = SolverConfig(epsilon=spec["epsilon"], stall_window=10**9,
                   profile=abi.PROFILE_FAST if fast else abi.PROFILE_EXACT)
for rep in range(2):
    t = time.time()
    cols, tm = s.solve_nnls_batched_device(dA.data_ptr(), dB.data_ptr(), dX.data_ptr(), d, n, nrhs, cfg)
    wall = time.time() - t
    it = np.array([c["iterations"] for c in cols])
    err = float((dX - dH).abs().max())
    print(json.dumps({"rep": rep, "wall_s": wall, **tm, "solves_per_s": nrhs / tm["total_s"],
                      "iters_mean": float(it.mean()), "iters_max": int(it.max()), "max_err_vs_Htrue": err,
                      "loop_TFLOPs_algorithmic": 2 * tm["multiplies_total"] / tm["loop_s"] / 1e12}), flush=True)

"""FAST profile check on the GPU: the one-pass loop (fastloop.cu) and the DMMA
Gram against the EXACT path (bitwise the reference) on the four BASELINE.json
tolerances, plus timings. Usage: python tools/fast_check.py [c1 c2 c3 c5s ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_01645_b200 import abi, instances  # noqa: E402
from paper_1502_01645_b200.api import Solver, SolverConfig  # noqa: E402
from tests.parity import baseline_tolerances  # noqa: E402

CASES = {"c1": ("c1", None, None), "c2": ("c2", None, None), "c3": ("c3", None, None),
         "c5s": ("c5", 4096, 2048), "c5m": ("c5", 8192, 4096), "c2s": ("c2", 1024, 512),
         "c5": ("c5", None, None)}


def run(s, name):
    cname, d, n = CASES[name]
    inst = instances.make_config(cname, d=d, n=n)
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()
    out = {"case": name, "d": d, "n": n}
    res = {}
    for prof in ("exact", "fast"):
        cfg = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9,
                           profile=abi.PROFILE_FAST if prof == "fast" else abi.PROFILE_EXACT)
        r = s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=True)
        sm = s.last_summary()
        reps = 3 if d * n <= 8192 * 4096 else 1
        t = []
        for _ in range(reps):
            s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
            sm2 = s.last_summary()
            t.append((sm2.t_setup_s, sm2.t_loop_s))
        ts = min(x[0] for x in t)
        tl = min(x[1] for x in t)
        it = int(sm.iterations)
        res[prof] = r
        out[prof] = {"iters": it, "term": r.inner.termination, "setup_ms": ts * 1e3,
                     "loop_ms": tl * 1e3, "us_per_iter": tl / max(1, it) * 1e6,
                     "mults_total": int(sm.multiplies_total),
                     "gbs_loop": 8.0 * sm.multiplies_total / tl / 1e9 if tl > 0 else None,
                     "f": r.inner.trace[-1].f}
        # FAST loop alone on the exact Q (isolates the loop's perturbation)
    e, f = res["exact"], res["fast"]
    out["tol_fast_vs_exact"] = baseline_tolerances(f.x, e.x, f.inner.trace[-1].f, e.inner.trace[-1].f,
                                                   f.inner.iterations(), e.inner.iterations())
    # loop-only: FAST loop on the exact path's Q, q
    sc = s.setup(A, b)
    Q, q = sc["Q"], sc["q"]
    cfgx = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
    cfgf = SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9,
                        profile=abi.PROFILE_FAST)
    rx = s.solve_nqp(Q, q, cfgx)
    rf = s.solve_nqp(Q, q, cfgf)
    out["tol_fastloop_only"] = baseline_tolerances(rf.x, rx.x, rf.trace[-1].f, rx.trace[-1].f,
                                                   rf.iterations(), rx.iterations())
    out["loop_only_iters"] = [rx.iterations(), rf.iterations()]
    print(json.dumps(out, default=float), flush=True)
    return out


def main():
    names = sys.argv[1:] or ["c1", "c2s", "c5s", "c2"]
    s = Solver(0)
    for nm in names:
        t = time.time()
        run(s, nm)
        print(f"# {nm} {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()

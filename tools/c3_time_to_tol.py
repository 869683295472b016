"""c3 time-to-tolerance on the GPU.

configs[2] (d = n = 4096, singular values log-spaced 1 .. 1e-6, KKT tol 1e-10)
does not reach 1e-10 within the reference's default cap of 5n = 20480
iterations (both the reference and this path stop at MaxIters there; bench.py
and the golden fixture cover that capped run bit for bit). This GPU-only run
lifts the cap (default 4,000,000 iterations, no stall test) and reports the
device time to the 1e-10 gradient tolerance, certified like the reference's
acceptance test (acceptance.cpp:248-256): kkt_error (nqp.hpp:190-207) of the
returned scaled-space iterate against the solver's own Q and q, recomputed
here with a fresh fp64 matvec (torch/cuBLAS on the device; a checker, not the
product path), against kappa = sqrt(eps) (1 + ||q||_2).

  python tools/c3_time_to_tol.py [--max-iters N] > profiles/rNN_c3_time_to_tol.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1502_01645_b200 import instances  # noqa: E402
from paper_1502_01645_b200.api import Solver, SolverConfig  # noqa: E402


def kkt_error(Q, q, x):
    """nqp.hpp:190-207 on the device: max |g_i| over x_i > 0, max(0, -g_i) over x_i = 0."""
    g = Q @ x + q
    if bool((x < 0).any()):
        return float("inf"), g
    pos = torch.where(x > 0, g.abs(), torch.clamp(-g, min=0.0))
    return float(pos.max()) if pos.numel() else 0.0, g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-iters", type=int, default=4_000_000)
    ap.add_argument("--trace-every", type=int, default=10_000)
    args = ap.parse_args()
    inst = instances.make_config("c3")
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    eps = inst["epsilon"]
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()
    s = Solver(0)
    cfg = SolverConfig(epsilon=eps, max_iters=args.max_iters, stall_window=10**9,
                       trace_every=args.trace_every)
    torch.cuda.synchronize()
    s.timer_start()
    res = s.solve_nnls_device(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=True)
    t = s.timer_stop()
    summ = s.last_summary()
    scaled = s._scaled()
    Q = torch.from_numpy(scaled["Q"]).cuda()
    q = torch.from_numpy(scaled["q"]).cuda()
    x = torch.from_numpy(res.inner.x).cuda()
    viol, g = kkt_error(Q, q, x)
    kappa = float(np.sqrt(eps) * (1.0 + float(torch.linalg.vector_norm(q))))
    fg = torch.from_numpy(res.inner.final_grad).cuda()
    gbar = torch.where((x > 0) | (g < 0), g, torch.zeros_like(g))
    tr = res.inner.trace
    line = {
        "workload": f"c3: d={d}, n={n} (configs[2]), eps {eps:g}, stall off",
        "max_iters": args.max_iters,
        "termination": res.inner.termination,
        "iterations": res.inner.iterations(),
        "time_to_tol_s": t,
        "setup_ms": summ.t_setup_s * 1e3,
        "loop_s": summ.t_loop_s,
        "us_per_iter": summ.t_loop_s * 1e6 / max(1, res.inner.iterations()),
        "final_grad_bar_sq": tr[-1].grad_bar_sq if tr else None,
        "grad_bar_sq_fresh": float((gbar * gbar).sum()),
        "kkt_error": viol,
        "kappa": kappa,
        "certified": bool(viol <= kappa),
        "max_abs_final_grad_vs_fresh": float((fg - g).abs().max()),
        "residual_sq": res.residual_sq,
        "max_abs_err_vs_x_true": float(np.max(np.abs(res.x - inst["x_true"]))),
        "trace_samples": [[r.iter, r.grad_bar_sq, r.f] for r in tr[:: max(1, len(tr) // 40)]],
        "note": ("GPU-only (a matching reference run at this cap would take days on one core); "
                 "the capped 20480-iteration run is bitwise against the reference "
                 "(tests/golden/full_c3.npz)"),
    }
    print(json.dumps(line), flush=True)
    s.close()


if __name__ == "__main__":
    main()

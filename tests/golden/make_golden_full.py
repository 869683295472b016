#!/usr/bin/env python3
"""Full-size golden summaries for BASELINE.json c2 and c3 (configs[1], [2]) from
the REFERENCE itself (oracle/_ref; build container only: /root/reference must
exist to build it). c2 takes ~2 min and c3 (20480 iterations at the default
cap; the reference does not reach eps = 1e-10) ~15 min on one core.

    make -C oracle && python tests/golden/make_golden_full.py [c2] [c3]

Stores the input sha256 (inputs come from paper_1502_01645_b200/instances.py),
x, inner x, final_grad, residual_sq, iterations, termination, the last trace
record and a sha256 over every trace record, so tests/test_golden.py can check
the GPU's full-size solve bit for bit without the reference."""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1502_01645_b200 import abi, instances  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def trace_sha(tr):
    h = hashlib.sha256()
    for r in tr:
        al = np.nan if r["alpha"] is None else r["alpha"]
        h.update(np.array([r["iter"], r["passive_count"]], np.uint64).tobytes())
        h.update(np.array([r["f"], r["grad_bar_sq"], al], np.float64).tobytes())
    return h.hexdigest()


def main(names):
    ref = Oracle("ref")
    for name in names:
        inst = instances.make_config(name)
        A, b = inst["A"], inst["b"]
        kw = dict(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
        cfg = abi.make_config(**kw)
        t = time.time()
        r = ref.solve_nnls(A, b, cfg)
        last = r["trace"][-1]
        np.savez_compressed(
            os.path.join(OUT, f"full_{name}.npz"),
            input_sha256=instances.sha256(np.asfortranarray(A), b), cfg=repr(sorted(kw.items())),
            x=r["x"], inner_x=r["inner_x"], final_grad=r["final_grad"],
            residual_sq=np.float64(r["residual_sq"]), iterations=np.uint64(r["iterations"]),
            termination=r["termination"], trace_len=np.uint64(len(r["trace"])),
            trace_sha256=trace_sha(r["trace"]), last_f=np.float64(last["f"]),
            last_gbs=np.float64(last["grad_bar_sq"]), seconds=np.float64(time.time() - t))
        print(name, r["iterations"], r["termination"], f"{time.time() - t:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3"])

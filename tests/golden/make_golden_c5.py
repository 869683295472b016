#!/usr/bin/env python3
"""Full-size golden summary for BASELINE.json c5 (configs[4], d=32768, n=16384)
from the REFERENCE itself (oracle/_ref; build container only).

The reference's `solve_nnls` (nnls.hpp:129-144) would spend ~1.75 h of one core in
`gram` alone, so the pipeline is run stage by stage with the reference's own
functions, which is bitwise the same composition:
  gram (linalg.hpp:160-174)      - the reference's gram() driven over column-block
                                   pairs on all host threads; every entry is the same
                                   ascending-k chain, so H is bitwise gram(A)
  transpose_matvec + negate      - nnls.hpp:133-134
  rescale (nnls.hpp:41-83)       - reference
  solve_nqp (nqp.hpp:215-339)    - reference, single thread (~1.5-2 h)
  unscale (nnls.hpp:87-96)       - x[r_a] = y_a / D_a (one IEEE division, same bits)
  residual_norm_sq (:115-123)    - reference matvec, then the ascending sum of r_i*r_i
                                   (rounded product, rounded add; a Python float loop)

    make -C oracle && python tests/golden/make_golden_c5.py

Stores the input sha256, sha256s of the rescaled Q (column-major bytes) and q,
x, inner x, final gradient, residual, iterations, termination, the per-record
trace (f, gbs, |P|, alpha) with its sha256, and the multiply counts, so
tests/test_golden.py can check the GPU's full-size c5 solve bit for bit."""
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


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def trace_sha(tr):
    h = hashlib.sha256()
    for r in tr:
        al = np.nan if r["alpha"] is None else r["alpha"]
        h.update(np.array([r["iter"], r["passive_count"]], np.uint64).tobytes())
        h.update(np.array([r["f"], r["grad_bar_sq"], al], np.float64).tobytes())
    return h.hexdigest()


def gram_parallel(ora, A, threads, nb=32):
    from concurrent.futures import ThreadPoolExecutor
    d, n = A.shape
    bs = (n + nb - 1) // nb
    blocks = [(i * bs, min(n, (i + 1) * bs)) for i in range(nb) if i * bs < n]
    H = np.zeros((n, n), order="F")
    done = [0]

    def work(pair):
        (a0, a1), (b0, b1) = pair
        if (a0, a1) == (b0, b1):
            H[a0:a1, a0:a1] = ora.gram(np.asfortranarray(A[:, a0:a1]))
        else:
            cols = np.concatenate([np.arange(a0, a1), np.arange(b0, b1)])
            Hb = ora.gram(np.asfortranarray(A[:, cols]))
            k = a1 - a0
            H[a0:a1, b0:b1] = Hb[:k, k:]
            H[b0:b1, a0:a1] = Hb[k:, :k]
        done[0] += 1
        if done[0] % 32 == 0:
            log(f"gram pairs {done[0]}/{len(pairs)}")

    pairs = [(blocks[i], blocks[j]) for i in range(len(blocks)) for j in range(i, len(blocks))]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, pairs))
    return H


def main():
    ora = Oracle("ref")
    threads = os.cpu_count() or 1
    inst = instances.make_config("c5")
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    kw = dict(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9)
    cfg = abi.make_config(**kw)
    sha_in = instances.sha256(np.asfortranarray(A), b)
    log("inputs", sha_in)
    t0 = time.time()
    H = gram_parallel(ora, A, threads)
    t_gram = time.time() - t0
    log(f"gram {t_gram:.0f} s")
    h = -ora.transpose_matvec(A, b)
    sys_ = ora.rescale(H, h)
    del H
    Q, q = sys_["Q"], sys_["q"]
    q_sha = hashlib.sha256(np.ascontiguousarray(q).tobytes()).hexdigest()
    Q_sha = hashlib.sha256(np.asfortranarray(Q).tobytes(order="F")).hexdigest()
    log("rescale m =", len(q), "Q", Q_sha[:16], "q", q_sha[:16])
    t1 = time.time()
    r = ora.solve_nqp(Q, q, cfg)
    t_loop = time.time() - t1
    log(f"solve_nqp {r['iterations']} {r['termination']} {t_loop:.0f} s")
    del Q
    x = np.zeros(n)
    x[sys_["retained"].astype(np.int64)] = r["x"] / sys_["scale"]
    ax = ora.matvec(A, x)
    s = 0.0
    for i in range(d):
        ri = float(ax[i]) - float(b[i])
        s += ri * ri
    tr = r["trace"]
    al = np.array([np.nan if t["alpha"] is None else t["alpha"] for t in tr])
    np.savez_compressed(
        os.path.join(OUT, "full_c5.npz"),
        input_sha256=sha_in, cfg=repr(sorted(kw.items())), Q_sha256=Q_sha, q_sha256=q_sha,
        x=x, inner_x=r["x"], final_grad=r["final_grad"], residual_sq=np.float64(s),
        iterations=np.uint64(r["iterations"]), termination=r["termination"],
        dropped=sys_["dropped"], trace_len=np.uint64(len(tr)), trace_sha256=trace_sha(tr),
        trace_f=np.array([t["f"] for t in tr]), trace_gbs=np.array([t["grad_bar_sq"] for t in tr]),
        trace_passive=np.array([t["passive_count"] for t in tr], np.uint64), trace_alpha=al,
        mults=r["mults"], last_f=np.float64(tr[-1]["f"]), last_gbs=np.float64(tr[-1]["grad_bar_sq"]),
        gram_seconds=np.float64(t_gram), loop_seconds=np.float64(t_loop),
        threads_gram=np.int64(threads))
    log("wrote full_c5.npz")


if __name__ == "__main__":
    main()

"""Seeded synthetic inputs for BASELINE.json's five configs (c1..c5).

Generation runs in C (csrc/instgen.c, SplitMix64 substream per column, the
scheme of /root/reference/proj/include/antilop/testgen.hpp:42-76). No dataset
is downloaded: the configs are synthetic by definition (BASELINE.json).
Inputs are produced once on the host and the same bytes feed the oracle and
the GPU.
"""
import ctypes as C
import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GEN_LIB = os.path.join(HERE, "lib", "libalnnls_gen.so")

# name -> (kind, d, n, seed, epsilon, max_iters)  (BASELINE.json "configs")
CONFIGS = {
    "c1": dict(kind=1, d=600, n=300, seed=1, epsilon=1e-8, max_iters=10000),
    "c2": dict(kind=2, d=8192, n=4096, seed=2, epsilon=1e-8, max_iters=None),
    "c3": dict(kind=3, d=4096, n=4096, seed=3, epsilon=1e-10, max_iters=None),
    "c4": dict(kind=4, d=20000, n=256, seed=4, epsilon=1e-8, max_iters=None, nrhs=65536),
    "c5": dict(kind=5, d=32768, n=16384, seed=5, epsilon=1e-8, max_iters=None),
}

_lib = None


def _gen():
    global _lib
    if _lib is None:
        if not os.path.exists(GEN_LIB):
            raise FileNotFoundError(f"{GEN_LIB} missing: run __graft_entry__.build() or make")
        L = C.CDLL(GEN_LIB)
        dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        L.alnnls_gen_matrix.argtypes = [dp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int]
        L.alnnls_gen_config.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, dp, dp, dp,
                                        C.c_int]
        L.alnnls_gen_htrue.argtypes = [dp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]
        L.alnnls_gen_c3_matrix.argtypes = [dp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        _lib = L
    return _lib


def _threads():
    return max(1, min(32, os.cpu_count() or 1))


def gen_matrix(d, n, seed, law="u01"):
    """d x n (Fortran order) with column j from substream(seed, j)."""
    laws = {"u01": 0, "normal": 1, "absnormal": 2}
    A = np.empty(d * n)
    _gen().alnnls_gen_matrix(A, d, n, seed, laws[law], _threads())
    return A.reshape(d, n, order="F")


def _haar(n, seed):
    """Haar-random orthogonal n x n: QR of a Gaussian with the sign fix."""
    G = gen_matrix(n, n, seed, "normal")
    Qm, R = np.linalg.qr(G)
    return Qm * np.sign(np.diag(R))[None, :]


def make_config(name, d=None, n=None, seed=None):
    """Returns dict(A (d x n, Fortran), b, x_true, cfg kwargs). d/n/seed override
    the config's shape for scaled-down parity cases with the same value laws."""
    spec = dict(CONFIGS[name])
    d = spec["d"] if d is None else d
    n = spec["n"] if n is None else n
    seed = spec["seed"] if seed is None else seed
    kind = spec["kind"]
    if kind == 4:
        raise ValueError("c4 is batched: use make_batched")
    A = np.empty(d * n)
    b = np.empty(d)
    x = np.empty(n)
    if kind == 3:
        # U diag(s) V^T with Haar U, V, assembled in C (deterministic on any host)
        _gen().alnnls_gen_c3_matrix(A, d, n, seed, _threads())
    _gen().alnnls_gen_config(kind, d, n, seed, A, b, x, _threads())
    return {
        "A": A.reshape(d, n, order="F"),
        "b": b,
        "x_true": x,
        "epsilon": spec["epsilon"],
        "max_iters": spec["max_iters"],
        "name": name,
        "seed": seed,
    }


def make_batched(d=None, n=None, nrhs=None, seed=None, col0=0):
    """c4: A (d x n, U[0,1)), H_true (n x nrhs, 40% zeros per column), B = A H_true.
    B is formed on the host here (tests, small nrhs); bench.py forms it on device."""
    spec = CONFIGS["c4"]
    d = spec["d"] if d is None else d
    n = spec["n"] if n is None else n
    nrhs = spec["nrhs"] if nrhs is None else nrhs
    seed = spec["seed"] if seed is None else seed
    A = gen_matrix(d, n, seed, "u01")
    H = gen_htrue(n, nrhs, seed, col0)
    B = np.asfortranarray(A @ H)
    return {"A": A, "H_true": H, "B": B, "epsilon": spec["epsilon"], "seed": seed}


def gen_htrue(n, nrhs, seed, col0=0):
    H = np.empty(n * nrhs)
    _gen().alnnls_gen_htrue(H, n, nrhs, seed, col0)
    return H.reshape(n, nrhs, order="F")


def sha256(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).reshape(-1).tobytes()
                 if a.flags["C_CONTIGUOUS"] else np.asfortranarray(a).tobytes(order="F"))
    return h.hexdigest()

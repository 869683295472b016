"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the parity checkers.

* ``Oracle("oracle")``: oracle/build/liboracle.so, the plain-C restatement of
  the reference hot path (oracle/antilop_oracle.c).
* ``Oracle("ref")``: oracle/_ref/libantilop_ref.so, the reference headers
  compiled in place (oracle/ref_shim.cpp, oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module. The product package never does.
"""
import ctypes as C
import os

import numpy as np

from paper_1502_01645_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "oracle": os.path.join(HERE, "build", "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libantilop_ref.so"),
}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class OracleOut(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("x_cap", C.c_uint64),
        ("inner_x", C.c_void_p), ("final_grad", C.c_void_p), ("vec_cap", C.c_uint64),
        ("trace", C.c_void_p), ("trace_cap", C.c_uint64),
        ("mults", C.c_void_p), ("mults_cap", C.c_uint64),
        ("scale", C.c_void_p), ("retained", C.c_void_p), ("dropped", C.c_void_p),
        ("summary", abi.Summary),
        ("error", C.c_char * 256),
    ]


def available(kind):
    return os.path.exists(LIBS[kind])


class OracleError(Exception):
    def __init__(self, status, msg, result=None):
        super().__init__(f"{abi.STATUS_NAMES[status]}: {msg}")
        self.status = status
        self.result = result


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _trace_list(buf, n):
    out = []
    for i in range(min(n, len(buf))):
        r = buf[i]
        out.append({"iter": r.iter, "f": r.f, "grad_bar_sq": r.grad_bar_sq,
                    "passive_count": r.passive_count, "elapsed": r.elapsed_s,
                    "alpha": r.alpha if r.has_alpha else None})
    return out


class Oracle:
    def __init__(self, kind="oracle"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        p = "oracle_" if kind == "oracle" else "ref_"
        self.p = p
        L = self.lib
        for name, args in {
            "gram": [C.c_uint64, C.c_uint64, _dp, _dp],
            "transpose_matvec": [C.c_uint64, C.c_uint64, _dp, _dp, _dp],
            "matvec": [C.c_uint64, C.c_uint64, _dp, _dp, _dp],
            "masked_matvec": [C.c_uint64, C.c_uint64, _dp, _dp, _up, C.c_uint64, _dp,
                              C.POINTER(C.c_uint64)],
            "rescale": [C.c_uint64, _dp, _dp, _dp, _dp, C.POINTER(OracleOut)],
            "solve_nqp": [C.c_uint64, _dp, _dp, C.c_void_p, C.POINTER(abi.Config),
                          C.POINTER(OracleOut)],
            "solve_nnls": [C.c_uint64, C.c_uint64, _dp, _dp, C.POINTER(abi.Config),
                           C.POINTER(OracleOut)],
            "solve_accelerated": [C.c_uint64, _dp, _dp, C.c_void_p, C.POINTER(abi.Config),
                                  C.POINTER(OracleOut)],
            "solve_anti_accelerated": [C.c_uint64, C.c_uint64, _dp, _dp, C.POINTER(abi.Config),
                                       C.POINTER(OracleOut)],
        }.items():
            f = getattr(L, p + name)
            f.argtypes = args
            f.restype = C.c_int
        for name in ("objective", "kkt_error"):
            f = getattr(L, p + name)
            f.argtypes = [C.c_uint64, _dp, _dp, _dp]
            f.restype = C.c_double
        f = getattr(L, p + "frobenius_norm")
        f.argtypes = [C.c_uint64, C.c_uint64, _dp]
        f.restype = C.c_double
        if kind == "ref":
            f = L.ref_solve_nnls_columns
            f.argtypes = [C.c_uint64, C.c_uint64, _dp, C.c_uint64, _dp, C.POINTER(abi.Config),
                          _dp, C.c_void_p, C.c_int]
            f.restype = C.c_int

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    # ---- dense kernels (linalg.hpp) ----
    def gram(self, A):
        A = np.asfortranarray(A, dtype=np.float64)
        d, n = A.shape
        H = np.empty(n * n)
        self._fn("gram")(d, n, A.reshape(-1, order="F"), H)
        return H.reshape(n, n, order="F")

    def transpose_matvec(self, M, v):
        M = np.asfortranarray(M, dtype=np.float64)
        y = np.empty(M.shape[1])
        self._fn("transpose_matvec")(M.shape[0], M.shape[1], M.reshape(-1, order="F"),
                                     np.ascontiguousarray(v, dtype=np.float64), y)
        return y

    def matvec(self, M, v):
        M = np.asfortranarray(M, dtype=np.float64)
        y = np.empty(M.shape[0])
        self._fn("matvec")(M.shape[0], M.shape[1], M.reshape(-1, order="F"),
                           np.ascontiguousarray(v, dtype=np.float64), y)
        return y

    def masked_matvec(self, M, v, mask, count=None):
        M = np.asfortranarray(M, dtype=np.float64)
        y = np.empty(M.shape[0])
        mk = np.ascontiguousarray(mask, dtype=np.uint64)
        cnt = C.c_uint64(count or 0)
        st = self._fn("masked_matvec")(M.shape[0], M.shape[1], M.reshape(-1, order="F"),
                                       np.ascontiguousarray(v, dtype=np.float64),
                                       mk if len(mk) else np.zeros(1, np.uint64), len(mk), y,
                                       C.byref(cnt))
        if st != abi.OK:
            raise OracleError(st, "masked_matvec: mask index out of range")
        return y, cnt.value

    def objective(self, Q, q, x):
        Q = np.asfortranarray(Q, dtype=np.float64)
        return self._fn("objective")(len(q), Q.reshape(-1, order="F"),
                                     np.ascontiguousarray(q, np.float64),
                                     np.ascontiguousarray(x, np.float64))

    def kkt_error(self, Q, q, x):
        Q = np.asfortranarray(Q, dtype=np.float64)
        return self._fn("kkt_error")(len(q), Q.reshape(-1, order="F"),
                                     np.ascontiguousarray(q, np.float64),
                                     np.ascontiguousarray(x, np.float64))

    # ---- rescale (nnls.hpp:41-83) ----
    def rescale(self, H, h):
        H = np.asfortranarray(H, dtype=np.float64)
        n = H.shape[0]
        Q = np.zeros(max(1, n * n))
        q = np.zeros(max(1, n))
        out = OracleOut()
        scale = np.zeros(max(1, n))
        ret = np.zeros(max(1, n), np.uint64)
        drop = np.zeros(max(1, n), np.uint64)
        out.scale, out.retained, out.dropped = _ptr(scale), _ptr(ret), _ptr(drop)
        st = self._fn("rescale")(n, H.reshape(-1, order="F"), np.ascontiguousarray(h, np.float64),
                                 Q, q, C.byref(out))
        if st != abi.OK:
            raise OracleError(st, out.error.decode())
        m = out.summary.m
        return {"Q": Q[:m * m].reshape(m, m, order="F"), "q": q[:m].copy(),
                "scale": scale[:m].copy(), "retained": ret[:m].copy(),
                "dropped": drop[:out.summary.n_dropped].copy()}

    # ---- solvers ----
    def _alloc(self, cfg, n, m):
        out = OracleOut()
        keep = {}
        tcap = abi.trace_capacity(cfg, m)
        keep["trace"] = (abi.IterRecord * tcap)()
        keep["x"] = np.zeros(max(1, n))
        keep["inner_x"] = np.zeros(max(1, m))
        keep["final_grad"] = np.zeros(max(1, m))
        mcap = (cfg.max_iters if cfg.has_max_iters else 5 * m) + 1
        keep["mults"] = np.zeros(max(1, mcap), np.uint64)
        keep["scale"] = np.zeros(max(1, n))
        keep["retained"] = np.zeros(max(1, n), np.uint64)
        keep["dropped"] = np.zeros(max(1, n), np.uint64)
        out.x, out.x_cap = _ptr(keep["x"]), n
        out.inner_x, out.final_grad, out.vec_cap = _ptr(keep["inner_x"]), _ptr(keep["final_grad"]), m
        out.trace, out.trace_cap = C.cast(keep["trace"], C.c_void_p), tcap
        out.mults, out.mults_cap = _ptr(keep["mults"]), mcap
        out.scale, out.retained, out.dropped = (_ptr(keep["scale"]), _ptr(keep["retained"]),
                                                _ptr(keep["dropped"]))
        return out, keep

    @staticmethod
    def _result(out, keep, nnls):
        s = out.summary
        r = {
            "termination": abi.TERMINATIONS[s.termination],
            "iterations": s.iterations,
            "trace": _trace_list(keep["trace"], s.trace_len),
            "trace_len": s.trace_len,
            "min_iterate": s.min_iterate,
            "final_grad": keep["final_grad"][:s.m].copy(),
            "mults": keep["mults"][:s.mult_len].copy(),
            "multiplies_total": s.multiplies_total,
            "m": s.m,
            "summary": s,
        }
        if nnls:
            r["x"] = keep["x"][:s.n].copy()
            r["inner_x"] = keep["inner_x"][:s.m].copy()
            r["residual_sq"] = s.residual_sq
            r["dropped"] = keep["dropped"][:s.n_dropped].copy()
        else:
            r["x"] = keep["x"][:s.m].copy()
        return r

    def solve_nqp(self, Q, q, cfg, start=None):
        Q = np.asfortranarray(Q, dtype=np.float64)
        m = Q.shape[0]
        out, keep = self._alloc(cfg, m, m)
        st_arr = None if start is None else np.ascontiguousarray(start, np.float64)
        st = self._fn("solve_nqp")(m, Q.reshape(-1, order="F"), np.ascontiguousarray(q, np.float64),
                                   _ptr(st_arr), C.byref(cfg), C.byref(out))
        if st != abi.OK:
            res = self._result(out, keep, False) if st == abi.ENUMERIC else None
            raise OracleError(st, out.error.decode(), res)
        return self._result(out, keep, False)

    def frobenius_norm(self, M):
        M = np.asfortranarray(M, dtype=np.float64)
        return self._fn("frobenius_norm")(M.shape[0], M.shape[1], M.reshape(-1, order="F"))

    def solve_accelerated(self, Q, q, cfg):
        """accelerated.hpp:21-117 (Nesterov baseline on an NQP)."""
        Q = np.asfortranarray(Q, dtype=np.float64)
        m = Q.shape[0]
        out, keep = self._alloc(cfg, m, m)
        st = self._fn("solve_accelerated")(m, Q.reshape(-1, order="F"),
                                           np.ascontiguousarray(q, np.float64), None,
                                           C.byref(cfg), C.byref(out))
        if st != abi.OK:
            res = self._result(out, keep, False) if st == abi.ENUMERIC else None
            raise OracleError(st, out.error.decode(), res)
        return self._result(out, keep, False)

    def solve_anti_accelerated(self, A, b, cfg):
        """accelerated.hpp:121-139 (Anti+Acc: rescale, then the Nesterov baseline)."""
        return self.solve_nnls(A, b, cfg, fn="solve_anti_accelerated")

    def solve_nnls(self, A, b, cfg, fn="solve_nnls"):
        A = np.asfortranarray(A, dtype=np.float64)
        d, n = A.shape
        out, keep = self._alloc(cfg, n, n)
        st = self._fn(fn)(d, n, A.reshape(-1, order="F"),
                                    np.ascontiguousarray(b, np.float64), C.byref(cfg), C.byref(out))
        if st != abi.OK:
            res = self._result(out, keep, True) if st == abi.ENUMERIC else None
            raise OracleError(st, out.error.decode(), res)
        return self._result(out, keep, True)

    def solve_nnls_columns(self, A, B, cfg, threads=1):
        """ref only: Gram once + per-column reference pipeline (bitwise = solve_nnls)."""
        A = np.asfortranarray(A, dtype=np.float64)
        B = np.asfortranarray(B, dtype=np.float64)
        d, n = A.shape
        k = B.shape[1]
        X = np.zeros(n * k)
        cols = (abi.ColumnResult * k)()
        st = self.lib.ref_solve_nnls_columns(d, n, A.reshape(-1, order="F"), k,
                                             B.reshape(-1, order="F"), C.byref(cfg), X,
                                             C.cast(cols, C.c_void_p), threads)
        if st != abi.OK:
            raise OracleError(st, "ref_solve_nnls_columns failed")
        return X.reshape(n, k, order="F"), cols

"""Python mirror of the reference's public solver API, backed by the C ABI.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/antilop/{linalg,nqp,nnls}.hpp):

    solve_nnls(A, b, config)            nnls.hpp:129-144
    solve_nqp(Q, q, config, start)      nqp.hpp:215-339
    gram / matvec / masked_matvec / transpose_matvec   linalg.hpp:160-219
    rescale(H, h)                       nnls.hpp:41-83

Errors: std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
antilop::NumericFailure -> NumericFailure (carries .trace). All compute runs on
the GPU through lib/libalnnls.so; there is no CPU fallback.
"""
import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi
from ._native import load

TERMINATIONS = abi.TERMINATIONS


class ColumnResults:
    """Per-column results of a batched solve (alnnls_column_result records): a sequence of
    dicts built on access, over one structured numpy copy of the records (`.array`), so a
    65536-column batch does not pay for 65536 Python dicts inside the call."""
    _DTYPE = np.dtype([("termination", "<i4"), ("numeric_failure", "<i4"), ("iterations", "<u8"),
                       ("residual_sq", "<f8"), ("f_final", "<f8"), ("gbs_final", "<f8"),
                       ("multiplies_total", "<u8")])

    def __init__(self, cols):
        assert self._DTYPE.itemsize == C.sizeof(abi.ColumnResult)
        self.array = np.frombuffer(cols, dtype=self._DTYPE).copy() if len(cols) else \
            np.zeros(0, dtype=self._DTYPE)

    def __len__(self):
        return len(self.array)

    def _dict(self, r):
        return {"termination": TERMINATIONS[int(r["termination"])],
                "numeric_failure": bool(r["numeric_failure"]), "iterations": int(r["iterations"]),
                "residual_sq": float(r["residual_sq"]), "f_final": float(r["f_final"]),
                "gbs_final": float(r["gbs_final"]),
                "multiplies_total": int(r["multiplies_total"])}

    def __getitem__(self, j):
        if isinstance(j, slice):
            return [self._dict(r) for r in self.array[j]]
        return self._dict(self.array[j])

    def __iter__(self):
        return (self._dict(r) for r in self.array)

    def __eq__(self, other):
        return list(self) == list(other)


class NumericFailure(RuntimeError):
    """antilop::NumericFailure (nqp.hpp:136-145)."""

    def __init__(self, what, trace):
        super().__init__(what)
        self.trace = trace


@dataclass
class SolverConfig:
    """antilop::SolverConfig (nqp.hpp:71-99) + the numerics profile extension."""
    epsilon: Optional[float] = None
    max_iters: Optional[int] = None
    time_cap: Optional[float] = None  # seconds
    stall_window: int = 50
    trace_every: int = 1
    nesterov_restart: bool = False    # accelerated baseline only (unused here)
    active_set_tol: Optional[float] = None  # active-set baseline only (unused here)
    profile: int = abi.PROFILE_EXACT

    def to_abi(self, record_multiplies=True):
        return abi.make_config(self.epsilon, self.max_iters, self.time_cap, self.stall_window,
                               self.trace_every, self.profile, record_multiplies,
                               self.nesterov_restart)

    def resolve_epsilon(self, n):
        if self.epsilon is not None:
            if not self.epsilon > 0.0:
                raise ValueError("SolverConfig: epsilon must be > 0")
            return self.epsilon
        return 1e-10 * n

    def resolve_max_iters(self, n):
        if self.max_iters is not None:
            if self.max_iters < 1:
                raise ValueError("SolverConfig: max_iters must be >= 1")
            return self.max_iters
        return 5 * n


@dataclass
class IterRecord:
    iter: int
    f: float
    grad_bar_sq: float
    passive_count: int
    elapsed: float
    alpha: Optional[float]


@dataclass
class SolveResult:
    x: np.ndarray
    trace: List[IterRecord]
    termination: str
    final_grad: np.ndarray
    min_iterate: float
    multiplies_per_iter: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    timings: dict = field(default_factory=dict)

    def iterations(self):
        return self.trace[-1].iter if self.trace else 0


@dataclass
class NnlsResult:
    x: np.ndarray
    residual_sq: float
    inner: SolveResult
    dropped_columns: List[int]
    timings: dict = field(default_factory=dict)


def _f64(a, name):
    a = np.asarray(a, dtype=np.float64)
    return a


def _fortran(M):
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise ValueError("DenseMatrix: expected a 2-D array")
    return np.asfortranarray(M)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class Solver:
    """One alnnls_ctx (device memory, stream, events) on one GPU.

    Single-threaded like the C context; use one Solver per thread/device."""

    def __init__(self, device=0):
        self.lib = load()
        self.ctx = C.c_void_p()
        st = self.lib.alnnls_create(C.byref(self.ctx), device)
        if st != abi.OK:
            raise RuntimeError(f"alnnls_create(device={device}) failed: {abi.STATUS_NAMES[st]} "
                               "(no sm_100 GPU visible; there is no CPU fallback)")
        self.device = device

    def close(self):
        if self.ctx:
            self.lib.alnnls_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- error mapping ------------------------------------------------------------
    def _raise(self, st, trace=None):
        msg = self.lib.alnnls_last_error(self.ctx).decode()
        if st == abi.EINVAL:
            raise ValueError(msg)
        if st == abi.ERANGE:
            raise IndexError(msg)
        if st == abi.ENUMERIC:
            raise NumericFailure(msg, trace if trace is not None else self._trace())
        raise RuntimeError(f"{abi.STATUS_NAMES[st]}: {msg}")

    def _check(self, st):
        if st != abi.OK:
            self._raise(st)

    def _vec(self, fn, n, dtype=np.float64):
        out = np.zeros(max(1, n), dtype=dtype)
        self._check(fn(self.ctx, _ptr(out), n))
        return out[:n]

    def _trace(self):
        s = self._summary
        buf = (abi.IterRecord * max(1, s.trace_len))()
        self._check(self.lib.alnnls_get_trace(self.ctx, C.cast(buf, C.c_void_p), s.trace_len))
        return [IterRecord(r.iter, r.f, r.grad_bar_sq, r.passive_count, r.elapsed_s,
                           r.alpha if r.has_alpha else None) for r in buf[:s.trace_len]]

    def _solve_result(self, nnls):
        s = self._summary
        m = s.m
        if nnls:
            x_inner = self._vec(self.lib.alnnls_get_inner_x, m)
        else:
            x_inner = self._vec(self.lib.alnnls_get_x, m)
        mults = self._vec(self.lib.alnnls_get_multiplies, s.mult_len, np.uint64)
        return SolveResult(
            x=x_inner,
            trace=self._trace(),
            termination=TERMINATIONS[s.termination],
            final_grad=self._vec(self.lib.alnnls_get_final_grad, m),
            min_iterate=s.min_iterate,
            multiplies_per_iter=mults,
            timings={"loop_s": s.t_loop_s, "phase_s": self.phase_times()},
        )

    def timer_start(self):
        """Records a CUDA event on the context's stream (device-side timing)."""
        self._check(self.lib.alnnls_timer_start(self.ctx))

    def timer_stop(self):
        """Seconds between timer_start and now, measured on the device."""
        out = C.c_double()
        self._check(self.lib.alnnls_timer_stop(self.ctx, C.byref(out)))
        return out.value

    def launch_count(self):
        """Number of this library's kernels launched on the context so far."""
        return int(self.lib.alnnls_launch_count(self.ctx))

    def loop_kernel(self):
        """Loop kernel of the last solve: "grid", "cluster", "small", "fast" or "none"."""
        k = int(self.lib.alnnls_last_loop_kernel(self.ctx))
        return {0: "none", 1: "grid", 2: "cluster", 3: "small", 4: "fast"}.get(k, str(k))

    def last_summary(self):
        return self._summary

    def phase_times(self):
        ns = np.zeros(8, np.uint64)
        self._check(self.lib.alnnls_get_phase_ns(self.ctx, _ptr(ns), 8))
        return [float(v) * 1e-9 for v in ns[:8]]

    # ---- solvers ------------------------------------------------------------------
    def solve_nnls(self, A, b, config: SolverConfig = SolverConfig()):
        A = _fortran(A)
        b = np.ascontiguousarray(_f64(b, "b")).reshape(-1)
        if A.shape[0] != b.shape[0]:
            raise ValueError("solve_nnls: A and b dimension mismatch")
        d, n = A.shape
        self._summary = abi.Summary()
        cfg = config.to_abi()
        st = self.lib.alnnls_solve_nnls(self.ctx, d, n, _ptr(A), _ptr(b), C.byref(cfg),
                                        C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._nnls_result()

    def solve_nnls_device(self, A_ptr, lda, d, n, b_ptr, config: SolverConfig = SolverConfig(),
                          fetch=True):
        """Inputs already in HBM (e.g. torch tensors' data_ptr()); A column-major."""
        self._summary = abi.Summary()
        cfg = config.to_abi()
        st = self.lib.alnnls_solve_nnls_device(self.ctx, d, n, C.c_void_p(A_ptr), lda,
                                               C.c_void_p(b_ptr), C.byref(cfg),
                                               C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._nnls_result() if fetch else self._summary

    def _nnls_result(self):
        s = self._summary
        x = self._vec(self.lib.alnnls_get_x, s.n)
        dropped = self._vec(self.lib.alnnls_get_dropped, s.n_dropped, np.uint64)
        inner = self._solve_result(True)
        return NnlsResult(x=x, residual_sq=s.residual_sq, inner=inner,
                          dropped_columns=[int(v) for v in dropped],
                          timings={"setup_s": s.t_setup_s, "loop_s": s.t_loop_s,
                                   "finish_s": s.t_finish_s, "total_s": s.t_total_s})

    # ---- multi-GPU exact setup by row blocks (include/alnnls.h) ----
    GRAM_TILE_DOUBLES = 16384

    def gram_tiles(self, n):
        return int(self.lib.alnnls_gram_tiles(n))

    def gram_rowblock_device(self, rows, n, A_ptr, lda, tile_lo, tile_hi, pin_ptr=0, pout_ptr=0,
                             H_ptr=0):
        """Continues the Gram tiles [tile_lo, tile_hi) over a row block (device pointers)."""
        self._check(self.lib.alnnls_gram_rowblock_device(
            self.ctx, rows, n, C.c_void_p(A_ptr), lda, tile_lo, tile_hi,
            C.c_void_p(pin_ptr) if pin_ptr else None, C.c_void_p(pout_ptr) if pout_ptr else None,
            C.c_void_p(H_ptr) if H_ptr else None))

    def atb_rowblock_device(self, rows, n, A_ptr, lda, b_ptr, pin_ptr, out_ptr):
        self._check(self.lib.alnnls_atb_rowblock_device(
            self.ctx, rows, n, C.c_void_p(A_ptr), lda, C.c_void_p(b_ptr),
            C.c_void_p(pin_ptr) if pin_ptr else None, C.c_void_p(out_ptr)))

    def solve_nnls_gram_device(self, n, H_ptr, atb_ptr, config: SolverConfig = SolverConfig(),
                               fetch=True):
        """rescale + solve_nqp + unscale from a finished Gram and A^T b chains."""
        self._summary = abi.Summary()
        cfg = config.to_abi()
        st = self.lib.alnnls_solve_nnls_gram_device(self.ctx, n, C.c_void_p(H_ptr),
                                                    C.c_void_p(atb_ptr), C.byref(cfg),
                                                    C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._nnls_result() if fetch else self._summary

    def gram_partial_device(self, rows, n, A_ptr, lda, b_ptr, H_ptr, atb_ptr,
                            profile=abi.PROFILE_FAST):
        """Partial Gram A_blk^T A_blk (n x n, both triangles) and A_blk^T b_blk of one
        row block, for the allreduce setup (rowblock.allreduce_setup)."""
        self._check(self.lib.alnnls_gram_partial_device(
            self.ctx, rows, n, C.c_void_p(A_ptr), lda, C.c_void_p(b_ptr) if b_ptr else None,
            int(profile), C.c_void_p(H_ptr), C.c_void_p(atb_ptr) if atb_ptr else None))

    def pack_upper_device(self, n, H_ptr, P_ptr):
        """Packed upper triangle (j(j+1)/2 + i) of the symmetric n x n dH into dP."""
        self._check(self.lib.alnnls_pack_upper_device(self.ctx, n, C.c_void_p(H_ptr),
                                                      C.c_void_p(P_ptr)))

    def unpack_upper_device(self, n, P_ptr, H_ptr):
        """dH (both triangles) from the packed upper triangle dP."""
        self._check(self.lib.alnnls_unpack_upper_device(self.ctx, n, C.c_void_p(P_ptr),
                                                        C.c_void_p(H_ptr)))

    def nmf(self, V, W0, outer_iters, config: SolverConfig = SolverConfig()):
        """NMF by alternating NNLS (alnnls_nmf): V (d x N) ~ W H, W >= 0, H >= 0.
        W0 (d x k, nonnegative) is the start. Returns (W, H, objective per outer
        iteration = ||V - W H||_F^2 after its H update)."""
        V = _fortran(V)
        W = np.array(_fortran(W0), order="F", copy=True)
        d, N = V.shape
        if W.shape[0] != d:
            raise ValueError("nmf: V and W dimension mismatch")
        k = W.shape[1]
        H = np.zeros((k, N), order="F")
        obj = np.zeros(max(1, outer_iters))
        cfg = config.to_abi(record_multiplies=False)
        self._check(self.lib.alnnls_nmf(self.ctx, d, N, k, _ptr(V), _ptr(W), _ptr(H), outer_iters,
                                        C.byref(cfg), _ptr(obj)))
        return W, H, obj[:outer_iters]

    def matmat_device(self, rows, inner, cols, A_ptr, lda, H_ptr, ldh, C_ptr, ldc):
        """C = A H on device pointers, column j bitwise matvec(A, H[:, j])."""
        self._check(self.lib.alnnls_matmat_device(self.ctx, rows, inner, cols, C.c_void_p(A_ptr),
                                                  lda, C.c_void_p(H_ptr), ldh, C.c_void_p(C_ptr),
                                                  ldc))

    def finish(self, A, b, y):
        """x = unscale(y, sys, n) and ||A x - b||^2 (nnls.hpp:141-142) with the rescale
        bookkeeping of the last setup / solve on this context."""
        A = _fortran(A)
        b = np.ascontiguousarray(_f64(b, "b")).reshape(-1)
        y = np.ascontiguousarray(_f64(y, "y")).reshape(-1)
        d, n = A.shape
        x = np.zeros(n)
        r = C.c_double(0.0)
        self._check(self.lib.alnnls_finish(self.ctx, d, n, _ptr(A), _ptr(b),
                                           _ptr(y) if len(y) else None, len(y), _ptr(x),
                                           C.byref(r)))
        return x, r.value

    def residual_rowblock_device(self, rows, n, A_ptr, lda, b_ptr, x_ptr, s_in=0.0):
        out = C.c_double(0.0)
        self._check(self.lib.alnnls_residual_rowblock_device(
            self.ctx, rows, n, C.c_void_p(A_ptr), lda, C.c_void_p(b_ptr), C.c_void_p(x_ptr),
            float(s_in), C.byref(out)))
        return out.value

    def solve_nnls_batched(self, A, B, config: SolverConfig = SolverConfig(), out=None):
        """solve_nnls(A, B[:, j], config) for every column j (bitwise, exact profile).
        Returns (X (n x nrhs), per-column results, summary timings). `out`: an optional
        Fortran-ordered float64 (n x nrhs) array that receives X (e.g. a pinned buffer a
        caller reuses across NMF half steps) instead of a fresh allocation."""
        A = _fortran(A)
        B = _fortran(B)
        if A.shape[0] != B.shape[0]:
            raise ValueError("solve_nnls: A and b dimension mismatch")
        d, n = A.shape
        k = B.shape[1]
        if out is not None:
            if (out.dtype != np.float64 or out.shape != (n, k) or not out.flags.f_contiguous
                    or not out.flags.writeable):
                raise ValueError("solve_nnls_batched: out must be a writable Fortran-ordered "
                                 "float64 (n x nrhs) array")
            X = out
        else:
            X = np.empty((n, k), order="F")  # the library writes every entry
        cols = (abi.ColumnResult * k)()
        self._summary = abi.Summary()
        cfg = config.to_abi(record_multiplies=False)
        st = self.lib.alnnls_solve_nnls_batched(self.ctx, d, n, _ptr(A), k, _ptr(B), C.byref(cfg),
                                                _ptr(X), C.cast(cols, C.c_void_p),
                                                C.byref(self._summary))
        if st != abi.OK:
            self._raise(st, trace=[])
        return X, ColumnResults(cols), self._timings()

    def solve_nnls_batched_device(self, A_ptr, B_ptr, X_ptr, d, n, nrhs,
                                  config: SolverConfig = SolverConfig(), fetch_cols=True):
        """Device-resident batched solve: A (d x n), B (d x nrhs), X (n x nrhs), column-major."""
        cols = (abi.ColumnResult * nrhs)() if fetch_cols else None
        self._summary = abi.Summary()
        cfg = config.to_abi(record_multiplies=False)
        st = self.lib.alnnls_solve_nnls_batched_device(
            self.ctx, d, n, C.c_void_p(A_ptr), nrhs, C.c_void_p(B_ptr), C.byref(cfg),
            C.c_void_p(X_ptr), C.cast(cols, C.c_void_p) if cols is not None else None,
            C.byref(self._summary))
        if st != abi.OK:
            self._raise(st, trace=[])
        return (ColumnResults(cols) if cols is not None else None), self._timings()

    @staticmethod
    def _col(c):
        return {"termination": TERMINATIONS[c.termination], "numeric_failure": bool(c.numeric_failure),
                "iterations": int(c.iterations), "residual_sq": c.residual_sq, "f_final": c.f_final,
                "gbs_final": c.gbs_final, "multiplies_total": int(c.multiplies_total)}

    def _timings(self):
        s = self._summary
        return {"setup_s": s.t_setup_s, "loop_s": s.t_loop_s, "finish_s": s.t_finish_s,
                "total_s": s.t_total_s, "multiplies_total": int(s.multiplies_total),
                "iterations_total": int(s.iterations)}

    def solve_nqp(self, Q, q, config: SolverConfig = SolverConfig(), start=None):
        Q = _fortran(Q)
        q = np.ascontiguousarray(_f64(q, "q")).reshape(-1)
        if Q.shape[0] != Q.shape[1]:
            raise ValueError("NqpProblem: Q must be square")
        if Q.shape[0] != q.shape[0]:
            raise ValueError("NqpProblem: Q and q dimension mismatch")
        m = q.shape[0]
        sp = None
        if start is not None:
            start = np.ascontiguousarray(_f64(start, "start")).reshape(-1)
            if start.shape[0] != m:
                raise ValueError("solve_nqp: start dimension mismatch")
            sp = _ptr(start)
        self._summary = abi.Summary()
        cfg = config.to_abi()
        st = self.lib.alnnls_solve_nqp(self.ctx, m, _ptr(Q), _ptr(q), sp, C.byref(cfg),
                                       C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._solve_result(False)

    # ---- Anti+Acc baseline (accelerated.hpp) -------------------------------
    def solve_anti_accelerated(self, A, b, config: SolverConfig = SolverConfig()):
        """solve_anti_accelerated (accelerated.hpp:121-139): rescale, Nesterov, unscale."""
        A = _fortran(A)
        b = np.ascontiguousarray(_f64(b, "b")).reshape(-1)
        if A.shape[0] != b.shape[0]:
            raise ValueError("solve_anti_accelerated: A and b dimension mismatch")
        d, n = A.shape
        self._summary = abi.Summary()
        cfg = config.to_abi(record_multiplies=False)
        st = self.lib.alnnls_solve_anti_accelerated(self.ctx, d, n, _ptr(A), _ptr(b), C.byref(cfg),
                                                    C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._nnls_result()

    def solve_anti_accelerated_device(self, A_ptr, lda, d, n, b_ptr,
                                      config: SolverConfig = SolverConfig(), fetch=True):
        self._summary = abi.Summary()
        cfg = config.to_abi(record_multiplies=False)
        st = self.lib.alnnls_solve_anti_accelerated_device(self.ctx, d, n, C.c_void_p(A_ptr), lda,
                                                           C.c_void_p(b_ptr), C.byref(cfg),
                                                           C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._nnls_result() if fetch else self._summary

    def solve_accelerated(self, Q, q, config: SolverConfig = SolverConfig()):
        """solve_accelerated (accelerated.hpp:21-117) on an NQP."""
        Q = _fortran(Q)
        q = np.ascontiguousarray(_f64(q, "q")).reshape(-1)
        if Q.shape[0] != Q.shape[1]:
            raise ValueError("NqpProblem: Q must be square")
        if Q.shape[0] != q.shape[0]:
            raise ValueError("NqpProblem: Q and q dimension mismatch")
        self._summary = abi.Summary()
        cfg = config.to_abi(record_multiplies=False)
        st = self.lib.alnnls_solve_accelerated(self.ctx, q.shape[0], _ptr(Q), _ptr(q), C.byref(cfg),
                                               C.byref(self._summary))
        if st != abi.OK:
            self._raise(st)
        return self._solve_result(False)

    # ---- setup and dense kernels ---------------------------------------------------------
    def setup(self, A, b):
        """rescale(gram(A), -A^T b) on device -> dict(Q, q, scale, retained, dropped)."""
        A = _fortran(A)
        b = np.ascontiguousarray(_f64(b, "b")).reshape(-1)
        self._summary = abi.Summary()
        self._check(self.lib.alnnls_setup(self.ctx, A.shape[0], A.shape[1], _ptr(A), _ptr(b),
                                          C.byref(self._summary)))
        return self._scaled()

    def rescale(self, H, h):
        H = _fortran(H)
        h = np.ascontiguousarray(_f64(h, "h")).reshape(-1)
        if H.shape[0] != H.shape[1]:
            raise ValueError("rescale: H must be square")
        if H.shape[0] != h.shape[0]:
            raise ValueError("rescale: H and h dimension mismatch")
        self._summary = abi.Summary()
        self._check(self.lib.alnnls_rescale(self.ctx, H.shape[0], _ptr(H), _ptr(h),
                                            C.byref(self._summary)))
        return self._scaled()

    def _scaled(self):
        s = self._summary
        m = s.m
        Qf = self._vec(self.lib.alnnls_get_Q, m * m)
        return {
            "Q": Qf.reshape(m, m, order="F"),
            "q": self._vec(self.lib.alnnls_get_q, m),
            "scale": self._vec(self.lib.alnnls_get_scale, m),
            "retained": self._vec(self.lib.alnnls_get_retained, m, np.uint64),
            "dropped": self._vec(self.lib.alnnls_get_dropped, s.n_dropped, np.uint64),
            "t_setup_s": s.t_setup_s,
        }

    def gram(self, A):
        A = _fortran(A)
        d, n = A.shape
        H = np.zeros(n * n)
        self._check(self.lib.alnnls_gram(self.ctx, d, n, _ptr(A), _ptr(H)))
        return H.reshape(n, n, order="F")

    def transpose_matvec(self, M, v):
        M = _fortran(M)
        v = np.ascontiguousarray(_f64(v, "v")).reshape(-1)
        if M.shape[0] != v.shape[0]:
            raise ValueError("transpose_matvec: dimension mismatch")
        y = np.zeros(M.shape[1])
        self._check(self.lib.alnnls_transpose_matvec(self.ctx, M.shape[0], M.shape[1], _ptr(M),
                                                     _ptr(v), _ptr(y)))
        return y

    def matvec(self, M, v):
        M = _fortran(M)
        v = np.ascontiguousarray(_f64(v, "v")).reshape(-1)
        if M.shape[1] != v.shape[0]:
            raise ValueError("matvec: dimension mismatch")
        y = np.zeros(M.shape[0])
        self._check(self.lib.alnnls_matvec(self.ctx, M.shape[0], M.shape[1], _ptr(M), _ptr(v),
                                           _ptr(y)))
        return y

    def masked_matvec(self, M, v, mask, multiply_count=None):
        """Returns y (and the incremented count when multiply_count is given)."""
        M = _fortran(M)
        v = np.ascontiguousarray(_f64(v, "v")).reshape(-1)
        if M.shape[1] != v.shape[0]:
            raise ValueError("masked_matvec: dimension mismatch")
        mk = np.ascontiguousarray(np.asarray(mask, dtype=np.uint64).reshape(-1))
        y = np.zeros(M.shape[0])
        cnt = C.c_uint64(multiply_count or 0)
        self._check(self.lib.alnnls_masked_matvec(
            self.ctx, M.shape[0], M.shape[1], _ptr(M), _ptr(v),
            _ptr(mk) if len(mk) else None, len(mk), _ptr(y), C.byref(cnt)))
        return (y, cnt.value) if multiply_count is not None else y


_default = {}


def device_count():
    """Visible CUDA devices (0 without a GPU)."""
    return int(load().alnnls_device_count())


def solve_nnls_batched_multi(solvers, A, B, config: SolverConfig = SolverConfig()):
    """Batched solve with the columns of B sharded over several contexts (one per
    GPU: alnnls_solve_nnls_batched_multi, one host thread per context, no
    collective). Returns (X, [per-column dict], summary)."""
    A = _fortran(A)
    B = _fortran(B)
    if A.shape[0] != B.shape[0]:
        raise ValueError("solve_nnls: A and b dimension mismatch")
    d, n = A.shape
    k = B.shape[1]
    X = np.zeros((n, k), order="F")
    cols = (abi.ColumnResult * k)()
    summ = abi.Summary()
    cfg = config.to_abi(record_multiplies=False)
    arr = (C.c_void_p * len(solvers))(*[s.ctx.value for s in solvers])
    lib = load()
    st = lib.alnnls_solve_nnls_batched_multi(arr, len(solvers), d, n, _ptr(A), k, _ptr(B),
                                             C.byref(cfg), _ptr(X), C.cast(cols, C.c_void_p),
                                             C.byref(summ))
    if st != abi.OK:
        solvers[0]._raise(st)
    return X, ColumnResults(cols), summ


def default_solver(device=0):
    if device not in _default:
        _default[device] = Solver(device)
    return _default[device]


def solve_nnls(A, b, config: SolverConfig = SolverConfig()):
    return default_solver().solve_nnls(A, b, config)


def solve_nqp(Q, q, config: SolverConfig = SolverConfig(), start=None):
    return default_solver().solve_nqp(Q, q, config, start)


# Host-side helpers the reference's tests call (nqp.hpp:149-157, :183-207). They are
# O(n) / O(n^2) checks, not the hot path, and are restated here in numpy.
def passive_mask(x, grad):
    x = np.asarray(x, np.float64)
    grad = np.asarray(grad, np.float64)
    if x.shape != grad.shape:
        raise ValueError("passive_mask: length mismatch")
    return [i for i in range(len(x)) if x[i] > 0.0 or grad[i] < 0.0]


def to_string(termination):
    return termination

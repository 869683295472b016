"""ctypes mirrors of the POD types in include/alnnls.h (the C ABI).

Kept in one place so the product bindings (``_native``) and the test-only
oracle bindings (``oracle/oracle.py``) agree on the layout.
"""
import ctypes as C

OK, EINVAL, ENUMERIC, ECUDA, ENOMEM, ENCCL, ERANGE, ECAPACITY, ENODEV = range(9)
STATUS_NAMES = ["OK", "EINVAL", "ENUMERIC", "ECUDA", "ENOMEM", "ENCCL", "ERANGE",
                "ECAPACITY", "ENODEV"]

# antilop::Termination order (nqp.hpp:47-54)
TERMINATIONS = ["EmptyPassiveSet", "GradientBelowEpsilon", "MaxIters", "TimeCap",
                "Stalled", "ZeroCurvature"]

PROFILE_EXACT, PROFILE_FAST = 0, 1


class Config(C.Structure):
    _fields_ = [
        ("has_epsilon", C.c_int32),
        ("epsilon", C.c_double),
        ("has_max_iters", C.c_int32),
        ("max_iters", C.c_uint64),
        ("has_time_cap", C.c_int32),
        ("time_cap_s", C.c_double),
        ("stall_window", C.c_uint64),
        ("trace_every", C.c_uint64),
        ("profile", C.c_int32),
        ("record_multiplies", C.c_int32),
        ("nesterov_restart", C.c_int32),
    ]


class IterRecord(C.Structure):
    _fields_ = [
        ("iter", C.c_uint64),
        ("f", C.c_double),
        ("grad_bar_sq", C.c_double),
        ("passive_count", C.c_uint64),
        ("elapsed_s", C.c_double),
        ("alpha", C.c_double),
        ("has_alpha", C.c_int64),
    ]


class Summary(C.Structure):
    _fields_ = [
        ("termination", C.c_int32),
        ("numeric_failure", C.c_int32),
        ("iterations", C.c_uint64),
        ("trace_len", C.c_uint64),
        ("mult_len", C.c_uint64),
        ("n", C.c_uint64),
        ("m", C.c_uint64),
        ("n_dropped", C.c_uint64),
        ("min_iterate", C.c_double),
        ("residual_sq", C.c_double),
        ("f_final", C.c_double),
        ("gbs_final", C.c_double),
        ("multiplies_total", C.c_uint64),
        ("t_setup_s", C.c_double),
        ("t_loop_s", C.c_double),
        ("t_finish_s", C.c_double),
        ("t_total_s", C.c_double),
    ]


class ColumnResult(C.Structure):
    _fields_ = [
        ("termination", C.c_int32),
        ("numeric_failure", C.c_int32),
        ("iterations", C.c_uint64),
        ("residual_sq", C.c_double),
        ("f_final", C.c_double),
        ("gbs_final", C.c_double),
        ("multiplies_total", C.c_uint64),
    ]


def make_config(epsilon=None, max_iters=None, time_cap=None, stall_window=50, trace_every=1,
                profile=PROFILE_EXACT, record_multiplies=True, nesterov_restart=False):
    """SolverConfig (nqp.hpp:71-99) as the POD the ABI takes; None = unset optional."""
    c = Config()
    c.has_epsilon = 0 if epsilon is None else 1
    c.epsilon = 0.0 if epsilon is None else float(epsilon)
    c.has_max_iters = 0 if max_iters is None else 1
    c.max_iters = 0 if max_iters is None else int(max_iters)
    c.has_time_cap = 0 if time_cap is None else 1
    c.time_cap_s = 0.0 if time_cap is None else float(time_cap)
    c.stall_window = int(stall_window)
    c.trace_every = int(trace_every)
    c.profile = int(profile)
    c.record_multiplies = 1 if record_multiplies else 0
    c.nesterov_restart = 1 if nesterov_restart else 0
    return c


def trace_capacity(cfg, m):
    """floor(max_iters / trace_every) + 2 records."""
    mi = cfg.max_iters if cfg.has_max_iters else 5 * m
    te = max(1, cfg.trace_every)
    return mi // te + 2

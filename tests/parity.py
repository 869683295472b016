"""Parity helpers shared by the tests: bitwise and BASELINE.json tolerances."""
import numpy as np


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def same_bits(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


def first_diff(a, b):
    a, b = bits(a), bits(b)
    idx = np.nonzero(a != b)[0]
    return int(idx[0]) if len(idx) else -1


def trace_tuples(trace):
    """(iter, f, gbs, |P|, alpha) per record from either an oracle dict list or api records."""
    out = []
    for r in trace:
        if isinstance(r, dict):
            out.append((r["iter"], r["f"], r["grad_bar_sq"], r["passive_count"], r["alpha"]))
        else:
            out.append((r.iter, r.f, r.grad_bar_sq, r.passive_count, r.alpha))
    return out


def assert_trace_bitwise(gpu_trace, ref_trace):
    g, r = trace_tuples(gpu_trace), trace_tuples(ref_trace)
    assert len(g) == len(r), f"trace length {len(g)} != {len(r)}"
    for k, (a, b) in enumerate(zip(g, r)):
        assert a[0] == b[0] and a[3] == b[3], f"record {k}: iter/|P| {a} vs {b}"
        assert same_bits([a[1]], [b[1]]), f"record {k}: f {a[1]!r} vs {b[1]!r}"
        assert same_bits([a[2]], [b[2]]), f"record {k}: gbs {a[2]!r} vs {b[2]!r}"
        if a[4] is None or b[4] is None:
            assert a[4] is None and b[4] is None, f"record {k}: alpha presence"
        else:
            assert same_bits([a[4]], [b[4]]), f"record {k}: alpha {a[4]!r} vs {b[4]!r}"


def baseline_tolerances(x_gpu, x_ref, f_gpu, f_ref, it_gpu, it_ref):
    """The four BASELINE.json tolerances."""
    x_gpu = np.asarray(x_gpu)
    x_ref = np.asarray(x_ref)
    rel_f = abs(f_gpu - f_ref) / max(abs(f_ref), 1e-300)
    dx = float(np.max(np.abs(x_gpu - x_ref))) if len(x_ref) else 0.0
    xs = max(1.0, float(np.max(np.abs(x_ref))) if len(x_ref) else 1.0)
    big = np.maximum(np.abs(x_gpu), np.abs(x_ref)) > 1e-12
    flips = int(np.sum(((x_gpu > 0) != (x_ref > 0)) & big))
    return {
        "rel_objective": rel_f,
        "objective_ok": rel_f <= 1e-10,
        "dx_inf": dx,
        "x_ok": dx <= 1e-8 * xs,
        "support_flips": flips,
        "support_ok": flips == 0,
        "iter_diff": abs(int(it_gpu) - int(it_ref)),
        "iter_ok": abs(int(it_gpu) - int(it_ref)) <= 1,
    }

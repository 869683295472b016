"""ctypes loader for lib/libalnnls.so (the C ABI of include/alnnls.h).

No fallback: if the library or an sm_100 device is missing, calls raise.
"""
import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ALNNLS_LIB") or os.path.join(HERE, "lib", "libalnnls.so")

# every symbol include/alnnls.h declares (tests check the .so exports them all)
EXPORTS = [
    "alnnls_abi_version", "alnnls_config_default", "alnnls_create", "alnnls_destroy",
    "alnnls_last_error", "alnnls_device_info", "alnnls_solve_nnls", "alnnls_solve_nqp",
    "alnnls_solve_nnls_device", "alnnls_solve_nqp_device", "alnnls_get_x", "alnnls_get_inner_x",
    "alnnls_get_final_grad", "alnnls_get_trace", "alnnls_get_multiplies", "alnnls_get_phase_ns",
    "alnnls_get_scale",
    "alnnls_get_retained", "alnnls_get_dropped", "alnnls_setup", "alnnls_get_Q", "alnnls_get_q",
    "alnnls_rescale", "alnnls_gram", "alnnls_transpose_matvec", "alnnls_matvec",
    "alnnls_masked_matvec", "alnnls_solve_nnls_batched", "alnnls_solve_nnls_batched_device",
    "alnnls_timer_start", "alnnls_timer_stop", "alnnls_launch_count", "alnnls_last_loop_kernel",
    "alnnls_gram_tiles", "alnnls_gram_rowblock_device", "alnnls_atb_rowblock_device",
    "alnnls_solve_nnls_gram_device", "alnnls_residual_rowblock_device",
    "alnnls_gram_partial_device",
    "alnnls_solve_accelerated", "alnnls_solve_accelerated_device", "alnnls_solve_anti_accelerated",
    "alnnls_solve_anti_accelerated_device",
    "alnnls_pack_upper_device", "alnnls_unpack_upper_device", "alnnls_finish",
    "alnnls_solve_nnls_batched_multi", "alnnls_device_count", "alnnls_matmat_device",
    "alnnls_nmf_device", "alnnls_nmf",
]

_lib = None

vp = C.c_void_p
u64 = C.c_uint64
i32 = C.c_int


def load():
    """Loads the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: the CUDA extension was not built "
                           "(run __graft_entry__.build() or `make`); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    sig = {
        "alnnls_abi_version": ([], i32),
        "alnnls_config_default": ([C.POINTER(abi.Config)], None),
        "alnnls_create": ([C.POINTER(vp), i32], i32),
        "alnnls_destroy": ([vp], None),
        "alnnls_last_error": ([vp], C.c_char_p),
        "alnnls_device_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)], i32),
        "alnnls_solve_nnls": ([vp, u64, u64, vp, vp, C.POINTER(abi.Config),
                               C.POINTER(abi.Summary)], i32),
        "alnnls_solve_nqp": ([vp, u64, vp, vp, vp, C.POINTER(abi.Config),
                              C.POINTER(abi.Summary)], i32),
        "alnnls_solve_nnls_device": ([vp, u64, u64, vp, u64, vp, C.POINTER(abi.Config),
                                      C.POINTER(abi.Summary)], i32),
        "alnnls_solve_nqp_device": ([vp, u64, vp, u64, vp, vp, C.POINTER(abi.Config),
                                     C.POINTER(abi.Summary)], i32),
        "alnnls_get_x": ([vp, vp, u64], i32),
        "alnnls_get_inner_x": ([vp, vp, u64], i32),
        "alnnls_get_final_grad": ([vp, vp, u64], i32),
        "alnnls_get_trace": ([vp, vp, u64], i32),
        "alnnls_get_multiplies": ([vp, vp, u64], i32),
        "alnnls_get_phase_ns": ([vp, vp, u64], i32),
        "alnnls_timer_start": ([vp], i32),
        "alnnls_timer_stop": ([vp, C.POINTER(C.c_double)], i32),
        "alnnls_launch_count": ([vp], u64),
        "alnnls_last_loop_kernel": ([vp], i32),
        "alnnls_get_scale": ([vp, vp, u64], i32),
        "alnnls_get_retained": ([vp, vp, u64], i32),
        "alnnls_get_dropped": ([vp, vp, u64], i32),
        "alnnls_setup": ([vp, u64, u64, vp, vp, C.POINTER(abi.Summary)], i32),
        "alnnls_get_Q": ([vp, vp, u64], i32),
        "alnnls_get_q": ([vp, vp, u64], i32),
        "alnnls_rescale": ([vp, u64, vp, vp, C.POINTER(abi.Summary)], i32),
        "alnnls_gram": ([vp, u64, u64, vp, vp], i32),
        "alnnls_transpose_matvec": ([vp, u64, u64, vp, vp, vp], i32),
        "alnnls_matvec": ([vp, u64, u64, vp, vp, vp], i32),
        "alnnls_masked_matvec": ([vp, u64, u64, vp, vp, vp, u64, vp, C.POINTER(u64)], i32),
        "alnnls_solve_nnls_batched": ([vp, u64, u64, vp, u64, vp, C.POINTER(abi.Config), vp, vp,
                                       C.POINTER(abi.Summary)], i32),
        "alnnls_solve_nnls_batched_device": ([vp, u64, u64, vp, u64, vp, C.POINTER(abi.Config),
                                              vp, vp, C.POINTER(abi.Summary)], i32),
        "alnnls_gram_tiles": ([u64], u64),
        "alnnls_solve_accelerated": ([vp, u64, vp, vp, C.POINTER(abi.Config),
                                      C.POINTER(abi.Summary)], i32),
        "alnnls_solve_accelerated_device": ([vp, u64, vp, u64, vp, C.POINTER(abi.Config),
                                             C.POINTER(abi.Summary)], i32),
        "alnnls_solve_anti_accelerated": ([vp, u64, u64, vp, vp, C.POINTER(abi.Config),
                                           C.POINTER(abi.Summary)], i32),
        "alnnls_solve_anti_accelerated_device": ([vp, u64, u64, vp, u64, vp, C.POINTER(abi.Config),
                                                  C.POINTER(abi.Summary)], i32),
        "alnnls_gram_rowblock_device": ([vp, u64, u64, vp, u64, u64, u64, vp, vp, vp], i32),
        "alnnls_atb_rowblock_device": ([vp, u64, u64, vp, u64, vp, vp, vp], i32),
        "alnnls_solve_nnls_gram_device": ([vp, u64, vp, vp, C.POINTER(abi.Config),
                                           C.POINTER(abi.Summary)], i32),
        "alnnls_residual_rowblock_device": ([vp, u64, u64, vp, u64, vp, vp, C.c_double,
                                             C.POINTER(C.c_double)], i32),
        "alnnls_gram_partial_device": ([vp, u64, u64, vp, u64, vp, i32, vp, vp], i32),
        "alnnls_pack_upper_device": ([vp, u64, vp, vp], i32),
        "alnnls_unpack_upper_device": ([vp, u64, vp, vp], i32),
        "alnnls_finish": ([vp, u64, u64, vp, vp, vp, u64, vp, C.POINTER(C.c_double)], i32),
        "alnnls_solve_nnls_batched_multi": ([C.POINTER(vp), i32, u64, u64, vp, u64, vp,
                                             C.POINTER(abi.Config), vp, vp,
                                             C.POINTER(abi.Summary)], i32),
        "alnnls_device_count": ([], i32),
        "alnnls_matmat_device": ([vp, u64, u64, u64, vp, u64, vp, u64, vp, u64], i32),
        "alnnls_nmf_device": ([vp, u64, u64, u64, vp, vp, vp, u64, C.POINTER(abi.Config), vp], i32),
        "alnnls_nmf": ([vp, u64, u64, u64, vp, vp, vp, u64, C.POINTER(abi.Config), vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L

"""ctypes declarations of include/cpd.h (names identical to the C ABI)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcpd.so")
CPD_NCCL_ID_BYTES = 128
CPD_MAX_RANK = 1024
CPD_MAX_ORDER = 8

STATUS = {0: "CPD_OK", 1: "CPD_ERR_INVALID_ARG", 2: "CPD_ERR_STATE", 3: "CPD_ERR_NUMERIC",
          4: "CPD_ERR_CUDA", 5: "CPD_ERR_NCCL", 6: "CPD_ERR_OOM", 7: "CPD_ERR_INTERNAL"}

EXPORTED_SYMBOLS = [
    "cpd_opts_default", "cpd_nccl_unique_id", "cp_als_init", "msdt_sweep", "dt_sweep", "pp_init",
    "pp_approx_sweep", "fitness", "cpd_pp_condition", "cpd_get_factor", "cpd_get_last_mttkrp",
    "cpd_set_factors", "cpd_get_phase_ms", "cpd_get_counters", "cpd_reset_counters",
    "cpd_debug_get_pp_operator", "cpd_last_error", "cpd_destroy", "cpd_gen_tensor", "cpd_ttm", "cpd_ttm_i8", "cpd_ttm_engine", "cpd_set_tensor",
    "cpd_last_sweep_status",
    "cpd_mttv", "cpd_gen_tensor_block", "cpd_get_filler_counters", "cpd_get_memory", "cpd_get_ttm_bytes", "cpd_local_group_create", "cpd_local_group_destroy", "cpd_set_profile_level",
]


class CPDError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


class cpd_opts(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p), ("pp_eps", C.c_double),
                ("reuse_root_in_pp_init", C.c_int), ("profile_phases", C.c_int), ("local_group", C.c_void_p),
                ("ttm_impl", C.c_int), ("grid", C.c_int * CPD_MAX_ORDER),
                ("fused_rs", C.c_int), ("msdt_levels", C.c_int)]


_lib = None
_P = C.c_void_p
_D = C.POINTER(C.c_double)


def load_library():
    """Load libcpd.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CPDError(4, f"{LIB_PATH} not built (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    sig = {
        "cpd_opts_default": (C.c_int, [C.POINTER(cpd_opts)]),
        "cpd_nccl_unique_id": (C.c_int, [_P]),
        "cp_als_init": (C.c_int, [C.POINTER(_P), C.c_int, C.POINTER(C.c_int64), C.c_int, _P,
                                  C.POINTER(_D), C.POINTER(cpd_opts)]),
        "msdt_sweep": (C.c_int, [_P, _D]),
        "dt_sweep": (C.c_int, [_P, _D]),
        "pp_init": (C.c_int, [_P]),
        "pp_approx_sweep": (C.c_int, [_P, _D, C.POINTER(C.c_int)]),
        "fitness": (C.c_int, [_P, _D]),
        "cpd_pp_condition": (C.c_int, [_P, C.POINTER(C.c_int)]),
        "cpd_get_factor": (C.c_int, [_P, C.c_int, _D]),
        "cpd_get_last_mttkrp": (C.c_int, [_P, C.c_int, _D]),
        "cpd_set_factors": (C.c_int, [_P, C.POINTER(_D)]),
        "cpd_get_phase_ms": (C.c_int, [_P, _D]),
        "cpd_get_counters": (C.c_int, [_P, _D]),
        "cpd_reset_counters": (C.c_int, [_P]),
        "cpd_get_filler_counters": (C.c_int, [_P, _D]),
        "cpd_get_memory": (C.c_int, [_P, _D]),
        "cpd_get_ttm_bytes": (C.c_int, [_P, _D]),
        "cpd_set_profile_level": (C.c_int, [_P, C.c_int]),
        "cpd_debug_get_pp_operator": (C.c_int, [_P, C.c_int, C.c_int, _D]),
        "cpd_last_error": (C.c_char_p, [_P]),
        "cpd_destroy": (C.c_int, [_P]),
        "cpd_gen_tensor": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int64), C.c_int64, C.c_int64, C.c_int,
                                     C.POINTER(_D), C.c_int, C.c_double, C.c_uint64, _P]),
        "cpd_gen_tensor_block": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.c_int, C.POINTER(_D), C.c_int, C.c_double,
                                           C.c_uint64, _P]),
        "cpd_ttm": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, _P, C.c_int, _P, _P]),
        "cpd_ttm_engine": (C.c_int, [_P, C.POINTER(C.c_int)]),
        "cpd_last_sweep_status": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_double)]),
        "cpd_set_tensor": (C.c_int, [_P]),
        "cpd_ttm_i8": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, _P, C.c_int, _P, C.c_int, _P]),
        "cpd_mttv": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int, _P, _P, C.c_int, _P]),
        "cpd_local_group_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
        "cpd_local_group_destroy": (C.c_int, [_P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status, ctx=None):
    if status != 0:
        msg = load_library().cpd_last_error(ctx).decode(errors="replace")
        raise CPDError(status, msg)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def dptr_array(arrs):
    arr = (_D * len(arrs))()
    for i, a in enumerate(arrs):
        arr[i] = dptr(a)
    return arr


def cpd_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(CPD_NCCL_ID_BYTES)
    check(load_library().cpd_nccl_unique_id(buf))
    return buf.raw


def _stream_ptr(stream):
    if stream is None:
        return None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def cpd_gen_tensor(T, shape, lo, hi, kind, At, noise_std, seed, stream=None):
    """Fill the torch CUDA tensor T (slab [lo,hi) of the last mode) with the synth recipe."""
    shp = (C.c_int64 * len(shape))(*shape)
    At = [np.ascontiguousarray(a, dtype=np.float64) for a in At] if At is not None else None
    arr = dptr_array(At) if At else None
    Rt = At[0].shape[1] if At else 0
    check(load_library().cpd_gen_tensor(C.c_void_p(T.data_ptr()), len(shape), shp, lo, hi, kind, arr, Rt,
                                        float(noise_std), C.c_uint64(seed), _stream_ptr(stream)))


def cpd_gen_tensor_block(T, shape, lo, hi, kind, At, noise_std, seed, stream=None):
    """Fill the torch CUDA tensor T with the block [lo_n, hi_n) of the synthetic tensor."""
    n = len(shape)
    shp, l, h = (C.c_int64 * n)(*shape), (C.c_int64 * n)(*lo), (C.c_int64 * n)(*hi)
    At = [np.ascontiguousarray(a, dtype=np.float64) for a in At] if At is not None else None
    arr = dptr_array(At) if At else None
    Rt = At[0].shape[1] if At else 0
    check(load_library().cpd_gen_tensor_block(C.c_void_p(T.data_ptr()), n, shp, l, h, kind, arr, Rt,
                                              float(noise_std), C.c_uint64(seed), _stream_ptr(stream)))


def cpd_ttm(T, pre, K, post, A, R, out, stream=None):
    check(load_library().cpd_ttm(C.c_void_p(T.data_ptr()), pre, K, post, C.c_void_p(A.data_ptr()), R,
                                 C.c_void_p(out.data_ptr()), _stream_ptr(stream)))


def cpd_ttm_i8(T, pre, K, post, A, R, out, use_digits=True, stream=None):
    check(load_library().cpd_ttm_i8(C.c_void_p(T.data_ptr()), pre, K, post, C.c_void_p(A.data_ptr()), R,
                                    C.c_void_p(out.data_ptr()), int(bool(use_digits)), _stream_ptr(stream)))


def cpd_mttv(X, pre, K, post, R, v, out, beta=0, stream=None):
    check(load_library().cpd_mttv(C.c_void_p(X.data_ptr()), pre, K, post, R, C.c_void_p(v.data_ptr()),
                                  C.c_void_p(out.data_ptr()), beta, _stream_ptr(stream)))


def cpd_local_group_create(world):
    g = C.c_void_p()
    check(load_library().cpd_local_group_create(world, C.byref(g)))
    return g


def cpd_local_group_destroy(g):
    load_library().cpd_local_group_destroy(g)

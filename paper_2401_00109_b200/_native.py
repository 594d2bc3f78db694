"""ctypes binding of libjabba_b200.so (include/jabba_b200.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libjabba_b200.so")

i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")

# every symbol include/jabba_b200.h declares
EXPORTS = [
    "jb_config_default", "jb_abi_version", "jb_last_error", "jb_context_create",
    "jb_context_destroy", "jb_plan_segments", "jb_fit_transform", "jb_fit_free",
    "jb_fit_n_segments", "jb_fit_n_pieces", "jb_fit_k", "jb_fit_layout",
    "jb_fit_reconstruct_size", "jb_fit_copy_pieces", "jb_fit_copy_symbolic", "jb_fit_stats",
    "jb_fit_inverse_transform", "jb_reconstruct_size", "jb_inverse_transform",
    "jb_symbol_token", "jb_profile_enable", "jb_profile_reset", "jb_profile_read",
    "jb_probe_fp64_tflops", "jb_mt19937_64_stream", "jb_sample_indices",
    "jb_fit_transform_dist", "jb_symbolize_with", "jb_seq_sum_nonneg", "jb_kmeans", "jb_mse",
]

# int32_t (*allgather)(void* user, const void* send, uint64_t bytes, void* recv)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class JbComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32),
                ("allgather", ALLGATHER_FN)]


class JbConfig(C.Structure):
    _fields_ = [
        ("tol", C.c_double), ("max_piece_len", C.c_int64), ("backend", C.c_int32),
        ("scl", C.c_double), ("k", C.c_uint64), ("r", C.c_double),
        ("max_iters", C.c_uint64), ("n_init", C.c_uint64), ("seed", C.c_uint64),
        ("alpha", C.c_double), ("sort_key", C.c_int32), ("early_stop", C.c_int32),
        ("has_alpha_len", C.c_int32), ("alpha_len", C.c_double),
        ("has_alpha_inc", C.c_int32), ("alpha_inc", C.c_double), ("eta", C.c_double),
        ("threads", C.c_uint32),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load libjabba_b200.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (make -C paper_2401_00109_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.jb_last_error.restype = C.c_char_p
    L.jb_abi_version.restype = C.c_int
    L.jb_config_default.argtypes = [C.POINTER(JbConfig)]
    L.jb_context_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.jb_context_destroy.argtypes = [vp]
    L.jb_plan_segments.argtypes = [i64p, C.c_int64, C.c_int32, C.c_int64, i64p, i64p,
                                   C.POINTER(C.c_int64)]
    L.jb_fit_transform.argtypes = [vp, vp, C.c_int64, C.c_int32, i64p, i64p, C.c_int64,
                                   C.c_int32, C.POINTER(JbConfig), C.POINTER(vp)]
    L.jb_fit_free.argtypes = [vp]
    for f in ("jb_fit_n_segments", "jb_fit_n_pieces", "jb_fit_reconstruct_size"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = C.c_int64
    L.jb_fit_k.argtypes = [vp]
    L.jb_fit_k.restype = C.c_uint64
    L.jb_fit_layout.argtypes = [vp]
    L.jb_fit_layout.restype = C.c_int32
    L.jb_fit_copy_pieces.argtypes = [vp, vp, vp, vp]
    L.jb_fit_copy_symbolic.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.jb_fit_stats.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                               C.POINTER(C.c_int32), vp]
    L.jb_fit_inverse_transform.argtypes = [vp, vp, vp, C.c_int32, vp]
    L.jb_reconstruct_size.argtypes = [i64p, C.c_int64, C.c_int32]
    L.jb_reconstruct_size.restype = C.c_int64
    L.jb_inverse_transform.argtypes = [vp, f64p, f64p, C.c_uint64, f64p, u32p, i64p, f64p, i64p,
                                       C.c_int64, C.c_int32, vp]
    L.jb_symbolize_with.argtypes = [vp, f64p, C.c_uint64, f64p, vp, vp, C.c_int64, C.c_int32,
                                    vp]
    L.jb_symbolize_with.restype = C.c_int
    L.jb_symbol_token.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p]
    L.jb_symbol_token.restype = C.c_int32
    L.jb_profile_enable.argtypes = [C.c_int32]
    L.jb_profile_read.argtypes = [C.c_char_p, vp, vp, C.c_int32]
    L.jb_profile_read.restype = C.c_int32
    L.jb_mt19937_64_stream.argtypes = [vp, C.c_uint64, C.c_uint64, vp]
    L.jb_mt19937_64_stream.restype = C.c_int
    L.jb_sample_indices.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, vp]
    L.jb_sample_indices.restype = C.c_int
    L.jb_seq_sum_nonneg.argtypes = [vp, vp, vp, C.c_int64, vp]
    L.jb_seq_sum_nonneg.restype = C.c_int
    L.jb_kmeans.argtypes = [vp, vp, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp,
                            vp, C.POINTER(C.c_uint64)]
    L.jb_kmeans.restype = C.c_int
    L.jb_mse.argtypes = [vp, vp, vp, C.c_int64, C.c_int32, C.POINTER(C.c_double)]
    L.jb_mse.restype = C.c_int
    L.jb_fit_transform_dist.argtypes = [vp, C.POINTER(JbComm), vp, C.c_int64, C.c_int32, i64p,
                                        i64p, C.c_int64, C.c_int64, C.c_int32,
                                        C.POINTER(JbConfig), C.POINTER(vp)]
    L.jb_fit_transform_dist.restype = C.c_int
    L.jb_probe_fp64_tflops.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.jb_probe_fp64_tflops.restype = C.c_int
    for name in ("jb_fit_transform", "jb_plan_segments", "jb_context_create",
                 "jb_fit_copy_pieces", "jb_fit_copy_symbolic", "jb_fit_stats",
                 "jb_fit_inverse_transform", "jb_inverse_transform"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def last_error() -> str:
    return lib().jb_last_error().decode(errors="replace")


def profile_enable(on: bool = True):
    lib().jb_profile_enable(1 if on else 0)


def profile_reset():
    lib().jb_profile_reset()


def profile_read() -> dict:
    """{kernel name: (total_ms, launches)} accumulated since the last reset."""
    cap = 64
    names = C.create_string_buffer(64 * cap)
    ms = np.zeros(cap, np.float64)
    cnt = np.zeros(cap, np.int64)
    n = lib().jb_profile_read(names, ms.ctypes.data, cnt.ctypes.data, cap)
    out = {}
    raw = names.raw
    for i in range(min(n, cap)):
        nm = raw[64 * i: 64 * i + 64].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out

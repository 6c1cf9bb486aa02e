"""ctypes binding of libsqr.so (the C ABI in include/sqr.h).

This is the reference-facing plumbing: every entry takes raw device pointers
(ints), sizes and a CUDA stream handle.  The library must be built in-tree
(``python -m paper_2008_04447_b200.build`` or ``__graft_entry__.build()``);
there is no fallback of any kind when it is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SQR_LIB selects an alternative in-tree build (kernel-variant experiments).
LIB_PATH = os.path.join(HERE, os.environ.get("SQR_LIB", "libsqr.so"))

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_ptr = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/sqr.h one to one.
SIGNATURES = {
    "sqr_version": (ctypes.c_char_p, []),
    "sqr_last_error": (ctypes.c_char_p, []),
    "sqr_device_sm_count": (c_int, []),
    "sqr_launch_count": (c_i64, []),
    "sqr_profile_enable": (c_int, [c_i64]),
    "sqr_profile_collect": (c_int, [c_ptr, c_ptr, c_int]),
    "sqr_profile_flops": (c_int, [c_ptr, c_int]),
    "sqr_profile_select": (c_int, [ctypes.c_uint32]),
    "sqr_debug_trace": (c_int, [c_ptr]),
    "sqr_gaussian": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_u64, c_u64, c_int, c_ptr]),
    "sqr_gemm_tn": (c_int, [c_i64, c_i64, c_i64, c_dbl, c_ptr, c_i64, c_ptr, c_i64, c_dbl, c_ptr, c_i64,
                            c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "sqr_gemm_nn": (c_int, [c_i64, c_i64, c_i64, c_dbl, c_ptr, c_i64, c_ptr, c_i64, c_dbl, c_ptr, c_i64,
                            c_ptr, c_i64, c_ptr]),
    "sqr_gemm_nn_ws": (c_int, [c_i64, c_i64, c_i64, c_dbl, c_ptr, c_i64, c_ptr, c_i64, c_dbl, c_ptr, c_i64,
                               c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "sqr_sample_qrcp": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_int,
                                c_ptr, c_ptr]),
    "sqr_sample_qrcp_workspace": (c_i64, [c_i64, c_i64]),
    "sqr_sample_qrcp_ws": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_int,
                                   c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_sample_qrcp_ws_sig": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_int,
                                       c_ptr, c_ptr, c_i64, c_ptr, ctypes.c_uint32, c_ptr]),
    "sqr_wait_resident": (c_int, [c_ptr, ctypes.c_uint32, c_int, c_ptr]),
    "sqr_apply_moves": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_panel_qr": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_int, c_ptr,
                             c_ptr]),
    "sqr_build_t": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "sqr_sample_update": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr]),
    "sqr_sample_update_prep": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr]),
    "sqr_sample_update_apply": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr,
                                        c_ptr]),
    "sqr_sample_update_b": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr,
                                    c_ptr]),
    "sqr_rqrcp_workspace": (c_i64, [c_i64, c_i64, c_i64, c_i64, c_i64]),
    "sqr_rqrcp": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_u64, c_ptr, c_i64, c_int, c_ptr,
                          c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_rqrcp_stream_r_workspace": (c_i64, [c_i64] * 5),
    "sqr_rqrcp_stream_r": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_u64, c_ptr, c_i64, c_int,
                                   c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "sqr_trqrcp_workspace": (c_i64, [c_i64, c_i64, c_i64, c_i64, c_i64]),
    "sqr_trqrcp": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_u64, c_ptr, c_i64, c_ptr, c_i64,
                           c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_qr_blocked_workspace": (c_i64, [c_i64, c_i64, c_i64, c_i64]),
    "sqr_qr_blocked": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_apply_wy": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_i64, c_int, c_ptr, c_i64,
                             c_ptr]),
    "sqr_block_workspace": (c_i64, [c_i64, c_i64, c_i64]),
    "sqr_copy_check": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr]),
    "sqr_copy_check_t": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr]),
    "sqr_copy_columns": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "sqr_panel_factor": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_int, c_ptr, c_ptr, c_i64,
                                 c_ptr]),
    "sqr_apply_block_update": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr,
                                       c_i64, c_ptr]),
    "sqr_transpose": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_int, c_ptr]),
    "sqr_unpack_reflectors": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "sqr_gather_rows": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_scatter_rows": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_ptr]),
    "sqr_peer_put": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_int, c_ptr, c_int, c_u64, c_ptr, c_ptr]),
    "sqr_peer_put_columns": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_int, c_ptr, c_int, c_u64,
                                     c_ptr, c_ptr]),
    "sqr_peer_wait": (c_int, [c_ptr, c_int, c_u64, c_ptr]),
    "sqr_trsm_right_upper": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_int, c_ptr]),
    "sqr_jacobi_svd": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_int, c_ptr, c_ptr]),
}

# struct sqr_status (include/sqr.h)
STATUS_DTYPE = np.dtype([
    ("stop", np.int32), ("reason", np.int32), ("achieved", np.int32), ("nblocks", np.int32),
    ("sample_achieved", np.int32), ("bhat", np.int32), ("nmoves", np.int32), ("pad_", np.int32),
    ("floor_sq", np.float64), ("aux", np.float64, (4,)),
])
STATUS_BYTES = STATUS_DTYPE.itemsize

STOP_REASONS = {0: "none", 1: "k_reached", 2: "sample_floor", 3: "sample_rank", 4: "panel_zero",
                5: "short_block", 6: "no_trailing", 7: "r11_singular"}

_lib = None


class LibraryMissing(ImportError):
    pass


def lib():
    """The loaded libsqr (raises loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2008_04447_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(SIGNATURES)


def check(rc: int, what: str = "libsqr") -> None:
    if rc != 0:
        msg = lib().sqr_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")


PROFILE_TAGS = ["gemm_tn", "gemm_nn", "sample_qrcp", "panel", "build_t", "apply_moves", "sample_update",
                "gaussian", "misc", "gemm_nn_beside_chain"]


def profile_collect():
    """{class: (ms, launches)} since sqr_profile_enable."""
    ms = (ctypes.c_double * 16)()
    cnt = (ctypes.c_int64 * 16)()
    lib().sqr_profile_collect(ms, cnt, 16)
    return {t: (ms[i], cnt[i]) for i, t in enumerate(PROFILE_TAGS)}


def profile_flops():
    """{class: flops} the drivers attributed since sqr_profile_enable (call before profile_collect resets)."""
    fl = (ctypes.c_double * 16)()
    lib().sqr_profile_flops(fl, 16)
    return {t: fl[i] for i, t in enumerate(PROFILE_TAGS)}

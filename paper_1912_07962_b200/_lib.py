"""ctypes binding of the C-ABI in ``include/slimb200.h``.

The product path has no CPU fallback: if ``libslimb200.so`` is missing the
import of :func:`lib` raises, and every solver call fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SLIM_LIB: an alternate in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("SLIM_LIB") or os.path.join(_HERE, "libslimb200.so")

SLIM_OK, SLIM_EINVAL, SLIM_ERANGE, SLIM_ENOTSPD = 0, 1, 2, 3
SLIM_ECUDA, SLIM_ENCCL, SLIM_ESTATE, SLIM_ENOMEM = 4, 5, 6, 7
SLIM_F64, SLIM_F32 = 0, 1
SLIM_DENSE_ROWMAJOR, SLIM_CSR_PERBLOCK, SLIM_GEN_SPLITMIX64 = 0, 1, 2
SLIM_HIST_FIXED = 5
SLIM_METHOD_SLIMLS, SLIM_METHOD_SG = 0, 1
SLIM_FLAG_FP64_FACTOR = 1

# every symbol include/slimb200.h declares (checked by tests/test_capi_exports.py)
EXPORTS = (
    "slim_create", "slim_destroy", "slim_last_error", "slim_abi_version",
    "slim_upload_dense", "slim_upload_csr_block", "slim_upload_csr_blocks", "slim_upload_csr", "slim_finalize_operator",
    "slim_set_rhs", "slim_gen_apply", "slim_set_x", "slim_get_x", "slim_set_references",
    "slim_set_divergence_limit", "slim_run", "slim_set_host_streaming", "slim_attach_stream_file", "slim_nccl_unique_id", "slim_comm_init",
    "slim_local_group_create", "slim_local_group_destroy", "slim_comm_init_local", "slim_set_factor_round_robin", "slim_set_method",
    "slim_dual_step", "slim_potrf", "slim_potrf_traced", "slim_block_residual", "slim_timing", "slim_set_profiling", "slim_set_timing_start", "slim_probe_stream",
    "slim_siddon2d_view", "slim_siddon3d_view",
    "slim_build_projector", "slim_apply", "slim_get_csr_block", "slim_nnz",
)


class SlimDesc(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int64), ("n_cols", C.c_int64), ("block_rows", C.c_int64),
        ("memory_r", C.c_int64), ("value_dtype", C.c_int32), ("layout", C.c_int32),
        ("device", C.c_int32), ("flags", C.c_int32), ("gen_seed", C.c_uint64),
        ("gen_n_total", C.c_int64), ("col_offset", C.c_int64),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double
_DP = C.POINTER(C.c_double)
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)

_SIGS = {
    "slim_create": (C.c_int, [C.POINTER(_P), C.POINTER(SlimDesc)]),
    "slim_destroy": (None, [_P]),
    "slim_last_error": (C.c_char_p, [_P]),
    "slim_abi_version": (C.c_int, []),
    "slim_upload_dense": (C.c_int, [_P, _P, _DP]),
    "slim_upload_csr_block": (C.c_int, [_P, _I64, _I64P, _I32P, _P, _DP]),
    "slim_upload_csr_blocks": (C.c_int, [_P, _I64, C.c_void_p, C.c_void_p, C.c_void_p, _DP]),
    "slim_upload_csr": (C.c_int, [_P, _I64P, _I32P, _P, _DP]),
    "slim_finalize_operator": (C.c_int, [_P]),
    "slim_set_rhs": (C.c_int, [_P, _DP]),
    "slim_gen_apply": (C.c_int, [_P, _DP, _DP]),
    "slim_set_x": (C.c_int, [_P, _DP]),
    "slim_get_x": (C.c_int, [_P, _DP]),
    "slim_set_references": (C.c_int, [_P, _I32, C.POINTER(_DP)]),
    "slim_set_divergence_limit": (C.c_int, [_P, _D]),
    "slim_run": (C.c_int, [_P, _I64P, _DP, _I64, _I64, _DP, _I64P, _I32P, _I64P, _DP]),
    "slim_set_host_streaming": (C.c_int, [_P, _I32]),
    "slim_attach_stream_file": (C.c_int, [_P, C.c_char_p]),
    "slim_comm_init": (C.c_int, [_P, _P, _I32, _I32]),
    "slim_nccl_unique_id": (C.c_int, [_P]),
    "slim_local_group_create": (C.c_void_p, [_I32]),
    "slim_local_group_destroy": (None, [_P]),
    "slim_comm_init_local": (C.c_int, [_P, _P, _I32]),
    "slim_dual_step": (C.c_int, [_I32, _DP, _I64, _I64, _DP, _I64, _D, _DP]),
    "slim_potrf": (C.c_int, [_I32, _DP, _I64, _DP]),
    "slim_potrf_traced": (C.c_int, [_I32, _DP, _I64, _DP, C.POINTER(C.c_uint64), _DP]),
    "slim_block_residual": (C.c_int, [_P, _I64, _DP, _DP, _DP]),
    "slim_timing": (C.c_int, [_P, _I32, _DP, _I64P]),
    "slim_set_profiling": (C.c_int, [_P, _I32]),
    "slim_set_timing_start": (C.c_int, [_P, _I64]),
    "slim_probe_stream": (C.c_int, [_P, _I32, _I32, _DP, _DP]),
    "slim_siddon2d_view": (C.c_int, [_D, _I64, _I64, _D, _I64P, _I32P, _DP]),
    "slim_siddon3d_view": (C.c_int, [_DP, _I64, _I64, _D, _I64P, _I32P, _DP]),
    "slim_build_projector": (C.c_int, [_P, _I32, _I64, _I64, _I64, _DP, _D, _I32P]),
    "slim_apply": (C.c_int, [_P, _DP, _DP]),
    "slim_nnz": (C.c_int, [_P, _I64P]),
    "slim_set_factor_round_robin": (C.c_int, [_P, _I32]),
    "slim_set_method": (C.c_int, [_P, _I32]),
    "slim_get_csr_block": (C.c_int, [_P, _I64, _I64P, _I32P, C.c_void_p]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load ``libslimb200.so`` (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1912_07962_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


class LinAlgError(np.linalg.LinAlgError):
    pass


def check(rc: int, ctx=None):
    """Map a C status code onto the reference's exception types."""
    if rc == SLIM_OK:
        return
    msg = lib().slim_last_error(ctx)
    msg = msg.decode() if msg else f"status {rc}"
    if rc == SLIM_EINVAL:
        raise ValueError(msg)
    if rc == SLIM_ERANGE:
        raise IndexError(msg)
    if rc == SLIM_ENOTSPD:
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_I32P)


def vptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)

"""ctypes binding of libjtb200.so (the C ABI in include/jt_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device is
usable, every entry point raises `DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import (
    DeviceError,
    InconsistentDivisionError,
    UnknownVariableError,
    ZeroMassError,
)

LIB_NAME = "libjtb200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

JT_OK, JT_ERR_BAD_ARG, JT_ERR_INCONSISTENT_DIVISION, JT_ERR_ZERO_MASS, JT_ERR_CUDA, JT_ERR_OOM, \
    JT_ERR_UNSUPPORTED = range(7)
JT_F32, JT_F64 = 0, 1
JT_MATERIALIZED, JT_SHARED_BASE = 0, 1

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p

# name -> (restype, argtypes); mirrors include/jt_b200.h one to one
SIGNATURES = {
    "jt_plan_create": (C.c_int, [C.c_int, _i32p, C.c_int, _i32p, _i32p, C.c_int, _i32p, _i32p, _i32p,
                                 C.c_int, _i32p, C.c_int, C.c_int, C.POINTER(_vp)]),
    "jt_plan_destroy": (None, [_vp]),
    "jt_plan_mapping_table": (C.c_int, [_vp, C.c_int, C.c_int, _i64p]),
    "jt_state_create": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "jt_state_destroy": (None, [_vp]),
    "jt_state_device_bytes": (C.c_int64, [_vp]),
    "jt_state_load": (C.c_int, [_vp, C.c_int, _f64p, _f64p]),
    "jt_state_store": (C.c_int, [_vp, C.c_int, _f64p, _f64p]),
    "jt_apply_evidence": (C.c_int, [_vp, C.c_int, _i32p, _i32p, _i32p, _i32p, _vp]),
    "jt_apply_evidence_device": (C.c_int, [_vp, C.c_int, _vp, C.c_int, _i32p, _i32p, _vp]),
    "jt_clear_evidence": (C.c_int, [_vp]),
    "jt_state_reset": (C.c_int, [_vp, _vp]),
    "jt_state_initialize": (C.c_int, [_vp, C.c_int, _i32p, _i32p, _i32p, _f64p]),
    "jt_message": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp]),
    "jt_propagate": (C.c_int, [_vp, _i32p, _vp]),
    "jt_query": (C.c_int, [_vp, C.c_int, _i32p, _i32p, C.c_int, _f64p, _vp]),
    "jt_query_device": (C.c_int, [_vp, C.c_int, _i32p, _i32p, C.c_int, _vp, _vp]),
    "jt_propagate_query": (C.c_int, [_vp, C.c_int, _i32p, C.c_int, _vp, _vp]),
    "jt_sync_error": (C.c_int, [_vp]),
    "jt_error_case": (C.c_int, [_vp]),
    "jt_state_clone": (C.c_int, [_vp, C.POINTER(_vp)]),
    "jt_error_string": (C.c_char_p, [C.c_int]),
    "jt_state_launch_count": (C.c_int64, [_vp]),
    "jt_run_message_mu": (C.c_int, [_f64p, C.c_int64, _f64p, C.c_int64, _f64p, C.c_int64, _vp, C.c_int64,
                                    _vp, C.c_int64, C.c_int, C.c_int]),
    "jt_debug_plan": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int64]),
    "jt_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str | None = None):
    """Load and type the shared library; raises DeviceError when it is absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or os.environ.get("JT_LIB") or LIB_PATH  # JT_LIB: kernel-variant sweeps (tools/)
        if not os.path.exists(p):
            raise DeviceError(
                f"{LIB_NAME} not built ({p}); run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib():
    return load_library()


def check(rc: int, what: str = ""):
    if rc == JT_OK:
        return
    msg = lib().jt_error_string(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == JT_ERR_INCONSISTENT_DIVISION:
        raise InconsistentDivisionError(msg)
    if rc == JT_ERR_ZERO_MASS:
        raise ZeroMassError(msg)
    if rc == JT_ERR_BAD_ARG:
        raise ValueError(msg)
    if rc == JT_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(msg)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def require_device():
    """The product path runs on a CUDA device only."""
    try:
        import torch  # plumbing: device discovery and streams
    except Exception as exc:  # pragma: no cover
        raise DeviceError(f"torch unavailable: {exc}") from exc
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
    load_library()


__all__ = ["lib", "load_library", "check", "require_device", "SIGNATURES", "UnknownVariableError"]

"""ctypes binding of libvegas_b200.so (the C ABI in include/vegas_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every entry point raises NativeLibraryError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import (ContractViolationError, NativeLibraryError, NonFiniteIntegrandError,
                     VegasError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VPB_LIB_PATH") or os.path.join(HERE, "_lib", "libvegas_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "vegas_b200.h")

VPB_OK = 0
VPB_ERR_CUDA = 1
VPB_ERR_INVALID = 2
VPB_ERR_NONFINITE = 3
VPB_ERR_ASSERT = 4
VPB_ERR_NCCL = 5
VPB_ERR_UNSUPPORTED = 6
ABI_VERSION = 3
VPB_FLAG_DETERMINISTIC = 1
MAX_PARAMS = 64
MAX_DIMS = 64


class VpbDesc(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int32),
        ("n_intervals", ctypes.c_int32),
        ("n_strat", ctypes.c_int64),
        ("n_eval", ctypes.c_int64),
        ("batch_size", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("integrand", ctypes.c_int32),
        ("n_params", ctypes.c_int32),
        ("params", ctypes.POINTER(ctypes.c_double)),
        ("bounds", ctypes.POINTER(ctypes.c_double)),
        ("device", ctypes.c_int32),
        ("max_it", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("flags", ctypes.c_int32),
    ]


_c = ctypes
_P = ctypes.c_void_p
_I32, _I64, _U64, _F64 = _c.c_int32, _c.c_int64, _c.c_uint64, _c.c_double

# vpb_allreduce_fn (vegas_b200.h): int fn(void *user, void *buf, int64_t count,
# int32_t dtype, int32_t op) -- the host exchange callback
ALLREDUCE_FN = _c.CFUNCTYPE(_c.c_int, _P, _P, _I64, _I32, _I32)
VPB_DT_F64, VPB_DT_I64 = 0, 1
VPB_OP_SUM, VPB_OP_MAX = 0, 1

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES = {
    "vpb_abi_version": [],
    "vpb_last_error": [],
    "vpb_is_specialised": [_I32, _I32],
    "vpb_device_count": [_c.POINTER(_I32)],
    "vpb_create": [_c.POINTER(VpbDesc), _c.POINTER(_P)],
    "vpb_destroy": [_P],
    "vpb_nccl_unique_id": [_c.c_char_p],
    "vpb_attach_nccl": [_P, _c.c_char_p, _I32, _I32],
    "vpb_set_shard": [_P, _I32, _I32],
    "vpb_attach_exchange": [_P, _I32, _I32, ALLREDUCE_FN, _P],
    "vpb_reset": [_P],
    "vpb_iterate": [_P, _I32],
    "vpb_history": [_P, _I32, _P, _P, _P, _c.POINTER(_I32)],
    "vpb_error_info": [_P, _c.POINTER(_I64), _P, _c.POINTER(_F64)],
    "vpb_phase_times": [_P, _c.POINTER(_F64), _c.POINTER(_F64), _c.POINTER(_F64)],
    "vpb_last_fill_ms": [_P, _c.POINTER(_F64)],
    "vpb_sync": [_P],
    "vpb_timing": [_P, _I32, _I32, _c.POINTER(_F64), _c.POINTER(_F64)],
    "vpb_fp64_peak": [_I32, _c.POINTER(_F64)],
    "vpb_fill_layout": [_P, _c.POINTER(_I32), _c.POINTER(_I32), _c.POINTER(_I32)],
    "vpb_fx_stats": [_P, _P],
    "vpb_set_edges": [_P, _P],
    "vpb_get_edges": [_P, _P],
    "vpb_set_allocation": [_P, _P],
    "vpb_get_plan": [_P, _P, _P],
    "vpb_get_spread": [_P, _P],
    "vpb_get_fill": [_P, _P, _P, _P, _P, _P],
    "vpb_get_run_base": [_P, _c.POINTER(_I64)],
    "vpb_set_run_base": [_P, _I64],
    "vpb_iteration_host": [_P, _P, _P, _c.POINTER(_F64), _c.POINTER(_F64), _c.POINTER(_I64)],
    "vpb_fill": [_P, _I64],
    "vpb_philox_host": [_P, _P, _P, _I64, _P],
    "vpb_uniform_at_host": [_P, _P, _P, _I64, _P],
    "vpb_sample_runs_host": [_U64, _I64, _I64, _I64, _I64, _P, _I64, _P, _I32, _I32, _I64,
                             _P, _P, _P, _P],
    "vpb_eval_host": [_I32, _P, _I32, _P, _I64, _I32, _P],
    "vpb_fill_host": [_P, _I64, _P, _I32, _I32, _I64, _U64, _I64, _I64, _I32, _P, _I32, _I64,
                      _I64, _P, _P, _P, _P, _P, _c.POINTER(_I64), _P, _c.POINTER(_F64)],
    "vpb_pairwise_sum_host": [_P, _I64, _c.POINTER(_F64)],
    "vpb_pow_host": [_P, _I64, _F64, _P],
    "vpb_update_evals_host": [_P, _I64, _F64, _I64, _P],
    "vpb_build_plan_host": [_P, _I64, _P],
    "vpb_compute_results_host": [_P, _P, _P, _I64, _c.POINTER(_F64), _c.POINTER(_F64), _P],
    "vpb_smooth_and_damp_host": [_P, _P, _I32, _I32, _F64, _P],
    "vpb_update_grid_host": [_P, _P, _I32, _I32, _P],
}
_RESTYPES = {"vpb_last_error": ctypes.c_char_p}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return LIB_PATH


def load():
    """Load the CUDA library (once).  Raises NativeLibraryError if missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2408_09229_b200.build` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        if lib.vpb_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libvegas_b200.so ABI version mismatch; rebuild")
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().vpb_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = ""):
    """Map a status code to the reference's exception types."""
    if rc == VPB_OK:
        return
    msg = last_error()
    where = f"{what}: " if what else ""
    if rc == VPB_ERR_INVALID:
        raise ContractViolationError(where + msg)
    if rc == VPB_ERR_ASSERT:
        raise AssertionError(where + msg)
    if rc == VPB_ERR_NONFINITE:
        raise NonFiniteIntegrandError([], float("nan"), None)
    if rc == VPB_ERR_UNSUPPORTED:
        raise VegasError(where + msg)
    raise NativeLibraryError(where + f"status {rc}: {msg}")


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)

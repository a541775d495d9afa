"""ctypes binding of ``libnfft45.so`` (the C ABI declared in ``include/nfft45.h``).

There is no CPU fallback: importing the product API without the built
library, or calling it without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NFFT45_LIB", os.path.join(_HERE, "lib", "libnfft45.so"))

_c_double_p = ctypes.c_void_p  # device/host pointers are passed as raw addresses
_i64 = ctypes.c_int64

# signature table: name -> (restype, argtypes)
_SIGS = {
    "nfft45_last_error": (ctypes.c_char_p, []),
    "nfft45_version": (ctypes.c_int, []),
    "nfft45_launch_count": (_i64, []),
    "nfft45_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "nfft45_profile_read": (ctypes.c_int, [ctypes.c_char_p, _i64]),
    "nfft45_validate_grid": (ctypes.c_int, [ctypes.c_void_p, _i64, ctypes.c_double, ctypes.c_void_p]),
    "nfft45_grid_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "nfft45_grid_destroy": (None, [ctypes.c_void_p]),
    "nfft45_grid_size": (_i64, [ctypes.c_void_p]),
    "nfft45_type1": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_type2": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_nonuniform_conv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_void_p, _i64,
                                              _i64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_type1_direct": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "nfft45_type2_direct": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "nfft45_dft": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_int, ctypes.c_void_p]),
    "nfft45_v_samples": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_v_samples_terms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, _i64, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_kernel_samples": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_kernel_coefficients": (ctypes.c_int, [ctypes.c_void_p, _i64, ctypes.c_double, ctypes.c_void_p,
                                                  ctypes.c_void_p]),
    "nfft45_derivative_coefficients": (ctypes.c_int, [ctypes.c_void_p, _i64, ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_min_abs": (ctypes.c_int, [ctypes.c_void_p, _i64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
    "nfft45_derivative_samples": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                                 ctypes.c_void_p]),
    "nfft45_plan_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "nfft45_plan_create_terms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, _i64, ctypes.c_int,
                                                ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "nfft45_plan_destroy": (None, [ctypes.c_void_p]),
    "nfft45_plan_table": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_type5": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_type4": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_void_p, ctypes.c_void_p]),
    "nfft45_refine_type5": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "nfft45_refine_type4": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "nfft45_solve_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _i64,
                                         ctypes.c_void_p, _i64, ctypes.c_int, ctypes.c_void_p]),
    "nfft45_solve_host_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _i64,
                                            ctypes.c_void_p, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "nfft45_ge_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_void_p, ctypes.c_double,
                                       ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
    "nfft45_cg_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, _i64, ctypes.c_double, _i64,
                                       ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_STATUS_TO_ERROR = {
    1: errors.OutOfRangeError,
    2: errors.DuplicateNodeError,
    3: errors.NonPositiveDampingError,
    4: errors.LengthMismatchError,
    5: errors.SizeMismatchError,
    6: errors.KernelOverflowError,
    7: errors.SingularDerivativeError,
    8: errors.NonConvergenceError,
    9: ValueError,
    10: errors.DeviceError,
    11: errors.DeviceError,
    12: errors.SingularMatrixError,
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes handle; raises if the build is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libnfft45.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (or `make -C paper_1604_06236_b200`). "
                    "There is no CPU fallback."
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int):
    """Raise the reference's exception class for a non-zero C status."""
    if status == 0:
        return
    msg = load().nfft45_last_error().decode("utf-8", "replace")
    raise _STATUS_TO_ERROR.get(status, errors.DeviceError)(msg)


def call(name: str, *args):
    status = getattr(_lib or load(), name)(*args)
    if status:
        check(status)


def profile_enable(on: bool):
    load().nfft45_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel name: (launches, total_ms)} recorded since profiling was enabled."""
    lib = load()
    buf = ctypes.create_string_buffer(1 << 20)
    lib.nfft45_profile_read(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.rsplit(" ", 2)
        out[name] = (int(cnt), float(ms))
    return out

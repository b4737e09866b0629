"""ctypes binding of ``libbcnrand_b200.so`` (the C ABI in include/bcnrand_b200.h).

The library is the product: every generating call runs the sm_100a kernels.
There is no Python or CPU fallback — if the library is missing the import of
any generating function raises, and with no CUDA device every generating call
fails with :class:`CudaError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbcnrand_b200.so")

_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_int = ctypes.c_int
_vp = ctypes.c_void_p
_pu64 = ctypes.POINTER(ctypes.c_uint64)

# (name, restype, argtypes) for every symbol declared in include/bcnrand_b200.h
SIGNATURES = [
    ("bcn_abi_version", _int, []),
    ("bcn_last_error", ctypes.c_char_p, []),
    ("bcn_engine_name", ctypes.c_char_p, [_int]),
    ("bcn_device_count", _int, []),
    ("bcn_l2_bytes", _u64, [_int]),
    ("bcn_auto_engine", _int, [_int]),
    ("bcn_launch_count", _u64, []),
    ("bcn_set_launch_config", _int, [_int, _int]),
    ("bcn_set_write_pacing", _int, [ctypes.c_double, _int, _int]),
    ("bcn_get_write_pacing", None, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_int),
                                    ctypes.POINTER(_int)]),
    ("bcn_write_pacing", ctypes.c_double, []),
    ("bcn_device_write_pacing", _int, [_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_int)]),
    ("bcn_pace_calibration", _int, [_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                    _int, ctypes.POINTER(_int)]),
    ("bcn_modpow2", _int, [_u64, _u64, _pu64]),
    ("bcn_seed_from_index", _int, [_u64, _pu64]),
    ("bcn_state_at", _int, [_u64, _u64, _pu64]),
    ("bcn_next", _int, [_pu64]),
    ("bcn_to_unit_interval", _int, [_u64, ctypes.POINTER(ctypes.c_double)]),
    ("bcn_make_plan", _int, [_u64, _u32, ctypes.POINTER(_u32), _pu64]),
    ("bcn_physical_index", _int, [_u64, _u32, _int, _u32, _u64, _pu64]),
    ("bcn_fill", _int, [_vp, _u64, _u64, _int, _u32, _int, _u64, _int, _u64, _int, _int, _vp]),
    ("bcn_fill_multi", _int, [ctypes.POINTER(_vp), _pu64, ctypes.POINTER(_int), _int, _u64, _int, _u64,
                              _u64, _int, ctypes.POINTER(_vp)]),
    ("bcn_deinterleave", _int, [_vp, _vp, _u64, _u32, _u32, _int, _vp]),
    ("bcn_seed_states", _int, [_vp, _vp, _vp, _u64, _u32, _int, _vp]),
    ("bcn_digest", _int, [_vp, _u64, _u32, _u64, _pu64, _int, _vp]),
    ("bcn_fill_constant", _int, [_vp, _u64, _u64, _int, _vp]),
    ("bcn_fill_noise", _int, [_vp, _u64, _u64, _int, _vp]),
    ("bcn_engine_check", _int, [_int, _vp, _vp, _vp, _u64, _u32, _int]),
    ("bcn_bench_fill", _int, [_u64, ctypes.c_uint32, _int, _u64, _int, _int, _int, _int,
                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    ("bcn_format_text", _int, [_vp, _u64, _vp, _u64, _pu64]),
    ("bcn_chi_square_uniformity", _int, [_vp, _u64, _int, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(_int), ctypes.POINTER(_int), _int, _vp]),
    ("bcn_monobit_mantissa", _int, [_vp, _u64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_int),
                                    ctypes.POINTER(_int), _int, _vp]),
    ("bcn_serial_correlation", _int, [_vp, _u64, _int, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(_int), _int, _vp]),
]

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the product library; raise loudly if missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1206_1187_b200.build` "
                    "or __graft_entry__.build(); there is no CPU fallback")
            handle = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise the mapped exception."""
    h = lib()
    st = getattr(h, name)(*args)
    if st:
        raise_for_status(st, h.bcn_last_error().decode(errors="replace"))

"""ctypes binding of include/sim3d_b200.h (the 3-D path's C-ABI).

The structs are parsed from the header with the same restricted-style parser
as the planar ABI (paper_2601_22074_b200/native.py) and cross-checked against
``s3_sizeof``. No fallback: a missing or stale library raises.
"""

from __future__ import annotations

import ctypes
import os

from .. import native as _n

_HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "sim3d_b200.h")
LIBRARY = os.environ.get("S3_LIBRARY") or os.path.join(_HERE, "_sim3d_b200.so")  # override: A/B of kernel builds

MACROS, _STRUCTS, _ORDER = _n._parse_header(HEADER)
globals().update({k: v for k, v in MACROS.items() if k.startswith("S3_")})
_TYPES = _n._build_types(_STRUCTS, _ORDER)
ModelT = _TYPES["s3_model"]
DataT = _TYPES["s3_data"]
LayoutT = _TYPES["s3_layout"]
TaskT = _TYPES["s3_task"]

_SIGNATURES = {
    "s3_abi_version": ([], ctypes.c_int),
    "s3_sizeof": ([ctypes.c_int], ctypes.c_size_t),
    "s3_last_error": ([], ctypes.c_char_p),
    "s3_plan": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "s3_step": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "s3_env_step": ([ctypes.c_void_p] * 5 + [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p], ctypes.c_int),
    "s3_motion_bodies": ([ctypes.c_void_p] * 5, ctypes.c_int),
    "s3_raycast": ([ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                    ctypes.c_double, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "s3_depth": ([ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                  ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                 ctypes.c_int),
}
EXPORTED = sorted(_SIGNATURES)
_LIB = None
LAUNCHES = {"count": 0}


class NativeError(RuntimeError):
    pass


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIBRARY):
            raise NativeError(f"CUDA extension {LIBRARY} is not built; run __graft_entry__.build()")
        so = ctypes.CDLL(LIBRARY)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(so, name)
            fn.argtypes = args
            fn.restype = res
        if so.s3_abi_version() != S3_ABI_VERSION:  # noqa: F821
            raise NativeError("stale sim3d extension: ABI version mismatch, rebuild it")
        for which, cls in ((0, ModelT), (1, DataT), (2, LayoutT), (3, TaskT)):
            if so.s3_sizeof(which) != ctypes.sizeof(cls):
                raise NativeError(f"struct layout mismatch for {cls.__name__}; rebuild the extension")
        _LIB = so
    return _LIB


def call(name: str, *args, launch: bool = False) -> None:
    if launch:
        LAUNCHES["count"] += 1
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise NativeError(f"{name} failed ({rc}): {lib().s3_last_error().decode(errors='replace')}")

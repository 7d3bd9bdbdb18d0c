"""ctypes binding of the C-ABI in include/stridesim_b200.h.

The struct layouts are not restated by hand: the header is parsed at import
time (it is written in a deliberately restricted one-field-per-line style)
and turned into ctypes.Structure classes, then ``ss_sizeof`` from the built
library cross-checks the sizes. There is no fallback: if the shared library
is missing or stale, ``lib()`` raises and nothing runs.
"""

from __future__ import annotations

import ctypes
import os
import re
from ctypes import byref  # noqa: F401  (re-exported for callers)

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
HEADER = os.path.join(_ROOT, "include", "stridesim_b200.h")
LIBRARY = os.path.join(_HERE, "_stridesim_b200.so")


class NativeError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# header -> ctypes


def _parse_header(path: str):
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    macros: dict[str, int] = {}
    for name, val in re.findall(r"#define\s+(\w+)\s+(0x[0-9A-Fa-f]+|-?\d+)u?\b", text):
        macros[name] = int(val, 0)
    structs: dict[str, list[tuple[str, str, list[int]]]] = {}
    order: list[str] = []
    for m in re.finditer(r"typedef\s+struct\s+(\w+)\s*\{(.*?)\}\s*(\w+)\s*;", text, flags=re.S):
        name = m.group(3)
        fields = []
        for line in m.group(2).split(";"):
            line = " ".join(line.split())
            if not line:
                continue
            fm = re.fullmatch(r"(const\s+)?([\w]+)\s*(\*?)\s*(\w+)((?:\[\w+\])*)", line)
            if fm is None:
                raise NativeError(f"cannot parse header field {line!r} in {name}")
            base, ptr, fname, dims = fm.group(2), fm.group(3), fm.group(4), fm.group(5)
            shape = [int(d) if d.isdigit() else macros[d] for d in re.findall(r"\[(\w+)\]", dims)]
            fields.append((fname, base + ptr, shape))
        structs[name] = fields
        order.append(name)
    return macros, structs, order


_SCALARS = {
    "double": ctypes.c_double,
    "int32_t": ctypes.c_int32,
    "uint32_t": ctypes.c_uint32,
    "int64_t": ctypes.c_int64,
    "uint64_t": ctypes.c_uint64,
    "uint8_t": ctypes.c_uint8,
}

MACROS, _STRUCTS, _ORDER = _parse_header(HEADER)
globals().update({k: v for k, v in MACROS.items() if k.startswith("SS_")})

_TYPES: dict[str, type] = {}
for _name in _ORDER:
    _fields = []
    for _fname, _ftype, _shape in _STRUCTS[_name]:
        if _ftype.endswith("*"):
            t = ctypes.c_void_p
        elif _ftype in _SCALARS:
            t = _SCALARS[_ftype]
        else:
            t = _TYPES[_ftype]
        for dim in reversed(_shape):
            t = t * dim
        _fields.append((_fname, t))
    _TYPES[_name] = type(_name, (ctypes.Structure,), {"_fields_": _fields})

EnvDesc = _TYPES["ss_env_desc"]
Uniforms = _TYPES["ss_uniforms"]
RngDrawArgs = _TYPES["ss_rng_draw_args"]
Terrain = _TYPES["ss_terrain"]
RtState = _TYPES["ss_rt_state"]
Launch = _TYPES["ss_launch"]

# ---------------------------------------------------------------------------
# library

_LIB = None

_SIGNATURES = {
    "ss_abi_version": ([], ctypes.c_int),
    "ss_sizeof": ([ctypes.c_int], ctypes.c_size_t),
    "ss_last_error": ([], ctypes.c_char_p),
    "ss_env_step": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "ss_rng_draw": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "ss_fk": ([ctypes.c_void_p] * 5 + [ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "ss_heights": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p], ctypes.c_int),
    "ss_randomize": (
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "ss_jit_compile": (
        [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t), ctypes.c_char_p, ctypes.c_size_t],
        ctypes.c_int,
    ),
    "ss_jit_load": ([ctypes.c_void_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
                    ctypes.c_int),
    "ss_jit_unload": ([ctypes.c_void_p], ctypes.c_int),
    "ss_env_step_jit": ([ctypes.c_void_p] * 4, ctypes.c_int),
    "ss_rt_launch": ([ctypes.c_void_p] * 5, ctypes.c_int),
    "ss_rt_poll": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32], ctypes.c_int),
    "ss_rt_release": ([ctypes.c_void_p], ctypes.c_int),
    "ss_actuator_eval": (
        [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_double,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p],
        ctypes.c_int,
    ),
}

EXPORTED = sorted(_SIGNATURES)


def lib():
    """Load the sm_100a extension (built by __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIBRARY):
            raise NativeError(
                f"CUDA extension {LIBRARY} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        so = ctypes.CDLL(LIBRARY)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(so, name)
            fn.argtypes = args
            fn.restype = res
        if so.ss_abi_version() != SS_ABI_VERSION:  # noqa: F821
            raise NativeError("stale extension: ABI version mismatch, rebuild it")
        for which, cls in ((0, EnvDesc), (1, Uniforms), (2, RngDrawArgs), (3, RtState), (4, Launch)):
            if so.ss_sizeof(which) != ctypes.sizeof(cls):
                raise NativeError(
                    f"struct layout mismatch for {cls.__name__}: C {so.ss_sizeof(which)} vs "
                    f"ctypes {ctypes.sizeof(cls)}; rebuild the extension"
                )
        _LIB = so
    return _LIB


LAUNCHES = {"count": 0}  # kernel launches issued through the C-ABI (bench.py reports them)


def call(name: str, *args) -> None:
    LAUNCHES["count"] += 1
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().ss_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")


def current_stream(device=None) -> int:
    """Raw cudaStream_t of the current stream (an int device index is the fast path)."""
    import torch

    if isinstance(device, int):
        return torch._C._cuda_getCurrentRawStream(device)
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    return None if t is None else t.data_ptr()

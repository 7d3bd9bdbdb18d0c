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


def _parse_header(path: str, overrides: dict | None = None):
    """Macros + struct field lists of the header. ``overrides`` pins macros
    (the SS_DCAP_* bounds of a specialized kernel's packed descriptor)."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    macros: dict[str, int] = dict(overrides or {})
    for name, val in re.findall(r"#define\s+(\w+)[ \t]+(0x[0-9A-Fa-f]+|-?\d+|[A-Za-z_]\w*)u?[ \t]*$", text,
                                flags=re.M):
        if name in macros:
            continue  # overridden, or an #ifndef default already seen
        if val[0].isalpha() or val[0] == "_":
            if val in macros:
                macros[name] = macros[val]  # alias of an earlier macro
        else:
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

def _build_types(structs, order) -> dict[str, type]:
    types: dict[str, type] = {}
    for name in order:
        fields = []
        for fname, ftype, shape in structs[name]:
            if ftype.endswith("*"):
                t = ctypes.c_void_p
            elif ftype in _SCALARS:
                t = _SCALARS[ftype]
            else:
                t = types[ftype]
            for dim in reversed(shape):
                t = t * dim
            fields.append((fname, t))
        types[name] = type(name, (ctypes.Structure,), {"_fields_": fields})
    return types


_TYPES = _build_types(_STRUCTS, _ORDER)

EnvDesc = _TYPES["ss_env_desc"]
Uniforms = _TYPES["ss_uniforms"]
RngDrawArgs = _TYPES["ss_rng_draw_args"]
Terrain = _TYPES["ss_terrain"]
RtState = _TYPES["ss_rt_state"]
Launch = _TYPES["ss_launch"]
StatsArgs = _TYPES["ss_stats_args"]

DCAPS = ("JOINTS", "FEET", "ACTION_TERMS", "ACTUATORS", "CMD", "RAYS", "GROUPS", "OBS_TERMS", "REWARDS",
         "TERMINATIONS", "EVENTS", "CURRICULUM", "FIELDS", "SLOTS", "MLP_LAYERS")
_PACKED: dict[tuple, type] = {}


def packed_desc_type(caps: dict) -> type:
    """ctypes class of ss_env_desc with SS_DCAP_<k> = caps[k] (a specialized
    kernel's parameter block)."""
    key = tuple(sorted(caps.items()))
    t = _PACKED.get(key)
    if t is None:
        _, structs, order = _parse_header(HEADER, {f"SS_DCAP_{k}": int(v) for k, v in caps.items()})
        t = _PACKED[key] = _build_types(structs, order)["ss_env_desc"]
    return t


def _copy_into(dst, src) -> None:
    """Field-by-field copy between two layouts of one struct; arrays are
    truncated to the destination's bounds (ctypes objects)."""
    for name, t in dst._fields_:
        sv = getattr(src, name)
        if isinstance(sv, ctypes.Structure):
            _copy_into(getattr(dst, name), sv)
        elif isinstance(sv, ctypes.Array):
            _copy_array(getattr(dst, name), sv)
        else:
            setattr(dst, name, sv)


def _copy_array(dst, src) -> None:
    n = len(dst)
    if n and isinstance(dst[0], (ctypes.Structure, ctypes.Array)):
        for i in range(n):
            if isinstance(dst[i], ctypes.Structure):
                _copy_into(dst[i], src[i])
            else:
                _copy_array(dst[i], src[i])
    else:
        dst[:n] = src[:n]


def pack_desc(desc, caps: dict):
    """The descriptor re-laid-out with the given SS_DCAP_* bounds."""
    out = packed_desc_type(caps)()
    _copy_into(out, desc)
    return out


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
    "ss_jit_set_desc_bytes": ([ctypes.c_void_p, ctypes.c_int64], ctypes.c_int),
    "ss_jit_set_smem": ([ctypes.c_void_p, ctypes.c_int32], ctypes.c_int),
    "ss_env_step_jit_packed": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_void_p], ctypes.c_int),
    "ss_rt_launch": ([ctypes.c_void_p] * 5, ctypes.c_int),
    "ss_rt_poll": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32], ctypes.c_int),
    "ss_rt_release": ([ctypes.c_void_p], ctypes.c_int),
    "ss_pipe_create": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                        ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "ss_pipe_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "ss_pipe_pre": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "ss_pipe_post": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "ss_pipe_wait": ([ctypes.c_void_p], ctypes.c_int),
    "ss_stats_pack": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
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
        for which, cls in ((0, EnvDesc), (1, Uniforms), (2, RngDrawArgs), (3, RtState), (4, Launch), (5, StatsArgs)):
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

"""Per-env specialization of the fused step kernel (NVRTC, sm_100a).

The reference re-specializes its substep whenever the model layout changes
(StepPipeline._rebuild, sim/physics.py:158-237). Here the analogous step is
a compile: every value the kernel reads from the term tables is turned into
a compile-time constant (the X-lists of csrc/ss_cfg.cuh, evaluated against
the env's descriptor), so NVRTC unrolls every term loop, folds topology and
parameters into immediates and keeps each world's arrays in registers. The
kernel source is the same ss_kernel.cuh the generic AOT build uses, so the
two agree bit for bit; device pointers and RNG keys stay runtime values.

Compiled cubins are cached in memory by source hash (and on disk under
$XDG_CACHE_HOME/paper_2601_22074_b200/jit, an optional speed-up only).
SS_JIT=0 in the environment selects the generic kernel.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import re

from . import native

_CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
_HEADERS = {
    "stridesim_b200.h": native.HEADER,
    "ss_device.cuh": os.path.join(_CSRC, "ss_device.cuh"),
    "ss_cfg.cuh": os.path.join(_CSRC, "ss_cfg.cuh"),
    "ss_kernel.cuh": os.path.join(_CSRC, "ss_kernel.cuh"),
}
OPTIONS = ["--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "-lineinfo", "-DSS_JIT=1", "-default-device",
           f"--include-path={_CSRC}", f"--include-path={os.path.dirname(native.HEADER)}"]
KERNEL = "ss_step_jit"


class JitUnsupported(RuntimeError):
    pass


def options() -> list[str]:
    opts = list(OPTIONS)
    if os.environ.get("SS_FMAD") == "1":  # experiment: let NVRTC contract a*b+c into FMA (not numpy's rounding)
        opts = [o if o != "--fmad=false" else "--fmad=true" for o in opts]
    if os.environ.get("SS_PROBES") == "1":
        opts.append("-DSS_PROBES=1")
    # experiment switches, e.g. SS_JIT_DEFINES="-DSS_PEEL_LAST_SUBSTEP=0"
    opts += os.environ.get("SS_JIT_DEFINES", "").split()
    return opts


def enabled() -> bool:
    return os.environ.get("SS_JIT", "1") != "0"


def _parse_lists():
    text = open(_HEADERS["ss_cfg.cuh"]).read()
    out = {}
    for macro, arity in (("SS_CFG_SCALARS", 3), ("SS_CFG_ARRAYS", 4), ("SS_CFG_ARRAYS2", 5)):
        body = text.split(f"#define {macro}(")[1].split("\n\n")[0]
        items = []
        for m in re.finditer(r"X[AB]?\(([^()]*(?:\([^()]*\)[^()]*)*)\)", body):
            parts = [p.strip() for p in m.group(1).split(",")]
            if len(parts) != arity:
                continue
            items.append(parts)
        out[macro] = items
    return out


_LISTS = _parse_lists()


def _bound(name: str) -> int:
    return int(name) if name.isdigit() else getattr(native, name)


def _lit(typ: str, v) -> str:
    if typ == "double":
        v = float(v)
        if not math.isfinite(v):
            raise JitUnsupported(f"non-finite constant {v}")
        return v.hex()
    if typ == "unsigned":
        return f"{int(v) & 0xFFFFFFFF}u"
    return str(int(v))


def config_source(d) -> str:
    """C++ source of the constexpr config struct for descriptor ``d``."""
    caps = {"kCapAct": d.n_actuators, "kCapActTerms": d.n_action_terms, "kCapTerms": d.n_terms,
            "kCapRewards": d.n_rewards, "kCapEvents": d.n_events, "kCapGroups": d.n_groups, "kCapObs": d.n_obs_terms}
    lines = ["struct JitCfg {", "  static constexpr bool kJit = true;", "  static constexpr int kUnroll = 64;"]
    lines += [f"  static constexpr int {k} = {int(v)};" for k, v in caps.items()]
    # shared-memory staging of the observation rows (one bulk copy per group)
    dims = [int(d.group[g].dim) for g in range(int(d.n_groups))]
    soff = [sum(dims[:g]) for g in range(len(dims))] + [0] * (native.SS_MAX_GROUPS - len(dims))
    block = block_size(d)
    stage = obs_staged(d, block)
    lines += [f"  static constexpr int kBlock = {block}, kStageObs = {stage}, kObsTotal = {max(sum(dims), 1)}, "
              f"kRays = {max(int(d.n_rays), 1)};",
              f"  static __device__ __forceinline__ int g_soff(const ss_env_desc&, int g) {{ constexpr int a[{native.SS_MAX_GROUPS}] = "
              f"{{{', '.join(str(x) for x in soff)}}}; return a[g]; }}"]
    lines += [staging_config(d, block, stage, sum(dims))]
    head = "  static __device__ __forceinline__"
    # Integers (counts, ids, flags, indices) become immediates: they drive the
    # unrolling and fold the term tables. Doubles stay kernel-parameter loads:
    # FP64 instructions read constant-bank operands directly, whereas a 64-bit
    # immediate costs two uniform moves per use.
    for typ, name, expr in _LISTS["SS_CFG_SCALARS"]:
        if typ == "double":
            lines.append(f"{head} {typ} {name}(const ss_env_desc& d) {{ return {expr}; }}")
            continue
        val = eval(expr, {"d": d})  # noqa: S307 -- expressions come from ss_cfg.cuh
        if name == "NW" and int(val) < const_worlds_min():
            # small envs share one build across world counts (tests, tools);
            # large ones fold N into every SoA offset (ptr[c*N + w])
            lines.append(f"{head} {typ} {name}(const ss_env_desc& d) {{ return {expr}; }}")
            continue
        lines.append(f"{head} {typ} {name}(const ss_env_desc&) {{ return {_lit(typ, val)}; }}")
    for typ, name, bound, expr in _LISTS["SS_CFG_ARRAYS"]:
        if typ == "double":
            lines.append(f"{head} {typ} {name}(const ss_env_desc& d, int i) {{ return {expr}; }}")
            continue
        n = _bound(bound)
        vals = [_lit(typ, eval(expr, {"d": d, "i": i})) for i in range(n)]  # noqa: S307
        lines.append(f"{head} {typ} {name}(const ss_env_desc&, int i) {{ constexpr {typ} a[{n}] = {{"
                     f"{', '.join(vals)}}}; return a[i]; }}")
    for typ, name, bt, bi, expr in _LISTS["SS_CFG_ARRAYS2"]:
        if typ == "double":
            lines.append(f"{head} {typ} {name}(const ss_env_desc& d, int t, int i) {{ return {expr}; }}")
            continue
        nt, ni = _bound(bt), _bound(bi)
        rows = []
        for t in range(nt):
            rows.append("{" + ", ".join(_lit(typ, eval(expr, {"d": d, "t": t, "i": i})) for i in range(ni)) + "}")  # noqa: S307
        lines.append(f"{head} {typ} {name}(const ss_env_desc&, int t, int i) {{ constexpr {typ} a[{nt}][{ni}] = {{"
                     f"{', '.join(rows)}}}; return a[t][i]; }}")
    lines.append("};")
    return "\n".join(lines)


def obs_staged(d, block: int) -> int:
    """Observation rows staged in shared memory (one TMA bulk copy per group) while they fit 48 KB."""
    total = sum(int(d.group[g].dim) for g in range(int(d.n_groups)))
    return int(total > 0 and block * total * 8 <= 48 * 1024 and os.environ.get("SS_STAGE_OBS", "1") != "0")


def dyn_smem_bytes(d) -> int:
    block = block_size(d)
    total = sum(int(d.group[g].dim) for g in range(int(d.n_groups)))
    return staging_layout(d, block, obs_staged(d, block), total)["dyn"]


def staging_layout(d, block: int, stage: int, obs_total: int) -> dict:
    """Shared-memory staging of the specialized kernel (ss_kernel.cuh): the observation rows (one TMA
    bulk copy per group), the hoisted model fields (Params columns) and, for large action vectors, the
    action / previous-action columns (ActArr). The three sit in static shared memory while they fit its
    48 KB; beyond that, in one dynamic block (up to SS_DYN_SMEM_MAX bytes) -- the large surrogates,
    whose register-resident copies spill."""
    km, na = max(int(d.model.n_joints), 1), max(int(d.n_actuators), 1)
    a = max(int(d.action_dim), 1)
    nv = 6 + 4 * km + 2 * na * km
    obs = stage * block * obs_total
    param = nv * block if os.environ.get("SS_PARAM_SMEM", "1") != "0" else 0
    ncol = 2 * a + km + 2 * max(int(d.n_rewards), 1)  # ss_kernel.cuh step_world: action, prev, targets, ep sums
    act_mode = os.environ.get("SS_ACT_SMEM", "1")  # "0" never, "1" from 8 actions, "all" always
    act = ncol * block if ((a >= 8 and act_mode != "0") or act_mode == "all") else 0
    static_max = 48 * 1024 - 64
    dyn_max = int(os.environ.get("SS_DYN_SMEM_MAX", str(112 * 1024)))  # 2 blocks per SM
    if (obs + param + act) * 8 <= static_max:
        return {"param": int(param > 0), "act": int(act > 0), "dyn": 0, "obs_off": 0, "param_off": 0, "act_off": 0,
                "act_cols": a}
    if act and (obs + param + act) * 8 <= dyn_max:
        return {"param": int(param > 0), "act": 1, "dyn": (obs + param + act) * 8, "obs_off": 0, "param_off": obs,
                "act_off": obs + param, "act_cols": a}
    # the biped's layout: params only while they fit the static budget
    param_fits = param and (obs + param) * 8 <= static_max
    return {"param": int(bool(param_fits)), "act": 0, "dyn": 0, "obs_off": 0, "param_off": 0, "act_off": 0,
            "act_cols": a}


def staging_config(d, block: int, stage: int, obs_total: int) -> str:
    L = staging_layout(d, block, stage, obs_total)
    km, na = max(int(d.model.n_joints), 1), max(int(d.n_actuators), 1)
    alone = int(os.environ.get("SS_PARAM_SMEM", "1") != "0" and (6 + 4 * km + 2 * na * km) * block * 8 + 64 <= 48 * 1024)
    return (f"  static constexpr int kParamSmemAlone = {alone};\n"
            f"  static constexpr int kParamSmem = {L['param']}, kActSmem = {L['act']}, kDynSmem = {L['dyn']}, "
            f"kDynObs = {L['obs_off']}, kDynParam = {L['param_off']}, kDynAct = {L['act_off']};")


def const_worlds_min() -> int:
    """World count from which N is compiled in as a constant (SS_CONST_N_MIN)."""
    return int(os.environ.get("SS_CONST_N_MIN", "1024"))


def block_size(d=None) -> int:
    """Threads per block of the specialized kernel (one world per thread). 64 spreads a partial wave over
    the most SMs (4096 worlds: 64 blocks); from 65,536 worlds, where the grid is many waves deep, 128 is
    faster (fewer, larger TMA row copies of the observation blocks; Velocity-Rough 262,144 worlds 162 ->
    156 us, 1,048,576 worlds 628 -> 583 us, tools/kab.py on one B200). SS_BLOCK overrides."""
    env = os.environ.get("SS_BLOCK")
    if env:
        return int(env)
    return 128 if d is not None and int(d.n_worlds) >= 65536 else 64


def min_blocks() -> int:
    """__launch_bounds__ min blocks per SM (0: let ptxas use every register)."""
    return int(os.environ.get("SS_MINB", "0"))


def desc_caps(d) -> dict:
    """SS_DCAP_* bounds of the packed descriptor for ``d``: the counts that
    exist (>= 1); stream slots rounded up to 8 so a new purpose rarely
    changes the layout."""
    k, f = int(d.model.n_joints), int(d.model.n_feet)
    fields = max([i + 1 for i in range(native.SS_MAX_FIELDS) if d.field[i].ptr] + [1])
    fsize = max([int(d.field[i].size) for i in range(fields)] + [1])
    slots = max([i + 1 for i in range(native.SS_MAX_SLOTS) if d.rng.counter[i]] + [1])
    slots = min(native.SS_MAX_SLOTS, -(-slots // 8) * 8)
    layers = max([int(d.actuator[a].n_layers) for a in range(int(d.n_actuators))] + [1])
    return {"JOINTS": max(k, fsize, 1), "FEET": max(f, 1), "ACTION_TERMS": max(int(d.n_action_terms), 1),
            "ACTUATORS": max(int(d.n_actuators), 1), "CMD": max(int(d.n_cmd), 1), "RAYS": max(int(d.n_rays), 1),
            "GROUPS": max(int(d.n_groups), 1), "OBS_TERMS": max(int(d.n_obs_terms), 1),
            "REWARDS": max(int(d.n_rewards), 1), "TERMINATIONS": max(int(d.n_terms), 1),
            "EVENTS": max(int(d.n_events), 1), "CURRICULUM": max(int(d.n_curriculum), 1), "FIELDS": fields,
            "SLOTS": slots, "MLP_LAYERS": layers}


SPLIT_PHYS = native.SS_ST_ACTION | native.SS_ST_APPLY | native.SS_ST_PUSH | native.SS_ST_PHYS | native.SS_ST_SENSOR
SPLIT_POST = (native.SS_ST_TERM | native.SS_ST_REWARD | native.SS_ST_CURRICULUM | native.SS_ST_RESET
              | native.SS_ST_COMMAND | native.SS_ST_EVENTS | native.SS_ST_OBS | native.SS_ST_PREV_AFTER)
KERNELS = {"main": (KERNEL, 0), "phys": (KERNEL + "_phys", SPLIT_PHYS), "post": (KERNEL + "_post", SPLIT_POST)}


def split_enabled(d) -> bool:
    """Step in two launches of kernels compiled for fixed stage sets (physics | terms + observations):
    each needs ~40 registers fewer than the whole body (244 -> 168 at block 128), 12 warps per SM
    instead of 8 -- and the second re-reads ~400 B per world the first wrote. Measured slower at every
    size (262,144 worlds 156 -> 162 us, 1,048,576 583 -> 622 us), so off unless SS_SPLIT=1
    (or SS_SPLIT=auto: from SS_SPLIT_MIN worlds). Bit-identical to the fused launch (tested)."""
    mode = os.environ.get("SS_SPLIT", "0")
    if mode in ("0", "1"):
        return mode == "1"
    return int(d.n_worlds) >= int(os.environ.get("SS_SPLIT_MIN", "65536"))


def kernel_source(d) -> str:
    k, f = int(d.model.n_joints), int(d.model.n_feet)
    caps = desc_caps(d)
    packed = ctypes.sizeof(native.packed_desc_type(caps))
    lines = [
        *[f"#define SS_DCAP_{c} {v}" for c, v in caps.items()],
        f"#define SS_DCAP_ACTION_COLS {max(int(d.action_dim), 1)}",
        '#include "stridesim_b200.h"',
        f'static_assert(sizeof(ss_env_desc) == {packed}, "packed descriptor layout differs from the host packing");',
        '#include "ss_kernel.cuh"',
        config_source(d),
    ]
    names = ["main"] + (["phys", "post"] if split_enabled(d) else [])
    for which in names:
        name, fs = KERNELS[which]
        lines += [
            f"extern \"C\" __global__ void __launch_bounds__({block_size(d)}"
            f"{', ' + str(min_blocks()) if min_blocks() else ''}) {name}(",
            "    const __grid_constant__ ss_env_desc d, const __grid_constant__ ss_uniforms u) {",
            f"  ss::step_body<JitCfg, {max(k, 1)}, {max(f, 1)}, {fs}u>(d, u);",
            "}",
        ]
    return "\n".join(lines) + "\n"


def _headers():
    names, srcs = [], []
    for name, path in _HEADERS.items():
        names.append(name.encode())
        srcs.append(open(path, "rb").read())
    return names, srcs


def _source_file(src: str) -> str:
    """Write the generated translation unit next to the cache so -lineinfo
    (and ncu --import-source) can resolve it; headers resolve to csrc/."""
    key = hashlib.sha256(src.encode()).hexdigest()[:16]
    path = os.path.join(_cache_dir(), f"ss_step_jit_{key}.cu")
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        if not os.path.exists(path):
            with open(path, "w") as fh:
                fh.write(src)
    except OSError:
        return "ss_step_jit.cu"
    return path


def compile_cubin(src: str) -> bytes:
    """NVRTC: source -> sm_100a cubin (no GPU needed)."""
    opts = [o.encode() for o in options()]
    c_opts = (ctypes.c_char_p * len(opts))(*opts)
    size = ctypes.c_size_t(0)
    log = ctypes.create_string_buffer(1 << 16)
    so = native.lib()
    name = _source_file(src).encode()
    rc = so.ss_jit_compile(src.encode(), name, 0, None, None, len(opts), c_opts, None, ctypes.byref(size),
                           log, len(log))
    if rc != 0:
        raise native.NativeError(f"NVRTC failed: {so.ss_last_error().decode()}\n{log.value.decode()[:4000]}")
    buf = ctypes.create_string_buffer(size.value)
    rc = so.ss_jit_compile(src.encode(), name, 0, None, None, len(opts), c_opts, buf, ctypes.byref(size),
                           log, len(log))
    if rc != 0:
        raise native.NativeError(f"NVRTC failed: {so.ss_last_error().decode()}")
    return buf.raw[: size.value]


def _cache_dir() -> str:
    base = os.environ.get("XDG_CACHE_HOME", os.path.join(os.path.expanduser("~"), ".cache"))
    return os.path.join(base, "paper_2601_22074_b200", "jit")


_MODULES: dict[str, int] = {}
STATS = {"compiled": 0, "disk_hits": 0, "memory_hits": 0}


def _store_cubin(path: str, cubin: bytes) -> None:
    """Atomically publish a cubin: a private temp file (mkstemp), fsync, rename (ranks of one node may
    share the cache directory; a reader sees the old file or the complete new one)."""
    import tempfile

    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path), prefix=".cubin.")
        try:
            with os.fdopen(fd, "wb") as fh:
                fh.write(cubin)
                fh.flush()
                os.fsync(fh.fileno())
            os.replace(tmp, path)
        except BaseException:
            os.unlink(tmp)
            raise
    except OSError:
        pass


def _load(cubin: bytes, d, name: str = KERNEL) -> int:
    handle = ctypes.c_void_p()
    native.call("ss_jit_load", cubin, len(cubin), name.encode(), block_size(d), ctypes.byref(handle))
    native.call("ss_jit_set_desc_bytes", handle, ctypes.sizeof(native.packed_desc_type(desc_caps(d))))
    dyn = dyn_smem_bytes(d)
    if dyn:
        native.call("ss_jit_set_smem", handle, dyn)
    return handle.value


def modules_for(d) -> dict:
    """Loaded kernel handles specialized for descriptor ``d`` on the current device (compiled on first
    use): {"main": whole step} and, for split envs, {"phys": ..., "post": ...}."""
    import torch

    src = kernel_source(d)
    key = hashlib.sha256((src + "|".join(options()) + "".join(open(p).read() for p in _HEADERS.values())).encode()).hexdigest()
    mkey = f"{key}@{torch.cuda.current_device()}"  # a module is loaded into one device's context
    hs = _MODULES.get(mkey)
    if hs is not None:
        STATS["memory_hits"] += 1
        return hs
    names = ["main"] + (["phys", "post"] if split_enabled(d) else [])
    path = os.path.join(_cache_dir(), key + ".cubin")
    hs = None
    try:
        with open(path, "rb") as fh:
            cubin = fh.read()
        hs = {w: _load(cubin, d, KERNELS[w][0]) for w in names}
        STATS["disk_hits"] += 1
    except (OSError, native.NativeError):
        hs = None  # absent or unloadable (e.g. truncated by a crashed writer): recompile
    if hs is None:
        cubin = compile_cubin(src)
        STATS["compiled"] += 1
        _store_cubin(path, cubin)
        hs = {w: _load(cubin, d, KERNELS[w][0]) for w in names}
    _MODULES[mkey] = hs
    return hs


def module_for(d) -> int:
    """Loaded kernel handle of the whole step specialized for descriptor ``d``."""
    return modules_for(d)["main"]

"""Offline (no GPU) inspection of a specialized step kernel: NVRTC-compile a
translation unit from tools/dump_jit_tu.py with the production options
(+ SS_JIT_DEFINES), print ptxas resource usage and the SASS size.

    python tools/jit_offline.py tools/tu/jit_tu_Velocity-Rough.cu [--sass out.sass]
"""
import argparse
import ctypes
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_22074_b200 import jit, native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("tu")
ap.add_argument("--sass", default=None)
ap.add_argument("--cubin", default=None, help="also write the cubin (nvdisasm -g for line info)")
args = ap.parse_args()
src = open(args.tu).read()
opts = [o.encode() for o in jit.options() + ["--ptxas-options=-v"]]
c_opts = (ctypes.c_char_p * len(opts))(*opts)
so = native.lib()
size = ctypes.c_size_t(0)
log = ctypes.create_string_buffer(1 << 20)
rc = so.ss_jit_compile(src.encode(), b"tu.cu", 0, None, None, len(opts), c_opts, None, ctypes.byref(size), log, len(log))
if rc != 0:
    sys.exit(log.value.decode()[:4000])
buf = ctypes.create_string_buffer(size.value)
so.ss_jit_compile(src.encode(), b"tu.cu", 0, None, None, len(opts), c_opts, buf, ctypes.byref(size), log, len(log))
for line in log.value.decode().splitlines():
    if "ptxas" in line and ("Used" in line or "spill" in line or "stack" in line):
        print(line.strip())
with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as fh:
    fh.write(buf.raw[: size.value])
if args.cubin:
    open(args.cubin, "wb").write(buf.raw[: size.value])
sass = subprocess.run(["cuobjdump", "-sass", fh.name], capture_output=True, text=True).stdout
os.unlink(fh.name)
ins = [l for l in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
print(f"SASS instructions: {len(ins)} ({len(ins) * 16 / 1024:.1f} KB)")
ops = {}
for l in ins:
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
    if m:
        op = m.group(2).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
print("top opcodes:", ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:16]))
if args.sass:
    open(args.sass, "w").write(sass)

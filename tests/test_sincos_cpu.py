"""The kernels' sin/cos (ss_device.cuh sincos_fast) is faithfully rounded.

The reference computes np.sin/np.cos (glibc) in sim/physics.py:31-40; the
CUDA path uses its own Cody-Waite + fdlibm-kernel sincos, so every result
must stay within 1 ulp of the exact value (long-double sinl/cosl here) --
the same accuracy class as glibc, which is what the parity tolerances
assume. Compiled for the host with nvcc; no GPU needed.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_sincos_fast_within_one_ulp(tmp_path):
    exe = tmp_path / "sincos_acc"
    subprocess.run(["nvcc", "-O2", "-std=c++17", os.path.join(ROOT, "tools/micro/sincos_acc.cu"), "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), "200000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "sin=-0 (-0)" in r.stdout  # sign of zero preserved

"""The heightfield lookup's division (ss_device.cuh div_rn) is exact.

terrain.py:135 divides positions by the sample spacing; the kernels form
the same correctly-rounded quotient from a hoisted reciprocal plus one FMA
correction (Markstein). Checked bit-for-bit against IEEE division for the
spacings a terrain config can use and for random divisors. Host-only.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_div_rn_matches_ieee_division(tmp_path):
    exe = tmp_path / "div_check"
    subprocess.run(["nvcc", "-O2", "-std=c++17", os.path.join(ROOT, "tools/micro/div_check.cu"), "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), "2000000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout

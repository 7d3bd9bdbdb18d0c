"""The reference's OWN test-suite (pkg/tests, unmodified) against this package on the GPU.

`tools/reftests/run.sh prepare` (build container) copies the reference's tests to
baseline/_ref_tests (git-ignored; it travels to the GPU box with the snapshot -- the box has no
/root/reference); `tools/reftests/run.sh` resolves `stridesim.*` to this package
(tools/reftests/stridesim) and runs them. The CLI / viewer files (test_cli, test_bridge,
test_config) are out of scope and not collected. Skipped when the copy is absent.
"""

import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isfile(os.path.join(ROOT, "baseline", "_ref_tests", "test_env.py")),
                    reason="reference tests not copied (tools/reftests/run.sh prepare)")
def test_reference_test_suite_passes_against_the_package():
    out = subprocess.run([os.path.join(ROOT, "tools", "reftests", "run.sh")], capture_output=True, text=True,
                         timeout=1200)
    tail = (out.stdout + out.stderr)[-3000:]
    m = re.search(r"(\d+) passed", tail)
    assert out.returncode == 0 and m and not re.search(r"\d+ (failed|error)", tail), tail
    assert int(m.group(1)) >= 178, tail

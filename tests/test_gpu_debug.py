"""GPU: the HD_DEBUG build of the library (the substitute for compute-sanitizer, which this
pool does not allow): device-side index bounds, the halo freshness check and the non-finite check
after every RK stage stay silent on valid runs and report a NaN as HD_ERR_STATE. Runs
tools/debug_checks.py in a subprocess against paper_2002_08110_b200/libhd_debug.so (built by build())."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2002_08110_b200", "libhd_debug.so")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhd_debug.so not built")
def test_debug_build_checks():
    env = dict(os.environ, HD_LIB_PATH=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_checks.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DEBUG-CHECKS OK" in r.stdout, r.stdout + r.stderr

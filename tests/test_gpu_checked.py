"""The device-check build (compute-sanitizer is closed on the GPU pool):
every persistent-kernel path, the chain, the QR path and the peer kernel run
with bounds asserts on the sampled reads / factor rows and time-outs on the
flag waits compiled in (paper_1701_06600_b200/libcprand_b200_check.so,
`make checklib`), in a subprocess; a failed check traps."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_device_checked_build_runs_every_path():
    lib = os.path.join(ROOT, "paper_1701_06600_b200", "libcprand_b200_check.so")
    assert os.path.exists(lib), "build the device-check library: make checklib"
    env = dict(os.environ, CPRAND_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_workload.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert "CPB_DCHECK failed" not in out, out[-4000:]
    assert p.returncode == 0 and "CHECKED OK" in p.stdout, out[-4000:]

"""Every default kernel family on small cases (scripts/sanitize_case.py), run twice per case in a fresh
process: finite D and gradients, no CUDA error.  (It was written for compute-sanitizer memcheck / racecheck;
the GPU pool refuses compute-sanitizer, so the out-of-bounds guard is this run plus the parity tests.)"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_kernel_families_run_clean():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize cases ok" in r.stdout, (r.stdout + r.stderr)[-3000:]

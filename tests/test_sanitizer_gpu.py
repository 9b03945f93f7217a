"""compute-sanitizer over small evaluations through every default kernel family (scripts/sanitize_case.py):
memcheck (out-of-bounds / misaligned global and shared accesses, leaks) and racecheck (shared-memory
hazards of the hand-rolled TMA / mbarrier / tcgen05 pipelines) must report no error."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.fail("compute-sanitizer not found")
    return exe


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_sanitizer_clean(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "9", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "sanitize cases ok" in r.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in (r.stdout + r.stderr), tail

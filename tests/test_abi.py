"""CPU tests of the C-ABI surface: the library loads and exports exactly the symbols
include/seqreg_b200.h declares (no CUDA call is made)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2001_06613_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "seqreg_b200.h"


def _declared():
    text = HEADER.read_text()
    return set(re.findall(r"SR_API\s+[\w\s\*]+?\b(sr_\w+)\s*\(", text))


def test_header_declarations_match_binding():
    assert _declared() == set(_lib.EXPORTS)


def test_library_exports_every_symbol():
    path = _lib.library_path()
    if not path.exists():
        pytest.fail(f"{path} not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = _declared() - exported
    assert not missing, missing
    # nothing else leaks from the library's namespace besides the ABI
    assert not {s for s in exported if s.startswith("sr") and not s.startswith("sr_")}


def test_library_loads_and_host_only_calls():
    lib = _lib.load_library()
    assert lib.sr_abi_version() == 1
    for k in (1, 3, 32, 100, 128):
        assert lib.sr_raw_size(k) == k * k + 3 * k + 1
        offs = [lib.sr_stats_offset(k, f) for f in range(10)]
        assert offs == sorted(offs) and offs[0] == 8
        assert lib.sr_stats_size(k) > offs[-1]
    assert lib.sr_stats_offset(4, 99) == -1
    assert lib.sr_status_string(3) == b"singular system"


def test_problem_struct_layout():
    import ctypes
    # sr_grid: int32 ndim, int32 dims[3], double spacing[3], double origin[3]
    assert ctypes.sizeof(_lib.SrGrid) == 4 + 12 + 24 + 24
    assert _lib.SrProblem.grid.offset == 0

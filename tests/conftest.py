"""Test configuration: the `gpu` marker (parity tests through the C-ABI on a B200) and
shared fixtures.  `-m "not gpu"` runs the oracle, host-logic and ABI-surface tests on CPU."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"
# the unmodified reference package, installed into baseline/_ref by __graft_entry__.build(); it travels
# to the GPU box with the repo (tests there never read /root/reference)
REF = ROOT / "baseline" / "_ref"
if str(REF) not in sys.path:
    sys.path.append(str(REF))


def ref_types():
    """The reference's Grid / Image / ImageSequence / AffineStack (the drop-in API takes the reference's
    own objects); fails the calling test when baseline/_ref is missing."""
    try:
        from seqreg.grid import Grid, Image, ImageSequence
        from seqreg.transform import AffineStack
    except ImportError as exc:
        pytest.fail(f"reference package not importable from baseline/_ref ({exc}); run build()")
    return Grid, Image, ImageSequence, AffineStack


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libseqreg_b200.so")


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN, allow_pickle=False)
    cases = {}
    for key in data.files:
        name, field = key.split("/", 1)
        cases.setdefault(name, {})[field] = data[key]
    return cases


def golden_frames(case):
    """Frames of a golden case (stored, or regenerated from the seeded synthetic config)."""
    if "frames" in case:
        return case["frames"]
    from paper_2001_06613_b200 import synth

    cfg_name, seed = str(case["synth"]).split(":")
    frames, _, _, _ = synth.make_sequence(synth.CONFIGS[cfg_name], seed=int(seed), device="cpu")
    return frames.numpy()

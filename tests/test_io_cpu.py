"""CPU: the STSQ1 reader raises the reference reader's exception class and message for every
malformed variant (tests/golden/stsq1_errors.json, recorded from seqreg.grid.read_sequence);
validation happens before any device work, so no GPU is needed."""

import json
from pathlib import Path

import pytest

from paper_2001_06613_b200 import io as sio
from tests.stsq1_cases import variants

GOLD = Path(__file__).resolve().parent / "golden"
ERRORS = json.loads((GOLD / "stsq1_errors.json").read_text())


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_reader_errors_match_reference(name, tmp_path):
    data = variants((GOLD / "small_seq.stsq1").read_bytes())[name]
    p = tmp_path / f"{name}.stsq1"
    p.write_bytes(data)
    cls, msg = ERRORS[name]
    with pytest.raises(ValueError) as ei:
        sio.read_sequence(p)
    assert type(ei.value).__name__ == cls
    assert str(ei.value) == msg
    # header errors are SequenceFormatErrors; the payload / sequence checks plain ValueErrors (grid.py:104-150)
    assert isinstance(ei.value, sio.SequenceFormatError) == (cls != "ValueError")

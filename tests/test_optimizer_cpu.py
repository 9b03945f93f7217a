"""CPU: the L-BFGS oracle restatement (oracle/seqreg_oracle.py, optimizer.py:59-168) reproduces
the reference optimizer's outcomes (tests/golden/lbfgs_golden.json, made by running seqreg), and
the Python mirror validates options with the reference's messages."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import seqreg_oracle as orc
from tests.lbfgs_problems import problems

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "lbfgs_golden.json").read_text())


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_oracle_lbfgs_matches_reference(name):
    fn, x0, opts = problems()[name]
    trace = []
    r = orc.lbfgs_minimize(fn, x0, trace=lambda *a: trace.append([float(v) for v in a]), **opts)
    gold = GOLDEN[name]
    assert (r["iterations"], r["objective_evaluations"], r["converged_reason"]) == (
        gold["iterations"], gold["objective_evaluations"], gold["converged_reason"])
    assert r["f_final"] == gold["f_final"]
    np.testing.assert_array_equal(r["x_final"], np.asarray(gold["x_final"]))
    assert trace == gold["trace"]


def test_oracle_nonfinite_start():
    with pytest.raises(ValueError, match="not finite at the starting point"):
        orc.lbfgs_minimize(lambda x: (float("inf"), x), np.zeros(3))


@pytest.mark.parametrize("kw,msg", [
    (dict(memory=0), "memory, max_iters, max_backtracks must be >= 1"),
    (dict(max_backtracks=0), "memory, max_iters, max_backtracks must be >= 1"),
    (dict(grad_tol=0.0), "tolerances must be > 0"),
    (dict(armijo_c1=1.0), r"armijo_c1 must be in \(0, 1\)"),
    (dict(backtrack_factor=0.0), r"backtrack_factor must be in \(0, 1\)"),
])
def test_options_validation_messages(kw, msg):
    from paper_2001_06613_b200.optimizer import OptimOptions
    with pytest.raises(ValueError, match=msg):
        OptimOptions(**kw)

"""Runs the reference optimizer (seqreg.optimizer.lbfgs_minimize, optimizer.py:76-168) on the
problems of tests/lbfgs_problems.py and writes tests/golden/lbfgs_golden.json.  Needs the
reference (PYTHONPATH=/root/reference/pkg/src); the GPU box never runs this.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_lbfgs_golden.py
"""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from seqreg.optimizer import ObjectiveEval, OptimOptions, lbfgs_minimize  # noqa: E402

from tests.lbfgs_problems import problems  # noqa: E402


def main():
    out = {}
    for name, (fn, x0, opts) in problems().items():
        trace = []
        res = lbfgs_minimize(lambda x: ObjectiveEval(*fn(x)), x0, OptimOptions(**opts),
                             trace=lambda *a: trace.append([float(v) for v in a]))
        out[name] = dict(iterations=res.iterations, objective_evaluations=res.objective_evaluations,
                         converged_reason=res.converged_reason, f_final=res.f_final, f_initial=res.f_initial,
                         x_final=np.asarray(res.x_final).tolist(), trace=trace)
        print(name, res.iterations, res.objective_evaluations, res.converged_reason, res.f_final)
    (ROOT / "tests" / "golden" / "lbfgs_golden.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

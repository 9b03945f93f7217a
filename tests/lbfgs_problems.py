"""Deterministic L-BFGS test problems shared by tests/golden/make_lbfgs_golden.py (which runs
the reference optimizer, optimizer.py:76-168, on them) and the oracle / device tests.

Each problem: name -> (objective(x) -> (f, g) in numpy fp64, x0, options dict).
"""

from __future__ import annotations

import numpy as np


def _quadratic(n=40, cond=100.0, seed=3):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.geomspace(1.0, cond, n)
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    b = rng.standard_normal(n)

    def f(x):
        ax = a @ x
        return 0.5 * x @ ax - b @ x, ax - b

    return f, np.zeros(n)


def _rosenbrock(m=4):
    def f(x):
        xo, xe = x[0::2], x[1::2]
        t1 = 10.0 * (xe - xo**2)
        t2 = 1.0 - xo
        val = float(np.sum(t1**2 + t2**2))
        g = np.zeros_like(x)
        g[0::2] = -40.0 * xo * t1 - 2.0 * t2
        g[1::2] = 20.0 * t1
        return val, g

    return f, np.tile([-1.2, 1.0], m)


def _logcosh(n=64, seed=5):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal(n) * 2.0
    w = rng.uniform(0.5, 2.0, n)

    def f(x):
        z = x - c
        return float(np.sum(w * np.log(np.cosh(z)))) + 1e-3 * float(x @ x), w * np.tanh(z) + 2e-3 * x

    return f, np.zeros(n)


def _nan_after_start(n=6):
    x0 = np.linspace(-1.0, 1.0, n)

    def f(x):
        if np.array_equal(x, x0):
            return float(x @ x), 2.0 * x
        return float("nan"), np.zeros_like(x)

    return f, x0


def _flat(n=5):
    def f(x):
        return 3.0, np.zeros_like(x)

    return f, np.ones(n)


def problems():
    q, q0 = _quadratic()
    r, r0 = _rosenbrock()
    lc, lc0 = _logcosh()
    nan, nan0 = _nan_after_start()
    fl, fl0 = _flat()
    return {
        "quadratic": (q, q0, {}),
        "quadratic_tight": (q, q0, dict(grad_tol=1e-10, f_tol=1e-14, max_iters=300)),
        "quadratic_mem1": (q, q0, dict(memory=1, max_iters=80)),
        "rosenbrock": (r, r0, dict(max_iters=400, grad_tol=1e-8, f_tol=1e-16)),
        "rosenbrock_maxit": (r, r0, dict(max_iters=7)),
        "logcosh": (lc, lc0, dict(grad_tol=1e-9, f_tol=1e-15, max_iters=200)),
        "line_search_failure": (nan, nan0, {}),
        "flat_start": (fl, fl0, {}),
    }

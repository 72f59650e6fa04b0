"""Host CGLS (the checker of kz_cgls and of make_inconsistent's x_LS).

TEST INFRASTRUCTURE ONLY (imported by tests/ alone; the package solves CGLS on
the device, csrc/kz_cgls.cu).  Restates cgls.py:18-75: conjugate gradients on
A^T A x = A^T b with products against A and A^T, the stop rule
||A^T (b - A x)|| <= tol ||A^T b|| checked on the recurred residual, one restart
from the iterate when the true normal-equations residual misses the target,
and a budget of 10 n + 100 iterations shared by both passes.
"""

from __future__ import annotations

import numpy as np


def _pass(A, b, x, target, budget):
    """One CGLS pass from x (cgls.py:18-39); returns (x, iterations used)."""
    r = b - A @ x
    s = A.T @ r
    p = s.copy()
    gamma = float(s @ s)
    used = 0
    while used < budget and np.sqrt(gamma) > target:
        t = A @ p
        delta = float(t @ t)
        if delta == 0.0:
            break
        step = gamma / delta
        x += step * p
        r -= step * t
        s = A.T @ r
        g_new = float(s @ s)
        p = s + (g_new / gamma) * p
        gamma = g_new
        used += 1
    return x, used


def cgls(A, b, tol=1e-10, max_it=None):
    """x_LS (cgls.py:42-75); raises RuntimeError when the budget runs out."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    budget = 10 * A.shape[1] + 100 if max_it is None else int(max_it)
    norm_atb = float(np.linalg.norm(A.T @ b))
    x = np.zeros(A.shape[1])
    if norm_atb == 0.0:
        return x
    target = tol * norm_atb
    left = budget
    for _ in range(2):
        x, used = _pass(A, b, x, target, left)
        left -= used
        if float(np.linalg.norm(A.T @ (A @ x - b))) <= target:
            return x
        if left <= 0:
            break
    raise RuntimeError(f"CGLS did not reach tol={tol} within {budget} iterations")

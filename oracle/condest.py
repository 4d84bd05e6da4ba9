"""Oracle: Hager's 1-norm estimates (condest.cpp:11-49).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import numpy as np


def estimate_norm_1(n: int, apply, apply_adjoint) -> float:
    """condest.cpp:11-41: every candidate is ||A x||_1 with ||x||_1 = 1, so the result never
    exceeds ||A||_1."""
    if n < 1:
        raise ValueError("estimate_norm_1: dimension must be positive")
    x = np.full(n, 1.0 / n, dtype=np.complex128)
    best = 0.0
    previous = -1
    for iteration in range(6):
        y = apply(x)
        estimate = float(np.sum(np.abs(y)))
        if iteration > 0 and estimate <= best:
            break
        best = max(best, estimate)
        a = np.abs(y)
        xi = np.where(a == 0.0, 1.0 + 0.0j, y / np.where(a == 0.0, 1.0, a))
        z = apply_adjoint(xi)
        pivot = int(np.argmax(np.abs(z)))
        if pivot == previous:
            break
        x = np.zeros(n, dtype=np.complex128)
        x[pivot] = 1.0
        previous = pivot
    return best


def estimate_condition_1norm(n: int, apply, apply_adjoint, solve, solve_adjoint) -> float:
    """condest.cpp:43-49."""
    return estimate_norm_1(n, apply, apply_adjoint) * estimate_norm_1(n, solve, solve_adjoint)

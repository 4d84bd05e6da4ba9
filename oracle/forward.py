"""Oracle: per-time contour forward solves and the pooled multi-time batch.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Restates /root/reference/proj/src/forward.cpp:17-198 (Crank-Nicolson,
forward.cpp:200-258, is a "next" row and not restated here).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .shifted_solver import (ConvergenceError, ShiftedPencil, ShiftedSolveOptions,
                             select_preconditioner_shifts, solve_shifted_direct,
                             solve_shifted_flexible, solve_shifted_single)
from .talbot import TalbotParams, build_contour, inverse_laplace_sum, qhat_step


@dataclass
class SolverConfig:
    """forward.hpp:18-23 (kind 'single' | 'flexible' | 'direct')."""

    kind: str = "flexible"
    variant: str = "gmres"
    tol: float = 1e-10
    maxit: int = 0


@dataclass
class ForwardProblem:
    """forward.hpp:27-35 (stiffness / mass instead of the AssembledOperators pointer)."""

    stiffness: object
    mass: object
    source: np.ndarray
    rate: float = 0.0
    initial_head: Optional[np.ndarray] = None
    times: List[float] = field(default_factory=list)
    n_quad: int = 40
    contour: TalbotParams = TalbotParams()


@dataclass
class TimeDiagnostics:
    """forward.hpp:37-41."""

    iterations: int = 0
    all_converged: bool = True
    shift_residuals: List[float] = field(default_factory=list)


@dataclass
class HeadSolution:
    """forward.hpp:43-46."""

    heads: np.ndarray
    diagnostics: List[TimeDiagnostics]


def _check_problem(problem: ForwardProblem) -> None:
    """forward.cpp:19-33."""
    if problem.stiffness is None or problem.mass is None:
        raise ValueError("solve_forward: missing operators")
    if len(problem.times) == 0:
        raise ValueError("solve_forward: no target times")
    previous = 0.0
    for t in problem.times:
        if not (t > 0.0):
            raise ValueError("solve_forward: times must be positive")
        if t < previous:
            raise ValueError("solve_forward: times must be ascending")
        previous = t


def solve_family(pencil, rhs, shifts, solver: SolverConfig, diag: Optional[TimeDiagnostics]):
    """forward.cpp:40-71."""
    if solver.kind == "direct":
        return solve_shifted_direct(pencil, rhs, shifts)
    options = ShiftedSolveOptions(variant=solver.variant, tol=solver.tol, maxit=solver.maxit,
                                  record_history=False)
    if solver.kind == "single":
        result = solve_shifted_single(pencil, rhs, shifts,
                                      select_preconditioner_shifts(shifts).taus[0], options)
    else:
        result = solve_shifted_flexible(pencil, rhs, shifts, select_preconditioner_shifts(shifts),
                                        options)
    if diag is not None:
        diag.iterations = max(diag.iterations, result.iterations)
        diag.all_converged = diag.all_converged and result.all_converged
        diag.shift_residuals += [st.true_residual for st in result.shifts]
    if not result.all_converged:
        raise ConvergenceError(
            f"shifted solve: {len(result.unconverged())} of {len(shifts)} shifts unconverged "
            f"after {result.iterations} iterations", result.unconverged())
    return result.solutions


def _with_initial(problem: ForwardProblem) -> bool:
    ih = problem.initial_head
    return ih is not None and len(ih) > 0 and float(np.max(np.abs(ih))) > 0.0


def solve_forward(problem: ForwardProblem, solver: SolverConfig = SolverConfig(),
                  pencil: Optional[ShiftedPencil] = None) -> HeadSolution:
    """forward.cpp:75-118."""
    _check_problem(problem)
    if pencil is None:
        pencil = ShiftedPencil(problem.stiffness, problem.mass)
    n_times = len(problem.times)
    with_initial = _with_initial(problem)
    heads = np.zeros((pencil.rows(), n_times))
    diags = [TimeDiagnostics() for _ in range(n_times)]
    rhs_source = np.asarray(problem.source, dtype=np.complex128)
    rhs_initial = pencil.apply_mass(np.asarray(problem.initial_head, dtype=np.complex128)) \
        if with_initial else None
    for it, t in enumerate(problem.times):
        contour = build_contour(problem.n_quad, t, problem.contour)
        shifts = list(contour.nodes)
        values = np.zeros((pencil.rows(), contour.n_half()), dtype=np.complex128)
        if problem.rate != 0.0:
            xs = solve_family(pencil, rhs_source, shifts, solver, diags[it])
            for k in range(contour.n_half()):
                values[:, k] = qhat_step(problem.rate, contour.nodes[k]) * xs[:, k]
        if with_initial:
            values += solve_family(pencil, rhs_initial, shifts, solver, diags[it])
        heads[:, it] = inverse_laplace_sum(contour, values)
    return HeadSolution(heads, diags)


def solve_forward_batch(problem: ForwardProblem, solver: SolverConfig = SolverConfig(),
                        pencil: Optional[ShiftedPencil] = None) -> HeadSolution:
    """forward.cpp:126-198: pooled shifts of all times, one flexible solve."""
    _check_problem(problem)
    if pencil is None:
        pencil = ShiftedPencil(problem.stiffness, problem.mass)
    n_times = len(problem.times)
    with_initial = _with_initial(problem)
    contours = [build_contour(problem.n_quad, t, problem.contour) for t in problem.times]
    pooled = [z for c in contours for z in c.nodes]
    schedule = select_preconditioner_shifts(pooled)
    pooled_diag = TimeDiagnostics()

    def solve_pooled(rhs):
        options = ShiftedSolveOptions(variant=solver.variant, tol=solver.tol, maxit=solver.maxit,
                                      record_history=False)
        if solver.kind == "direct":
            return solve_shifted_direct(pencil, rhs, pooled)
        result = solve_shifted_flexible(pencil, rhs, pooled, schedule, options)
        pooled_diag.iterations = max(pooled_diag.iterations, result.iterations)
        pooled_diag.all_converged = pooled_diag.all_converged and result.all_converged
        pooled_diag.shift_residuals += [st.true_residual for st in result.shifts]
        if not result.all_converged:
            raise ConvergenceError(
                f"batch solve: {len(result.unconverged())} of {len(pooled)} pooled shifts "
                f"unconverged after {result.iterations} iterations", result.unconverged())
        return result.solutions

    x_source = solve_pooled(np.asarray(problem.source, dtype=np.complex128)) \
        if problem.rate != 0.0 else None
    x_initial = solve_pooled(pencil.apply_mass(np.asarray(problem.initial_head,
                                                          dtype=np.complex128))) \
        if with_initial else None
    heads = np.zeros((pencil.rows(), n_times))
    offset = 0
    for it, contour in enumerate(contours):
        values = np.zeros((pencil.rows(), contour.n_half()), dtype=np.complex128)
        for k in range(contour.n_half()):
            if problem.rate != 0.0:
                values[:, k] = qhat_step(problem.rate, contour.nodes[k]) * x_source[:, offset + k]
            if with_initial:
                values[:, k] += x_initial[:, offset + k]
        heads[:, it] = inverse_laplace_sum(contour, values)
        offset += contour.n_half()
    return HeadSolution(heads, [pooled_diag] * n_times)


def crank_nicolson(stiffness, mass, source, rate: float, initial_head, dt: float, sample_times,
                   return_steps: bool = False):
    """forward.cpp:200-258: one factorisation of M + dt/2 K (SimplicialLDLT there, SuperLU
    here) reused for every step; samples by linear interpolation between the two states
    around each sample time."""
    import scipy.sparse.linalg as spla
    if not dt > 0.0:
        raise ValueError("crank_nicolson: dt must be positive")
    if len(sample_times) == 0:
        raise ValueError("crank_nicolson: no sample times")
    t_end = max(sample_times)
    lhs = (mass + (0.5 * dt) * stiffness).tocsc()
    solver = spla.splu(lhs)
    rhs_op = (mass - (0.5 * dt) * stiffness).tocsr()
    forcing = dt * rate * np.asarray(source, dtype=np.float64)
    n = stiffness.shape[0]
    head = np.zeros(n) if initial_head is None or len(initial_head) == 0 else np.asarray(initial_head, dtype=np.float64)
    samples = np.zeros((n, len(sample_times)))
    filled = [False] * len(sample_times)

    def record(t_prev, head_prev, t_now, head_now):
        for s, target in enumerate(sample_times):
            if filled[s]:
                continue
            if target <= t_now + 1e-9 * dt:
                if abs(target - t_now) <= 1e-9 * dt or t_now == t_prev:
                    samples[:, s] = head_now
                else:
                    w = (target - t_prev) / (t_now - t_prev)
                    samples[:, s] = (1.0 - w) * head_prev + w * head_now
                filled[s] = True

    record(0.0, head, 0.0, head)
    steps = 0
    t = 0.0
    while t < t_end - 1e-9 * dt:
        head_prev = head
        head = solver.solve(rhs_op @ head + forcing)
        t_prev = t
        t += dt
        steps += 1
        record(t_prev, head_prev, t, head)
    return (samples, steps) if return_steps else samples

"""Oracle: the geostatistical Gauss-Newton inversion (inversion.hpp:17-91, inversion.cpp:17-201).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Dense NumPy restatement: jittered
Cholesky of Q (cpp:17-33), misfit / prior term / objective (cpp:58-76), the saddle-point step
with step halving (cpp:78-148) and the outer loop with its stopping rules (cpp:150-186).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np


class FactorizationError(RuntimeError):
    pass


@dataclass
class InversionProblem:
    """inversion.hpp:17-27 (predict / jacobian_and_predict: s -> h, s -> (J, h))."""

    y: np.ndarray
    r_diag: np.ndarray
    drift: np.ndarray   # X, n_s x p
    prior: np.ndarray   # Q, n_s x n_s
    predict: Callable
    jacobian_and_predict: Callable


@dataclass
class GnOptions:
    """inversion.hpp:29-34."""

    max_gn: int = 15
    rtol: float = 1e-3
    damping: bool = True
    max_halvings: int = 5


@dataclass
class GnIterate:
    """inversion.hpp:36-47."""

    s: np.ndarray = None
    beta: np.ndarray = None
    xi: np.ndarray = None
    objective: float = 0.0
    misfit: float = 0.0
    prior: float = 0.0
    step_norm: float = 0.0
    alpha: float = 1.0
    saddle_residual: float = 0.0
    drift_violation: float = 0.0


@dataclass
class InversionResult:
    s_hat: np.ndarray = None
    beta_hat: np.ndarray = None
    history: List[GnIterate] = field(default_factory=list)
    converged: bool = False
    stop_reason: str = ""


def jittered_cholesky(q: np.ndarray) -> np.ndarray:
    """inversion.cpp:17-33: 1e-10 x max diag, doubled, up to six retries."""
    scale = float(np.max(np.diag(q)))
    jitter = 1e-10 * scale
    for attempt in range(7):
        work = q.copy()
        if attempt > 0:
            work[np.diag_indices_from(work)] += jitter
            jitter *= 2.0
        try:
            return np.linalg.cholesky(work)
        except np.linalg.LinAlgError:
            continue
    raise FactorizationError("GaussNewtonSolver: prior Cholesky failed after max jitter")


def check_problem(problem: InversionProblem) -> None:
    """inversion.cpp:35-48."""
    n_s = problem.prior.shape[0]
    if problem.prior.shape[1] != n_s or problem.drift.shape[0] != n_s:
        raise ValueError("InversionProblem: Q and X dimensions disagree")
    if np.any(problem.r_diag <= 0.0):
        raise ValueError("InversionProblem: R diagonal must be positive")
    if problem.r_diag.size != problem.y.size:
        raise ValueError("InversionProblem: R and y dimensions disagree")


class GaussNewtonSolver:
    """inversion.hpp:51-79."""

    def __init__(self, problem: InversionProblem):
        check_problem(problem)
        self.problem = problem
        self.prior_chol = jittered_cholesky(problem.prior)

    def misfit(self, predictions) -> float:
        r = self.problem.y - predictions
        return 0.5 * float(np.sum(r * r / self.problem.r_diag))

    def prior_term(self, s, beta) -> float:
        import scipy.linalg as sla
        anomaly = s - self.problem.drift @ beta
        white = sla.solve_triangular(self.prior_chol, anomaly, lower=True)
        return 0.5 * float(white @ white)

    def objective(self, s, beta) -> float:
        return self.misfit(self.problem.predict(s)) + self.prior_term(s, beta)

    def step(self, s, beta, options: GnOptions = GnOptions()) -> GnIterate:
        """inversion.cpp:78-148."""
        pb = self.problem
        jac, pred = pb.jacobian_and_predict(s)
        n_y, p = pb.y.size, pb.drift.shape[1]
        jq = jac @ pb.prior
        jx = jac @ pb.drift
        saddle = np.zeros((n_y + p, n_y + p))
        saddle[:n_y, :n_y] = jq @ jac.T
        saddle[np.arange(n_y), np.arange(n_y)] += pb.r_diag
        saddle[:n_y, n_y:] = jx
        saddle[n_y:, :n_y] = jx.T
        rhs = np.zeros(n_y + p)
        rhs[:n_y] = pb.y - pred + jac @ s
        try:
            sol = np.linalg.solve(saddle, rhs)
        except np.linalg.LinAlgError:
            sol = np.full(n_y + p, np.nan)
        if not np.all(np.isfinite(sol)):
            raise FactorizationError(
                "gauss_newton_step: saddle system solve failed (rank-deficient J Q J^T + R or J X block)")
        it = GnIterate()
        it.xi = sol[:n_y]
        it.beta = sol[n_y:]
        it.saddle_residual = float(np.linalg.norm(saddle @ sol - rhs) / np.linalg.norm(rhs))
        xn = np.linalg.norm(it.xi)
        it.drift_violation = float(np.linalg.norm(jx.T @ it.xi) / xn) if p > 0 and xn > 0.0 else 0.0
        s_full = pb.drift @ it.beta + jq.T @ it.xi
        objective_old = self.misfit(pred) + self.prior_term(s, beta)
        alpha = 1.0
        accepted = False
        for _ in range((options.max_halvings if options.damping else 0) + 1):
            s_trial = s + alpha * (s_full - s)
            beta_trial = beta + alpha * (it.beta - beta)
            obj = self.objective(s_trial, beta_trial)
            if obj <= objective_old or not options.damping:
                it.s, it.beta, it.objective = s_trial, beta_trial, obj
                it.misfit = self.misfit(pb.predict(s_trial))
                it.prior = it.objective - it.misfit
                it.alpha = alpha
                accepted = True
                break
            alpha *= 0.5
        if not accepted:
            it.s, it.beta, it.objective = s, beta, objective_old
            it.misfit = self.misfit(pred)
            it.prior = objective_old - it.misfit
            it.alpha = 0.0
        it.step_norm = float(np.linalg.norm(it.s - s))
        return it

    def invert(self, s0, beta0, options: GnOptions = GnOptions()) -> InversionResult:
        """inversion.cpp:150-186."""
        if options.max_gn < 1:
            raise ValueError("invert: max_gn must be at least 1")
        res = InversionResult()
        s, beta = s0, beta0
        objective_prev = self.objective(s, beta)
        for _ in range(options.max_gn):
            it = self.step(s, beta, options)
            s, beta = it.s, it.beta
            res.history.append(it)
            if it.alpha == 0.0:
                res.converged = False
                res.stop_reason = "step stalled: damping could not decrease the objective"
                break
            rel_step = it.step_norm / max(float(np.linalg.norm(s)), 1e-300)
            rel_decrease = (objective_prev - it.objective) / max(abs(objective_prev), 1e-300)
            objective_prev = it.objective
            if rel_step <= options.rtol:
                res.converged = True
                res.stop_reason = "relative step norm below rtol"
                break
            if 0.0 <= rel_decrease <= options.rtol:
                res.converged = True
                res.stop_reason = "relative objective decrease below rtol"
                break
        if not res.stop_reason:
            res.stop_reason = "max_gn reached"
        res.s_hat, res.beta_hat = s, beta
        return res


def grid_covariance(shape, h, variance, corr_lengths) -> np.ndarray:
    """The dense exponential covariance var exp(-|(dx/l0, dy/l1[, dz/l2])|) between the cell
    centres of an FD grid (x fastest) -- fields.cpp:18-38 on the grid, anisotropic lengths."""
    axes = [np.arange(n) * h for n in shape]
    pts = np.stack([g.ravel() for g in np.meshgrid(*axes, indexing="ij")], axis=1)
    pts = pts.reshape(*shape, len(shape)).transpose(*reversed(range(len(shape))), len(shape)).reshape(-1, len(shape))
    d = (pts[:, None, :] - pts[None, :, :]) / np.asarray(corr_lengths)[: len(shape)]
    return variance * np.exp(-np.sqrt((d * d).sum(-1)))

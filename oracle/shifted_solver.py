"""Oracle: flexible shifted FOM/GMRES (FGMRES-Sh, Algorithm 1) and its helpers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Restates /root/reference/proj/src/shifted_solver.cpp and
include/laptomo/shifted_solver.hpp; the factorisation plugin
(src/factorization.cpp:14-39, Eigen SparseLU<COLAMD>) is SuperLU with COLAMD.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

BREAKDOWN_TOL = 1e-14  # shifted_solver.cpp:17


class FactorizationError(RuntimeError):
    """errors.hpp:14-17."""


class ConvergenceError(RuntimeError):
    """errors.hpp:20-25: carries the unconverged shift indices."""

    def __init__(self, what: str, unconverged: List[int]):
        super().__init__(what)
        self.unconverged_shifts = list(unconverged)


@dataclass
class PreconditionerSchedule:
    """shifted_solver.hpp:25-33."""

    taus: List[complex]
    pattern: List[int]

    def tau_at(self, iteration: int) -> complex:
        return self.taus[self.pattern[iteration % len(self.pattern)]]


def single_tau_schedule(tau: complex) -> PreconditionerSchedule:
    """shifted_solver.cpp:81-83."""
    return PreconditionerSchedule([complex(tau)], [0])


def select_preconditioner_shifts(shifts) -> PreconditionerSchedule:
    """shifted_solver.cpp:85-104: tau1 = min Re (ties: smaller Im, then index),
    tau2 = max Re; pattern [0,0,0,1,1]; single schedule when tau1 == tau2."""
    shifts = [complex(s) for s in shifts]
    if not shifts:
        raise ValueError("select_preconditioner_shifts: empty shift list")

    def less(a: complex, b: complex) -> bool:
        if a.real != b.real:
            return a.real < b.real
        return a.imag < b.imag

    i_min = i_max = 0
    for i in range(1, len(shifts)):
        if less(shifts[i], shifts[i_min]):
            i_min = i
        if less(shifts[i_max], shifts[i]):
            i_max = i
    tau1, tau2 = shifts[i_min], shifts[i_max]
    if tau1 == tau2:
        return single_tau_schedule(tau1)
    return PreconditionerSchedule([tau1, tau2], [0, 0, 0, 1, 1])


@dataclass
class ShiftedSolveOptions:
    """shifted_solver.hpp:44-50 (variant 'gmres' | 'fom')."""

    variant: str = "gmres"
    tol: float = 1e-10
    maxit: int = 0
    keep_basis: bool = False
    record_history: bool = True


@dataclass
class ShiftStatus:
    """shifted_solver.hpp:52-58."""

    converged: bool = False
    iteration: int = 0
    estimate: float = math.inf
    true_residual: float = math.nan
    history: List[float] = field(default_factory=list)


@dataclass
class FlexibleBasisState:
    """shifted_solver.hpp:63-74."""

    V: np.ndarray
    U: np.ndarray
    Hbar: np.ndarray
    taus: np.ndarray
    beta: float

    def steps(self) -> int:
        return int(self.Hbar.shape[1])

    def shifted_hessenberg(self, z: complex) -> np.ndarray:
        return shifted_hessenberg(self.Hbar, self.taus, self.steps(), z)


@dataclass
class ShiftedSolveResult:
    """shifted_solver.hpp:76-84."""

    solutions: np.ndarray
    iterations: int = 0
    all_converged: bool = False
    shifts: List[ShiftStatus] = field(default_factory=list)
    basis: Optional[FlexibleBasisState] = None

    def unconverged(self) -> List[int]:
        return [k for k, s in enumerate(self.shifts) if not s.converged]


class SparseComplexFactorization:
    """factorization.hpp:19-27 / factorization.cpp:14-33 (SuperLU, COLAMD)."""

    def __init__(self, matrix):
        matrix = sp.csc_matrix(matrix, dtype=np.complex128)
        try:
            self._lu = spla.splu(matrix, permc_spec="COLAMD")
        except RuntimeError as exc:  # singular
            raise FactorizationError("sparse LU factorization failed") from exc

    def rows(self) -> int:
        return self._lu.shape[0]

    def solve(self, rhs):
        return self._lu.solve(np.asarray(rhs, dtype=np.complex128))

    def solve_adjoint(self, rhs):
        return self._lu.solve(np.asarray(rhs, dtype=np.complex128), trans="H")


def factorize_sparse(matrix) -> SparseComplexFactorization:
    """factorization.cpp:37-39."""
    return SparseComplexFactorization(matrix)


class ShiftedPencil:
    """shifted_solver.hpp:88-104, shifted_solver.cpp:106-128."""

    def __init__(self, stiffness, mass):
        self.stiffness = sp.csr_matrix(stiffness, dtype=np.complex128)
        self.mass = sp.csr_matrix(mass, dtype=np.complex128)
        self._cache: list = []

    def rows(self) -> int:
        return self.stiffness.shape[0]

    def apply(self, z, x):
        return self.stiffness @ x + z * (self.mass @ x)

    def apply_adjoint(self, z, x):
        return self.stiffness @ x + np.conj(z) * (self.mass @ x)

    def apply_mass(self, x):
        return self.mass @ x

    def factorization(self, tau) -> SparseComplexFactorization:
        tau = complex(tau)
        for cached_tau, fact in self._cache:
            if cached_tau == tau:
                return fact
        shifted = (self.stiffness + tau * self.mass).tocsc()
        fact = factorize_sparse(shifted)
        self._cache.append((tau, fact))
        return fact

    def factorization_count(self) -> int:
        return len(self._cache)


def shifted_hessenberg(hbar, taus, m: int, z: complex) -> np.ndarray:
    """shifted_solver.cpp:26-34: Hbar_m(z; T_m) = [I; 0] + Hbar_m (z I - T_m)."""
    hz = np.array(hbar[: m + 1, :m], dtype=np.complex128, copy=True)
    for l in range(m):
        hz[:, l] *= (z - taus[l])
        hz[l, l] += 1.0
    return hz


def _small_solve_fom(hz, beta):
    """shifted_solver.cpp:36-51 (PartialPivLU on the square top)."""
    m = hz.shape[1]
    rhs = np.zeros(m, dtype=np.complex128)
    rhs[0] = beta
    with np.errstate(all="ignore"):
        try:
            y = np.linalg.solve(hz[:m, :], rhs)
        except np.linalg.LinAlgError:
            return None, math.inf
    if not np.all(np.isfinite(y)):
        return None, math.inf
    return y, abs(hz[m, m - 1] * y[m - 1])


def _small_solve_gmres(hz, beta):
    """shifted_solver.cpp:53-65 (Householder QR least squares)."""
    m = hz.shape[1]
    rhs = np.zeros(m + 1, dtype=np.complex128)
    rhs[0] = beta
    with np.errstate(all="ignore"):
        q, r = np.linalg.qr(hz, mode="reduced")
        try:
            y = np.linalg.solve(r, q.conj().T @ rhs)
        except np.linalg.LinAlgError:
            return None, math.inf
    if not np.all(np.isfinite(y)):
        return None, math.inf
    return y, float(np.linalg.norm(rhs - hz @ y))


def run_flexible(pencil: ShiftedPencil, b, shifts, schedule: PreconditionerSchedule,
                 options: ShiftedSolveOptions) -> ShiftedSolveResult:
    """shifted_solver.cpp:132-287, step for step."""
    b = np.asarray(b, dtype=np.complex128)
    n = pencil.rows()
    shifts = [complex(s) for s in shifts]
    n_shifts = len(shifts)
    result = ShiftedSolveResult(np.zeros((n, n_shifts), dtype=np.complex128))
    result.shifts = [ShiftStatus() for _ in range(n_shifts)]
    if n_shifts == 0:
        result.all_converged = True
        return result
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        for st in result.shifts:
            st.converged, st.estimate, st.true_residual = True, 0.0, 0.0
        result.all_converged = True
        return result

    maxit = min(n, options.maxit) if options.maxit > 0 else min(n, 10 * n_shifts)
    small = _small_solve_fom if options.variant == "fom" else _small_solve_gmres

    V = np.zeros((n, maxit + 1), dtype=np.complex128)
    U = np.zeros((n, maxit), dtype=np.complex128)
    hbar = np.zeros((maxit + 1, maxit), dtype=np.complex128)
    taus = np.zeros(maxit, dtype=np.complex128)
    V[:, 0] = b / beta
    verify_at = [options.tol] * n_shifts
    n_converged = 0
    m = 0
    breakdown = False

    j = 0
    while j < maxit and n_converged < n_shifts:
        tau = schedule.tau_at(j)
        taus[j] = tau
        U[:, j] = pencil.factorization(tau).solve(V[:, j])
        s = pencil.apply_mass(U[:, j])
        # MGS with one conditional re-orthogonalisation (cpp:196-210).
        norm_before = float(np.linalg.norm(s))
        for i in range(j + 1):
            hij = np.vdot(V[:, i], s)
            hbar[i, j] = hij
            s = s - hij * V[:, i]
        if np.linalg.norm(s) < norm_before / math.sqrt(2.0):
            for i in range(j + 1):
                corr = np.vdot(V[:, i], s)
                hbar[i, j] += corr
                s = s - corr * V[:, i]
        h_next = float(np.linalg.norm(s))
        hbar[j + 1, j] = h_next
        m = j + 1
        breakdown = h_next <= BREAKDOWN_TOL * norm_before
        if not breakdown:
            V[:, j + 1] = s / h_next

        for k in range(n_shifts):
            status = result.shifts[k]
            if status.converged:
                continue
            hz = shifted_hessenberg(hbar, taus, m, shifts[k])
            y, est = small(hz, beta)
            if y is None:
                if options.record_history:
                    status.history.append(status.estimate)
                continue
            status.estimate = est / beta
            if options.record_history:
                status.history.append(status.estimate)
            if status.estimate <= verify_at[k] or breakdown:
                x = U[:, :m] @ y
                true_rel = float(np.linalg.norm(b - pencil.apply(shifts[k], x))) / beta
                if true_rel <= options.tol or breakdown:
                    status.converged = True
                    status.iteration = m
                    status.true_residual = true_rel
                    result.solutions[:, k] = x
                    n_converged += 1
                else:
                    verify_at[k] = status.estimate / 2.0
        if breakdown:
            break
        j += 1

    result.iterations = m
    result.all_converged = n_converged == n_shifts
    if options.keep_basis:
        Vk = V[:, : m + 1].copy()
        if breakdown:
            Vk[:, m] = 0.0
        result.basis = FlexibleBasisState(Vk, U[:, :m].copy(), hbar[: m + 1, :m].copy(),
                                          taus[:m].copy(), beta)
    if not result.all_converged and m > 0:
        for k in range(n_shifts):
            status = result.shifts[k]
            if status.converged:
                continue
            hz = shifted_hessenberg(hbar, taus, m, shifts[k])
            y, _ = small(hz, beta)
            if y is not None:
                x = U[:, :m] @ y
                status.true_residual = float(np.linalg.norm(b - pencil.apply(shifts[k], x))) / beta
                result.solutions[:, k] = x
    return result


def solve_shifted_flexible(pencil, b, shifts, schedule, options=None) -> ShiftedSolveResult:
    """shifted_solver.cpp:291-299."""
    if not schedule.taus or not schedule.pattern:
        raise ValueError("solve_shifted_flexible: empty preconditioner schedule")
    return run_flexible(pencil, b, shifts, schedule, options or ShiftedSolveOptions())


def solve_shifted_single(pencil, b, shifts, tau, options=None) -> ShiftedSolveResult:
    """shifted_solver.cpp:310-314."""
    return run_flexible(pencil, b, shifts, single_tau_schedule(tau), options or ShiftedSolveOptions())


def solve_shifted_direct(pencil, b, shifts) -> np.ndarray:
    """shifted_solver.cpp:324-332: one factorisation per shift."""
    out = np.zeros((pencil.rows(), len(shifts)), dtype=np.complex128)
    for k, z in enumerate(shifts):
        out[:, k] = pencil.factorization(z).solve(np.asarray(b, dtype=np.complex128))
    return out


def residual_estimate(state: FlexibleBasisState, z: complex, y_fom) -> float:
    """shifted_solver.cpp:334-343."""
    m = state.steps()
    if m < 1 or len(y_fom) != m:
        raise ValueError("residual_estimate: FOM coefficients of length m required")
    h_next = state.Hbar[m, m - 1]
    tau_m = state.taus[m - 1]
    return abs(h_next * (z - tau_m) * y_fom[m - 1])

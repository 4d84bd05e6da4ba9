"""Python mirror of the reference's public solver API (namespace laptomo,
/root/reference/proj/include/laptomo), backed by the sm_100a library through
the C ABI (include/laptomo_gpu.h).  Same names, argument meaning and error
behaviour as the reference:

  build_contour / inverse_laplace_sum / qhat_step        talbot.hpp:46-63
  select_preconditioner_shifts / single_tau_schedule     shifted_solver.hpp:36-42
  ShiftedPencil (apply, apply_adjoint, apply_mass,
                 factorization, factorization_count)     shifted_solver.hpp:88-104
  solve_shifted_flexible / _single / _direct,
  residual_estimate                                      shifted_solver.hpp:110-138
  solve_forward / solve_forward_batch                    forward.hpp:52-61
  solve_adjoint_fields, ThtExperiment, ThtForwardModel,
  assemble_jacobian                                      jacobian.hpp:22-101

Exceptions: std::invalid_argument -> ValueError, FactorizationError,
ConvergenceError (with .unconverged_shifts).

Difference at the boundary: the reference's ShiftedPencil takes assembled
sparse (K, M); here a pencil is built from a structured grid plus per-cell log
fields (`Grid`, the cell-centred FD discretisation of the BASELINE configs),
and assembled on the device.  Solutions of batched calls are RHS-major.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import capi
from .capi import (ConvergenceError, FactorizationError, LtComplex, check, cptr, dptr, lc, lib)

__all__ = [
    "ConvergenceError", "FactorizationError", "Context", "TalbotParams", "TalbotContour", "build_contour",
    "inverse_laplace_sum", "qhat_step", "PreconditionerSchedule", "single_tau_schedule",
    "select_preconditioner_shifts", "Grid", "Mesh2D", "build_mesh", "ShiftedPencil", "ShiftedSolveOptions",
    "ShiftStatus",
    "FlexibleBasisState", "ShiftedSolveResult", "solve_shifted_flexible", "solve_shifted_single",
    "solve_shifted_direct", "residual_estimate", "SolverConfig", "ForwardProblem", "TimeDiagnostics",
    "HeadSolution", "solve_forward", "solve_forward_batch", "solve_adjoint_fields", "ThtExperiment",
    "JacobianResult", "ThtForwardModel", "assemble_jacobian", "default_context",
]


# ---- context ------------------------------------------------------------------------------
class Context:
    """One device + one stream (lt_ctx)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().lt_ctx_create(device, C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        check(lib().lt_ctx_synchronize(self._h))

    def stream(self) -> int:
        return int(lib().lt_ctx_stream(self._h) or 0)

    def set_profiling(self, enabled: bool):
        check(lib().lt_ctx_set_profiling(self._h, int(enabled)))

    def reset_profile(self):
        check(lib().lt_ctx_reset_profile(self._h))

    def set_profile_sampling(self, every: int):
        check(lib().lt_ctx_set_profile_sampling(self._h, int(every)))

    def launch_count(self) -> int:
        return int(lib().lt_ctx_launch_count(self._h))

    def profile(self):
        """{kernel class: (total_ms, launches, algorithmic_bytes)}."""
        n = lib().lt_ctx_profile(self._h, 0, None, None, None, None)
        if n <= 0:
            return {}
        names = C.create_string_buffer(64 * n)
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        by = np.zeros(n)
        lib().lt_ctx_profile(self._h, n, names, dptr(ms), cnt.ctypes.data_as(capi.PI64), dptr(by))
        out = {}
        for i in range(n):
            name = names.raw[64 * i: 64 * (i + 1)].split(b"\0", 1)[0].decode()
            out[name] = (float(ms[i]), int(cnt[i]), float(by[i]))
        return out

    def close(self):
        if self._h:
            lib().lt_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---- talbot ------------------------------------------------------------------------------
@dataclass(frozen=True)
class TalbotParams:
    sigma0: float = -0.6122
    mu0: float = 0.5017
    nu: float = 0.2645 / 0.5017
    alpha: float = 0.6407

    def c(self) -> capi.LtTalbotParams:
        return capi.LtTalbotParams(self.sigma0, self.mu0, self.nu, self.alpha)


@dataclass
class TalbotContour:
    n_quad: int
    time: float
    sigma: float
    mu: float
    nu: float
    alpha: float
    thetas: np.ndarray
    nodes: np.ndarray
    dnodes: np.ndarray
    weights: np.ndarray

    def n_half(self) -> int:
        return int(self.nodes.shape[0])


def build_contour(n_quad: int, time: float, params: TalbotParams = TalbotParams()) -> TalbotContour:
    nh = max(n_quad // 2, 0)
    th = np.zeros(max(nh, 1))
    z = np.zeros(max(nh, 1), dtype=np.complex128)
    dz = np.zeros_like(z)
    w = np.zeros_like(z)
    p = params.c()
    check(lib().lt_talbot_build(int(n_quad), float(time), C.byref(p), dptr(th), cptr(z), cptr(dz), cptr(w)))
    scale = n_quad / time
    return TalbotContour(n_quad, time, params.sigma0 * scale, params.mu0 * scale, params.nu, params.alpha,
                         th[:nh], z[:nh], dz[:nh], w[:nh])


def inverse_laplace_sum(contour: TalbotContour, values):
    """2 Re sum_k w_k F_k (talbot.cpp:82-94); host arithmetic on caller data, as in the
    reference (the device drivers recombine in basis form on the GPU)."""
    values = np.asarray(values)
    if values.ndim == 1:
        if values.shape[0] != contour.n_half():
            raise ValueError("inverse_laplace_sum: one value per retained node required")
        return float(2.0 * np.sum(contour.weights * values).real)
    if values.shape[1] != contour.n_half():
        raise ValueError("inverse_laplace_sum: one column per retained node required")
    return 2.0 * (values @ contour.weights).real


def qhat_step(q0: float, z: complex) -> complex:
    out = LtComplex()
    check(lib().lt_qhat_step(float(q0), lc(z), C.byref(out)))
    return complex(out.re, out.im)


# ---- fields ------------------------------------------------------------------------------
def sample_field_grid(ctx: "Context", shape: Sequence[int], h: float, variance: float,
                      corr_lengths: Sequence[float], mean: float, seed: int = 0,
                      noise: Optional[np.ndarray] = None) -> np.ndarray:
    """sample_field_on_mesh (fields.hpp:41-44, fields.cpp:84-123) on a structured grid, by
    circulant embedding on the device (lt_sample_field_grid): a GRF with covariance
    variance * exp(-|r / l|) on the cell centres, flat, x fastest.  `noise` (complex, shape
    2 * shape reversed, i.e. x fastest over the doubled grid) replaces the Philox normals."""
    dim = len(shape)
    sh = (C.c_int * dim)(*[int(v) for v in shape])
    cl = np.ascontiguousarray(np.asarray(corr_lengths, dtype=np.float64))
    if cl.size != dim:
        raise ValueError("sample_field_grid: one correlation length per axis")
    out = np.empty(int(np.prod(shape)), dtype=np.float64)
    nz = None
    if noise is not None:
        nz = np.ascontiguousarray(noise, dtype=np.complex128).ravel()
        if nz.size != int(np.prod([2 * v for v in shape])):
            raise ValueError("sample_field_grid: noise must hold prod(2 * shape) values")
    check(lib().lt_sample_field_grid(ctx._h, dim, sh, float(h), float(variance), dptr(cl), float(mean),
                                     int(seed), cptr(nz) if nz is not None else None, capi.LT_MEM_HOST,
                                     dptr(out)))
    return out


# ---- schedule ----------------------------------------------------------------------------
@dataclass
class PreconditionerSchedule:
    taus: List[complex]
    pattern: List[int]

    def tau_at(self, iteration: int) -> complex:
        return self.taus[self.pattern[iteration % len(self.pattern)]]


def single_tau_schedule(tau: complex) -> PreconditionerSchedule:
    return PreconditionerSchedule([complex(tau)], [0])


def select_preconditioner_shifts(shifts) -> PreconditionerSchedule:
    s = np.ascontiguousarray(np.asarray(list(shifts), dtype=np.complex128))
    taus = np.zeros(2, dtype=np.complex128)
    nt = C.c_int()
    pat = (C.c_int * 5)()
    pl = C.c_int()
    check(lib().lt_select_preconditioner_shifts(cptr(s) if s.size else None, int(s.size), cptr(taus),
                                                C.byref(nt), pat, C.byref(pl)))
    return PreconditionerSchedule([complex(t) for t in taus[: nt.value]], list(pat[: pl.value]))


# ---- pencil ------------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    """Cell-centred grid: shape (nx, ny[, nz]) cells of spacing h; cell a = (k ny + j) nx + i."""

    shape: tuple
    h: float

    @property
    def dim(self) -> int:
        return len(self.shape)

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.shape))

    def c(self) -> capi.LtGrid:
        shp = (C.c_int * 3)(*(list(self.shape) + [1] * (3 - len(self.shape))))
        return capi.LtGrid(capi.LT_GRID_FD_CELL, self.dim, shp, float(self.h))


@dataclass(frozen=True)
class Mesh2D:
    """The reference's structured P1 mesh (build_mesh, mesh.hpp:17-27 / mesh.cpp:14-52) as a
    device pencil geometry: per-element log fields (element 2c lower, 2c+1 upper triangle of
    cell c), unknowns = interior nodes in ascending node order (the reference's free dofs)."""

    n_per_side: int
    side_length: float

    @property
    def dim(self) -> int:
        return 2

    @property
    def n_elements(self) -> int:
        return 2 * (self.n_per_side - 1) ** 2

    @property
    def n_cells(self) -> int:  # parameters per log field
        return self.n_elements

    @property
    def n_free(self) -> int:
        return (self.n_per_side - 2) ** 2

    def spacing(self) -> float:
        return self.side_length / (self.n_per_side - 1)

    def c(self) -> capi.LtGrid:
        shp = (C.c_int * 3)(self.n_per_side, self.n_per_side, 1)
        return capi.LtGrid(capi.LT_GRID_P1_TRI, 2, shp, float(self.spacing()))


def build_mesh(n_per_side: int, side_length: float) -> Mesh2D:
    """mesh.cpp:14-20 argument checks."""
    if n_per_side < 2:
        raise ValueError("build_mesh: n_per_side must be at least 2")
    if not (side_length > 0.0):
        raise ValueError("build_mesh: side length must be positive")
    return Mesh2D(int(n_per_side), float(side_length))


class _Factorization:
    """SparseComplexFactorization view (factorization.hpp:19-27) of a prepared tau."""

    def __init__(self, pencil: "ShiftedPencil", tau: complex):
        self.pencil, self.tau = pencil, complex(tau)

    def rows(self) -> int:
        return self.pencil.rows()

    def solve(self, rhs):
        return self.pencil._solve(self.tau, rhs, adjoint=False)

    def solve_adjoint(self, rhs):
        return self.pencil._solve(self.tau, rhs, adjoint=True)


def _as_batch(x, n: int):
    x = np.asarray(x, dtype=np.complex128)
    single = x.ndim == 1
    xb = np.ascontiguousarray(x.reshape(1, n) if single else x)
    if xb.shape[-1] != n:
        raise ValueError("vector length does not match the pencil")
    return xb, single


class ShiftedPencil:
    """The pencil (K, M) of a grid and per-cell log fields, assembled on the device."""

    def __init__(self, grid: Grid, log_kappa, log_storativity, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.grid = grid
        lk = np.ascontiguousarray(np.asarray(log_kappa, dtype=np.float64).ravel())
        ls = np.ascontiguousarray(np.asarray(log_storativity, dtype=np.float64).ravel())
        if lk.size != grid.n_cells or ls.size != grid.n_cells:
            raise ValueError("assemble: one kappa and one storativity value per element")
        self._h = C.c_void_p()
        g = grid.c()
        check(lib().lt_pencil_create_grid(self.ctx.handle, C.byref(g), dptr(lk), dptr(ls), capi.LT_MEM_HOST,
                                          C.byref(self._h)))

    @classmethod
    def from_csr(cls, grid, stiffness, mass, ctx: Optional[Context] = None) -> "ShiftedPencil":
        """ShiftedPencil(K, M) (shifted_solver.hpp:90): an assembled sparse pair (SciPy sparse,
        any format) declared on `grid` (Grid for the FD operator, Mesh2D for the reference's P1
        pair on build_mesh's interior nodes); checked against that stencil on the host and
        converted to it (lt_pencil_create_csr)."""
        import scipy.sparse as sp
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.grid = grid
        K = sp.csr_matrix(stiffness)
        M = sp.csr_matrix(mass)
        n = K.shape[0]
        if K.shape != (n, n) or M.shape != (n, n):
            raise ValueError("ShiftedPencil(K, M): square matrices of equal size required")
        keep = []

        def sparse(A):
            outer = np.ascontiguousarray(A.indptr.astype(np.int64))
            inner = np.ascontiguousarray(A.indices.astype(np.int64))
            vals = np.ascontiguousarray(A.data.astype(np.float64))
            keep.extend([outer, inner, vals])
            return capi.LtSparse(outer.ctypes.data, inner.ctypes.data, dptr(vals), 8)

        ks, ms = sparse(K), sparse(M)
        self._h = C.c_void_p()
        g = grid.c()
        check(lib().lt_pencil_create_csr(self.ctx.handle, C.byref(g), int(n), C.byref(ks), C.byref(ms),
                                         C.byref(self._h)))
        return self

    @property
    def handle(self):
        return self._h

    def rows(self) -> int:
        return int(lib().lt_pencil_rows(self._h))

    def parameters(self) -> int:
        return int(lib().lt_pencil_parameters(self._h))

    def levels(self) -> int:
        return int(lib().lt_pencil_levels(self._h))

    def _apply(self, fn, args, x):
        n = self.rows()
        xb, single = _as_batch(x, n)
        y = np.zeros_like(xb)
        check(fn(self._h, *args, cptr(xb), cptr(y), xb.shape[0], capi.LT_MEM_HOST))
        return y[0] if single else y

    def apply(self, z, x):
        return self._apply(lib().lt_pencil_apply, (lc(z),), x)

    def apply_adjoint(self, z, x):
        return self._apply(lib().lt_pencil_apply_adjoint, (lc(z),), x)

    def apply_mass(self, x):
        return self._apply(lib().lt_pencil_apply_mass, (), x)

    def prepare(self, taus):
        t = np.ascontiguousarray(np.asarray(list(taus), dtype=np.complex128))
        check(lib().lt_pencil_prepare(self._h, cptr(t), int(t.size)))

    def factorization(self, tau) -> _Factorization:
        self.prepare([tau])
        return _Factorization(self, tau)

    def factorization_count(self) -> int:
        return int(lib().lt_pencil_factorization_count(self._h))

    def set_inner_tolerance(self, rel_tol: float, max_iterations: int = 200):
        check(lib().lt_pencil_set_inner_tolerance(self._h, float(rel_tol), int(max_iterations)))

    def _solve(self, tau, rhs, adjoint: bool):
        fn = lib().lt_pencil_solve_adjoint if adjoint else lib().lt_pencil_solve
        return self._apply(fn, (lc(tau),), rhs)

    def point_weights(self, point):
        pt = np.ascontiguousarray(np.asarray(point, dtype=np.float64))
        idx = np.zeros(8, dtype=np.int64)
        w = np.zeros(8)
        cnt = C.c_int()
        check(lib().lt_pencil_point_weights(self._h, dptr(pt), idx.ctypes.data_as(capi.PI64), dptr(w),
                                            C.byref(cnt)))
        out = np.zeros(self.rows())
        out[idx[: cnt.value]] = w[: cnt.value]
        return out

    def close(self):
        if self._h:
            lib().lt_pencil_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- shifted solver ----------------------------------------------------------------------
@dataclass
class ShiftedSolveOptions:
    variant: str = "gmres"
    tol: float = 1e-10
    maxit: int = 0
    keep_basis: bool = False
    record_history: bool = True

    def c(self) -> capi.LtSolveOptions:
        return capi.LtSolveOptions(capi.LT_VARIANT_FOM if self.variant == "fom" else capi.LT_VARIANT_GMRES,
                                   float(self.tol), int(self.maxit), int(self.keep_basis),
                                   int(self.record_history))


@dataclass
class ShiftStatus:
    converged: bool = False
    iteration: int = 0
    estimate: float = math.inf
    true_residual: float = math.nan
    history: List[float] = field(default_factory=list)


@dataclass
class FlexibleBasisState:
    V: np.ndarray
    U: np.ndarray
    Hbar: np.ndarray
    taus: np.ndarray
    beta: float

    def steps(self) -> int:
        return int(self.Hbar.shape[1])

    def shifted_hessenberg(self, z):
        m = self.steps()
        hz = self.Hbar[: m + 1, :m].copy()
        for l in range(m):
            hz[:, l] *= (z - self.taus[l])
            hz[l, l] += 1.0
        return hz


@dataclass
class ShiftedSolveResult:
    solutions: np.ndarray
    iterations: int = 0
    all_converged: bool = False
    shifts: List[ShiftStatus] = field(default_factory=list)
    basis: Optional[FlexibleBasisState] = None

    def unconverged(self) -> List[int]:
        return [k for k, s in enumerate(self.shifts) if not s.converged]


def _run(pencil: ShiftedPencil, b, shifts, schedule: PreconditionerSchedule, options: ShiftedSolveOptions):
    n = pencil.rows()
    bb, single = _as_batch(b, n)
    B = bb.shape[0]
    sh = np.ascontiguousarray(np.asarray(list(shifts), dtype=np.complex128))
    ns = int(sh.size)
    taus = np.ascontiguousarray(np.asarray(schedule.taus, dtype=np.complex128))
    pat = (C.c_int * max(len(schedule.pattern), 1))(*schedule.pattern)
    opt = options.c()
    x = np.zeros((B, ns, n), dtype=np.complex128)
    status = (capi.LtShiftStatus * max(B * ns, 1))()
    iters = (C.c_int * B)()
    maxit = options.maxit if options.maxit > 0 else 10 * ns
    maxit = min(n, maxit)
    hist = np.full(B * ns * max(maxit, 1), np.nan) if options.record_history else None
    check(lib().lt_solve_shifted(pencil.handle, cptr(bb), B, cptr(sh) if ns else None, ns,
                                 cptr(taus) if taus.size else None, int(taus.size), pat, len(schedule.pattern),
                                 C.byref(opt), capi.LT_MEM_HOST, cptr(x) if ns else None, status, iters,
                                 dptr(hist) if hist is not None else None))
    results = []
    for r in range(B):
        res = ShiftedSolveResult(np.ascontiguousarray(x[r].T), int(iters[r]))
        for k in range(ns):
            st = status[r * ns + k]
            h = []
            if hist is not None:
                hv = hist[(r * ns + k) * maxit: (r * ns + k + 1) * maxit]
                h = [float(v) for v in hv[: int(iters[r])] if not np.isnan(v)]
            res.shifts.append(ShiftStatus(bool(st.converged), int(st.iteration), float(st.estimate),
                                          float(st.true_residual), h))
        res.all_converged = all(s.converged for s in res.shifts)
        if options.keep_basis:
            res.basis = _basis(pencil, r)
        results.append(res)
    return results[0] if single else results


def _basis(pencil: ShiftedPencil, r: int) -> FlexibleBasisState:
    n = pencil.rows()
    m = C.c_int()
    beta = C.c_double()
    check(lib().lt_last_basis(pencil.handle, r, C.byref(m), C.byref(beta), None, None, None, None))
    m = m.value
    V = np.zeros((m + 1, n), dtype=np.complex128)
    U = np.zeros((max(m, 1), n), dtype=np.complex128)
    H = np.zeros((max(m, 1), m + 1), dtype=np.complex128)  # column-major (m+1) x m
    T = np.zeros(max(m, 1), dtype=np.complex128)
    check(lib().lt_last_basis(pencil.handle, r, None, None, cptr(V), cptr(U), cptr(H), cptr(T)))
    return FlexibleBasisState(V.T.copy(), U[:m].T.copy(), H[:m].T.copy(), T[:m].copy(), beta.value)


def solve_shifted_flexible(pencil: ShiftedPencil, b, shifts, schedule: PreconditionerSchedule,
                           options: Optional[ShiftedSolveOptions] = None):
    """shifted_solver.cpp:291-299; `b` may be (n,) or (B, n) (lockstep batch)."""
    if not schedule.taus or not schedule.pattern:
        raise ValueError("solve_shifted_flexible: empty preconditioner schedule")
    return _run(pencil, b, shifts, schedule, options or ShiftedSolveOptions())


def solve_shifted_single(pencil: ShiftedPencil, b, shifts, tau, options: Optional[ShiftedSolveOptions] = None):
    return _run(pencil, b, shifts, single_tau_schedule(tau), options or ShiftedSolveOptions())


def solve_shifted_direct(pencil: ShiftedPencil, b, shifts):
    """shifted_solver.cpp:324-332: n x n_shifts (per RHS)."""
    n = pencil.rows()
    bb, single = _as_batch(b, n)
    sh = np.ascontiguousarray(np.asarray(list(shifts), dtype=np.complex128))
    x = np.zeros((bb.shape[0], sh.size, n), dtype=np.complex128)
    check(lib().lt_solve_shifted_direct(pencil.handle, cptr(bb), bb.shape[0], cptr(sh), int(sh.size),
                                        capi.LT_MEM_HOST, cptr(x)))
    out = [np.ascontiguousarray(x[r].T) for r in range(bb.shape[0])]
    return out[0] if single else out


def residual_estimate(state: FlexibleBasisState, z, y_fom) -> float:
    """shifted_solver.cpp:334-343 (lt_residual_estimate)."""
    m = state.steps()
    H = np.ascontiguousarray(state.Hbar.T.astype(np.complex128))  # column-major (m+1) x m
    T = np.ascontiguousarray(np.asarray(state.taus, dtype=np.complex128))
    y = np.ascontiguousarray(np.asarray(y_fom, dtype=np.complex128).ravel())
    out = np.zeros(1)
    check(lib().lt_residual_estimate(cptr(H) if H.size else None, cptr(T) if T.size else None, int(m), lc(z),
                                     cptr(y) if y.size else None, int(y.size), dptr(out)))
    return float(out[0])


# ---- forward -----------------------------------------------------------------------------
_KIND = {"single": capi.LT_SOLVER_SINGLE, "flexible": capi.LT_SOLVER_FLEXIBLE, "direct": capi.LT_SOLVER_DIRECT}


@dataclass
class SolverConfig:
    kind: str = "flexible"
    variant: str = "gmres"
    tol: float = 1e-10
    maxit: int = 0

    def c(self) -> capi.LtSolverConfig:
        return capi.LtSolverConfig(_KIND[self.kind],
                                   capi.LT_VARIANT_FOM if self.variant == "fom" else capi.LT_VARIANT_GMRES,
                                   float(self.tol), int(self.maxit))


@dataclass
class ForwardProblem:
    """forward.hpp:27-35 (the pencil carries the operators)."""

    source: np.ndarray
    rate: float = 0.0
    initial_head: Optional[np.ndarray] = None
    times: List[float] = field(default_factory=list)
    n_quad: int = 40
    contour: TalbotParams = TalbotParams()


@dataclass
class TimeDiagnostics:
    iterations: int = 0
    all_converged: bool = True
    shift_residuals: List[float] = field(default_factory=list)


@dataclass
class HeadSolution:
    heads: np.ndarray
    diagnostics: List[TimeDiagnostics]


def _forward(pencil: ShiftedPencil, problem: ForwardProblem, solver: SolverConfig, pooled: bool,
             receivers=None):
    n = pencil.rows()
    times = np.ascontiguousarray(np.asarray(problem.times, dtype=np.float64))
    if times.size == 0:
        raise ValueError("solve_forward: no target times")
    src = np.ascontiguousarray(np.asarray(problem.source, dtype=np.float64).reshape(1, n))
    rates = np.array([float(problem.rate)])
    ih = None
    if problem.initial_head is not None and len(problem.initial_head) > 0:
        ih = np.ascontiguousarray(np.asarray(problem.initial_head, dtype=np.float64).reshape(1, n))
    heads = np.zeros((times.size, n))
    diag = (capi.LtTimeDiag * times.size)()
    nh = problem.n_quad // 2
    resid = np.full(times.size * max(nh, 1), np.nan)
    cp = problem.contour.c()
    sc = solver.c()
    rec = None
    n_rec = 0
    dd = None
    if receivers is not None:
        rec = np.ascontiguousarray(np.asarray(receivers, dtype=np.float64))
        n_rec = rec.shape[0]
        dd = np.zeros(n_rec * times.size)
    check(lib().lt_forward(pencil.handle, dptr(src), dptr(rates), 1, dptr(ih) if ih is not None else None,
                           dptr(times), int(times.size), int(problem.n_quad), C.byref(cp), C.byref(sc), int(pooled),
                           capi.LT_MEM_HOST, dptr(heads), dptr(rec) if rec is not None else None, n_rec,
                           dptr(dd) if dd is not None else None, diag, dptr(resid)))
    diags = [TimeDiagnostics(int(diag[t].iterations), bool(diag[t].all_converged),
                             [float(v) for v in resid[t * nh:(t + 1) * nh]]) for t in range(times.size)]
    sol = HeadSolution(np.ascontiguousarray(heads.T), diags)
    if receivers is not None:
        return sol, dd.reshape(n_rec, times.size)
    return sol


def solve_forward_sources(pencil: ShiftedPencil, sources, rates, times, n_quad: int, receivers,
                          solver: SolverConfig = SolverConfig(), pooled: bool = False,
                          contour: TalbotParams = TalbotParams()):
    """solve_forward (forward.cpp:75-118) for n_src pumping sources that share the times, contour
    and solver, batched in lockstep on the device (one lt_forward call): drawdown at the
    receiver points, (n_src, n_rec, n_times), and the per-time diagnostics.  `sources` are
    points (the multilinear weights are formed by the library, lt_pencil_point_weights)."""
    n = pencil.rows()
    src_w = np.ascontiguousarray(np.stack([pencil.point_weights(q) for q in sources]).astype(np.float64))
    rates = np.ascontiguousarray(np.asarray(rates, dtype=np.float64))
    times = np.ascontiguousarray(np.asarray(times, dtype=np.float64))
    rec = np.ascontiguousarray(np.asarray(receivers, dtype=np.float64))
    n_src, n_rec = src_w.shape[0], rec.shape[0]
    assert src_w.shape[1] == n and rates.size == n_src
    dd = np.zeros(n_src * n_rec * times.size)
    diag = (capi.LtTimeDiag * times.size)()
    cp = contour.c()
    sc = solver.c()
    check(lib().lt_forward(pencil.handle, dptr(src_w), dptr(rates), n_src, None, dptr(times), int(times.size),
                           int(n_quad), C.byref(cp), C.byref(sc), int(pooled), capi.LT_MEM_HOST, None, dptr(rec),
                           n_rec, dptr(dd), diag, None))
    diags = [TimeDiagnostics(int(diag[t].iterations), bool(diag[t].all_converged)) for t in range(times.size)]
    return dd.reshape(n_src, n_rec, times.size), diags


def solve_forward(pencil: ShiftedPencil, problem: ForwardProblem, solver: SolverConfig = SolverConfig()):
    """forward.cpp:75-118."""
    return _forward(pencil, problem, solver, False)


def solve_forward_batch(pencil: ShiftedPencil, problem: ForwardProblem, solver: SolverConfig = SolverConfig()):
    """forward.cpp:126-198."""
    return _forward(pencil, problem, solver, True)


def solve_adjoint_fields(pencil: ShiftedPencil, receiver, contour: TalbotContour, solver: SolverConfig):
    """jacobian.cpp:47-55: (K + z_k M) psi_k = -e_r, n x n_half."""
    rhs = -np.asarray(receiver, dtype=np.complex128)
    if np.linalg.norm(rhs) == 0.0:
        return np.zeros((pencil.rows(), contour.n_half()), dtype=np.complex128)
    shifts = list(contour.nodes)
    opts = ShiftedSolveOptions(variant=solver.variant, tol=solver.tol, maxit=solver.maxit, record_history=False)
    if solver.kind == "direct":
        return solve_shifted_direct(pencil, rhs, shifts)
    sched = select_preconditioner_shifts(shifts)
    if solver.kind == "single":
        res = solve_shifted_single(pencil, rhs, shifts, sched.taus[0], opts)
    else:
        res = solve_shifted_flexible(pencil, rhs, shifts, sched, opts)
    if not res.all_converged:
        raise ConvergenceError(capi.LT_ERR_NOT_CONVERGED,
                               f"adjoint solve: {len(res.unconverged())} of {len(shifts)} shifts unconverged "
                               f"after {res.iterations} iterations", res.unconverged())
    return res.solutions


def crank_nicolson(pencil: ShiftedPencil, source, rate: float, initial_head, dt: float, sample_times,
                   return_steps: bool = False):
    """crank_nicolson (forward.cpp:200-258) on the device: n x n_samples heads.  `source` may be
    (n,) or (n_src, n) with `rate` a scalar or n_src rates (lockstep problems: then
    (n_src, n, n_samples))."""
    n = pencil.rows()
    src = np.ascontiguousarray(np.asarray(source, dtype=np.float64).reshape(-1, n))
    ns = src.shape[0]
    rates = np.ascontiguousarray(np.broadcast_to(np.asarray(rate, dtype=np.float64), (ns,)).copy())
    times = np.ascontiguousarray(np.asarray(list(sample_times), dtype=np.float64))
    ih = None
    if initial_head is not None and len(initial_head) > 0:
        ih = np.ascontiguousarray(np.broadcast_to(np.asarray(initial_head, dtype=np.float64).reshape(-1, n), (ns, n)).copy())
    out = np.zeros((ns, max(times.size, 1), n))
    steps = C.c_int()
    check(lib().lt_crank_nicolson(pencil.handle, dptr(src), dptr(rates), ns, dptr(ih) if ih is not None else None,
                                  float(dt), dptr(times) if times.size else None, int(times.size), capi.LT_MEM_HOST,
                                  dptr(out), C.byref(steps)))
    samples = np.ascontiguousarray(np.transpose(out, (0, 2, 1)))
    samples = samples[0] if np.asarray(source).ndim == 1 else samples
    return (samples, steps.value) if return_steps else samples


def estimate_condition_1norm(pencil: ShiftedPencil, z) -> float:
    """estimate_condition_1norm (condest.cpp:43-49) of K + z M on the device (the actions are the
    pencil's apply / adjoint and its shift-and-invert solve / adjoint)."""
    na, ni, cond = C.c_double(), C.c_double(), C.c_double()
    check(lib().lt_pencil_condest(pencil.handle, lc(z), C.byref(na), C.byref(ni), C.byref(cond)))
    return float(cond.value)


def estimate_norms_1(pencil: ShiftedPencil, z):
    """(||K + zM||_1 estimate, ||(K + zM)^-1||_1 estimate)."""
    na, ni, cond = C.c_double(), C.c_double(), C.c_double()
    check(lib().lt_pencil_condest(pencil.handle, lc(z), C.byref(na), C.byref(ni), C.byref(cond)))
    return float(na.value), float(ni.value)


# ---- Jacobian ----------------------------------------------------------------------------
@dataclass
class ThtExperiment:
    """jacobian.hpp:22-42 on a Grid (points are 2-/3-vectors)."""

    grid: Grid
    sources: List[Sequence[float]]
    rates: List[float]
    receivers: List[Sequence[float]]
    times: List[float]
    n_quad: int = 20
    contour: TalbotParams = TalbotParams()
    solver: SolverConfig = field(default_factory=SolverConfig)
    include_storativity: bool = False
    storativity_z_factor: bool = True

    def n_measurements(self) -> int:
        return len(self.sources) * len(self.receivers) * len(self.times)

    def measurement_index(self, source: int, receiver: int, time: int) -> int:
        return (source * len(self.receivers) + receiver) * len(self.times) + time

    def c(self):
        keep = {
            "src": np.ascontiguousarray(np.asarray(self.sources, dtype=np.float64).ravel()),
            "rates": np.ascontiguousarray(np.asarray(self.rates, dtype=np.float64)),
            "rec": np.ascontiguousarray(np.asarray(self.receivers, dtype=np.float64).ravel()),
            "times": np.ascontiguousarray(np.asarray(self.times, dtype=np.float64)),
        }
        ex = capi.LtExperiment()
        lib().lt_experiment_defaults(C.byref(ex))
        ex.sources = dptr(keep["src"])
        ex.rates = dptr(keep["rates"])
        ex.n_src = len(self.sources)
        ex.receivers = dptr(keep["rec"])
        ex.n_rec = len(self.receivers)
        ex.times = dptr(keep["times"])
        ex.n_times = len(self.times)
        ex.n_quad = int(self.n_quad)
        ex.contour = self.contour.c()
        ex.solver = self.solver.c()
        ex.include_storativity = int(self.include_storativity)
        ex.storativity_z_factor = int(self.storativity_z_factor)
        return ex, keep


@dataclass
class JacobianResult:
    jacobian: np.ndarray
    predictions: np.ndarray


class ThtForwardModel:
    """jacobian.hpp:79-97."""

    def __init__(self, experiment: ThtExperiment, log_storativity, ctx: Optional[Context] = None):
        if not experiment.sources or not experiment.receivers or not experiment.times:
            raise ValueError("ThtForwardModel: experiment must be nonempty")
        if len(experiment.rates) != len(experiment.sources):
            raise ValueError("ThtForwardModel: one rate per source required")
        ls = np.asarray(log_storativity, dtype=np.float64)
        if ls.size != experiment.grid.n_cells:
            raise ValueError("ThtForwardModel: one storativity value per element required")
        self.experiment = experiment
        self.log_storativity = ls
        self.ctx = ctx or default_context()

    def n_measurements(self) -> int:
        return self.experiment.n_measurements()

    def n_parameters(self) -> int:
        n = self.experiment.grid.n_cells
        return 2 * n if self.experiment.include_storativity else n

    def pencil(self, log_kappa, log_storativity=None) -> ShiftedPencil:
        ls = self.log_storativity if log_storativity is None else log_storativity
        return ShiftedPencil(self.experiment.grid, log_kappa, ls, self.ctx)

    def predict(self, log_kappa):
        return self.predict_with(log_kappa, self.log_storativity)

    def predict_with(self, log_kappa, log_storativity):
        pencil = self.pencil(log_kappa, log_storativity)
        ex, keep = self.experiment.c()
        out = np.zeros(self.n_measurements())
        check(lib().lt_predict(pencil.handle, C.byref(ex), dptr(out)))
        pencil.close()
        return out

    def jacobian(self, log_kappa) -> JacobianResult:
        pencil = self.pencil(log_kappa)
        ex, keep = self.experiment.c()
        J = np.zeros((self.n_measurements(), self.n_parameters()))
        pred = np.zeros(self.n_measurements())
        check(lib().lt_jacobian(pencil.handle, C.byref(ex), dptr(J), dptr(pred)))
        pencil.close()
        return JacobianResult(J, pred)


def assemble_jacobian(experiment: ThtExperiment, log_kappa, log_storativity) -> JacobianResult:
    return ThtForwardModel(experiment, log_storativity).jacobian(log_kappa)

"""Oracle: adjoint-state Laplace-domain Jacobian.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Restates /root/reference/proj/src/jacobian.cpp (P1 discretisation, exactly
as the reference) and applies the same orchestration to the FD
discretisation of oracle/fd.py (the BASELINE configs).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import fd as fdmod
from . import fem
from .forward import ForwardProblem, SolverConfig, solve_forward
from .shifted_solver import (ConvergenceError, ShiftedPencil, ShiftedSolveOptions,
                             select_preconditioner_shifts, solve_shifted_direct,
                             solve_shifted_flexible, solve_shifted_single)
from .talbot import TalbotParams, build_contour, inverse_laplace_sum, qhat_step


def _solve_family_or_throw(pencil, rhs, shifts, solver: SolverConfig, what: str):
    """jacobian.cpp:19-43."""
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
    if not result.all_converged:
        raise ConvergenceError(
            f"{what}: {len(result.unconverged())} of {len(shifts)} shifts unconverged after "
            f"{result.iterations} iterations", result.unconverged())
    return result.solutions


def solve_adjoint_fields(pencil, receiver, contour, solver: SolverConfig):
    """jacobian.cpp:47-55: (K + z_k M) psi_k = -e_r."""
    rhs = -np.asarray(receiver, dtype=np.complex128)
    if np.linalg.norm(rhs) == 0.0:
        return np.zeros((pencil.rows(), contour.n_half()), dtype=np.complex128)
    return _solve_family_or_throw(pencil, rhs, list(contour.nodes), solver, "adjoint solve")


def sensitivity_row_conductivity(mesh, ops, forward_fields, adjoint_fields, contour, kappa):
    """jacobian.cpp:57-87 (vectorised over elements)."""
    if forward_fields.shape[1] != contour.n_half() or adjoint_fields.shape[1] != contour.n_half():
        raise ValueError("sensitivity_row: fields do not match the contour")
    grads = fem.element_basis_gradients(mesh)  # (E, 3, 2)
    area = fem.element_areas(mesh)
    dof = ops.node_to_free[mesh.elements]  # (E, 3)
    mask = dof >= 0
    dof_c = np.where(mask, dof, 0)
    accum = np.zeros(mesh.n_elements(), dtype=np.complex128)
    for k in range(contour.n_half()):
        phi = np.where(mask, forward_fields[dof_c, k], 0.0)
        psi = np.where(mask, adjoint_fields[dof_c, k], 0.0)
        gp = np.einsum("ei,eid->ed", phi, grads)
        gq = np.einsum("ei,eid->ed", psi, grads)
        accum += contour.weights[k] * (gp[:, 0] * gq[:, 0] + gp[:, 1] * gq[:, 1])
    return 2.0 * accum.real * np.asarray(kappa) * area


def sensitivity_row_storativity(mesh, ops, forward_fields, adjoint_fields, contour, storativity,
                                include_z_factor: bool):
    """jacobian.cpp:89-125."""
    if forward_fields.shape[1] != contour.n_half() or adjoint_fields.shape[1] != contour.n_half():
        raise ValueError("sensitivity_row: fields do not match the contour")
    area = fem.element_areas(mesh)
    dof = ops.node_to_free[mesh.elements]
    mask = dof >= 0
    dof_c = np.where(mask, dof, 0)
    pattern = np.ones((3, 3)) + np.eye(3)
    accum = np.zeros(mesh.n_elements(), dtype=np.complex128)
    for k in range(contour.n_half()):
        phi = np.where(mask, forward_fields[dof_c, k], 0.0)
        psi = np.where(mask, adjoint_fields[dof_c, k], 0.0)
        integral = np.einsum("ei,ij,ej->e", phi, pattern, psi) * area / 12.0
        zf = contour.nodes[k] if include_z_factor else 1.0
        accum += contour.weights[k] * zf * integral
    return 2.0 * accum.real * np.asarray(storativity)


@dataclass
class ThtExperiment:
    """jacobian.hpp:22-42.  `discretisation` is a fem.Mesh2D (the reference's P1
    path) or an fd.Grid (the BASELINE FD extension); points are 2-/3-vectors."""

    discretisation: object
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


@dataclass
class JacobianResult:
    jacobian: np.ndarray
    predictions: np.ndarray


class ThtForwardModel:
    """jacobian.hpp:79-97, jacobian.cpp:127-247."""

    def __init__(self, experiment: ThtExperiment, log_storativity):
        self.experiment = experiment
        self.log_storativity = np.asarray(log_storativity, dtype=np.float64)
        disc = experiment.discretisation
        if disc is None:
            raise ValueError("ThtForwardModel: missing mesh")
        if not experiment.sources or not experiment.receivers or not experiment.times:
            raise ValueError("ThtForwardModel: experiment must be nonempty")
        if len(experiment.rates) != len(experiment.sources):
            raise ValueError("ThtForwardModel: one rate per source required")
        self.is_fd = isinstance(disc, fdmod.Grid)
        n_param = disc.n_cells if self.is_fd else disc.n_elements()
        if self.log_storativity.shape[0] != n_param:
            raise ValueError("ThtForwardModel: one storativity value per element required")
        self.n_elem = n_param
        if self.is_fd:
            self.source_weights = [fdmod.point_weights(disc, p) for p in experiment.sources]
            self.receiver_weights = [fdmod.point_weights(disc, p) for p in experiment.receivers]
        else:
            self.source_weights = [fem.point_source(disc, p[0], p[1]) for p in experiment.sources]
            self.receiver_weights = [fem.point_source(disc, p[0], p[1])
                                     for p in experiment.receivers]

    def n_measurements(self) -> int:
        return self.experiment.n_measurements()

    def n_parameters(self) -> int:
        return 2 * self.n_elem if self.experiment.include_storativity else self.n_elem

    def _assemble(self, kappa, storativity):
        disc = self.experiment.discretisation
        if self.is_fd:
            return fdmod.assemble_fd(disc, kappa, storativity)
        return fem.assemble(disc, kappa, storativity)

    def predict(self, log_kappa):
        return self.predict_with(log_kappa, self.log_storativity)

    def predict_with(self, log_kappa, log_storativity):
        """jacobian.cpp:158-187."""
        exp = self.experiment
        ops = self._assemble(np.exp(log_kappa), np.exp(log_storativity))
        pencil = ShiftedPencil(ops.stiffness, ops.mass)
        out = np.zeros(self.n_measurements())
        for s in range(len(exp.sources)):
            problem = ForwardProblem(ops.stiffness, ops.mass,
                                     ops.restrict_to_free(self.source_weights[s]),
                                     rate=exp.rates[s], times=list(exp.times), n_quad=exp.n_quad,
                                     contour=exp.contour)
            heads = solve_forward(problem, exp.solver, pencil=pencil)
            for r in range(len(exp.receivers)):
                e_r = ops.restrict_to_free(self.receiver_weights[r])
                for t in range(len(exp.times)):
                    out[exp.measurement_index(s, r, t)] = e_r @ heads.heads[:, t]
        return out

    def jacobian(self, log_kappa) -> JacobianResult:
        """jacobian.cpp:189-247."""
        exp = self.experiment
        kappa = np.exp(np.asarray(log_kappa, dtype=np.float64))
        storativity = np.exp(self.log_storativity)
        ops = self._assemble(kappa, storativity)
        pencil = ShiftedPencil(ops.stiffness, ops.mass)
        n_src, n_rec, n_times = len(exp.sources), len(exp.receivers), len(exp.times)
        J = np.zeros((self.n_measurements(), self.n_parameters()))
        pred = np.zeros(self.n_measurements())
        for t in range(n_times):
            contour = build_contour(exp.n_quad, exp.times[t], exp.contour)
            shifts = list(contour.nodes)
            forward_fields = []
            for s in range(n_src):
                b = ops.restrict_to_free(self.source_weights[s]).astype(np.complex128)
                fields = _solve_family_or_throw(pencil, b, shifts, exp.solver, "forward solve")
                for k in range(contour.n_half()):
                    fields[:, k] *= qhat_step(exp.rates[s], contour.nodes[k])
                forward_fields.append(fields)
            for r in range(n_rec):
                e_r = ops.restrict_to_free(self.receiver_weights[r]).astype(np.complex128)
                adjoint = solve_adjoint_fields(pencil, e_r, contour, exp.solver)
                for s in range(n_src):
                    row = exp.measurement_index(s, r, t)
                    if self.is_fd:
                        rk, rs = fdmod.sensitivity_rows_fd(
                            ops, forward_fields[s], adjoint, contour.weights, contour.nodes,
                            exp.include_storativity, exp.storativity_z_factor)
                        J[row, : self.n_elem] = rk
                        if exp.include_storativity:
                            J[row, self.n_elem:] = rs
                    else:
                        mesh = exp.discretisation
                        J[row, : self.n_elem] = sensitivity_row_conductivity(
                            mesh, ops, forward_fields[s], adjoint, contour, kappa)
                        if exp.include_storativity:
                            J[row, self.n_elem:] = sensitivity_row_storativity(
                                mesh, ops, forward_fields[s], adjoint, contour, storativity,
                                exp.storativity_z_factor)
                    at_receiver = forward_fields[s].T @ e_r
                    pred[row] = inverse_laplace_sum(contour, at_receiver)
        return JacobianResult(J, pred)


def assemble_jacobian(experiment: ThtExperiment, log_kappa, log_storativity) -> JacobianResult:
    """jacobian.cpp:249-254."""
    return ThtForwardModel(experiment, log_storativity).jacobian(log_kappa)

"""Oracle pinning: forward / adjoint / Jacobian known answers and invariants from the
reference SPEC (acceptance 8 at reduced size), on the reference's own P1
discretisation and on the FD extension used by the BASELINE configs."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import fd as ofd
from oracle import fem
from oracle import forward as F
from oracle import jacobian as J
from oracle import shifted_solver as S
from oracle import talbot as T


def _p1_ops(n=21, L=100.0, kappa=1e-4, s=1e-5, field=None):
    mesh = fem.build_mesh(n, L)
    k = np.full(mesh.n_elements(), kappa) if field is None else kappa * np.exp(field)
    ops = fem.assemble(mesh, k, np.full(mesh.n_elements(), s))
    return mesh, ops


def _eig_head(K, M, b, q0, t):
    lam, V = sla.eigh(K.toarray(), M.toarray())  # M-orthonormal eigenvectors
    coef = (V.T @ b) * q0 * (1.0 - np.exp(-lam * t)) / lam
    return V @ coef


def test_zero_rate_zero_head():
    mesh, ops = _p1_ops(9)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    sol = F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 0.0, None, [60.0, 600.0], 20))
    assert np.all(sol.heads == 0.0)


@pytest.mark.parametrize("kind", ["flexible", "single", "direct"])
def test_p1_forward_matches_eigendecomposition(kind):  # SPEC.md:334 (21^2, constant fields)
    mesh, ops = _p1_ops(21)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    times = [60.0, 300.0, 1200.0]
    sol = F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 8.5e-4, None, times, 40),
                          F.SolverConfig(kind=kind))
    for it, t in enumerate(times):
        ref = _eig_head(ops.stiffness, ops.mass, b, 8.5e-4, t)
        assert np.linalg.norm(sol.heads[:, it] - ref) <= 1e-8 * np.linalg.norm(ref)


def test_fd_forward_matches_eigendecomposition():
    grid = ofd.Grid((16, 12), 6.25)
    ops = ofd.assemble_fd(grid, np.full(grid.n_cells, 1e-4), np.full(grid.n_cells, 1e-5))
    b = ofd.point_weights(grid, (50.0, 37.5))
    times = [60.0, 600.0]
    sol = F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 1e-3, None, times, 32))
    for it, t in enumerate(times):
        ref = _eig_head(ops.stiffness, ops.mass, b, 1e-3, t)
        assert np.linalg.norm(sol.heads[:, it] - ref) <= 1e-8 * np.linalg.norm(ref)


def test_batch_of_one_time_equals_single_time():
    rng = np.random.default_rng(4)
    mesh, ops = _p1_ops(15, field=0.8 * rng.standard_normal(2 * 14 * 14))
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    prob = F.ForwardProblem(ops.stiffness, ops.mass, b, 1e-3, None, [300.0], 40)
    a = F.solve_forward(prob)
    c = F.solve_forward_batch(prob)
    assert np.max(np.abs(a.heads - c.heads)) <= 1e-12 * np.max(np.abs(a.heads))


def test_batch_duplicate_times_identical_columns():
    mesh, ops = _p1_ops(11)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    sol = F.solve_forward_batch(F.ForwardProblem(ops.stiffness, ops.mass, b, 1e-3, None, [300.0, 300.0], 20))
    assert np.array_equal(sol.heads[:, 0], sol.heads[:, 1])


def test_initial_head_family():  # forward.cpp:85-96, 112-114
    mesh, ops = _p1_ops(11)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    xy = mesh.nodes[ops.free_nodes]
    phi0 = np.sin(math.pi * xy[:, 0] / 100.0) * np.sin(math.pi * xy[:, 1] / 100.0)  # smooth phi0
    t = 120.0
    sol = F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 0.0, phi0, [t], 40))
    lam, V = sla.eigh(ops.stiffness.toarray(), ops.mass.toarray())
    ref = V @ (np.exp(-lam * t) * (V.T @ (ops.mass @ phi0)))
    assert np.linalg.norm(sol.heads[:, 0] - ref) <= 1e-8 * np.linalg.norm(ref)


def test_forward_argument_checks():  # forward.cpp:19-33
    mesh, ops = _p1_ops(5)
    b = np.zeros(ops.n_free())
    with pytest.raises(ValueError):
        F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 1.0, None, [], 20))
    with pytest.raises(ValueError):
        F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 1.0, None, [2.0, 1.0], 20))
    with pytest.raises(ValueError):
        F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, 1.0, None, [-1.0], 20))


def test_adjoint_zero_receiver_and_direct():
    mesh, ops = _p1_ops(11)
    pencil = S.ShiftedPencil(ops.stiffness, ops.mass)
    c = T.build_contour(20, 300.0)
    z = J.solve_adjoint_fields(pencil, np.zeros(ops.n_free()), c, F.SolverConfig())
    assert np.all(z == 0)
    e = ops.restrict_to_free(fem.point_source(mesh, 40.0, 50.0))
    psi = J.solve_adjoint_fields(pencil, e, c, F.SolverConfig())
    direct = S.solve_shifted_direct(pencil, -e.astype(complex), list(c.nodes))
    assert np.max(np.abs(psi - direct)) <= 1e-8 * np.max(np.abs(direct))


def _fd_check(model, log_kappa, log_s, include_s, step=1e-5):
    """Central differences of the predictions w.r.t. every parameter."""
    res = model.jacobian(log_kappa)
    n = len(log_kappa)
    fd = np.zeros_like(res.jacobian)
    for e in range(n):
        d = np.zeros(n)
        d[e] = step
        fd[:, e] = (model.predict_with(log_kappa + d, log_s) - model.predict_with(log_kappa - d, log_s)) / (2 * step)
        if include_s:
            fd[:, n + e] = (model.predict_with(log_kappa, log_s + d) - model.predict_with(log_kappa, log_s - d)) / (2 * step)
    return res, fd


def _assert_fd(Jm, fd):
    big = np.abs(Jm) > 1e-3 * np.max(np.abs(Jm), axis=1, keepdims=True)
    rel = np.abs(Jm - fd)[big] / np.abs(Jm)[big]
    assert rel.max() <= 1e-4, rel.max()


def test_p1_jacobian_matches_finite_differences():  # SPEC.md:407, 419, acceptance 8 (reduced)
    rng = np.random.default_rng(8)
    mesh = fem.build_mesh(9, 100.0)
    lk = np.log(1e-4) + 0.8 * rng.standard_normal(mesh.n_elements())
    ls = np.full(mesh.n_elements(), np.log(1e-5))
    exp = J.ThtExperiment(mesh, [(50.0, 50.0)], [8.5e-4], [(37.5, 50.0), (62.5, 37.5), (25.0, 75.0)],
                          [480.0, 600.0], n_quad=20, include_storativity=True)
    model = J.ThtForwardModel(exp, ls)
    res, fd = _fd_check(model, lk, ls, True)
    _assert_fd(res.jacobian, fd)
    assert np.allclose(res.predictions, model.predict(lk), rtol=1e-10)


def test_fd_jacobian_matches_finite_differences():
    rng = np.random.default_rng(9)
    grid = ofd.Grid((8, 8), 12.5)
    lk = np.log(1e-4) + 0.8 * rng.standard_normal(grid.n_cells)
    ls = np.log(1e-5) + 0.3 * rng.standard_normal(grid.n_cells)
    exp = J.ThtExperiment(grid, [(50.0, 50.0)], [8.5e-4], [(31.25, 56.25), (68.75, 43.75)],
                          [300.0, 900.0], n_quad=20, include_storativity=True)
    model = J.ThtForwardModel(exp, ls)
    res, fd = _fd_check(model, lk, ls, True)
    _assert_fd(res.jacobian, fd)


def test_fd_jacobian_3d_matches_finite_differences():
    rng = np.random.default_rng(10)
    grid = ofd.Grid((5, 4, 4), 10.0)
    lk = np.log(1e-4) + 0.5 * rng.standard_normal(grid.n_cells)
    ls = np.full(grid.n_cells, np.log(1e-5))
    exp = J.ThtExperiment(grid, [(25.0, 20.0, 20.0)], [1e-3], [(15.0, 25.0, 15.0)], [200.0],
                          n_quad=20, include_storativity=True)
    model = J.ThtForwardModel(exp, ls)
    res, fd = _fd_check(model, lk, ls, True)
    _assert_fd(res.jacobian, fd)


@pytest.mark.parametrize("disc", ["p1", "fd"])
def test_reciprocity(disc):
    rng = np.random.default_rng(12)
    if disc == "p1":
        d = fem.build_mesh(11, 100.0)
        n = d.n_elements()
    else:
        d = ofd.Grid((10, 10), 10.0)
        n = d.n_cells
    lk = np.log(1e-4) + 0.5 * rng.standard_normal(n)
    ls = np.full(n, np.log(1e-5))
    a, b = (35.0, 45.0), (65.0, 55.0)
    e1 = J.ThtExperiment(d, [a], [1e-3], [b], [400.0], n_quad=20)
    e2 = J.ThtExperiment(d, [b], [1e-3], [a], [400.0], n_quad=20)
    r1 = J.assemble_jacobian(e1, lk, ls).jacobian
    r2 = J.assemble_jacobian(e2, lk, ls).jacobian
    assert np.max(np.abs(r1 - r2)) <= 1e-10 * np.max(np.abs(r1))


def test_single_row_and_duplicate_times():
    mesh = fem.build_mesh(9, 100.0)
    n = mesh.n_elements()
    lk = np.full(n, np.log(1e-4))
    ls = np.full(n, np.log(1e-5))
    exp = J.ThtExperiment(mesh, [(50.0, 50.0)], [1e-3], [(37.5, 62.5)], [600.0, 600.0], n_quad=20)
    r = J.assemble_jacobian(exp, lk, ls)
    assert r.jacobian.shape == (2, n) and np.array_equal(r.jacobian[0], r.jacobian[1])
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    pencil = S.ShiftedPencil(ops.stiffness, ops.mass)
    c = T.build_contour(20, 600.0)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0)).astype(complex)
    phi = S.solve_shifted_flexible(pencil, b, list(c.nodes), S.select_preconditioner_shifts(list(c.nodes))).solutions
    phi = phi * (1e-3 / c.nodes)[None, :]
    e = ops.restrict_to_free(fem.point_source(mesh, 37.5, 62.5))
    psi = J.solve_adjoint_fields(pencil, e, c, F.SolverConfig())
    row = J.sensitivity_row_conductivity(mesh, ops, phi, psi, c, np.exp(lk))
    assert np.max(np.abs(row - r.jacobian[0])) <= 1e-12 * np.max(np.abs(row))


def test_model_argument_checks():  # jacobian.cpp:127-139
    mesh = fem.build_mesh(5, 1.0)
    n = mesh.n_elements()
    with pytest.raises(ValueError):
        J.ThtForwardModel(J.ThtExperiment(mesh, [], [], [(0.5, 0.5)], [1.0]), np.zeros(n))
    with pytest.raises(ValueError):
        J.ThtForwardModel(J.ThtExperiment(mesh, [(0.5, 0.5)], [], [(0.5, 0.5)], [1.0]), np.zeros(n))
    with pytest.raises(ValueError):
        J.ThtForwardModel(J.ThtExperiment(mesh, [(0.5, 0.5)], [1.0], [(0.5, 0.5)], [1.0]), np.zeros(n + 1))

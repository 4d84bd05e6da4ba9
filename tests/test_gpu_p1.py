"""Device path on the reference's own P1 discretisation (build_mesh + assemble,
mesh.cpp / assembly.cpp) vs the oracle's line-faithful restatement of the reference:
operator, shift-and-invert, FGMRES-Sh, forward heads and the Jacobian rows
(sensitivity_row_conductivity / _storativity)."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem
from oracle import forward as ofw
from oracle import jacobian as ojac
from oracle import shifted_solver as oss
from oracle import talbot as otal
from paper_1409_2556_b200 import laptomo as L

from .helpers import jacobian_errors, rel

pytestmark = pytest.mark.gpu


def _case(n, side, var, seed, kappa=1e-4, s=1e-5):
    rng = np.random.default_rng(seed)
    mesh = fem.build_mesh(n, side)
    lk = np.log(kappa) + np.sqrt(var) * rng.standard_normal(mesh.n_elements())
    ls = np.log(s) + 0.2 * rng.standard_normal(mesh.n_elements())
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    dmesh = L.build_mesh(n, side)
    return mesh, dmesh, lk, ls, ops


@pytest.mark.parametrize("n", [5, 21, 33])
def test_p1_operator_matches_reference_assembly(n):
    mesh, dmesh, lk, ls, ops = _case(n, 100.0, 0.8, n)
    p = L.ShiftedPencil(dmesh, lk, ls)
    assert p.rows() == ops.n_free()
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, ops.n_free())) + 1j * rng.standard_normal((2, ops.n_free()))
    z = 0.3 - 0.7j
    for r in range(2):
        assert rel(p.apply(z, x[r]), ops.stiffness @ x[r] + z * (ops.mass @ x[r])) <= 1e-14
        assert rel(p.apply_mass(x[r]), ops.mass @ x[r]) <= 1e-14


def test_p1_point_weights_match_point_source():
    mesh, dmesh, lk, ls, ops = _case(11, 100.0, 0.5, 3)
    p = L.ShiftedPencil(dmesh, lk, ls)
    for pt in [(50.0, 50.0), (33.3, 71.2), (5.0, 95.0), (12.0, 3.0)]:
        ref = ops.restrict_to_free(fem.point_source(mesh, *pt))
        assert np.max(np.abs(p.point_weights(pt) - ref)) <= 1e-15


@pytest.mark.parametrize("tau", [-0.04 + 0.03j, 0.002 + 0.0005j])
def test_p1_shift_and_invert(tau):
    mesh, dmesh, lk, ls, ops = _case(65, 100.0, 1.6, 5)
    p = L.ShiftedPencil(dmesh, lk, ls)
    rng = np.random.default_rng(2)
    v = rng.standard_normal(ops.n_free()) + 1j * rng.standard_normal(ops.n_free())
    u = p.factorization(tau).solve(v)
    ref = spla.splu((ops.stiffness + tau * ops.mass).tocsc(), permc_spec="COLAMD").solve(v)
    assert rel(u, ref) <= 1e-10


@pytest.mark.parametrize("kind", ["single", "flexible"])
def test_p1_paper_regime_shifted_solve(kind):
    """Paper regime (100 m domain, kappa 1e-4, S 1e-5, t = 5 min, N_z = 40):
    tens of outer iterations, exercising basis growth and the freeze / back-off logic."""
    mesh, dmesh, lk, ls, ops = _case(41, 100.0, 1.6, 7)
    p = L.ShiftedPencil(dmesh, lk, ls)
    opencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
    c = otal.build_contour(40, 300.0)
    shifts = list(c.nodes)
    sched = oss.select_preconditioner_shifts(shifts)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0)).astype(complex)
    if kind == "single":
        ref = oss.solve_shifted_single(opencil, b, shifts, sched.taus[0])
        got = L.solve_shifted_single(p, b, shifts, sched.taus[0])
    else:
        ref = oss.solve_shifted_flexible(opencil, b, shifts, sched)
        got = L.solve_shifted_flexible(p, b, shifts, L.PreconditionerSchedule(sched.taus, sched.pattern))
    assert ref.iterations >= 5
    assert got.all_converged and ref.all_converged
    assert abs(got.iterations - ref.iterations) <= 1
    direct = oss.solve_shifted_direct(opencil, b, shifts)
    for k in range(len(shifts)):
        assert got.shifts[k].true_residual <= 1e-10
        assert rel(got.solutions[:, k], direct[:, k]) <= 1e-8


def test_p1_forward_drawdown_matches_reference():
    mesh, dmesh, lk, ls, ops = _case(101, 100.0, 1.6, 11)
    p = L.ShiftedPencil(dmesh, lk, ls)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    times = [60.0, 300.0, 1200.0]
    prob = L.ForwardProblem(b, 8.5e-4, None, times, 40)
    sol, dd = L._forward(p, prob, L.SolverConfig(kind="flexible"), False, receivers=np.array([[70.0, 70.0], [40.0, 50.0]]))
    ref = ofw.solve_forward(ofw.ForwardProblem(ops.stiffness, ops.mass, b, 8.5e-4, None, times, 40))
    for r, q in enumerate([(70.0, 70.0), (40.0, 50.0)]):
        e = ops.restrict_to_free(fem.point_source(mesh, *q))
        assert np.max(np.abs(dd[r] - e @ ref.heads) / np.abs(e @ ref.heads)) <= 1e-8
    assert rel(sol.heads, ref.heads) <= 1e-8
    for t in range(len(times)):
        assert abs(sol.diagnostics[t].iterations - ref.diagnostics[t].iterations) <= 1


def test_p1_jacobian_matches_reference_rows():
    """SPEC acceptance-8 style experiment on the reference's P1 operator: 1 source x 36
    receivers x 3 times on a 21^2 mesh (§5.3), both blocks."""
    mesh, dmesh, lk, ls, ops = _case(21, 100.0, 0.8, 13)
    recs = [(x, y) for y in np.linspace(20, 80, 6) for x in np.linspace(20, 80, 6)]
    times = [480.0, 600.0, 1200.0]
    ex = L.ThtExperiment(dmesh, [(50.0, 50.0)], [8.5e-4], recs, times, 20, include_storativity=True)
    oex = ojac.ThtExperiment(mesh, [(50.0, 50.0)], [8.5e-4], recs, times, 20, include_storativity=True)
    got = L.ThtForwardModel(ex, ls).jacobian(lk)
    ref = ojac.ThtForwardModel(oex, ls).jacobian(lk)
    assert np.max(np.abs(got.predictions - ref.predictions) / np.abs(ref.predictions)) <= 1e-8
    row, entry, s_err = jacobian_errors(got.jacobian, ref.jacobian, mesh.n_elements(), False)
    assert row <= 1e-8 and entry <= 1e-8, (row, entry)
    # storativity block: per row, relative to the whole row (at early times some S-rows are
    # ~1e-12 of their kappa-row and carry only the solve's rounding in absolute terms)
    ne = mesh.n_elements()
    Js, Rs = got.jacobian[:, ne:], ref.jacobian[:, ne:]
    assert np.max(np.linalg.norm(Js - Rs, axis=1) / np.linalg.norm(ref.jacobian, axis=1)) <= 1e-8


def test_p1_unit_square_config0_statistics():
    """BASELINE configs[0] statistics on the reference's mesh: 101^2 nodes on the unit square."""
    from paper_1409_2556_b200 import inputs
    cfg = inputs.config(0)
    mesh = fem.build_mesh(101, 1.0)
    cent = fem.element_centroids(mesh)
    # sample the GRF on the 100x100 cells and give both triangles of a cell its value
    lk_cells, _ = cfg.fields()
    lk = np.repeat(lk_cells, 2)
    ls = np.full(mesh.n_elements(), np.log(1e-5))
    assert cent.shape[0] == lk.size
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    p = L.ShiftedPencil(L.build_mesh(101, 1.0), lk, ls)
    b = ops.restrict_to_free(fem.point_source(mesh, 0.5, 0.5))
    prob = L.ForwardProblem(b, 1e-4, None, cfg.times, cfg.n_quad)
    got = L.solve_forward(p, prob, L.SolverConfig(kind="single"))
    ref = ofw.solve_forward(ofw.ForwardProblem(ops.stiffness, ops.mass, b, 1e-4, None, cfg.times, cfg.n_quad),
                            ofw.SolverConfig(kind="single"))
    assert rel(got.heads, ref.heads) <= 1e-8

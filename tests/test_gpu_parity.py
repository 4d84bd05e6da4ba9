"""Device path vs the CPU oracle on the same seeded inputs (parity proper).

All calls go through the C ABI (paper_1409_2556_b200.laptomo -> liblaptomo_gpu.so).
Tolerances (north_star): drawdown and Jacobian entries 1e-8 relative in FP64,
same per-shift tolerance 1e-10.
"""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import forward as ofw
from oracle import jacobian as ojac
from oracle import shifted_solver as oss
from oracle import talbot as otal
from paper_1409_2556_b200 import inputs
from paper_1409_2556_b200 import laptomo as L

from .helpers import fd_case, jacobian_errors, rel

pytestmark = pytest.mark.gpu


def _pencil(cfg, lk, ls):
    return L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)


@pytest.mark.parametrize("index,shape", [(0, (40, 30)), (2, (32, 32)), (4, (12, 10, 8))])
def test_stencil_apply_matches_csr(index, shape):
    cfg, lk, ls, grid, ops = fd_case(index, shape)
    p = _pencil(cfg, lk, ls)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, grid.n_cells)) + 1j * rng.standard_normal((3, grid.n_cells))
    z = -0.3 + 0.2j
    y = p.apply(z, x)
    for r in range(3):
        ref = ops.stiffness @ x[r] + z * (ops.mass @ x[r])
        assert rel(y[r], ref) <= 1e-14
        assert rel(p.apply_mass(x[r]), ops.mass @ x[r]) <= 1e-15
        assert rel(p.apply_adjoint(z, x[r]), ops.stiffness @ x[r] + np.conj(z) * (ops.mass @ x[r])) <= 1e-14


# (100, 100) runs the natural-layout TMA kernels; (64, 40, 24), (96, 20, 18) and (128, 72, 12)
# the colour-split ones (rows of >= 64 cells, nx % 4 == 0; partial tiles in x, y and z; on
# two levels for (128, 72, 12)) with the pair transfers; the others the register-pipelined ones
@pytest.mark.parametrize("index,shape", [(0, (100, 100)), (4, (16, 16, 16)), (3, (32, 32, 16)), (4, (64, 40, 24)),
                                         (3, (96, 20, 18)), (4, (128, 72, 12))])
def test_preconditioner_solve_matches_sparse_lu(index, shape):
    cfg, lk, ls, grid, ops = fd_case(index, shape)
    p = _pencil(cfg, lk, ls)
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    sched = oss.select_preconditioner_shifts(list(contour.nodes))
    rng = np.random.default_rng(3)
    v = rng.standard_normal(grid.n_cells) + 1j * rng.standard_normal(grid.n_cells)
    for tau in sched.taus:
        u = p.factorization(tau).solve(v)
        A = (ops.stiffness + tau * ops.mass).tocsc()
        ref = spla.splu(A, permc_spec="COLAMD").solve(v)
        assert rel(u, ref) <= 1e-10, tau
        ua = p.factorization(tau).solve_adjoint(v)
        refa = spla.splu((ops.stiffness + np.conj(tau) * ops.mass).tocsc()).solve(v)
        assert rel(ua, refa) <= 1e-10
    assert p.factorization_count() == len(sched.taus)


@pytest.mark.parametrize("kind", ["single", "flexible"])
@pytest.mark.parametrize("variant", ["gmres", "fom"])
def test_shifted_solve_matches_oracle(kind, variant):
    cfg, lk, ls, grid, ops = fd_case(2, (48, 48))
    p = _pencil(cfg, lk, ls)
    opencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
    contour = otal.build_contour(cfg.n_quad, cfg.times[1])
    shifts = list(contour.nodes)
    sched = oss.select_preconditioner_shifts(shifts)
    b = ofd_point(grid, cfg.sources[0])
    opts = oss.ShiftedSolveOptions(variant=variant)
    gopts = L.ShiftedSolveOptions(variant=variant)
    if kind == "single":
        ref = oss.solve_shifted_single(opencil, b, shifts, sched.taus[0], opts)
        got = L.solve_shifted_single(p, b, shifts, sched.taus[0], gopts)
    else:
        ref = oss.solve_shifted_flexible(opencil, b, shifts, sched, opts)
        got = L.solve_shifted_flexible(p, b, shifts, L.PreconditionerSchedule(sched.taus, sched.pattern), gopts)
    assert got.all_converged and ref.all_converged
    assert got.iterations == ref.iterations
    direct = oss.solve_shifted_direct(opencil, b, shifts)
    for k in range(len(shifts)):
        assert got.shifts[k].iteration == ref.shifts[k].iteration
        assert got.shifts[k].true_residual <= 1e-10
        assert rel(got.solutions[:, k], ref.solutions[:, k]) <= 1e-8
        assert rel(got.solutions[:, k], direct[:, k]) <= 1e-8


def ofd_point(grid, point):
    from oracle import fd as ofd
    return ofd.point_weights(grid, point).astype(np.complex128)


def test_shift_equal_tau_is_exact_in_one_iteration():
    # z = tau -> exact solve at iteration 1
    cfg, lk, ls, grid, ops = fd_case(0, (32, 32))
    p = _pencil(cfg, lk, ls)
    tau = -0.2 + 0.1j
    b = ofd_point(grid, (0.5, 0.5))
    res = L.solve_shifted_single(p, b, [tau], tau)
    assert res.all_converged and res.shifts[0].iteration == 1
    ref = spla.spsolve((ops.stiffness + tau * ops.mass).tocsc(), b)
    assert rel(res.solutions[:, 0], ref) <= 1e-10


def test_batched_rhs_equal_individual():
    cfg, lk, ls, grid, ops = fd_case(2, (32, 32))
    p = _pencil(cfg, lk, ls)
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    shifts = list(contour.nodes)
    sched = oss.select_preconditioner_shifts(shifts)
    s = L.PreconditionerSchedule(sched.taus, sched.pattern)
    bs = np.stack([ofd_point(grid, q) for q in cfg.sources[:3]])
    batch = L.solve_shifted_flexible(p, bs, shifts, s)
    for r in range(3):
        one = L.solve_shifted_flexible(p, bs[r], shifts, s)
        assert one.iterations == batch[r].iterations
        assert rel(batch[r].solutions, one.solutions) <= 1e-12


def test_forward_config0_full_size_drawdown():
    """BASELINE configs[0] at full size: drawdown at the 16 receivers vs the oracle."""
    cfg, lk, ls, grid, ops = fd_case(0)
    p = _pencil(cfg, lk, ls)
    b = ofd_point(grid, cfg.sources[0]).real
    solver = L.SolverConfig(kind="single")
    sol, dd = L._forward(p, L.ForwardProblem(b, cfg.rates[0], None, cfg.times, cfg.n_quad), solver, False,
                         receivers=np.array(cfg.receivers))
    oprob = ofw.ForwardProblem(ops.stiffness, ops.mass, b, cfg.rates[0], None, cfg.times, cfg.n_quad)
    ref = ofw.solve_forward(oprob, ofw.SolverConfig(kind="single"))
    from oracle import fd as ofd
    for r, q in enumerate(cfg.receivers):
        e = ofd.point_weights(grid, q)
        ref_r = e @ ref.heads
        assert np.max(np.abs(dd[r] - ref_r) / np.abs(ref_r)) <= 1e-8
    assert rel(sol.heads, ref.heads) <= 1e-8
    for t in range(len(cfg.times)):
        assert sol.diagnostics[t].iterations == ref.diagnostics[t].iterations
        assert sol.diagnostics[t].all_converged


def test_forward_batch_pooled_matches_oracle():
    cfg, lk, ls, grid, ops = fd_case(1, (64, 64), n_times=3)
    p = _pencil(cfg, lk, ls)
    b = ofd_point(grid, cfg.sources[5]).real
    prob = L.ForwardProblem(b, 1e-4, None, cfg.times, cfg.n_quad)
    got = L.solve_forward_batch(p, prob)
    oprob = ofw.ForwardProblem(ops.stiffness, ops.mass, b, 1e-4, None, cfg.times, cfg.n_quad)
    ref = ofw.solve_forward_batch(oprob)
    assert rel(got.heads, ref.heads) <= 1e-8
    assert got.diagnostics[0].iterations == ref.diagnostics[0].iterations


def test_forward_with_initial_head():
    cfg, lk, ls, grid, ops = fd_case(0, (40, 40), n_times=2)
    p = _pencil(cfg, lk, ls)
    b = ofd_point(grid, (0.5, 0.5)).real
    rng = np.random.default_rng(1)
    phi0 = rng.standard_normal(grid.n_cells) * 1e-3
    prob = L.ForwardProblem(b, 1e-4, phi0, cfg.times, cfg.n_quad)
    got = L.solve_forward(p, prob, L.SolverConfig(kind="flexible"))
    oprob = ofw.ForwardProblem(ops.stiffness, ops.mass, b, 1e-4, phi0, cfg.times, cfg.n_quad)
    ref = ofw.solve_forward(oprob)
    assert rel(got.heads, ref.heads) <= 1e-8


def _experiment(cfg, grid_o, include_s):
    g = L.Grid(tuple(cfg.shape), cfg.h)
    solver = L.SolverConfig(kind=cfg.solver_kind)
    ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                         solver=solver, include_storativity=include_s)
    oex = ojac.ThtExperiment(grid_o, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                             solver=ofw.SolverConfig(kind=cfg.solver_kind), include_storativity=include_s)
    return ex, oex


def test_jacobian_config2_reduced():
    """BASELINE configs[2] statistics on 48^2 with all 9 sources x 25 receivers, 2 times."""
    cfg, lk, ls, grid, ops = fd_case(2, (48, 48), n_times=2)
    ex, oex = _experiment(cfg, grid, True)
    got = L.ThtForwardModel(ex, ls).jacobian(lk)
    ref = ojac.ThtForwardModel(oex, ls).jacobian(lk)
    assert np.max(np.abs(got.predictions - ref.predictions) / np.abs(ref.predictions)) <= 1e-8
    row, entry, s_err = jacobian_errors(got.jacobian, ref.jacobian, grid.n_cells, True)
    assert row <= 1e-8 and entry <= 1e-8 and s_err <= 1e-8, (row, entry, s_err)


def test_jacobian_3d_reduced():
    """BASELINE configs[4] statistics on 12^3, 3 sources x 5 receivers, 2 times."""
    cfg, lk, ls, grid, ops = fd_case(4, (12, 12, 12), n_src=3, n_rec=5, n_times=2)
    ex, oex = _experiment(cfg, grid, True)
    got = L.ThtForwardModel(ex, ls).jacobian(lk)
    ref = ojac.ThtForwardModel(oex, ls).jacobian(lk)
    assert np.max(np.abs(got.predictions - ref.predictions) / np.abs(ref.predictions)) <= 1e-8
    row, entry, s_err = jacobian_errors(got.jacobian, ref.jacobian, grid.n_cells, True)
    assert row <= 1e-8 and entry <= 1e-8 and s_err <= 1e-8, (row, entry, s_err)


@pytest.mark.parametrize("shape,n_src,n_rec", [((16, 16, 16), 16, 64), ((14, 14, 14), 5, 7)])
def test_jacobian_3d_tiles(shape, n_src, n_rec):
    """The tensor-core Jacobian's tile paths: 4-cell tiles with the full 16 x 64 item set
    (every consumer warp and both source m-tiles live), and the 2-cell fallback (nx % 4 != 0)."""
    cfg, lk, ls, grid, ops = fd_case(4, shape, n_src=n_src, n_rec=n_rec, n_times=1)
    ex, oex = _experiment(cfg, grid, True)
    got = L.ThtForwardModel(ex, ls).jacobian(lk)
    ref = ojac.ThtForwardModel(oex, ls).jacobian(lk)
    assert np.max(np.abs(got.predictions - ref.predictions) / np.abs(ref.predictions)) <= 1e-8
    row, entry, s_err = jacobian_errors(got.jacobian, ref.jacobian, grid.n_cells, True)
    assert row <= 1e-8 and entry <= 1e-8 and s_err <= 1e-8, (row, entry, s_err)


def test_predict_matches_jacobian_predictions():
    cfg, lk, ls, grid, ops = fd_case(2, (32, 32), n_src=2, n_rec=3, n_times=2)
    ex, _ = _experiment(cfg, grid, False)
    model = L.ThtForwardModel(ex, ls)
    pred = model.predict(lk)
    jr = model.jacobian(lk)
    assert rel(pred, jr.predictions) <= 1e-9


@pytest.mark.parametrize("index", [1, 2, 3, 4])
def test_full_size_self_checks(index):
    """BASELINE configs[1..4] at their full sizes (512^2 .. 128^3), where the oracle cannot run: size-independent
    properties of the discrete model.  (1) Scaling both kappa and S by e^eps scales (K + zM) and
    hence every shifted solution by e^-eps, so each Jacobian row sums to minus its prediction
    (kappa block + S block; the oracle satisfies it to 8e-12 at 12^3).  (2) Reciprocity: swapping
    the source and receiver points leaves the predictions unchanged (K, M symmetric, the same
    point weights for both)."""
    cfg = inputs.config(index)
    lk, ls = cfg.fields()
    g = L.Grid(tuple(cfg.shape), cfg.h)
    src, rec, times = cfg.sources[:2], cfg.receivers[:2], cfg.times[:1]
    solver = L.SolverConfig(kind=cfg.solver_kind)
    ex = L.ThtExperiment(g, src, [1e-4] * 2, rec, times, cfg.n_quad, solver=solver, include_storativity=True)
    model = L.ThtForwardModel(ex, ls)
    jr = model.jacobian(lk)
    assert jr.jacobian.shape == (4, 2 * g.n_cells)
    row_sum = jr.jacobian.sum(axis=1)
    assert np.max(np.abs(row_sum + jr.predictions)) <= 1e-8 * np.max(np.abs(jr.predictions))
    ex_swapped = L.ThtExperiment(g, rec, [1e-4] * 2, src, times, cfg.n_quad, solver=solver)
    pred_swapped = L.ThtForwardModel(ex_swapped, ls).predict(lk).reshape(2, 2)
    pred = jr.predictions.reshape(2, 2)
    assert np.max(np.abs(pred - pred_swapped.T)) <= 1e-8 * np.max(np.abs(pred))

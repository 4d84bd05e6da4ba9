"""Crank-Nicolson (forward.cpp:200-258) and the condition estimate (condest.cpp:11-49) on the
device against the oracle."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import condest as ocd
from oracle import fem, fields
from oracle import forward as ofw
from paper_1409_2556_b200 import laptomo as L

from .helpers import fd_case, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("index,shape", [(0, (40, 32)), (4, (16, 16, 12))])
def test_crank_nicolson_matches_oracle_fd(index, shape):
    cfg, lk, ls, grid, ops = fd_case(index, shape)
    from oracle import fd as ofd
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    b = ofd.point_weights(grid, tuple(0.45 * m * cfg.h for m in cfg.shape))
    times = [0.0, 250.0, 1000.0, 1730.0]
    rng = np.random.default_rng(2)
    h0 = 1e-3 * rng.standard_normal(grid.n_cells)
    got, steps = L.crank_nicolson(p, b, 1e-4, h0, 50.0, times, return_steps=True)
    ref, rsteps = ofw.crank_nicolson(ops.stiffness, ops.mass, b, 1e-4, h0, 50.0, times, return_steps=True)
    assert steps == rsteps == 35
    assert np.array_equal(got[:, 0], h0)
    for s in range(1, len(times)):
        assert rel(got[:, s], ref[:, s]) <= 1e-9


def test_crank_nicolson_lockstep_sources_and_laplace_crosscheck():
    """Two sources in lockstep; SPEC acceptance 2 on the device: Richardson-calibrated CN vs the
    Laplace forward solve on the reference's P1 41^2 Franke mesh, 1e-3."""
    mesh = fem.build_mesh(41, 100.0)
    lk = fields.franke_field(mesh, 1.6, np.log(1e-4))
    ls = np.full(mesh.n_elements(), np.log(1e-5))
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    p = L.ShiftedPencil(L.build_mesh(41, 100.0), lk, ls)
    b1 = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    b2 = ops.restrict_to_free(fem.point_source(mesh, 30.0, 65.0))
    t = 300.0
    h1 = L.crank_nicolson(p, np.stack([b1, b2]), [8.5e-4, 4e-4], None, 2.0, [t])
    h2 = L.crank_nicolson(p, b1, 8.5e-4, None, 1.0, [t])
    ref2 = ofw.crank_nicolson(ops.stiffness, ops.mass, b2, 4e-4, None, 2.0, [t])
    assert rel(h1[1][:, 0], ref2[:, 0]) <= 1e-9
    lap = L.solve_forward(p, L.ForwardProblem(b1, 8.5e-4, None, [t], 40)).heads[:, 0]
    rich = (4.0 * h2[:, 0] - h1[0][:, 0]) / 3.0
    assert np.linalg.norm(rich - lap) / np.linalg.norm(lap) <= 1e-3
    with pytest.raises(ValueError):
        L.crank_nicolson(p, b1, 1.0, None, -1.0, [t])


@pytest.mark.parametrize("z", [-0.03 + 0.02j, 0.5 - 0.2j])
def test_condition_estimate_matches_oracle_and_bounds_kappa(z):
    cfg, lk, ls, grid, ops = fd_case(0, (24, 20))
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    A = (ops.stiffness + z * ops.mass).tocsc()
    AH = (ops.stiffness + np.conj(z) * ops.mass).tocsc()
    lu, luh = spla.splu(A), spla.splu(AH)
    n = grid.n_cells
    na_ref = ocd.estimate_norm_1(n, lambda x: A @ x, lambda x: AH @ x)
    ni_ref = ocd.estimate_norm_1(n, lu.solve, luh.solve)
    na, ni = L.estimate_norms_1(p, z)
    assert abs(na - na_ref) <= 1e-12 * na_ref
    assert abs(ni - ni_ref) <= 1e-8 * ni_ref
    cond = L.estimate_condition_1norm(p, z)
    Ad = A.toarray()
    exact = np.linalg.norm(Ad, 1) * np.linalg.norm(np.linalg.inv(Ad), 1)
    assert cond <= exact * (1 + 1e-8) and cond >= 0.1 * exact

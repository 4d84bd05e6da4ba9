"""The Gauss-Newton step on the device (inversion.cpp:50-186) against the
oracle: the exact FFT grid prior against the dense Q, the reference's dense-Q path, and one
geostatistical step of a THT inversion with the device Jacobian."""
import numpy as np
import pytest

from oracle import fd as ofd
from oracle import forward as ofw
from oracle import inversion as oinv
from oracle import jacobian as ojac
from paper_1409_2556_b200 import inputs
from paper_1409_2556_b200 import inversion as I
from paper_1409_2556_b200 import laptomo as L

pytestmark = pytest.mark.gpu


def _linear(shape, dims_h, seed=3, n_y=15, two_blocks=True):
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    h = dims_h
    blocks = [(1.3, (0.5, 0.4, 0.3)[: len(shape)]), (0.6, (0.3, 0.7, 0.2)[: len(shape)])][: 2 if two_blocks else 1]
    Qb = [oinv.grid_covariance(shape, h, v, l) for v, l in blocks]
    nb = len(blocks)
    Q = np.zeros((nb * n, nb * n))
    for b in range(nb):
        Q[b * n:(b + 1) * n, b * n:(b + 1) * n] = Qb[b]
    G = rng.standard_normal((n_y, nb * n))
    X = np.zeros((nb * n, nb))
    for b in range(nb):
        X[b * n:(b + 1) * n, b] = 1.0
    s_true = rng.standard_normal(nb * n)
    y = G @ s_true + 0.01 * rng.standard_normal(n_y)
    R = np.full(n_y, 1e-3)
    gp = I.GridPrior(L.Grid(tuple(shape), h), [v for v, _ in blocks], [l for _, l in blocks])
    return G, Q, X, R, y, gp


@pytest.mark.parametrize("shape,h", [((7, 6), 0.2), ((5, 4, 3), 0.25)])
def test_linear_step_grid_prior_equals_dense_and_oracle(shape, h):
    G, Q, X, R, y, gp = _linear(shape, h)
    pred = lambda s: G @ s  # noqa: E731
    jac = lambda s: (G, G @ s)  # noqa: E731
    s0 = 0.1 * np.ones(G.shape[1])
    b0 = np.zeros(X.shape[1])
    ref = oinv.GaussNewtonSolver(oinv.InversionProblem(y, R, X, Q, pred, jac)).step(s0, b0)
    dense = I.GaussNewtonSolver(I.InversionProblem(y, R, X, Q, pred, jac)).step(s0, b0)
    grid = I.GaussNewtonSolver(I.InversionProblem(y, R, X, gp, pred, jac)).step(s0, b0)
    for got in (dense, grid):
        assert got.alpha == ref.alpha
        assert np.max(np.abs(got.s - ref.s)) <= 1e-9 * np.max(np.abs(ref.s))
        assert np.max(np.abs(got.beta - ref.beta)) <= 1e-9 * max(1.0, np.max(np.abs(ref.beta)))
        assert np.max(np.abs(got.xi - ref.xi)) <= 1e-8 * np.max(np.abs(ref.xi))
        assert abs(got.objective - ref.objective) <= 1e-8 * abs(ref.objective)
        assert abs(got.prior - ref.prior) <= 1e-7 * abs(ref.prior)
        assert got.saddle_residual <= 1e-10


def test_invert_matches_oracle_history():
    G, Q, X, R, y, gp = _linear((6, 6), 0.2, seed=5, two_blocks=False)
    pred = lambda s: G @ s  # noqa: E731
    jac = lambda s: (G, G @ s)  # noqa: E731
    s0 = np.zeros(G.shape[1])
    b0 = np.zeros(1)
    ref = oinv.GaussNewtonSolver(oinv.InversionProblem(y, R, X, Q, pred, jac)).invert(s0, b0)
    got = I.GaussNewtonSolver(I.InversionProblem(y, R, X, gp, pred, jac)).invert(s0, b0)
    assert got.converged == ref.converged and got.stop_reason == ref.stop_reason
    assert len(got.history) == len(ref.history)
    assert np.max(np.abs(got.s_hat - ref.s_hat)) <= 1e-9 * np.max(np.abs(ref.s_hat))


def test_tht_gauss_newton_step_with_device_jacobian():
    """One geostatistical step (§5, inversion.cpp:78-148) of a 2-D THT inversion for
    ln kappa: the device forward model (lt_jacobian_slice straight into the step's device
    buffer, lt_predict) with the FFT grid prior, against the oracle forward model with the dense
    prior."""
    cfg = inputs.config(2).scaled((14, 12), n_src=2, n_rec=3, n_times=2)
    lk_true, ls_true = cfg.fields()
    g = L.Grid(tuple(cfg.shape), cfg.h)
    n = g.n_cells
    ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                         solver=L.SolverConfig(kind="flexible"), include_storativity=False)
    model = L.ThtForwardModel(ex, ls_true)
    predict, djac, order = I.tht_handles(model)
    y = predict(lk_true)
    y = y + 0.01 * np.max(np.abs(y)) * np.random.default_rng(9).standard_normal(y.size)
    R = np.full(y.size, (0.01 * np.max(np.abs(y))) ** 2)
    X = np.ones((n, 1))
    var, corr = 2.0, (0.1, 0.1)
    gp = I.GridPrior(g, [var], [corr])
    s0 = np.full(n, -9.0)
    b0 = np.array([-9.0])
    got = I.GaussNewtonSolver(I.InversionProblem(y, R, X, gp, predict, djac)).step(s0, b0)
    # oracle: the same experiment, dense prior, rows in the same (time-major) order
    grid = ofd.Grid(tuple(cfg.shape), cfg.h)
    oex = ojac.ThtExperiment(grid, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                             solver=ofw.SolverConfig(kind="flexible"), include_storativity=False)
    omodel = ojac.ThtForwardModel(oex, ls_true)
    pairs = len(cfg.sources) * len(cfg.receivers)
    nt = len(cfg.times)
    perm = np.array([q * nt + t for t in range(nt) for q in range(pairs)])

    def opred(s):
        return omodel.predict(s)[perm]

    def ojacf(s):
        r = omodel.jacobian(s)
        return r.jacobian[perm], r.predictions[perm]

    Q = oinv.grid_covariance(cfg.shape, cfg.h, var, corr)
    ref = oinv.GaussNewtonSolver(oinv.InversionProblem(y, R, X, Q, opred, ojacf)).step(s0, b0)
    assert got.alpha == ref.alpha
    assert np.max(np.abs(got.s - ref.s)) <= 1e-6 * np.max(np.abs(ref.s - s0))
    assert abs(got.objective - ref.objective) <= 1e-6 * abs(ref.objective)
    assert got.objective < oinv.GaussNewtonSolver(oinv.InversionProblem(y, R, X, Q, opred, ojacf)).objective(s0, b0)

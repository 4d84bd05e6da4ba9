"""The oracle's Gauss-Newton inversion (inversion.cpp) on a linear problem, where one undamped
step lands on the closed-form MAP estimate of the geostatistical approach (CPU)."""
import numpy as np
import pytest

from oracle import inversion as oinv


def linear_problem(seed=0, n_y=12, shape=(6, 5)):
    rng = np.random.default_rng(seed)
    n_s = int(np.prod(shape))
    Q = oinv.grid_covariance(shape, 0.2, 1.3, (0.5, 0.4))
    G = rng.standard_normal((n_y, n_s))
    X = np.ones((n_s, 1))
    s_true = rng.standard_normal(n_s)
    y = G @ s_true + 0.01 * rng.standard_normal(n_y)
    R = np.full(n_y, 1e-4)
    return oinv.InversionProblem(y, R, X, Q, lambda s: G @ s, lambda s: (G, G @ s)), G, Q, X, R, y


def test_linear_step_is_the_map_estimate():
    pb, G, Q, X, R, y = linear_problem()
    it = oinv.GaussNewtonSolver(pb).step(np.zeros(G.shape[1]), np.zeros(1))
    # closed form (Kitanidis 1995): [G Q G^T + R, G X; (G X)^T, 0] [xi; beta] = [y; 0]
    n_y = y.size
    A = np.block([[G @ Q @ G.T + np.diag(R), G @ X], [(G @ X).T, np.zeros((1, 1))]])
    sol = np.linalg.solve(A, np.concatenate([y, [0.0]]))
    s_map = X @ sol[n_y:] + Q @ G.T @ sol[:n_y]
    assert it.alpha == 1.0
    assert np.allclose(it.s, s_map, rtol=0, atol=1e-10 * np.abs(s_map).max())
    assert it.saddle_residual <= 1e-12 and it.drift_violation <= 1e-8


def test_invert_stops_and_checks():
    pb, G, Q, X, R, y = linear_problem(1)
    res = oinv.GaussNewtonSolver(pb).invert(np.zeros(G.shape[1]), np.zeros(1), oinv.GnOptions(max_gn=5))
    assert res.converged and len(res.history) == 2
    assert res.stop_reason in ("relative step norm below rtol", "relative objective decrease below rtol")
    bad = oinv.InversionProblem(y, -R, X, Q, pb.predict, pb.jacobian_and_predict)
    with pytest.raises(ValueError):
        oinv.GaussNewtonSolver(bad)
    with pytest.raises(ValueError):
        oinv.GaussNewtonSolver(pb).invert(np.zeros(G.shape[1]), np.zeros(1), oinv.GnOptions(max_gn=0))

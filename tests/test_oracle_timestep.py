"""The oracle's Crank-Nicolson integrator (forward.cpp:200-258) and Hager condition estimate
(condest.cpp:11-49) against the reference SPEC's known answers (CPU)."""
import numpy as np
import pytest

from oracle import condest as ocd
from oracle import fem, fields
from oracle import forward as ofw


def test_condest_identity_and_diagonal():
    # SPEC.md: identity -> 1; diag(1, 1e-6) -> 1e6 exactly (estimator exact on diagonal matrices)
    I = lambda x: x  # noqa: E731
    assert ocd.estimate_condition_1norm(5, I, I, I, I) == pytest.approx(1.0, abs=1e-15)
    d = np.array([1.0, 1e-6])
    A = lambda x: d * x  # noqa: E731
    Ai = lambda x: x / d  # noqa: E731
    assert ocd.estimate_condition_1norm(2, A, A, Ai, Ai) == pytest.approx(1e6, rel=1e-15)
    with pytest.raises(ValueError):
        ocd.estimate_norm_1(0, I, I)


def test_condest_lower_bound_on_random_complex_matrices():
    """SPEC.md acceptance 10: 100 seeded 50 x 50 complex matrices: estimate <= exact kappa_1
    always, >= 0.1 exact in >= 90% of the seeds."""
    good = 0
    for seed in range(100):
        rng = np.random.default_rng(seed)
        A = rng.standard_normal((50, 50)) + 1j * rng.standard_normal((50, 50))
        Ai = np.linalg.inv(A)
        est = ocd.estimate_condition_1norm(50, lambda x: A @ x, lambda x: A.conj().T @ x, lambda x: Ai @ x,
                                           lambda x: Ai.conj().T @ x)
        exact = np.linalg.norm(A, 1) * np.linalg.norm(Ai, 1)
        assert est <= exact * (1 + 1e-12)
        good += est >= 0.1 * exact
    assert good >= 90


def test_crank_nicolson_matches_laplace_forward():
    """SPEC.md acceptance 2: 41^2 mesh, Franke field variance 1.6, t = 5 min: the Laplace-domain
    forward solve (N_z = 40, flexible, tol 1e-10) and the Richardson-calibrated Crank-Nicolson
    (dt and dt/2) agree to 1e-3 relative L2."""
    mesh = fem.build_mesh(41, 100.0)
    lk = fields.franke_field(mesh, 1.6, np.log(1e-4))
    ls = np.full(mesh.n_elements(), np.log(1e-5))
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    t = 300.0
    lap = ofw.solve_forward(ofw.ForwardProblem(ops.stiffness, ops.mass, b, 8.5e-4, None, [t], 40)).heads[:, 0]
    h1, s1 = ofw.crank_nicolson(ops.stiffness, ops.mass, b, 8.5e-4, None, 2.0, [t], return_steps=True)
    h2 = ofw.crank_nicolson(ops.stiffness, ops.mass, b, 8.5e-4, None, 1.0, [t])
    rich = (4.0 * h2[:, 0] - h1[:, 0]) / 3.0
    assert s1 == 150
    assert np.linalg.norm(rich - lap) / np.linalg.norm(lap) <= 1e-3
    # interpolated sample between steps, and the t = 0 sample is the initial head
    mid = ofw.crank_nicolson(ops.stiffness, ops.mass, b, 8.5e-4, None, 2.0, [0.0, 299.0, t])
    assert np.all(mid[:, 0] == 0.0)
    assert np.linalg.norm(mid[:, 1] - 0.5 * (h1[:, 0] + ofw.crank_nicolson(
        ops.stiffness, ops.mass, b, 8.5e-4, None, 2.0, [298.0])[:, 0])) <= 1e-12 * np.linalg.norm(h1)
    with pytest.raises(ValueError):
        ofw.crank_nicolson(ops.stiffness, ops.mass, b, 8.5e-4, None, 0.0, [t])
    with pytest.raises(ValueError):
        ofw.crank_nicolson(ops.stiffness, ops.mass, b, 8.5e-4, None, 1.0, [])

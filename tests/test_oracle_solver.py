"""Oracle pinning: shifted-solver known answers and invariants from the reference
SPEC and acceptance criterion 7."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import shifted_solver as S
from oracle import talbot as T


def _pencil(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    K = A @ A.T + n * np.eye(n)
    M = np.diag(rng.uniform(0.5, 2.0, n))
    return sp.csr_matrix(K), sp.csr_matrix(M), rng


def test_schedule_examples():
    s = S.select_preconditioner_shifts([1 + 1j, 5 + 2j])
    assert s.taus == [1 + 1j, 5 + 2j] and s.pattern == [0, 0, 0, 1, 1]
    assert [s.tau_at(j) for j in range(6)] == [1 + 1j] * 3 + [5 + 2j] * 2 + [1 + 1j]
    single = S.select_preconditioner_shifts([2 + 3j])
    assert single.taus == [2 + 3j] and single.pattern == [0]
    with pytest.raises(ValueError):
        S.select_preconditioner_shifts([])


def test_schedule_ties():  # shifted_solver.cpp:89-92: ties -> smaller imaginary part, then index
    s = S.select_preconditioner_shifts([1 + 2j, 1 + 1j, 3 + 0j, 3 - 1j, 3 - 1j])
    assert s.taus == [1 + 1j, 3 + 0j]


def test_shift_equal_tau_exact_at_iteration_one():
    K, M, rng = _pencil(12, 0)
    b = rng.standard_normal(12) + 0j
    tau = 0.7 + 0.4j
    res = S.solve_shifted_single(S.ShiftedPencil(K, M), b, [tau], tau)
    assert res.all_converged and res.shifts[0].iteration == 1
    assert np.allclose(res.solutions[:, 0], np.linalg.solve((K + tau * M).toarray(), b), rtol=1e-12)


def test_diagonal_5x5_matches_direct():
    K = sp.diags([1.0, 2.0, 3.0, 4.0, 5.0]).tocsr()
    M = sp.identity(5, format="csr")
    shifts = [0.5 + 1j, 1.5 + 0.5j, 2.0 + 2j]
    b = np.arange(1, 6).astype(complex)
    p = S.ShiftedPencil(K, M)
    res = S.solve_shifted_flexible(p, b, shifts, S.select_preconditioner_shifts(shifts))
    direct = S.solve_shifted_direct(p, b, shifts)
    assert res.all_converged
    assert np.max(np.abs(res.solutions - direct)) <= 1e-12 * np.max(np.abs(direct))


def test_single_tau_schedule_reproduces_single():
    K, M, rng = _pencil(30, 1)
    b = rng.standard_normal(30) + 0j
    shifts = list(T.build_contour(16, 1.0).nodes * 3.0)
    tau = shifts[0]
    p = S.ShiftedPencil(K, M)
    a = S.solve_shifted_single(p, b, shifts, tau)
    c = S.solve_shifted_flexible(p, b, shifts, S.single_tau_schedule(tau))
    assert a.iterations == c.iterations
    assert np.max(np.abs(a.solutions - c.solutions)) <= 1e-12 * np.max(np.abs(a.solutions))


@pytest.mark.parametrize("seed", range(10))
def test_fom_residual_estimate_equals_true_residual(seed):  # SPEC.md:273-275, acceptance 7
    K, M, rng = _pencil(20, 100 + seed)
    b = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    shifts = list(rng.uniform(0.1, 2.0, 4) + 1j * rng.uniform(0.1, 2.0, 4))
    sched = S.select_preconditioner_shifts(shifts)
    p = S.ShiftedPencil(K, M)
    opts = S.ShiftedSolveOptions(variant="fom", maxit=5, tol=1e-300, keep_basis=True)
    res = S.solve_shifted_flexible(p, b, shifts, sched, opts)
    st = res.basis
    m = st.steps()
    for k, z in enumerate(shifts):
        hz = st.shifted_hessenberg(z)
        rhs = np.zeros(m, dtype=complex)
        rhs[0] = st.beta
        y = np.linalg.solve(hz[:m, :], rhs)
        x = st.U @ y
        true = np.linalg.norm(b - p.apply(z, x))
        eta = S.residual_estimate(st, z, y)
        floor = 1e-13 * np.linalg.norm(b)  # z = tau_m gives eta = 0 and a rounding-level true residual
        assert abs(eta - true) <= 1e-10 * true + floor
        if true <= 1e3 * floor:
            continue
        # FOM residual collinear with v_{m+1}
        r = b - p.apply(z, x)
        cos = abs(np.vdot(st.V[:, m], r)) / (np.linalg.norm(r) * np.linalg.norm(st.V[:, m]))
        assert abs(cos - 1) <= 1e-10


def test_residual_estimate_vanishes_at_tau():
    K, M, rng = _pencil(15, 3)
    b = rng.standard_normal(15) + 0j
    tau = 0.9 + 0.2j
    res = S.solve_shifted_single(S.ShiftedPencil(K, M), b, [2 + 1j], tau,
                                 S.ShiftedSolveOptions(maxit=3, tol=1e-300, keep_basis=True))
    st = res.basis
    assert S.residual_estimate(st, tau, np.ones(st.steps())) == 0.0
    with pytest.raises(ValueError):
        S.residual_estimate(st, tau, np.ones(st.steps() + 1))


def test_arnoldi_relation_orthogonality_monotone_history():  # SPEC.md:281-290, acceptance 7
    K, M, rng = _pencil(60, 5)
    b = rng.standard_normal(60) + 1j * rng.standard_normal(60)
    shifts = list(T.build_contour(20, 0.5).nodes)
    p = S.ShiftedPencil(K, M)
    res = S.solve_shifted_flexible(p, b, shifts, S.select_preconditioner_shifts(shifts),
                                   S.ShiftedSolveOptions(keep_basis=True))
    st = res.basis
    V = st.V
    assert np.max(np.abs(V.conj().T @ V - np.eye(V.shape[1]))) <= 1e-8
    Kd, Md = K.toarray(), M.toarray()
    for z in (0.3 + 0.1j, 1.0 + 2.0j, -0.2 + 0.5j):
        lhs = (Kd + z * Md) @ st.U
        rhs = V @ st.shifted_hessenberg(z)
        scale = (np.linalg.norm(Kd) + abs(z) * np.linalg.norm(Md)) * np.linalg.norm(st.U)
        assert np.linalg.norm(lhs - rhs) <= 1e-10 * scale
    for k, s in enumerate(res.shifts):
        h = np.array(s.history)
        assert np.all(np.diff(h) <= 1e-12 * h[:-1] + 1e-300)  # GMRES residuals nonincreasing
        assert s.converged and s.true_residual <= 1e-10  # frozen-shift correctness
        x = res.solutions[:, k]
        assert np.linalg.norm(b - p.apply(shifts[k], x)) / np.linalg.norm(b) <= 1e-10


def test_zero_rhs_converges_immediately():  # shifted_solver.cpp:147-156
    K, M, _ = _pencil(8, 9)
    res = S.solve_shifted_flexible(S.ShiftedPencil(K, M), np.zeros(8, complex), [1j, 2j],
                                   S.select_preconditioner_shifts([1j, 2j]))
    assert res.all_converged and res.iterations == 0
    assert all(s.estimate == 0.0 and s.true_residual == 0.0 for s in res.shifts)


def test_empty_schedule_rejected():  # shifted_solver.cpp:295-297
    K, M, _ = _pencil(5, 1)
    with pytest.raises(ValueError):
        S.solve_shifted_flexible(S.ShiftedPencil(K, M), np.ones(5, complex), [1j],
                                 S.PreconditionerSchedule([], []))


def test_unconverged_best_effort():  # shifted_solver.cpp:270-285
    K, M, rng = _pencil(40, 11)
    b = rng.standard_normal(40) + 0j
    shifts = [5 + 5j, -3 + 1j]
    res = S.solve_shifted_single(S.ShiftedPencil(K, M), b, shifts, 0.1 + 0.1j,
                                 S.ShiftedSolveOptions(maxit=2))
    assert not res.all_converged and res.unconverged()
    for k in res.unconverged():
        assert not math.isnan(res.shifts[k].true_residual)
        assert np.any(res.solutions[:, k] != 0)


def test_factorization_cache_by_exact_tau():  # shifted_solver.cpp:120-128
    K, M, _ = _pencil(6, 2)
    p = S.ShiftedPencil(K, M)
    p.factorization(1 + 1j)
    p.factorization(1 + 1j)
    p.factorization(1 + 1.0000001j)
    assert p.factorization_count() == 2

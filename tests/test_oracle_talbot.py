"""Oracle pinning: contour / quadrature known answers from the reference SPEC
 and acceptance criterion 1."""
import math

import numpy as np
import pytest

from oracle import talbot as T


def test_inverse_laplace_of_exponential_decay():
    # F(z) = 1/(z+1), t = 1, N_z = 24 -> e^-1 within 1e-8
    c = T.build_contour(24, 1.0)
    assert abs(T.inverse_laplace_sum(c, 1.0 / (c.nodes + 1.0)) - math.exp(-1.0)) <= 1e-8


@pytest.mark.parametrize("t", [1e-3, 1.0, 1e2, 1e5])
def test_inverse_laplace_of_heaviside(t):
    # F(z) = 1/z, N_z = 32 -> 1 within 1e-8, any t
    c = T.build_contour(32, t)
    assert abs(T.inverse_laplace_sum(c, 1.0 / c.nodes) - 1.0) <= 1e-8


def test_zero_values_give_zero():
    c = T.build_contour(16, 2.0)
    assert T.inverse_laplace_sum(c, np.zeros(8, dtype=complex)) == 0.0


def test_qhat_step():
    assert T.qhat_step(1.0, 2.0) == 0.5
    assert T.qhat_step(0.0, 1 + 1j) == 0
    with pytest.raises(ValueError):
        T.qhat_step(1.0, 0.0)


def test_contour_argument_checks():
    with pytest.raises(ValueError):
        T.build_contour(7, 1.0)
    with pytest.raises(ValueError):
        T.build_contour(2, 1.0)
    with pytest.raises(ValueError):
        T.build_contour(8, 0.0)


def test_midpoints_and_upper_half():
    c = T.build_contour(20, 300.0)
    assert np.allclose(c.thetas, (np.arange(10) + 0.5) * 2 * math.pi / 20)
    assert np.all(c.nodes.imag > 0)
    assert c.n_half() == 10


def test_time_scaling_halves_nodes():
    # t doubled -> every node's real and imaginary part halved
    a = T.build_contour(40, 300.0)
    b = T.build_contour(40, 600.0)
    assert np.allclose(b.nodes, a.nodes / 2, rtol=1e-14, atol=0)


def test_theta_zero_limit():
    # SPEC.md:179 with the code's alpha: z(0) = sigma + mu / alpha (talbot.cpp:31)
    p = T.TalbotParams()
    z = T.contour_point(p, 32, 1.0, 0.0)
    assert abs(z - (p.sigma0 * 32 + p.mu0 * 32 / p.alpha)) < 1e-12
    assert T.contour_derivative(p, 32, 1.0, 0.0) == complex(0.0, p.mu0 * 32 * p.nu)


def test_real_crossing_encloses_origin():
    p = T.TalbotParams()
    assert p.sigma0 + p.mu0 / p.alpha > 0


def test_conjugate_symmetry_full_contour():
    # the full N_z-node sum has a negligible imaginary part
    n, t = 32, 1.0
    p = T.TalbotParams()
    thetas = (np.arange(n) + 0.5) * 2 * math.pi / n - math.pi
    z = np.array([T.contour_point(p, n, t, th) for th in thetas])
    dz = np.array([T.contour_derivative(p, n, t, th) for th in thetas])
    w = -1j / n * np.exp(z * t) * dz
    full = np.sum(w / (z + 0.3))
    assert abs(full.imag) <= 1e-10 * abs(full.real)
    half = T.inverse_laplace_sum(T.build_contour(n, t), 1.0 / (T.build_contour(n, t).nodes + 0.3))
    assert abs(full.real - half) <= 1e-12 * abs(half)


def test_exponential_convergence():
    # acceptance 1: log-error linear in N_z with negative slope, R^2 >= 0.98
    ns = np.arange(8, 33, 4)
    errs = []
    for n in ns:
        c = T.build_contour(int(n), 1.0)
        errs.append(max(abs(T.inverse_laplace_sum(c, 1.0 / (c.nodes + 1.0)) - math.exp(-1.0)), 1e-12))
    errs = np.array(errs)
    keep = errs > 1e-12  # fit the geometric decay before the 1e-12 floor
    y = np.log(errs[keep])
    ns = ns[keep]
    assert keep.sum() >= 4
    A = np.vstack([ns, np.ones_like(ns)]).T
    coef, res, *_ = np.linalg.lstsq(A, y, rcond=None)
    r2 = 1 - res[0] / np.sum((y - y.mean()) ** 2)
    assert coef[0] < 0 and r2 >= 0.98

"""Oracle: cotangent (Talbot-type) contour and quadrature.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Restates /root/reference/proj/src/talbot.cpp and include/laptomo/talbot.hpp.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class TalbotParams:
    """talbot.hpp:23-28 (defaults: optimised cotangent-contour constants)."""

    sigma0: float = -0.6122
    mu0: float = 0.5017
    nu: float = 0.2645 / 0.5017
    alpha: float = 0.6407


@dataclass
class TalbotContour:
    """talbot.hpp:33-43: upper-half nodes only."""

    n_quad: int
    time: float
    sigma: float
    mu: float
    nu: float
    alpha: float
    thetas: np.ndarray = field(repr=False)
    nodes: np.ndarray = field(repr=False)
    dnodes: np.ndarray = field(repr=False)
    weights: np.ndarray = field(repr=False)

    def n_half(self) -> int:
        return int(self.nodes.shape[0])


def _check(n_quad: int, time: float) -> None:
    # talbot.cpp:14-21
    if n_quad < 4 or n_quad % 2 != 0:
        raise ValueError("build_contour: n_quad must be even and at least 4")
    if not (time > 0.0):
        raise ValueError("build_contour: time must be positive")


def contour_point(params: TalbotParams, n_quad: int, time: float, theta: float) -> complex:
    """talbot.cpp:25-33."""
    scale = n_quad / time
    sigma = params.sigma0 * scale
    mu = params.mu0 * scale
    a = params.alpha
    cot_term = 1.0 / a if theta == 0.0 else theta * math.cos(a * theta) / math.sin(a * theta)
    return complex(sigma + mu * cot_term, mu * params.nu * theta)


def contour_derivative(params: TalbotParams, n_quad: int, time: float, theta: float) -> complex:
    """talbot.cpp:35-47."""
    scale = n_quad / time
    mu = params.mu0 * scale
    a = params.alpha
    if theta == 0.0:
        dcot = 0.0
    else:
        s = math.sin(a * theta)
        dcot = math.cos(a * theta) / s - a * theta / (s * s)
    return complex(mu * dcot, mu * params.nu)


def build_contour(n_quad: int, time: float, params: TalbotParams = TalbotParams()) -> TalbotContour:
    """talbot.cpp:49-80: midpoint angles theta_k = (k + 1/2) 2 pi / N, k < N/2,
    weights w_k = -(i/N) e^{z_k t} z'_k."""
    _check(n_quad, time)
    scale = n_quad / time
    n_half = n_quad // 2
    spacing = 2.0 * math.pi / n_quad
    thetas = np.empty(n_half)
    nodes = np.empty(n_half, dtype=np.complex128)
    dnodes = np.empty(n_half, dtype=np.complex128)
    weights = np.empty(n_half, dtype=np.complex128)
    for k in range(n_half):
        theta = (k + 0.5) * spacing
        z = contour_point(params, n_quad, time, theta)
        dz = contour_derivative(params, n_quad, time, theta)
        thetas[k] = theta
        nodes[k] = z
        dnodes[k] = dz
        weights[k] = (-1j / float(n_quad)) * np.exp(z * time) * dz
    return TalbotContour(n_quad, time, params.sigma0 * scale, params.mu0 * scale, params.nu,
                         params.alpha, thetas, nodes, dnodes, weights)


def inverse_laplace_sum(contour: TalbotContour, values: np.ndarray):
    """talbot.cpp:82-94.  `values` is a length-n_half vector (scalar transform)
    or an n x n_half matrix (one column per retained node)."""
    values = np.asarray(values)
    if values.ndim == 1:
        if values.shape[0] != contour.n_half():
            raise ValueError("inverse_laplace_sum: one value per retained node required")
        return float(2.0 * np.sum(contour.weights * values).real)
    if values.shape[1] != contour.n_half():
        raise ValueError("inverse_laplace_sum: one column per retained node required")
    return 2.0 * (values @ contour.weights).real


def qhat_step(q0: float, z: complex) -> complex:
    """talbot.cpp:96-101."""
    if z == 0:
        raise ValueError("qhat_step: z must be nonzero")
    return q0 / z

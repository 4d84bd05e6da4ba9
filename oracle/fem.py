"""Oracle: structured P1 mesh, exact P1 assembly, point weights.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Restates /root/reference/proj/src/mesh.cpp and src/assembly.cpp (vectorised,
same arithmetic per entry).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class Mesh2D:
    """mesh.hpp:17-27."""

    n_per_side: int
    side_length: float
    nodes: np.ndarray  # (n_nodes, 2)
    elements: np.ndarray  # (n_elements, 3) CCW
    dirichlet_nodes: np.ndarray

    def n_nodes(self) -> int:
        return int(self.nodes.shape[0])

    def n_elements(self) -> int:
        return int(self.elements.shape[0])

    def spacing(self) -> float:
        return self.side_length / (self.n_per_side - 1)


def build_mesh(n_per_side: int, side_length: float) -> Mesh2D:
    """mesh.cpp:14-52: node a = j n + i; element 2c = (a, b, c), 2c+1 = (a, c, d)."""
    if n_per_side < 2:
        raise ValueError("build_mesh: n_per_side must be at least 2")
    if not (side_length > 0.0):
        raise ValueError("build_mesh: side length must be positive")
    n = n_per_side
    h = side_length / (n - 1)
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    nodes = np.stack([ii.ravel() * h, jj.ravel() * h], axis=1).astype(np.float64)
    on_b = (ii == 0) | (ii == n - 1) | (jj == 0) | (jj == n - 1)
    dirichlet = np.flatnonzero(on_b.ravel())
    cj, ci = np.meshgrid(np.arange(n - 1), np.arange(n - 1), indexing="ij")
    a = (cj * n + ci).ravel()
    b = (cj * n + ci + 1).ravel()
    c = ((cj + 1) * n + ci + 1).ravel()
    d = ((cj + 1) * n + ci).ravel()
    elements = np.empty((2 * a.size, 3), dtype=np.int64)
    elements[0::2] = np.stack([a, b, c], axis=1)
    elements[1::2] = np.stack([a, c, d], axis=1)
    return Mesh2D(n, float(side_length), nodes, elements, dirichlet)


def element_areas(mesh: Mesh2D) -> np.ndarray:
    """mesh.cpp:54-62 for every element."""
    p0 = mesh.nodes[mesh.elements[:, 0]]
    p1 = mesh.nodes[mesh.elements[:, 1]]
    p2 = mesh.nodes[mesh.elements[:, 2]]
    u = p1 - p0
    v = p2 - p0
    return 0.5 * (u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0])


def element_area(mesh: Mesh2D, e: int) -> float:
    return float(element_areas(mesh)[e])


def element_centroids(mesh: Mesh2D) -> np.ndarray:
    """mesh.cpp:64-75."""
    return mesh.nodes[mesh.elements].mean(axis=1)


def element_basis_gradients(mesh: Mesh2D) -> np.ndarray:
    """mesh.cpp:77-89 for every element: (n_elements, 3, 2)."""
    p0 = mesh.nodes[mesh.elements[:, 0]]
    p1 = mesh.nodes[mesh.elements[:, 1]]
    p2 = mesh.nodes[mesh.elements[:, 2]]
    two_area = 2.0 * element_areas(mesh)
    g = np.empty((mesh.n_elements(), 3, 2))
    g[:, 0, 0] = (p1[:, 1] - p2[:, 1]) / two_area
    g[:, 0, 1] = (p2[:, 0] - p1[:, 0]) / two_area
    g[:, 1, 0] = (p2[:, 1] - p0[:, 1]) / two_area
    g[:, 1, 1] = (p0[:, 0] - p2[:, 0]) / two_area
    g[:, 2, 0] = (p0[:, 1] - p1[:, 1]) / two_area
    g[:, 2, 1] = (p1[:, 0] - p0[:, 0]) / two_area
    return g


def point_source(mesh: Mesh2D, x: float, y: float) -> np.ndarray:
    """mesh.cpp:91-125: P1 barycentric weights of the containing triangle."""
    L = mesh.side_length
    tol = 1e-12 * L
    if x < -tol or x > L + tol or y < -tol or y > L + tol:
        raise ValueError("point_source: point lies outside the domain")
    x = min(max(x, 0.0), L)
    y = min(max(y, 0.0), L)
    n = mesh.n_per_side
    h = mesh.spacing()
    ci = min(int(math.floor(x / h)), n - 2)
    cj = min(int(math.floor(y / h)), n - 2)
    xi = x / h - ci
    eta = y / h - cj
    a = cj * n + ci
    b = cj * n + ci + 1
    c = (cj + 1) * n + ci + 1
    d = (cj + 1) * n + ci
    w = np.zeros(mesh.n_nodes())
    if xi >= eta:
        w[a] = 1.0 - xi
        w[b] = xi - eta
        w[c] = eta
    else:
        w[a] = 1.0 - eta
        w[c] = xi
        w[d] = eta - xi
    return w


@dataclass
class AssembledOperators:
    """assembly.hpp:22-35."""

    stiffness: sp.csr_matrix
    mass: sp.csr_matrix
    free_nodes: np.ndarray
    node_to_free: np.ndarray

    def n_free(self) -> int:
        return int(self.free_nodes.size)

    def restrict_to_free(self, full):
        return np.asarray(full)[self.free_nodes]

    def prolong_to_full(self, free):
        free = np.asarray(free)
        out = np.zeros(self.node_to_free.size, dtype=free.dtype)
        out[self.free_nodes] = free
        return out


def _check_fields(mesh, kappa, storativity):
    """assembly.cpp:14-22."""
    kappa = np.asarray(kappa, dtype=np.float64)
    storativity = np.asarray(storativity, dtype=np.float64)
    if kappa.shape[0] != mesh.n_elements() or storativity.shape[0] != mesh.n_elements():
        raise ValueError("assemble: one kappa and one storativity value per element")
    if np.any(kappa <= 0.0) or np.any(storativity <= 0.0):
        raise ValueError("assemble: kappa and storativity must be positive")
    return kappa, storativity


def _triplets(mesh, kappa, storativity):
    """assembly.cpp:24-41: K_ij = k_e A_e grad_i.grad_j, M_ij = s_e A_e (1+d_ij)/12."""
    area = element_areas(mesh)
    g = element_basis_gradients(mesh)
    gg = np.einsum("eid,ejd->eij", g, g)
    kv = kappa[:, None, None] * area[:, None, None] * gg
    mass_pattern = (np.ones((3, 3)) + np.eye(3)) / 12.0
    mv = storativity[:, None, None] * area[:, None, None] * mass_pattern[None]
    rows = np.repeat(mesh.elements[:, :, None], 3, axis=2)
    cols = np.repeat(mesh.elements[:, None, :], 3, axis=1)
    return rows.ravel(), cols.ravel(), kv.ravel(), mv.ravel()


def assemble_full(mesh: Mesh2D, kappa, storativity):
    """assembly.cpp:115-127."""
    kappa, storativity = _check_fields(mesh, kappa, storativity)
    r, c, kv, mv = _triplets(mesh, kappa, storativity)
    n = mesh.n_nodes()
    K = sp.coo_matrix((kv, (r, c)), shape=(n, n)).tocsr()
    M = sp.coo_matrix((mv, (r, c)), shape=(n, n)).tocsr()
    return K, M


def assemble(mesh: Mesh2D, kappa, storativity) -> AssembledOperators:
    """assembly.cpp:69-113: symmetric Dirichlet elimination."""
    kappa, storativity = _check_fields(mesh, kappa, storativity)
    on_b = np.zeros(mesh.n_nodes(), dtype=bool)
    on_b[mesh.dirichlet_nodes] = True
    free_nodes = np.flatnonzero(~on_b)
    node_to_free = -np.ones(mesh.n_nodes(), dtype=np.int64)
    node_to_free[free_nodes] = np.arange(free_nodes.size)
    r, c, kv, mv = _triplets(mesh, kappa, storativity)
    fr, fc = node_to_free[r], node_to_free[c]
    keep = (fr >= 0) & (fc >= 0)
    nf = free_nodes.size
    K = sp.coo_matrix((kv[keep], (fr[keep], fc[keep])), shape=(nf, nf)).tocsr()
    M = sp.coo_matrix((mv[keep], (fr[keep], fc[keep])), shape=(nf, nf)).tocsr()
    return AssembledOperators(K, M, free_nodes, node_to_free)

"""Oracle: cell-centred finite-volume (FD) discretisation for the BASELINE configs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference discretises with P1 FEM only (`src/assembly.cpp:24-113`); the
BASELINE configs ask for cell-centred finite differences (5-point 2-D,
7-point 3-D).  This module is the documented extension (SURVEY.md Appendix
A), written to be consistent with the P1
scaling of the reference:

* face transmissibility  T_f = 2 k_a k_b / (k_a + k_b) * h^(d-2)  (harmonic mean),
* Dirichlet boundary face T_f = 2 k_a h^(d-2)  (zero ghost value at h/2),
* M = S_a h^d  (diagonal),
* sources / receivers: multilinear interpolation weights on cell centres
  (partition of unity, the FD analogue of `point_source`, mesh.cpp:91-125),
* discrete adjoint sensitivities, the FD analogue of
  `sensitivity_row_conductivity/storativity` (jacobian.cpp:57-125):
    J_k[a] = 2 Re sum_k w_k sum_{f ∋ a} (dT_f/dln k_a) (phi_a - phi_b)(psi_a - psi_b),
      dT_f/dln k_a = T_f k_b / (k_a + k_b) (interior), T_f (boundary, ghost 0),
    J_S[a] = 2 Re sum_k w_k z_k^p S_a h^d phi_a psi_a.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Tuple

import numpy as np
import scipy.sparse as sp


@dataclass(frozen=True)
class Grid:
    """Cell-centred grid on [0, n_x h] x [0, n_y h] (x [0, n_z h]); cell index
    a = (k n_y + j) n_x + i (x fastest)."""

    shape: Tuple[int, ...]  # (nx, ny) or (nx, ny, nz)
    h: float

    @property
    def dim(self) -> int:
        return len(self.shape)

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.shape))

    def array_shape(self) -> Tuple[int, ...]:
        """NumPy C-order shape with x fastest: (nz, ny, nx) / (ny, nx)."""
        return tuple(reversed(self.shape))


@dataclass
class FdOperators:
    """The FD pencil plus the face data the sensitivity rows need."""

    stiffness: sp.csr_matrix
    mass: sp.csr_matrix
    kappa: np.ndarray  # per cell (array_shape)
    storativity: np.ndarray
    grid: Grid

    def n_free(self) -> int:
        return self.grid.n_cells

    # Every cell is a free unknown (Dirichlet sits on the faces).
    def restrict_to_free(self, full):
        return np.asarray(full)

    def prolong_to_full(self, free):
        return np.asarray(free)


def _axes(grid: Grid):
    """NumPy axis of each physical direction: x is the last array axis."""
    d = grid.dim
    return [d - 1 - ax for ax in range(d)]


def face_transmissibilities(grid: Grid, kappa: np.ndarray):
    """Per direction: an array with n_dir + 1 faces along that direction
    (index 0 and n_dir are the Dirichlet boundary faces)."""
    kappa = np.asarray(kappa, dtype=np.float64).reshape(grid.array_shape())
    scale = grid.h ** (grid.dim - 2)
    faces = []
    for ax in _axes(grid):
        ka = np.take(kappa, range(0, kappa.shape[ax] - 1), axis=ax)
        kb = np.take(kappa, range(1, kappa.shape[ax]), axis=ax)
        interior = 2.0 * ka * kb / (ka + kb) * scale
        first = 2.0 * np.take(kappa, [0], axis=ax) * scale
        last = 2.0 * np.take(kappa, [kappa.shape[ax] - 1], axis=ax) * scale
        faces.append(np.concatenate([first, interior, last], axis=ax))
    return faces


def assemble_fd(grid: Grid, kappa, storativity) -> FdOperators:
    kappa = np.asarray(kappa, dtype=np.float64).reshape(grid.array_shape())
    storativity = np.asarray(storativity, dtype=np.float64).reshape(grid.array_shape())
    if np.any(kappa <= 0.0) or np.any(storativity <= 0.0):
        raise ValueError("assemble: kappa and storativity must be positive")
    n = grid.n_cells
    idx = np.arange(n).reshape(grid.array_shape())
    faces = face_transmissibilities(grid, kappa)
    diag = np.zeros(grid.array_shape())
    rows, cols, vals = [], [], []
    for ax, T in zip(_axes(grid), faces):
        nd = kappa.shape[ax]
        lo = np.take(T, range(0, nd), axis=ax)       # face on the low side of each cell
        hi = np.take(T, range(1, nd + 1), axis=ax)   # face on the high side
        diag += lo + hi
        t_int = np.take(T, range(1, nd), axis=ax)
        a = np.take(idx, range(0, nd - 1), axis=ax).ravel()
        b = np.take(idx, range(1, nd), axis=ax).ravel()
        rows += [a, b]
        cols += [b, a]
        vals += [-t_int.ravel(), -t_int.ravel()]
    rows.append(idx.ravel())
    cols.append(idx.ravel())
    vals.append(diag.ravel())
    K = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    M = sp.diags(storativity.ravel() * grid.h ** grid.dim).tocsr()
    return FdOperators(K, M, kappa, storativity, grid)


def point_weights(grid: Grid, point) -> np.ndarray:
    """Multilinear weights on the cell centres (i + 1/2) h; the point must lie
    in the hull of the cell centres."""
    point = np.asarray(point, dtype=np.float64)
    if point.shape[0] != grid.dim:
        raise ValueError("point_weights: dimension mismatch")
    w = np.zeros(grid.n_cells)
    base, fracs = [], []
    for d in range(grid.dim):
        xi = point[d] / grid.h - 0.5
        n = grid.shape[d]
        tol = 1e-12 * n
        if xi < -tol or xi > (n - 1) + tol:
            raise ValueError("point_weights: point lies outside the cell-centre hull")
        xi = min(max(xi, 0.0), float(n - 1))
        i0 = min(int(math.floor(xi)), max(n - 2, 0))
        base.append(i0)
        fracs.append(xi - i0)
    for corner in range(1 << grid.dim):
        weight = 1.0
        idx = []
        for d in range(grid.dim):
            bit = (corner >> d) & 1
            weight *= fracs[d] if bit else 1.0 - fracs[d]
            idx.append(base[d] + bit)
        if weight == 0.0:
            continue
        stride = 1
        flat = 0
        for d in range(grid.dim):
            flat += idx[d] * stride
            stride *= grid.shape[d]
        w[flat] += weight
    return w


def sensitivity_rows_fd(ops: FdOperators, forward_fields: np.ndarray, adjoint_fields: np.ndarray,
                        weights: np.ndarray, nodes: np.ndarray, include_storativity: bool,
                        z_factor: bool = True):
    """J_k and J_S rows (Appendix A).  fields: (n_cells, n_half) complex."""
    grid = ops.grid
    shp = grid.array_shape()
    kappa = ops.kappa
    scale = grid.h ** (grid.dim - 2)
    acc = np.zeros(shp, dtype=np.complex128)
    n_half = forward_fields.shape[1]
    for k in range(n_half):
        phi = forward_fields[:, k].reshape(shp)
        psi = adjoint_fields[:, k].reshape(shp)
        contrib = np.zeros(shp, dtype=np.complex128)
        for ax in _axes(grid):
            nd = shp[ax]
            sl_a = [slice(None)] * grid.dim
            sl_b = [slice(None)] * grid.dim
            sl_a[ax] = slice(0, nd - 1)
            sl_b[ax] = slice(1, nd)
            sl_a, sl_b = tuple(sl_a), tuple(sl_b)
            ka, kb = kappa[sl_a], kappa[sl_b]
            T = 2.0 * ka * kb / (ka + kb) * scale
            prod = (phi[sl_a] - phi[sl_b]) * (psi[sl_a] - psi[sl_b])
            contrib[sl_a] += T * kb / (ka + kb) * prod
            contrib[sl_b] += T * ka / (ka + kb) * prod
            # Boundary faces: ghost value 0, dT/dln k_a = T = 2 k_a h^(d-2).
            first = [slice(None)] * grid.dim
            last = [slice(None)] * grid.dim
            first[ax] = slice(0, 1)
            last[ax] = slice(nd - 1, nd)
            first, last = tuple(first), tuple(last)
            contrib[first] += 2.0 * kappa[first] * scale * phi[first] * psi[first]
            contrib[last] += 2.0 * kappa[last] * scale * phi[last] * psi[last]
        acc += weights[k] * contrib
    row_k = (2.0 * acc.real).ravel()
    row_s = None
    if include_storativity:
        acc_s = np.zeros(grid.n_cells, dtype=np.complex128)
        for k in range(n_half):
            zf = nodes[k] if z_factor else 1.0
            acc_s += weights[k] * zf * forward_fields[:, k] * adjoint_fields[:, k]
        row_s = 2.0 * acc_s.real * ops.storativity.ravel() * grid.h ** grid.dim
    return row_k, row_s

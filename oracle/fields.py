"""Oracle: the reference's test fields for the paper-regime known answers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Restates /root/reference/proj/src/fields.cpp:
  franke_function   fields.cpp:125-131
  franke_field      fields.cpp:133-150 (element centroids mapped to the unit square, affinely
                    rescaled to the target variance and mean)
  covariance_matrix fields.cpp:18-38, sample_field fields.cpp:62-81 and sample_field_on_mesh
                    fields.cpp:83-123 (exact jittered-Cholesky draw up to max_exact_points
                    centroids, else an exact draw on a coarse point grid interpolated
                    bilinearly).  The reference draws its standard normals with
                    std::mt19937_64 + std::normal_distribution (implementation-defined); here
                    they come from NumPy PCG64, so realisations differ from a reference binary
                    while the law (and the paper-regime iteration bands) are the same.
"""
from __future__ import annotations

import numpy as np

from .fem import Mesh2D, element_centroids


def franke_function(x, y):
    """fields.cpp:125-131."""
    t1 = 0.75 * np.exp(-((9 * x - 2) ** 2 + (9 * y - 2) ** 2) / 4.0)
    t2 = 0.75 * np.exp(-((9 * x + 1) ** 2) / 49.0 - (9 * y + 1) / 10.0)
    t3 = 0.5 * np.exp(-((9 * x - 7) ** 2 + (9 * y - 3) ** 2) / 4.0)
    t4 = -0.2 * np.exp(-((9 * x - 4) ** 2) - (9 * y - 7) ** 2)
    return t1 + t2 + t3 + t4


def franke_field(mesh: Mesh2D, target_variance: float, mean_log: float) -> np.ndarray:
    """fields.cpp:133-150: per-element log values."""
    if not target_variance > 0.0:
        raise ValueError("franke_field: target variance must be positive")
    c = element_centroids(mesh)
    raw = franke_function(c[:, 0] / mesh.side_length, c[:, 1] / mesh.side_length)
    mean = raw.mean()
    var = np.mean((raw - mean) ** 2)
    return mean_log + np.sqrt(target_variance / var) * (raw - mean)


def covariance_matrix(points: np.ndarray, theta: float, corr_length: float) -> np.ndarray:
    """fields.cpp:18-38."""
    d = np.sqrt(((points[:, None, :] - points[None, :, :]) ** 2).sum(-1))
    return theta * np.exp(-d / corr_length)


def _jittered_cholesky(q: np.ndarray) -> np.ndarray:
    """fields.cpp:44-59."""
    jitter = 1e-10 * np.max(np.diag(q))
    for attempt in range(7):
        work = q.copy()
        if attempt > 0:
            work[np.diag_indices_from(work)] += jitter
            jitter *= 2.0
        try:
            return np.linalg.cholesky(work)
        except np.linalg.LinAlgError:
            continue
    raise RuntimeError("sample_field: covariance Cholesky failed after max jitter")


def sample_field(covariance: np.ndarray, mean_log: float, seed: int) -> np.ndarray:
    """fields.cpp:62-81 (normals from PCG64(seed))."""
    n = covariance.shape[0]
    if np.max(np.abs(covariance)) == 0.0:
        return np.full(n, mean_log)
    chol = _jittered_cholesky(covariance)
    zeta = np.random.Generator(np.random.PCG64(seed)).standard_normal(n)
    return chol @ zeta + mean_log


def sample_field_on_mesh(mesh: Mesh2D, theta: float, corr_length: float, mean_log: float, seed: int,
                         max_exact_points: int = 4096) -> np.ndarray:
    """fields.cpp:83-123."""
    cent = element_centroids(mesh)
    if cent.shape[0] <= max_exact_points:
        return sample_field(covariance_matrix(cent, theta, corr_length), mean_log, seed)
    ng = max(2, int(np.floor(np.sqrt(float(max_exact_points)))))
    L = mesh.side_length
    hg = L / (ng - 1)
    gi, gj = np.meshgrid(np.arange(ng), np.arange(ng), indexing="xy")
    grid = np.stack([gi.ravel() * hg, gj.ravel() * hg], axis=1)  # row j * ng + i
    coarse = sample_field(covariance_matrix(grid, theta, corr_length), 0.0, seed)
    x = np.clip(cent[:, 0], 0.0, L)
    y = np.clip(cent[:, 1], 0.0, L)
    ci = np.minimum(np.floor(x / hg).astype(int), ng - 2)
    cj = np.minimum(np.floor(y / hg).astype(int), ng - 2)
    xi = x / hg - ci
    eta = y / hg - cj
    v00 = coarse[cj * ng + ci]
    v10 = coarse[cj * ng + ci + 1]
    v01 = coarse[(cj + 1) * ng + ci]
    v11 = coarse[(cj + 1) * ng + ci + 1]
    return mean_log + (1 - xi) * (1 - eta) * v00 + xi * (1 - eta) * v10 + (1 - xi) * eta * v01 + xi * eta * v11

"""Seeded synthetic inputs for the BASELINE configs.

BASELINE.json names no public dataset: seeded Gaussian random fields with the
stated statistics stand in for it.  Fields are drawn by circulant embedding
(FFT, NumPy PCG64), which replaces the reference's dense-Cholesky sampler
(`src/fields.cpp:45-123`; infeasible beyond ~10^4 points).  This is input
generation, not the hot path; both the GPU path and the CPU oracle consume
the same arrays.

Choices marked † in SURVEY.md §8d (unspecified by BASELINE.json) are frozen
here and repeated in DESIGN.md.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np


def grf_exponential(shape: Sequence[int], h: float, variance: float,
                    corr_lengths: Sequence[float], mean: float, seed: int,
                    noise: Optional[np.ndarray] = None) -> np.ndarray:
    """Stationary GRF with covariance var * exp(-|r / l|) (anisotropic l),
    sampled on cell centres by circulant embedding on a torus twice the grid.
    Returns an array in C order with x fastest: shape reversed(shape).
    `noise` (complex, indexed (x, y[, z]) over the doubled grid) replaces the PCG64 normals
    (the device generator lt_sample_field_grid is checked against this with shared noise)."""
    dim = len(shape)
    ext = [2 * n for n in shape]
    axes = []
    for d in range(dim):
        m = ext[d]
        lag = np.minimum(np.arange(m), m - np.arange(m)) * h
        axes.append(lag / corr_lengths[d])
    grids = np.meshgrid(*axes, indexing="ij")
    r = np.sqrt(sum(g * g for g in grids))
    cov = variance * np.exp(-r)
    lam = np.fft.fftn(cov).real
    lam = np.maximum(lam, 0.0)  # clip the (tiny) negative embedding modes
    if noise is None:
        rng = np.random.Generator(np.random.PCG64(seed))
        xi = rng.standard_normal(ext) + 1j * rng.standard_normal(ext)
    else:
        xi = np.asarray(noise, dtype=np.complex128).reshape(ext)
    total = float(np.prod(ext))
    field_c = np.fft.ifftn(np.sqrt(lam) * xi) * math.sqrt(total)
    sample = field_c.real[tuple(slice(0, n) for n in shape)]
    out = mean + sample  # indexed (x, y[, z])
    return np.ascontiguousarray(np.transpose(out))  # -> (z, y, x) / (y, x)


def lattice(values: Sequence[float], dim: int = 2, z: Optional[float] = None) -> List[Tuple]:
    pts = [(x, y) for y in values for x in values]
    if dim == 3:
        pts = [(x, y, z) for (x, y) in pts]
    return pts


@dataclass
class ThtConfig:
    name: str
    shape: Tuple[int, ...]
    h: float
    log_kappa: dict
    log_storativity: dict  # {"const": ln S} or GRF statistics
    sources: List[Tuple]
    receivers: List[Tuple]
    rates: List[float]
    times: List[float]
    n_quad: int
    solver_kind: str  # "single" | "flexible"
    jacobian: bool
    tol: float = 1e-10
    description: str = ""

    @property
    def dim(self) -> int:
        return len(self.shape)

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.shape))

    def fields(self):
        """(log_kappa, log_storativity) as flat float64 arrays (x fastest)."""
        lk = self.log_kappa
        log_kappa = grf_exponential(self.shape, self.h, lk["var"], lk["corr"], lk["mean"],
                                    lk["seed"]).ravel()
        ls = self.log_storativity
        if "const" in ls:
            log_s = np.full(self.n_cells, ls["const"])
        else:
            log_s = grf_exponential(self.shape, self.h, ls["var"], ls["corr"], ls["mean"],
                                    ls["seed"]).ravel()
        return log_kappa, log_s

    def scaled(self, shape: Tuple[int, ...], n_src: Optional[int] = None,
               n_rec: Optional[int] = None, n_times: Optional[int] = None) -> "ThtConfig":
        """Same statistics and geometry on a smaller grid (parity-test / CPU-sample size)."""
        extent = [n * self.h for n in self.shape]
        h = extent[0] / shape[0]
        out = ThtConfig(**{**self.__dict__})
        out.shape = tuple(shape)
        out.h = h
        out.name = f"{self.name}@{'x'.join(map(str, shape))}"
        if n_src is not None:
            out.sources = self.sources[:n_src]
            out.rates = self.rates[:n_src]
        if n_rec is not None:
            out.receivers = self.receivers[:n_rec]
        if n_times is not None:
            out.times = self.times[:n_times]
        return out


LN_S_1E5 = math.log(1e-5)


def _uniform_points(n: int, seed: int, lo: float = 0.05, hi: float = 0.95) -> List[Tuple]:
    rng = np.random.Generator(np.random.PCG64(seed))
    return [tuple(p) for p in rng.uniform(lo, hi, size=(n, 2))]


def config(index: int) -> ThtConfig:
    """The five BASELINE configs, all on [0,1]^2 / [0,1]^2 x [0, Lz]."""
    if index == 0:
        return ThtConfig(
            "c0-2d-forward-100x100", (100, 100), 0.01,
            {"mean": -9.0, "var": 1.0, "corr": (0.2, 0.2), "seed": 0}, {"const": LN_S_1E5},
            [(0.5, 0.5)], lattice([0.2, 0.4, 0.6, 0.8]), [1e-4],
            list(np.logspace(2, 5, 5)), 32, "single", False,
            description="BASELINE configs[0]")
    if index == 1:
        return ThtConfig(
            "c1-2d-batch-512x512", (512, 512), 1.0 / 512,
            {"mean": -9.0, "var": 1.0, "corr": (0.2, 0.2), "seed": 1}, {"const": LN_S_1E5},
            lattice([0.2, 0.4, 0.6, 0.8]), _uniform_points(32, 101), [1e-4] * 16,
            list(np.logspace(2, 5, 8)), 32, "flexible", False,
            description="BASELINE configs[1]")
    if index == 2:
        return ThtConfig(
            "c2-2d-jacobian-256x256", (256, 256), 1.0 / 256,
            {"mean": -9.0, "var": 2.0, "corr": (0.1, 0.1), "seed": 2},
            {"mean": -11.0, "var": 0.5, "corr": (0.1, 0.1), "seed": 3},
            lattice([0.25, 0.5, 0.75]), lattice([1 / 6, 2 / 6, 3 / 6, 4 / 6, 5 / 6]), [1e-4] * 9,
            list(np.logspace(2, 5, 5)), 24, "flexible", True,
            description="BASELINE configs[2]")
    if index == 3:
        return ThtConfig(
            "c3-3d-forward-128x128x64", (128, 128, 64), 1.0 / 128,
            {"mean": -9.0, "var": 1.0, "corr": (0.2, 0.2, 0.05), "seed": 4}, {"const": LN_S_1E5},
            lattice([0.25, 0.75], 3, 0.25), lattice([i / 9 for i in range(1, 9)], 3, 0.25),
            [1e-4] * 4, list(np.logspace(2, 6, 6)), 32, "flexible", False,
            description="BASELINE configs[3]")
    if index == 4:
        return ThtConfig(
            "c4-3d-jacobian-128^3", (128, 128, 128), 1.0 / 128,
            {"mean": -9.0, "var": 1.0, "corr": (0.2, 0.2, 0.05), "seed": 5},
            {"mean": LN_S_1E5, "var": 1.0, "corr": (0.2, 0.2, 0.05), "seed": 6},
            lattice([0.2, 0.4, 0.6, 0.8], 3, 0.5), lattice([i / 9 for i in range(1, 9)], 3, 0.5),
            [1e-4] * 16, list(np.logspace(2, 6, 4)), 32, "flexible", True,
            description="BASELINE configs[4] (headline)")
    raise ValueError(f"unknown config {index}")


def reduced(index: int, shape: Tuple[int, ...], n_src: Optional[int] = None,
            receivers: Optional[Sequence[int]] = None, n_times: Optional[int] = None) -> ThtConfig:
    """Config `index`'s statistics on a smaller box for the oracle parity fixtures.

    The spacing is h = 1 / shape[0] (unit extent along x, like every config), the other extents
    are shape[d] * h, the fields are drawn on the new grid with the same GRF statistics and
    seeds, and the source / receiver points are mapped linearly into the box (p_d * new extent /
    old extent), so the lattices keep their layout.  `receivers` selects receiver indices."""
    base = config(index)
    old_ext = [n * base.h for n in base.shape]
    h = 1.0 / shape[0]
    new_ext = [n * h for n in shape]
    scale = [new_ext[d] / old_ext[d] for d in range(len(shape))]

    def move(p):
        return tuple(float(p[d]) * scale[d] for d in range(len(shape)))

    out = ThtConfig(**{**base.__dict__})
    out.shape = tuple(shape)
    out.h = h
    out.name = f"{base.name}@box{'x'.join(map(str, shape))}"
    src = base.sources if n_src is None else base.sources[:n_src]
    out.sources = [move(p) for p in src]
    out.rates = base.rates[:len(src)]
    rec = base.receivers if receivers is None else [base.receivers[i] for i in receivers]
    out.receivers = [move(p) for p in rec]
    if n_times is not None:
        out.times = base.times[:n_times]
    return out

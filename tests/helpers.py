"""Shared test helpers: build the same seeded case for the oracle (CPU, SciPy)
and the device path (C ABI)."""
from __future__ import annotations

import numpy as np

from oracle import fd as ofd
from paper_1409_2556_b200 import inputs


def fd_case(index: int, shape=None, n_src=None, n_rec=None, n_times=None):
    cfg = inputs.config(index)
    if shape is not None or n_src is not None or n_rec is not None or n_times is not None:
        cfg = cfg.scaled(tuple(shape) if shape is not None else cfg.shape, n_src, n_rec, n_times)
    lk, ls = cfg.fields()
    grid = ofd.Grid(tuple(cfg.shape), cfg.h)
    ops = ofd.assemble_fd(grid, np.exp(lk), np.exp(ls))
    return cfg, lk, ls, grid, ops


def rel(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm((a - b).ravel())
    s = np.linalg.norm(b.ravel())
    return float(d / s) if s > 0 else float(d)


def jacobian_errors(J, Jref, n_cells: int, include_s: bool):
    """Per-row normwise error of the kappa block, entrywise error on entries above
    1e-3 of the row max (SPEC.md:547 floor convention), S block normwise relative to
    the kappa block norm (it is round-off in these configs)."""
    Jk, Rk = J[:, :n_cells], Jref[:, :n_cells]
    row_norm = np.max(np.linalg.norm(Jk - Rk, axis=1) / np.linalg.norm(Rk, axis=1))
    mask = np.abs(Rk) > 1e-3 * np.max(np.abs(Rk), axis=1, keepdims=True)
    entry = np.max(np.abs(Jk - Rk)[mask] / np.abs(Rk)[mask])
    s_err = 0.0
    if include_s:
        Js, Rs = J[:, n_cells:], Jref[:, n_cells:]
        s_err = float(np.max(np.linalg.norm(Js - Rs, axis=1) / np.linalg.norm(Rk, axis=1)))
    return float(row_norm), float(entry), s_err

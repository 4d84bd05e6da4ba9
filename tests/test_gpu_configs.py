"""Every BASELINE config through the production kernels against the CPU oracle's fixtures
(tests/golden/configs, made by scripts/make_config_golden.py; the oracle is the SciPy
restatement of the reference path).

  c1  configs[1] at full size (512^2, 16 sources batched x 32 receivers x 8 times, per-time
      flexible): every drawdown;
  c2  configs[2] at full size (256^2, 9 x 25 x 5, N = 24, both blocks): every prediction, every
      row normwise through a Gaussian sketch, 8 rows entrywise;
  c3  configs[3] statistics on the 64 x 64 x 16 box (colour-split V-cycle, TMA operator and
      transfers): every drawdown of 4 sources x 64 receivers x 6 times;
  c4  configs[4] statistics on the 64 x 32 x 24 box (as c3 plus the 4-cell tensor-core
      Jacobian): 16 sources x 8 receivers x 4 times, as c2.

Metric (north_star): drawdown and predictions 1e-8 relative per entry; the
kappa block of J per row normwise 1e-8 and entrywise 1e-8 on entries above 1e-3 of the row
max; the S block normwise relative to the kappa block (it is round-off in these configs).
All calls go through the C ABI.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1409_2556_b200 import laptomo as L

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "scripts"))
import make_config_golden as G  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-8


def fixture(name):
    d = np.load(ROOT / "tests" / "golden" / "configs" / f"{name}.npz")
    cfg = G.case(name)
    lk, ls = cfg.fields()
    assert G.field_hash(lk, ls) == str(d["field_sha256"]), "input generator drifted from the fixture"
    assert np.allclose(d["receivers"], np.array(cfg.receivers)) and np.allclose(d["times"], cfg.times)
    return d, cfg, lk, ls


def drawdown_errors(got, ref):
    """Per-entry relative error of every drawdown (source, receiver, time)."""
    return np.abs(got - ref) / np.abs(ref)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_forward_drawdown(name):
    d, cfg, lk, ls = fixture(name)
    p = L.ShiftedPencil(L.Grid(tuple(cfg.shape), cfg.h), lk, ls)
    got, diags = L.solve_forward_sources(p, cfg.sources, cfg.rates, cfg.times, cfg.n_quad, cfg.receivers,
                                         L.SolverConfig(kind=cfg.solver_kind))
    ref = d["drawdown"]
    assert got.shape == ref.shape
    assert all(dg.all_converged for dg in diags)
    err = drawdown_errors(got, ref)
    assert np.max(err) <= TOL, (np.max(err), np.unravel_index(np.argmax(err), err.shape))


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_jacobian(name):
    d, cfg, lk, ls = fixture(name)
    g = L.Grid(tuple(cfg.shape), cfg.h)
    ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                         solver=L.SolverConfig(kind=cfg.solver_kind), include_storativity=True)
    jr = L.ThtForwardModel(ex, ls).jacobian(lk)
    n = g.n_cells
    pred_err = np.abs(jr.predictions - d["predictions"]) / np.abs(d["predictions"])
    assert np.max(pred_err) <= TOL, np.max(pred_err)
    # every row normwise through the sketch: ||(J - Jref) G|| / ||Jref G|| estimates the row's
    # relative error (16 Gaussian columns: within a factor ~1.5 of the true ratio)
    sk = jr.jacobian @ G.sketch_matrix(jr.jacobian.shape[1])
    ref_sk = d["sketch"]
    row_err = np.linalg.norm(sk - ref_sk, axis=1) / np.linalg.norm(ref_sk, axis=1)
    assert np.max(row_err) <= TOL, np.max(row_err)
    # row norms of both blocks; the S block relative to the kappa block
    kn = np.linalg.norm(jr.jacobian[:, :n], axis=1)
    assert np.max(np.abs(kn - d["row_norm_kappa"]) / d["row_norm_kappa"]) <= TOL
    sn = np.linalg.norm(jr.jacobian[:, n:], axis=1)
    assert np.max(np.abs(sn - d["row_norm_s"]) / d["row_norm_kappa"]) <= TOL
    # entrywise on the significant entries of 8 full rows
    ptr = d["full_ptr"]
    for q, r in enumerate(d["full_rows"]):
        idx, val = d["full_idx"][ptr[q]:ptr[q + 1]], d["full_val"][ptr[q]:ptr[q + 1]]
        e = np.abs(jr.jacobian[r, idx] - val) / np.abs(val)
        assert np.max(e) <= TOL, (r, np.max(e))

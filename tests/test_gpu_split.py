"""The device side of the split Jacobian build in one process: the slice's
items solved in two parts (lt_split_solve), every slab's basis rows exported with their halo
(lt_split_export) and concatenated as the all-to-all delivers them, the slab columns assembled
(lt_jacobian_assemble_slab): equal to the one-call slice (lt_jacobian_slice).  The
collective itself is covered on CPU (tests/test_multirank.py, gloo, world size 2); one GPU
cannot stand in for two ranks of NCCL."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from paper_1409_2556_b200 import capi, inputs
from paper_1409_2556_b200 import laptomo as L
from paper_1409_2556_b200.split_build import DeviceBackend, partition, slabs, view

pytestmark = pytest.mark.gpu


CASES = {
    "3d": lambda: inputs.config(4).scaled((16, 12, 10), n_src=4, n_rec=6, n_times=2),  # 4-cell tensor-core tiles
    # the c4 box of tests/golden/configs (TMA operator, colour-split V-cycle), 16 x 8 items
    "3d-box": lambda: inputs.reduced(4, (64, 32, 24), receivers=list(range(0, 64, 8)), n_times=2),
    "2d": lambda: inputs.config(2).scaled((40, 36), n_src=3, n_rec=5, n_times=2),  # planes = rows
}


@pytest.mark.parametrize("case,parts", [("3d", 2), ("3d-box", 3), ("2d", 2)])
def test_split_parts_and_slabs_equal_the_full_slice(case, parts):
    cfg = CASES[case]()
    n_src, n_rec = len(cfg.sources), len(cfg.receivers)
    lk, ls = cfg.fields()
    g = L.Grid(tuple(cfg.shape), cfg.h)
    ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                         solver=L.SolverConfig(kind=cfg.solver_kind), include_storativity=True)
    p = L.ShiftedPencil(g, lk, ls)
    t = 1
    exc, keep = ex.c()
    n = g.n_cells
    pairs = n_src * n_rec
    Jfull = np.zeros((pairs, 2 * n))
    pred = np.zeros(pairs)
    capi.check(capi.lib().lt_jacobian_slice(p.handle, C.byref(exc), t, capi.LT_MEM_HOST, capi.dptr(Jfull),
                                            capi.dptr(pred)))
    be = DeviceBackend(p, ex, t)
    item_parts = partition(be.n_items, parts)
    hs = [be.solve(*r) for r in item_parts]
    m = max(be.columns(h) for h in hs)
    coef = [be.coefficients(h, m) for h in hs]
    Y = np.concatenate([c[0] for c in coef])
    mu = np.concatenate([c[1] for c in coef])
    got = np.zeros_like(Jfull)
    for (p0, p1) in slabs(be.n_planes, parts):
        v0, v1 = view(p0, p1, be.n_planes)
        cells = (v1 - v0) * be.plane_cells
        blocks = [be.export(h, v0, v1, m).view(m, r1 - r0, cells, 2) for h, (r0, r1) in zip(hs, item_parts)]
        U = torch.cat(blocks, dim=1).contiguous()
        J = be.assemble((p0, p1), U, m, Y, mu).cpu().numpy()
        c = (p1 - p0) * be.plane_cells
        got[:, p0 * be.plane_cells: p1 * be.plane_cells] = J[:, :c]
        got[:, n + p0 * be.plane_cells: n + p1 * be.plane_cells] = J[:, c:]
    predictions = np.concatenate([be.predictions(h) for h in hs]).ravel()
    for h in hs:
        be.release(h)
    scale = np.linalg.norm(Jfull[:, :n], axis=1, keepdims=True)
    assert np.max(np.abs(got - Jfull) / scale) <= 1e-12
    assert np.max(np.abs(predictions - pred) / np.abs(pred)) <= 1e-12

"""Golden fixtures (tests/golden, made by scripts/make_golden.py): the oracle reproduces
them (CPU), and the device path reproduces the FD ones through the C ABI (GPU)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import fd as ofd
from oracle import fem
from oracle import forward as F
from oracle import jacobian as J
from oracle import talbot as T

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return np.load(G / name)


def test_oracle_contours():
    d = load("talbot_contours.npz")
    for i in range(int(d["count"])):
        c = T.build_contour(int(d[f"n{i}"]), float(d[f"t{i}"]))
        assert np.max(np.abs(c.nodes - d[f"nodes{i}"])) <= 1e-15 * np.max(np.abs(c.nodes))
        assert np.max(np.abs(c.weights - d[f"weights{i}"])) <= 1e-13 * np.max(np.abs(c.weights))


def test_oracle_fd2d_forward():
    d = load("fd2d_forward.npz")
    grid = ofd.Grid(tuple(int(v) for v in d["shape"]), float(d["h"]))
    ops = ofd.assemble_fd(grid, np.exp(d["log_kappa"]), np.exp(d["log_storativity"]))
    b = ofd.point_weights(grid, d["source"])
    for kind in ("single", "flexible"):
        sol = F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, float(d["rate"]), None, list(d["times"]),
                                               int(d["n_quad"])), F.SolverConfig(kind=kind))
        assert np.max(np.abs(sol.heads - d[f"heads_{kind}"])) <= 1e-12 * np.max(np.abs(d[f"heads_{kind}"]))


def test_oracle_fd3d_jacobian():
    d = load("fd3d_jacobian.npz")
    grid = ofd.Grid(tuple(int(v) for v in d["shape"]), float(d["h"]))
    exp = J.ThtExperiment(grid, [tuple(p) for p in d["sources"]], list(d["rates"]), [tuple(p) for p in d["receivers"]],
                          list(d["times"]), int(d["n_quad"]), include_storativity=True)
    res = J.ThtForwardModel(exp, d["log_storativity"]).jacobian(d["log_kappa"])
    assert np.max(np.abs(res.jacobian - d["jacobian"])) <= 1e-10 * np.max(np.abs(d["jacobian"]))
    assert np.max(np.abs(res.predictions - d["predictions"]) / np.abs(d["predictions"])) <= 1e-10


def test_oracle_p1_jacobian():
    d = load("p1_jacobian.npz")
    mesh = fem.build_mesh(int(d["n_per_side"]), float(d["side"]))
    exp = J.ThtExperiment(mesh, [(50.0, 50.0)], [8.5e-4], [(30.0, 50.0), (70.0, 60.0)], [300.0, 600.0], n_quad=20,
                          include_storativity=True)
    res = J.ThtForwardModel(exp, d["log_storativity"]).jacobian(d["log_kappa"])
    assert np.max(np.abs(res.jacobian - d["jacobian"])) <= 1e-10 * np.max(np.abs(d["jacobian"]))


# ---- device path against the same fixtures ---------------------------------------------
@pytest.mark.gpu
def test_gpu_fd2d_forward_golden():
    from paper_1409_2556_b200 import laptomo as L
    d = load("fd2d_forward.npz")
    shape = tuple(int(v) for v in d["shape"])
    grid = ofd.Grid(shape, float(d["h"]))
    p = L.ShiftedPencil(L.Grid(shape, float(d["h"])), d["log_kappa"], d["log_storativity"])
    b = ofd.point_weights(grid, d["source"])
    for kind in ("single", "flexible"):
        sol, dd = L._forward(p, L.ForwardProblem(b, float(d["rate"]), None, list(d["times"]), int(d["n_quad"])),
                             L.SolverConfig(kind=kind), False, receivers=d["receivers"])
        ref = d[f"drawdown_{kind}"]
        assert np.max(np.abs(dd - ref) / np.abs(ref)) <= 1e-8
        assert [t.iterations for t in sol.diagnostics] == list(d[f"iterations_{kind}"])


@pytest.mark.gpu
def test_gpu_fd3d_jacobian_golden():
    from paper_1409_2556_b200 import laptomo as L
    d = load("fd3d_jacobian.npz")
    shape = tuple(int(v) for v in d["shape"])
    ex = L.ThtExperiment(L.Grid(shape, float(d["h"])), [tuple(p) for p in d["sources"]], list(d["rates"]),
                         [tuple(p) for p in d["receivers"]], list(d["times"]), int(d["n_quad"]),
                         include_storativity=True)
    res = L.ThtForwardModel(ex, d["log_storativity"]).jacobian(d["log_kappa"])
    n = int(np.prod(shape))
    Rk = d["jacobian"][:, :n]
    Jk = res.jacobian[:, :n]
    assert np.max(np.linalg.norm(Jk - Rk, axis=1) / np.linalg.norm(Rk, axis=1)) <= 1e-8
    Rs = d["jacobian"][:, n:]
    assert np.max(np.linalg.norm(res.jacobian[:, n:] - Rs, axis=1) / np.linalg.norm(Rk, axis=1)) <= 1e-8
    assert np.max(np.abs(res.predictions - d["predictions"]) / np.abs(d["predictions"])) <= 1e-8

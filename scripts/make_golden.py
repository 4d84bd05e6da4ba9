"""Generates tests/golden/*.npz: small seeded cases solved by the CPU oracle (SciPy
restatement of the reference path).  The reference itself cannot be built here (Eigen is
absent), so these fixtures pin the oracle against regressions and carry the exact inputs
the device path is checked on (tests/test_golden.py, tests/test_gpu_golden.py).

    python scripts/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import fd as ofd  # noqa: E402
from oracle import fem  # noqa: E402
from oracle import forward as F  # noqa: E402
from oracle import jacobian as J  # noqa: E402
from oracle import talbot as T  # noqa: E402
from paper_1409_2556_b200 import inputs  # noqa: E402

OUT = ROOT / "tests" / "golden"


def contours():
    cases = [(24, 1.0), (32, 100.0), (32, 1e5), (20, 300.0), (40, 3600.0)]
    d = {}
    for i, (n, t) in enumerate(cases):
        c = T.build_contour(n, t)
        d[f"n{i}"] = np.array(n)
        d[f"t{i}"] = np.array(t)
        d[f"nodes{i}"] = c.nodes
        d[f"weights{i}"] = c.weights
    np.savez_compressed(OUT / "talbot_contours.npz", count=np.array(len(cases)), **d)


def fd2d_forward():
    cfg = inputs.config(0).scaled((24, 20), n_times=3)
    lk, ls = cfg.fields()
    grid = ofd.Grid(cfg.shape, cfg.h)
    ops = ofd.assemble_fd(grid, np.exp(lk), np.exp(ls))
    b = ofd.point_weights(grid, cfg.sources[0])
    out = {}
    for kind in ("single", "flexible"):
        sol = F.solve_forward(F.ForwardProblem(ops.stiffness, ops.mass, b, cfg.rates[0], None, cfg.times,
                                               cfg.n_quad), F.SolverConfig(kind=kind))
        rec = np.array([ofd.point_weights(grid, q) @ sol.heads for q in cfg.receivers])
        out[f"heads_{kind}"] = sol.heads
        out[f"drawdown_{kind}"] = rec
        out[f"iterations_{kind}"] = np.array([d.iterations for d in sol.diagnostics])
    np.savez_compressed(OUT / "fd2d_forward.npz", shape=np.array(cfg.shape), h=np.array(cfg.h), log_kappa=lk,
                        log_storativity=ls, source=np.array(cfg.sources[0]), rate=np.array(cfg.rates[0]),
                        receivers=np.array(cfg.receivers), times=np.array(cfg.times), n_quad=np.array(cfg.n_quad),
                        **out)


def fd3d_jacobian():
    cfg = inputs.config(4).scaled((8, 8, 6), n_src=2, n_rec=3, n_times=2)
    lk, ls = cfg.fields()
    grid = ofd.Grid(cfg.shape, cfg.h)
    exp = J.ThtExperiment(grid, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                          include_storativity=True)
    res = J.ThtForwardModel(exp, ls).jacobian(lk)
    np.savez_compressed(OUT / "fd3d_jacobian.npz", shape=np.array(cfg.shape), h=np.array(cfg.h), log_kappa=lk,
                        log_storativity=ls, sources=np.array(cfg.sources), rates=np.array(cfg.rates),
                        receivers=np.array(cfg.receivers), times=np.array(cfg.times), n_quad=np.array(cfg.n_quad),
                        jacobian=res.jacobian, predictions=res.predictions)


def p1_forward_jacobian():
    rng = np.random.default_rng(21)
    mesh = fem.build_mesh(11, 100.0)
    lk = np.log(1e-4) + 0.8 * rng.standard_normal(mesh.n_elements())
    ls = np.full(mesh.n_elements(), np.log(1e-5))
    exp = J.ThtExperiment(mesh, [(50.0, 50.0)], [8.5e-4], [(30.0, 50.0), (70.0, 60.0)], [300.0, 600.0],
                          n_quad=20, include_storativity=True)
    res = J.ThtForwardModel(exp, ls).jacobian(lk)
    np.savez_compressed(OUT / "p1_jacobian.npz", n_per_side=np.array(11), side=np.array(100.0), log_kappa=lk,
                        log_storativity=ls, jacobian=res.jacobian, predictions=res.predictions)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    contours()
    fd2d_forward()
    fd3d_jacobian()
    p1_forward_jacobian()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
